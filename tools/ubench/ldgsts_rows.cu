// Feasibility of a 2-CTA-per-panel x + y pass on all 148 SMs: stream a 1024 x 1e6 fp32 matrix
// as 128-byte-wide panels (32 columns x 512 rows per CTA, two CTAs per panel) with cp.async
// (LDGSTS, 16 B per thread-instruction; no TMA row-rate limit) through a ring of NS sets in
// shared memory; every element is read once from shared memory by the consumer warps (a sum)
// so the loads cannot be elided.  Prints the achieved bandwidth for a few ring depths.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kRows = 512, kCols = 32, kThreads = 512;
constexpr int kSetBytes = kRows * kCols * 4;   // 64 KB

template <int NS>
__global__ void __launch_bounds__(kThreads, 1) stream_kernel(const float* __restrict__ S, int64_t n, int64_t m,
                                                              float* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int half = blockIdx.x & 1;
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int64_t panels = m / kCols;
  const int64_t row0 = (int64_t)half * kRows;
  float acc = 0.f;
  auto issue = [&](int64_t p, int set) {
    if (p < panels) {
      const int64_t col = p * kCols;
      unsigned char* dst = sm + (size_t)set * kSetBytes;
      // 512 rows x 8 pieces of 16 B = 4096 pieces, 8 per thread
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int piece = threadIdx.x + q * kThreads;
        const int r = piece >> 3, c = (piece & 7) * 4;
        const float* src = S + (row0 + r) * m + col + c;
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + (r * kCols + c) * 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t j = 0;
  const int64_t np = (panels - pair + npairs - 1) / npairs;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) issue(pair + (int64_t)s * npairs, s);
  for (j = 0; j < np; ++j) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
    __syncthreads();
    issue(pair + (j + NS - 1) * npairs, (int)((j + NS - 1) % NS));
    const float4* src = reinterpret_cast<const float4*>(sm + (size_t)(j % NS) * kSetBytes);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 v = src[threadIdx.x + q * kThreads];
      acc += v.x + v.y + v.z + v.w;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (acc == 123.456f) out[0] = acc;
}

int main() {
  const int64_t n = 1024, m = 1000000;
  float* S;
  float* out;
  cudaMalloc(&S, n * m * 4);
  cudaMalloc(&out, 4);
  cudaMemset(S, 0, n * m * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](auto kern, int ns) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * kSetBytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(a);
      kern<<<sms & ~1, kThreads, ns * kSetBytes>>>(S, n, m, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 3) printf("NS=%d: %.3f ms, %.0f GB/s (%s)\n", ns, ms, n * m * 4 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(stream_kernel<2>, 2);
  run(stream_kernel<3>, 3);
  return 0;
}
