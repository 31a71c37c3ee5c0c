// Microbenchmark: sustained fp64 tensor-core (mma.sync.m8n8k4.f64) rate per GPU, register-only
// operands, W warps per CTA, one CTA per SM (148 CTAs), 32 independent accumulators per warp (the
// SYRK's 8 x 4 fragment grid).  Prints TF/s and the SM clock the run averaged (clock64 / wall).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__global__ void peak(int iters, double* out, long long* clk) {
  double acc[8][4][2];
  double af[8], bf[4];
  for (int a = 0; a < 8; ++a) af[a] = 1e-3 * (threadIdx.x + a);
  for (int b = 0; b < 4; ++b) bf[b] = 1e-3 * (threadIdx.x - b);
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma(acc[a][b], af[a], bf[b]);
  }
  long long c1 = clock64();
  double s = 0;
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 4; ++b) s += acc[a][b][0] + acc[a][b][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* clk;
  cudaMalloc(&out, sizeof(double) * sms * 1024);
  cudaMalloc(&clk, sizeof(long long) * sms);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      peak<<<sms, warps * 32>>>(iters, out, clk);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long c;
      cudaMemcpy(&c, clk, sizeof(c), cudaMemcpyDeviceToHost);
      const double flop = 2.0 * 256 * 32 * (double)iters * warps * sms;
      const double fma_clk_sm = 256.0 * 32 * iters * warps / (double)c;
      printf("warps %2d  %.2f ms  %.1f TF/s  %.1f FMA/clk/SM  ~%.0f MHz\n", warps, ms, flop / (ms * 1e-3) / 1e12,
             fma_clk_sm, c / (ms * 1e3));
    }
  }
  return cudaGetLastError() != cudaSuccess;
}
