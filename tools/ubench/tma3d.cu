// Microbenchmark: TMA load throughput from a row-major n x m fp32 matrix (4 MB row pitch)
// into SWIZZLE_128B K-block atoms, with G K-blocks per request via a 3-D tensor map
// {32 cols, rows, m/32 groups} (G = 1 is the plain 2-D 128-B-row box).  Every CTA streams its
// own (row block, K range), as the SYRK does; each row block is read by ~19 CTAs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2310_17556_b200/csrc/tc_ptx.cuh"
using namespace fs;
constexpr int kAtom = 128 * 128;   // one K-block of one row block: 16 KB
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               ::"r"(ptx::smem_u32(dst)), "l"(map), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap map, int iters, int G, int stages) {
  extern __shared__ uint8_t sm_[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * G * kAtom);
  if (threadIdx.x == 0) { for (int s = 0; s < stages; ++s) ptx::mbar_init(&full[s], 1); ptx::fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int row0 = (blockIdx.x % 8) * 128;
  const int g0 = (blockIdx.x / 8) * iters * G;
  const uint32_t bytes = G * kAtom;
  for (int i = 0; i < stages && i < iters; ++i) {
    ptx::mbar_arrive_expect_tx(&full[i], bytes);
    tma3(sm + i * G * kAtom, &map, &full[i], 0, row0, g0 + i * G);
  }
  for (int i = 0; i < iters; ++i) {
    const int s = i % stages;
    ptx::mbar_wait(&full[s], (i / stages) & 1);
    const int nx = i + stages;
    if (nx < iters) {
      ptx::mbar_arrive_expect_tx(&full[s], bytes);
      tma3(sm + s * G * kAtom, &map, &full[s], 0, row0, g0 + nx * G);
    }
  }
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  const size_t n = 1024, m = 1000000;
  float* S; cudaMalloc(&S, n * m * 4); cudaMemset(S, 0, n * m * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int G : {1, 2, 4}) {
    for (CUtensorMapL2promotion prom : {CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B}) {
      CUtensorMap map;
      cuuint64_t gdim[3] = {32, n, m / 32}, gstr[2] = {m * 4, 128};
      cuuint32_t box[3] = {32, 128, (cuuint32_t)G}, es[3] = {1, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, S, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) { printf("encode failed %d\n", r); return 1; }
      const int stages = 8 / G;
      const int iters = 1600 / G;   // 19 CTAs per row block x 1600 K-blocks <= 31250
      for (int grid : {148, 296 / 2}) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        k<<<grid, 128, stages * G * kAtom + 2048>>>(map, iters, G, stages);
        cudaEventRecord(a);
        k<<<grid, 128, stages * G * kAtom + 2048>>>(map, iters, G, stages);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double bytes = (double)grid * iters * G * kAtom;
        printf("G=%d promo=%s grid %3d: %.3f ms  %.1f GB/s  %.2f B/clk/SM  err=%s\n", G,
               prom == CU_TENSOR_MAP_L2_PROMOTION_L2_128B ? "128" : "256", grid, ms, bytes / ms / 1e6,
               bytes / ms / 1e6 / grid / 1.965, cudaGetErrorString(cudaGetLastError()));
        break;
      }
    }
  }
  return 0;
}
