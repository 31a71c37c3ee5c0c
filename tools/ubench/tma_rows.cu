// Microbenchmark: TMA load throughput of 128-row x 128-B boxes (SWIZZLE_128B) from
// (A) a row-major matrix with a 4 MB row pitch (the SYRK's access pattern) and
// (B) the same bytes laid out contiguously (box = 16 KB contiguous).  6-stage ring per CTA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2310_17556_b200/csrc/tc_ptx.cuh"
using namespace fs;
constexpr int kStages = 6, kBox = 128 * 128;
__global__ void __launch_bounds__(128, 1) tma_kernel(const __grid_constant__ CUtensorMap map, int iters, int contiguous, int nrowblk) {
  extern __shared__ uint8_t sm_[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kBox);
  if (threadIdx.x == 0) { for (int s = 0; s < kStages; ++s) ptx::mbar_init(&full[s], 1); ptx::fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int row0 = (blockIdx.x % nrowblk) * 128;
  // prologue
  for (int i = 0; i < kStages && i < iters; ++i) {
    ptx::mbar_arrive_expect_tx(&full[i], kBox);
    if (contiguous) ptx::tma_load_2d(sm + i * kBox, &map, &full[i], 0, (blockIdx.x * iters + i) * 128);
    else ptx::tma_load_2d(sm + i * kBox, &map, &full[i], i * 32, row0);
  }
  for (int i = 0; i < iters; ++i) {
    const int s = i % kStages;
    ptx::mbar_wait(&full[s], (i / kStages) & 1);
    const int nx = i + kStages;
    if (nx < iters) {
      ptx::mbar_arrive_expect_tx(&full[s], kBox);
      if (contiguous) ptx::tma_load_2d(sm + s * kBox, &map, &full[s], 0, (blockIdx.x * iters + nx) * 128);
      else ptx::tma_load_2d(sm + s * kBox, &map, &full[s], nx * 32, row0);
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
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kBox + 2048);
  const int iters = 4000;
  for (int variant = 0; variant < 2; ++variant) {
    CUtensorMap map;
    cuuint64_t gdim[2], gstr[1];
    if (variant == 0) { gdim[0] = m; gdim[1] = n; gstr[0] = m * 4; }          // row pitch 4 MB
    else { gdim[0] = 32; gdim[1] = n * m / 32; gstr[0] = 128; }                 // contiguous boxes
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, S, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", r); return 1; }
    for (int grid : {148, 74, 16}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      // variant 1: make each CTA walk its own contiguous region (coordinates as rows of 32 floats)
      tma_kernel<<<grid, 128, kStages * kBox + 2048>>>(map, iters, variant, 8);
      cudaEventRecord(a);
      tma_kernel<<<grid, 128, kStages * kBox + 2048>>>(map, iters, variant, 8);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double bytes = (double)grid * iters * kBox;
      printf("variant %s grid %3d: %.3f ms  %.1f GB/s total  %.2f B/clk/SM @1.965GHz  err=%s\n",
             variant == 0 ? "strided-rows" : "contiguous ", grid, ms, bytes / ms / 1e6,
             bytes / ms / 1e6 / grid / 1.965, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
