// Microbenchmark: HBM throughput of a full read of a row-major n x m fp32 matrix (4 MB row pitch)
// when each CTA streams column panels W x 128 B wide over all rows, in 64-row chunks of W
// 128B-swizzled TMA boxes (the x+y pass's access pattern for W = 1).  24-slot ring per CTA, no
// compute: the number is the DRAM efficiency of W*128-byte row segments.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2310_17556_b200/csrc/tc_ptx.cuh"
using namespace fs;
constexpr int kSlots = 24, kChunk = 64 * 128;
__global__ void __launch_bounds__(32, 1) seg_kernel(const __grid_constant__ CUtensorMap map, int n, int64_t m, int W) {
  extern __shared__ uint8_t sm_[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kSlots * kChunk);
  if (threadIdx.x == 0) { for (int s = 0; s < kSlots; ++s) ptx::mbar_init(&full[s], 1); ptx::fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int64_t panels = (m / 32 + W - 1) / W;
  const int nch = n / 64;
  uint32_t issued = 0, done = 0;
  for (int64_t q = blockIdx.x; q < panels; q += gridDim.x)
    for (int c = 0; c < nch; ++c)
      for (int w = 0; w < W; ++w) {
        if (issued >= kSlots) {                      // retire the oldest
          const uint32_t s = done % kSlots;
          ptx::mbar_wait(&full[s], (done / kSlots) & 1);
          ++done;
        }
        const uint32_t s = issued % kSlots;
        ptx::mbar_arrive_expect_tx(&full[s], kChunk);
        ptx::tma_load_2d(sm + s * kChunk, &map, &full[s], (int)((q * W + w) * 32), c * 64);
        ++issued;
      }
  while (done < issued) { const uint32_t s = done % kSlots; ptx::mbar_wait(&full[s], (done / kSlots) & 1); ++done; }
}
// unswizzled 2-D boxes of Wb-byte rows (8 KB per box)
__global__ void __launch_bounds__(32, 1) wide_kernel(const __grid_constant__ CUtensorMap map, int n, int64_t m, int Wb,
                                                     int slots = kSlots, int R = 0) {
  extern __shared__ uint8_t sm_[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kSlots * kChunk);
  if (threadIdx.x == 0) { for (int s = 0; s < kSlots; ++s) ptx::mbar_init(&full[s], 1); ptx::fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int64_t cols = Wb / 4, panels = m / cols;
  if (R == 0) R = kChunk / Wb;
  const int nch = (n + R - 1) / R;
  uint32_t issued = 0, done = 0;
  for (int64_t q = blockIdx.x; q < panels; q += gridDim.x)
    for (int c = 0; c < nch; ++c) {
      if (issued >= (uint32_t)slots) {
        const uint32_t s = done % slots;
        ptx::mbar_wait(&full[s], (done / slots) & 1);
        ++done;
      }
      const uint32_t s = issued % slots;
      ptx::mbar_arrive_expect_tx(&full[s], R * Wb);
      ptx::tma_load_2d(sm + s * kChunk, &map, &full[s], (int)(q * cols), c * R);
      ++issued;
    }
  while (done < issued) { const uint32_t s = done % slots; ptx::mbar_wait(&full[s], (done / slots) & 1); ++done; }
}
// same stream through 1-D bulk copies: one Wb-byte row segment per copy, the 32 lanes of the
// producer warp issuing the rows of a chunk in parallel (chunk = 8 KB = 8192/Wb rows)
__global__ void __launch_bounds__(32, 1) bulk_kernel(const float* S, int n, int64_t m, int Wb) {
  extern __shared__ uint8_t sm_[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kSlots * kChunk);
  const int lane = threadIdx.x;
  if (lane == 0) { for (int s = 0; s < kSlots; ++s) ptx::mbar_init(&full[s], 1); ptx::fence_mbar_init(); }
  __syncthreads();
  const int64_t cols = Wb / 4;
  const int64_t panels = m / cols;
  const int R = kChunk / Wb, nch = n / R;
  uint32_t issued = 0, done = 0;
  for (int64_t q = blockIdx.x; q < panels; q += gridDim.x)
    for (int c = 0; c < nch; ++c) {
      if (issued >= kSlots) {
        const uint32_t s = done % kSlots;
        ptx::mbar_wait(&full[s], (done / kSlots) & 1);
        ++done;
      }
      const uint32_t s = issued % kSlots;
      if (lane == 0) ptx::mbar_arrive_expect_tx(&full[s], kChunk);
      __syncwarp();
      for (int r = lane; r < R; r += 32)
        ptx::bulk_load(sm + s * kChunk + r * Wb, S + (int64_t)(c * R + r) * m + q * cols, Wb, &full[s]);
      ++issued;
    }
  while (done < issued) { const uint32_t s = done % kSlots; ptx::mbar_wait(&full[s], (done / kSlots) & 1); ++done; }
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
  const int smem = kSlots * kChunk + 2048;
  cudaFuncSetAttribute(seg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  CUtensorMap map;
  cuuint64_t gdim[2] = {m, n}, gstr[1] = {m * 4};
  cuuint32_t box[2] = {32, 64}, es[2] = {1, 1};
  for (auto l2 : {CU_TENSOR_MAP_L2_PROMOTION_L2_256B}) {
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, S, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) { printf("encode failed\n"); return 1; }
    for (int W : {1, 2, 4, 8, 16, 32})
      for (int grid : {148}) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        seg_kernel<<<grid, 32, smem>>>(map, n, m, W);
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) seg_kernel<<<grid, 32, smem>>>(map, n, m, W);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
        printf("l2promo %d W %2d (%5d B segments) grid %d: %.3f ms  %.0f GB/s  err=%s\n", (int)l2, W, W * 128, grid, ms,
               n * m * 4.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
  }
  cudaFuncSetAttribute(wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // unswizzled boxes with wider rows: Wb-byte rows x (8192/Wb) rows per box
  for (int Wb : {128, 256, 512, 1024}) {
    cuuint32_t box2[2] = {(cuuint32_t)(Wb / 4), (cuuint32_t)(8192 / Wb)};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, S, gdim, gstr, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
      printf("encode failed\n"); return 1; }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    wide_kernel<<<148, 32, smem>>>(map, n, m, Wb);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) wide_kernel<<<148, 32, smem>>>(map, n, m, Wb);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
    printf("tma2d-noswizzle %5d B rows: %.3f ms  %.0f GB/s  err=%s\n", Wb, ms, n * m * 4.0 / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    cuuint32_t box2[2] = {64, 30};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, S, gdim, gstr, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int grid : {132, 148})
      for (int slots : {4, 8, 12, 16, 24}) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        wide_kernel<<<grid, 32, smem>>>(map, n, m, 256, slots, 30);
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) wide_kernel<<<grid, 32, smem>>>(map, n, m, 256, slots, 30);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
        printf("256Bx30 boxes grid %d slots %2d (%3d KB in flight): %.3f ms  %.0f GB/s  err=%s\n", grid, slots,
               slots * 30 * 256 / 1024, ms, n * m * 4.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
  }
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int Wb : {128, 256, 512, 1024, 2048, 4096}) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    bulk_kernel<<<148, 32, smem>>>(S, n, m, Wb);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) bulk_kernel<<<148, 32, smem>>>(S, n, m, Wb);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
    printf("bulk1d %5d B segments: %.3f ms  %.0f GB/s  err=%s\n", Wb, ms, n * m * 4.0 / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
