// trsv.cu — z <- L^-T (L^-1 z) with the lower Cholesky factor (fp64).
//
// Replaces solvers.py:111 (solve_triangular(L, t1, lower=True, trans='N')) and
// solvers.py:114 (trans='T') — the two LAPACK dtrtrs calls of _chol_apply.
// One CTA of 1024 threads, 32-wide diagonal blocks solved by one warp with shuffles,
// off-diagonal updates by all warps with coalesced row reads of L (L2-resident).
#include "common.cuh"
#include "kernels.h"

namespace fs {
namespace {

constexpr int kB = 32;
constexpr int kThreads = 1024;

__global__ void __launch_bounds__(kThreads)
trsv_pair_kernel(const double* __restrict__ L, int64_t n, int64_t ld, double* __restrict__ z,
                 const int64_t* status) {
  if (status && *(volatile const int64_t*)status != 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kThreads / 32;
  // ---- forward: L z' = z ----
  for (int64_t kb = 0; kb < n; kb += kB) {
    const int bs = (int)(n - kb < kB ? n - kb : kB);
    if (warp == 0) {
      double val = lane < bs ? z[kb + lane] : 0.0;
      for (int j = 0; j < bs; ++j) {
        if (lane == j) val = val / L[(kb + j) * ld + kb + j];
        const double zj = __shfl_sync(0xffffffffu, val, j);
        if (lane > j && lane < bs) val = fma(-L[(kb + lane) * ld + kb + j], zj, val);
      }
      if (lane < bs) z[kb + lane] = val;
    }
    __syncthreads();
    const double zb = lane < bs ? z[kb + lane] : 0.0;
    for (int64_t i = kb + bs + warp; i < n; i += kWarps) {
      double p = lane < bs ? L[i * ld + kb + lane] * zb : 0.0;
      p = warp_sum(p);
      if (lane == 0) z[i] -= p;
    }
    __syncthreads();
  }
  // ---- backward: L^T z = z' ----
  const int64_t nblk = (n + kB - 1) / kB;
  for (int64_t blk = nblk - 1; blk >= 0; --blk) {
    const int64_t kb = blk * kB;
    const int bs = (int)(n - kb < kB ? n - kb : kB);
    if (warp == 0) {
      double val = lane < bs ? z[kb + lane] : 0.0;
      for (int j = bs - 1; j >= 0; --j) {
        if (lane == j) val = val / L[(kb + j) * ld + kb + j];
        const double zj = __shfl_sync(0xffffffffu, val, j);
        if (lane < j) val = fma(-L[(kb + j) * ld + kb + lane], zj, val);
      }
      if (lane < bs) z[kb + lane] = val;
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < kb; i += kThreads) {
      double s = 0.0;
      for (int j = 0; j < bs; ++j) s = fma(L[(kb + j) * ld + i], z[kb + j], s);
      z[i] -= s;
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t trsv_pair(const double* L, int64_t n, int64_t ldL, double* z, const int64_t* d_status,
                      cudaStream_t st, int* launches) {
  trsv_pair_kernel<<<1, kThreads, 0, st>>>(L, n, ldL, z, d_status);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace fs
