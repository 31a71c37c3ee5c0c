// trsv.cu — z <- L^-T (L^-1 z) with the lower Cholesky factor (fp64).
//
// Replaces solvers.py:111 (solve_triangular(L, t1, lower=True, trans='N')) and
// solvers.py:114 (trans='T') — the two LAPACK dtrtrs calls of _chol_apply.
// Blocked substitution over 64-row blocks using the inverted diagonal blocks Linv_BB that
// potrf already produced: each block step is an off-diagonal GEMV (coalesced row reads of L,
// L2-resident) followed by a 64x64 GEMV with Linv_BB — no dependent global-load chains.
// One CTA of 1024 threads; deterministic (fixed reduction order).
#include "common.cuh"
#include "kernels.h"

namespace fs {
namespace {

constexpr int kNB = 64;
constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads)
trsv_pair_kernel(const double* __restrict__ L, int64_t n, int64_t ld, const double* __restrict__ Linv,
                 double* __restrict__ z, const int64_t* status) {
  __shared__ double t[kNB];
  __shared__ double part[kWarps][kNB];
  if (status && *(volatile const int64_t*)status != 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (int)((n + kNB - 1) / kNB);
  // ---------------- forward: L z' = z ----------------
  for (int B = 0; B < nb; ++B) {
    const int64_t r0 = (int64_t)B * kNB;
    const int b = (int)(n - r0 < kNB ? n - r0 : kNB);
    for (int r = warp; r < kNB; r += kWarps) {         // t_r = z_r - L[r, :r0] z[:r0]
      double s = 0.0;
      if (r < b) {
        const double* row = L + (r0 + r) * ld;
        for (int64_t c = lane; c < r0; c += 32) s = fma(row[c], z[c], s);
      }
      s = warp_sum(s);
      if (lane == 0) t[r] = (r < b) ? z[r0 + r] - s : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < 4 * kNB) {                          // z_B = Linv_BB t
      const int r = threadIdx.x >> 2, q = threadIdx.x & 3;
      const double* li = Linv + (size_t)B * kNB * kNB + r * kNB;
      double s = 0.0;
      for (int c = q; c <= r; c += 4) s = fma(li[c], t[c], s);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (q == 0 && r < b) z[r0 + r] = s;
    }
    __syncthreads();
  }
  // ---------------- backward: L^T z = z' ----------------
  for (int B = nb - 1; B >= 0; --B) {
    const int64_t r0 = (int64_t)B * kNB;
    const int b = (int)(n - r0 < kNB ? n - r0 : kNB);
    // part[w][c] = sum over rows i >= r0 + 64 owned by warp w of L[i][r0 + c] z[i]
    double a0 = 0.0, a1 = 0.0;
    for (int64_t i = r0 + kNB + warp; i < n; i += kWarps) {
      const double zi = z[i];
      const double* row = L + i * ld + r0;
      if (2 * lane < b) a0 = fma(row[2 * lane], zi, a0);
      if (2 * lane + 1 < b) a1 = fma(row[2 * lane + 1], zi, a1);
    }
    part[warp][2 * lane] = a0;
    part[warp][2 * lane + 1] = a1;
    __syncthreads();
    if (threadIdx.x < kNB) {
      const int c = threadIdx.x;
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s += part[w][c];
      t[c] = (c < b) ? z[r0 + c] - s : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < 4 * kNB) {                          // z_B = Linv_BB^T t
      const int c = threadIdx.x >> 2, q = threadIdx.x & 3;
      const double* li = Linv + (size_t)B * kNB * kNB;
      double s = 0.0;
      for (int r = c + q; r < kNB; r += 4) s = fma(li[r * kNB + c], t[r], s);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (q == 0 && c < b) z[r0 + c] = s;
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t trsv_pair(const double* L, int64_t n, int64_t ldL, const double* Linv, double* z,
                      const int64_t* d_status, cudaStream_t st, int* launches) {
  trsv_pair_kernel<<<1, kThreads, 0, st>>>(L, n, ldL, Linv, z, d_status);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace fs
