// apply.cu — Y = T X on the fp64 tensor cores: an r x n fp64 matrix applied to the rows of an
// n x m score-layout matrix (row-major, unit column stride, fp32 or fp64).
//
// The m x r factor products of the comparison routes are this shape:
//   thin_svd_eigh   V^T = (U / sigma)^T S            (solvers.py:272-276: V = A^T B -> dgemm)
//   svda (CQR)      Q^T = L^-1 S, V^T = W^T Q^T      (the QR-then-SVD route of thin_svd_direct)
// so they run on this package's own kernel instead of a library GEMM.  Every product t_ik x_kc is
// an IEEE fp64 FMA (fp32 X is widened exactly) on mma.sync.m8n8k4.f64.
//
// 128 x 128 output tiles, 256 threads = 8 warps of 64 x 32 (8 x 4 m8n8 fragments: 64 fp64
// accumulators per thread), K (= n, the contraction runs over the ROWS of X) in 32-deep stages,
// double-buffered through shared memory with register staging.  The X stage is stored transposed
// ([column][k], pitch 36 doubles) so the .col B fragments read it like the SYRK's B rows; a warp
// stores 32 consecutive k of one column per instruction (conflict-free).  A lower-triangular T
// (the CholeskyQR steps' L^-1) stops each row tile's K loop at its last row: ~half the products.  Tiles sharing a column
// panel of X are adjacent in the launch order, so X streams from HBM about once and T (r x n
// doubles) stays in L2.  The bound is the fp64 tensor rate (2 r n m flops).
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace fs {
namespace {

constexpr int kT = 128;
constexpr int kK = 32;
constexpr int kLd = kK + 4;
constexpr int kThreads = 256;
constexpr int kStageDoubles = 2 * kT * kLd;
constexpr size_t kSmemBytes = 2 * kStageDoubles * sizeof(double);   // 147 KB

FS_DEVINL void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

FS_DEVINL void stage_mma(double (&acc)[8][4][2], const double* A, const double* B, int wr, int wc, int fr, int fk) {
#pragma unroll
  for (int ks = 0; ks < kK; ks += 4) {
    double af[8], bf[4];
#pragma unroll
    for (int a = 0; a < 8; ++a) af[a] = A[(wr + 8 * a + fr) * kLd + ks + fk];
#pragma unroll
    for (int b = 0; b < 4; ++b) bf[b] = B[(wc + 8 * b + fr) * kLd + ks + fk];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma(acc[a][b], af[a], bf[b]);
  }
}

// T stage: rows [r0, r0+128) x k [k0, k0+32) -> A[row][k].  Thread t: row t >> 1, 16 k's.
struct LoadT {
  double v[16];
  FS_DEVINL void load(const double* __restrict__ T, int64_t r, int64_t n, int64_t ldT, int64_t r0, int64_t k0,
                      bool vec) {
    const int row = threadIdx.x >> 1, c = (threadIdx.x & 1) * 16;
    const int64_t gr = r0 + row, gc = k0 + c;
    if (gr < r && vec && gc + 16 <= n) {
      const double2* p = reinterpret_cast<const double2*>(T + gr * ldT + gc);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double2 f = __ldg(p + q);
        v[2 * q] = f.x; v[2 * q + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = (gr < r && gc + e < n) ? __ldg(T + gr * ldT + gc + e) : 0.0;
    }
  }
  FS_DEVINL void store(double* __restrict__ A) const {
    const int row = threadIdx.x >> 1, c = (threadIdx.x & 1) * 16;
    double2* d = reinterpret_cast<double2*>(A + row * kLd + c);
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = make_double2(v[2 * q], v[2 * q + 1]);
  }
};

// X stage: rows k [k0, k0+32) x columns [c0, c0+128) -> B[column][k] (transposed).
// Thread t: k = t & 31, columns (t >> 5) * 16 ... +16 (64 contiguous bytes of fp32 X).
template <typename T>
struct LoadX {
  double v[16];
  FS_DEVINL void load(const T* __restrict__ X, int64_t n, int64_t m, int64_t ldX, int64_t k0, int64_t c0, bool vec) {
    const int k = threadIdx.x & 31, cb = (threadIdx.x >> 5) * 16;
    const int64_t gk = k0 + k, gc = c0 + cb;
    if (gk < n && vec && gc + 16 <= m) {
      const T* p = X + gk * ldX + gc;
      if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(p) + q);
          v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double2 f = __ldg(reinterpret_cast<const double2*>(p) + q);
          v[2 * q] = f.x; v[2 * q + 1] = f.y;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = (gk < n && gc + e < m) ? (double)__ldg(X + gk * ldX + gc + e) : 0.0;
    }
  }
  FS_DEVINL void store(double* __restrict__ B) const {
    const int k = threadIdx.x & 31, cb = (threadIdx.x >> 5) * 16;
#pragma unroll
    for (int j = 0; j < 16; ++j) B[(cb + j) * kLd + k] = v[j];
  }
};

template <typename TX>
__global__ void __launch_bounds__(kThreads, 1)
apply_rows_kernel(const double* __restrict__ T, int64_t r, int64_t n, int64_t ldT, const TX* __restrict__ X, int64_t m,
                  int64_t ldX, double* __restrict__ Y, int64_t ldY, int tiles_r, int vecT, int vecX, int lower) {
  extern __shared__ __align__(16) double dsm[];
  const int64_t r0 = (int64_t)(blockIdx.x % tiles_r) * kT;
  const int64_t c0 = (int64_t)(blockIdx.x / tiles_r) * kT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 2) * 64, wc = (warp & 3) * 32;
  const int fr = lane >> 2, fk = lane & 3;
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  LoadT lt;
  LoadX<TX> lx;
  lt.load(T, r, n, ldT, r0, 0, vecT);
  lx.load(X, n, m, ldX, 0, c0, vecX);
  lt.store(dsm);
  lx.store(dsm + kT * kLd);
  __syncthreads();
  int buf = 0;
  // lower-triangular T: rows [r0, r0 + 128) have no entries past column r0 + 127
  const int64_t kend = lower ? (r0 + kT < n ? r0 + kT : n) : n;
  for (int64_t k0 = 0; k0 < kend; k0 += kK) {
    const bool more = k0 + kK < kend;
    if (more) {
      lt.load(T, r, n, ldT, r0, k0 + kK, vecT);
      lx.load(X, n, m, ldX, k0 + kK, c0, vecX);
    }
    const double* A = dsm + buf * kStageDoubles;
    stage_mma(acc, A, A + kT * kLd, wr, wc, fr, fk);
    if (more) {
      double* nxt = dsm + (buf ^ 1) * kStageDoubles;
      lt.store(nxt);
      lx.store(nxt + kT * kLd);
    }
    __syncthreads();
    buf ^= 1;
  }
  // accumulator fragment (m8n8 f64): rows fr, columns 2 (lane & 3) + {0, 1}
  const int cc = 2 * (lane & 3);
  const bool pair_ok = (ldY & 1) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t gi = r0 + wr + 8 * a + fr, gj = c0 + wc + 8 * b + cc;
      if (gi >= r) continue;
      double* y = Y + gi * ldY + gj;
      if (pair_ok && gj + 1 < m) {
        *reinterpret_cast<double2*>(y) = make_double2(acc[a][b][0], acc[a][b][1]);
      } else {
        if (gj < m) y[0] = acc[a][b][0];
        if (gj + 1 < m) y[1] = acc[a][b][1];
      }
    }
}

}  // namespace

cudaError_t apply_rows(bool x_f64, const double* T, int64_t r, int64_t n, int64_t ldT, const void* X, int64_t m,
                       int64_t ldX, double* Y, int64_t ldY, cudaStream_t st, int* launches, bool lower) {
  if (r < 1 || n < 1 || m < 1) return cudaErrorInvalidValue;
  const int64_t tiles_r = (r + kT - 1) / kT, tiles_c = (m + kT - 1) / kT;
  if (tiles_r * tiles_c > INT32_MAX) return cudaErrorInvalidValue;
  const int vecT = ((reinterpret_cast<uintptr_t>(T) | (uintptr_t)(ldT * 8)) & 15) == 0 ? 1 : 0;
  const int vecX = ((reinterpret_cast<uintptr_t>(X) | (uintptr_t)(ldX * (x_f64 ? 8 : 4))) & 15) == 0 ? 1 : 0;
  const unsigned grid = (unsigned)(tiles_r * tiles_c);
  if (x_f64) {
    cudaFuncSetAttribute(apply_rows_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    apply_rows_kernel<double><<<grid, kThreads, kSmemBytes, st>>>(T, r, n, ldT, (const double*)X, m, ldX, Y, ldY,
                                                                  (int)tiles_r, vecT, vecX, lower ? 1 : 0);
  } else {
    cudaFuncSetAttribute(apply_rows_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    apply_rows_kernel<float><<<grid, kThreads, kSmemBytes, st>>>(T, r, n, ldT, (const float*)X, m, ldX, Y, ldY,
                                                                 (int)tiles_r, vecT, vecX, lower ? 1 : 0);
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace fs
