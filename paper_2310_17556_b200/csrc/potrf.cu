// potrf.cu — fp64 lower Cholesky of the damped Gram matrix W (n x n, row-major), in place.
//
// Replaces solvers.py:74-90 (scipy get_lapack_funcs('potrf') -> LAPACK dpotrf(lower=1,
// clean=1)).  Same failure contract: the first column j whose updated pivot is not strictly
// positive (or is NaN) sets the device status word to j+1 (LAPACK info), which the host maps
// to FactorizationError(pivot=j) (solvers.py:82-87).  The upper triangle is never written
// (fs_unpack_lower leaves it exactly zero: clean=1, test_solvers.py:455).
//
// Blocked right-looking algorithm with 64-wide block columns, ONE launch per block column:
//   step k, CTA (I,J) for k < J <= I:   X_I = A_Ik Linv_kk^T   (the TRSM as a GEMM with the
//   inverted diagonal block; X_J likewise), A_IJ -= X_I X_J^T, and
//     * the CTA with J == k+1 stores X_I as the panel L_Ik (double-buffered panel, copied into
//       W by the next step, so no CTA ever overwrites data another CTA of its step still reads)
//     * the CTA with I == J == k+1 factors the freshly updated diagonal block AND inverts it
//       in the same sweep (next step's Linv, also kept for the TRSV pair).
// The diagonal block: recursive 2x2 split into 32x32 halves; each half is factored by one
// warp with its rows in registers, the pivot column broadcast by shuffles, and the inverse
// accumulated alongside (right-looking forward substitution on the identity) — no barriers,
// no shared-memory round trips; the off-diagonal pieces are 32^3 GEMMs by the whole CTA.
// Every kernel first checks the status word, so a breakdown stops the remaining work.
// Deterministic: fixed operation order, no atomics.
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <mutex>

namespace fs {
namespace {

constexpr int kNB = 64;
constexpr int kThreads = 256;
constexpr int kLd = kNB + 4;   // padded smem row (68: conflict-free DMMA fragment loads)

// ---------------------------------------------------------------- block-level helpers

// ---- warp-level 32x32 kernels on smem windows (kLd-strided); lane i owns row i.  Runtime
// loops keep the code small: these run once per diagonal block, so straight-line unrolled
// code would be instruction-cache bound. ----

// X (32x32 window) = inverse of the lower-triangular window L; upper part of X set to zero.
__device__ void warp_inv32(const double* L, double* X) {
  const int lane = threadIdx.x & 31;
#pragma unroll 4
  for (int c = 0; c < 32; ++c) X[lane * kLd + c] = (lane == c) ? 1.0 : 0.0;
  __syncwarp();
#pragma unroll 1
  for (int p = 0; p < 32; ++p) {
    if (lane <= p) X[p * kLd + lane] /= L[p * kLd + p];     // finalize row p (columns c <= p)
    __syncwarp();
    if (lane > p) {
      const double lip = L[lane * kLd + p];
#pragma unroll 4
      for (int c = 0; c <= p; ++c) X[lane * kLd + c] = fma(-lip, X[p * kLd + c], X[lane * kLd + c]);
    }
    __syncwarp();
  }
}

// C[r][c] = (-)sum_p A[r][p] * B[p][c] on 32x32 windows (all 256 threads, 2x2 each).
template <bool kNegate>
__device__ void gemm32_nn(const double* A, const double* B, double* C) {
  const int r = (threadIdx.x >> 4) * 2, c = (threadIdx.x & 15) * 2;
  double s00 = 0, s01 = 0, s10 = 0, s11 = 0;
#pragma unroll 8
  for (int p = 0; p < 32; ++p) {
    const double a0 = A[r * kLd + p], a1 = A[(r + 1) * kLd + p];
    const double b0 = B[p * kLd + c], b1 = B[p * kLd + c + 1];
    s00 = fma(a0, b0, s00); s01 = fma(a0, b1, s01); s10 = fma(a1, b0, s10); s11 = fma(a1, b1, s11);
  }
  if (kNegate) { s00 = -s00; s01 = -s01; s10 = -s10; s11 = -s11; }
  C[r * kLd + c] = s00; C[r * kLd + c + 1] = s01; C[(r + 1) * kLd + c] = s10; C[(r + 1) * kLd + c + 1] = s11;
}

// X = L^-1 for the lower 64x64 L in smem (upper part of L ignored); T is scratch.
//   Linv00 = inv(L00), Linv11 = inv(L11) (warps 0 and 1 concurrently), X10 = -Linv11 L10 Linv00
__device__ void invert_64(const double (*L)[kLd], double (*X)[kLd], double (*T)[kLd]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 2) {
    const int o = 32 * warp;
    warp_inv32(&L[o][o], &X[o][o]);
    for (int c = 0; c < 32; ++c) X[lane][32 + c] = 0.0;
  }
  __syncthreads();
  gemm32_nn<false>(&L[32][0], &X[0][0], &T[0][0]);            // M = L10 Linv00
  __syncthreads();
  gemm32_nn<true>(&X[32][32], &T[0][0], &X[32][0]);           // X10 = -Linv11 M
  __syncthreads();
}

// 1/d and 1/sqrt(d) without the library's special-case subroutines: hardware approximation
// + Newton steps (~1 ulp for positive normal d; the pivot test rejects everything else).
__device__ __forceinline__ double fast_rcp(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double fast_rsqrt(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double h = 0.5 * d * y * y;            // y (1.5 - d y^2 / 2), twice
  y = fma(y, 1.5 - h, 0.0);
  h = 0.5 * d * y * y;
  return y * (1.5 - h);
}

// One warp factors the lower 32x32 window A (stride kLd) in place, A = L L^T, and writes
// X = L^-1.  Lane r keeps row r of A and column r of the inverse's right-hand side in
// registers.  Unscaled (LDL^T) sweep: step j publishes the raw column A[.][j] in a
// double-buffered smem vector (one store per lane); every lane reads the pivot and the rows
// c > j back with 16-byte broadcast loads; A[r][c] -= (A[r][j] / d_j) A[c][j] and the
// inverse's forward substitution on the unit-lower factor s[c] -= A[c][j] (x_j / d_j) share
// each load.  The sqrt scaling is applied once at the end: L[r][c] = A[r][c] / sqrt(d_c),
// X[r][c] = x~[r][c] / sqrt(d_r).  Straight-line code (no early exit, no per-lane
// predicates); entries a[c] with c > lane are never read back.  Returns the first
// non-positive (or NaN) pivot, or -1.  (A shuffle broadcast measured slower: 2 SHFL per
// double, tools/ubench/chol32_steps.cu.)
// (single-warp version, kept for tools/ubench/chol64_phases.cu and potrf_parts.cu)
[[maybe_unused]] __device__ __noinline__ int warp_chol_inv32(double* A, double* X, double (*colbuf)[32]) {
  const int lane = threadIdx.x & 31;
  double a[32], sx[32], dj[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    a[c] = (c <= lane) ? A[lane * kLd + c] : 0.0;
    sx[c] = (c == lane) ? 1.0 : 0.0;
  }
  int fail = -1;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    double* cb = colbuf[j & 1];
    cb[lane] = a[j];
    __syncwarp();
    const double d = cb[j];
    fail = (fail < 0 && !(d > 0.0)) ? j : fail;
    const double dinv = fast_rcp(d);
    dj[j] = d;                             // the sqrt scaling is formed after the sweep (off the chain)
    const double t = a[j] * dinv;
    const double y = sx[j] * dinv;
#pragma unroll
    for (int c = (j + 1) & ~1; c < 32; c += 2) {
      const double2 lc = *reinterpret_cast<const double2*>(cb + c);
      if (c > j) {
        a[c] = fma(-t, lc.x, a[c]);
        sx[c] = fma(-lc.x, y, sx[c]);
      }
      a[c + 1] = fma(-t, lc.y, a[c + 1]);
      sx[c + 1] = fma(-lc.y, y, sx[c + 1]);
    }
  }
  if (fail < 0) {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const double rsq = fast_rsqrt(dj[c]);
      A[lane * kLd + c] = (c <= lane) ? a[c] * rsq : 0.0;
      X[c * kLd + lane] = sx[c] * rsq;
    }
  }
  return fail;
}

// The same factorisation + inverse with TWO warps (threads 0-63): thread (h, r) keeps row r's
// columns c = 2i + h (i < 16) of A and of the inverse's right-hand side, so each warp issues half
// of a step's fp64 updates.  Step j: the half owning column j publishes A[.][j] and x~[.][j]
// (double-buffered), one 64-thread named barrier, then every thread updates its columns c > j.
__device__ __noinline__ int chol_inv32_2w(double* A, double* X, double (*colbuf)[32], double (*ybuf)[32]) {
  const int r = threadIdx.x & 31, h = (threadIdx.x >> 5) & 1;
  double a[16], sx[16], dj[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = 2 * i + h;
    a[i] = (c <= r) ? A[r * kLd + c] : 0.0;
    sx[i] = (c == r) ? 1.0 : 0.0;
  }
  int fail = -1;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    double* cb = colbuf[j & 1];
    double* yb = ybuf[j & 1];
    if (h == (j & 1)) {
      cb[r] = a[j >> 1];
      yb[r] = sx[j >> 1];
    }
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const double d = cb[j];
    fail = (fail < 0 && !(d > 0.0)) ? j : fail;
    const double dinv = fast_rcp(d);
    if (h == (j & 1)) dj[j >> 1] = d;
    const double t = cb[r] * dinv;
    const double y = yb[r] * dinv;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int c = 2 * i + h;
      if (2 * i + 1 > j && c > j) {          // (the first test is compile-time)
        const double lc = cb[c];
        a[i] = fma(-t, lc, a[i]);
        sx[i] = fma(-lc, y, sx[i]);
      }
    }
  }
  if (fail < 0) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int c = 2 * i + h;
      const double rsq = fast_rsqrt(dj[i]);
      A[r * kLd + c] = (c <= r) ? a[i] * rsq : 0.0;
      X[c * kLd + r] = sx[i] * rsq;
    }
  }
  return fail;
}

// C = A B^T (kNT) or A B on 32x32 windows (stride kLd) on the fp64 tensor cores (mma.sync m8n8k4 f64): warp w owns the
// two 8x8 output tiles (w/2, 2(w%2)) and (w/2, 2(w%2)+1); eight k-steps of 4.
template <bool kNT>
__device__ void gemm32_dmma(const double* A, const double* B, double acc[2][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tr = (warp >> 1) * 8, tc = (warp & 1) * 16;
  const int fr = lane >> 2, fk = lane & 3;
  acc[0][0] = acc[0][1] = acc[1][0] = acc[1][1] = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < 32; k0 += 4) {
    const double a = A[(tr + fr) * kLd + k0 + fk];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      // B operand (4 x 8, "col"): element (k, col) = kNT ? B[col][k] : B[k][col]
      const int col = tc + 8 * j + fr;
      const double b = kNT ? B[col * kLd + k0 + fk] : B[(k0 + fk) * kLd + col];
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1])
                   : "d"(a), "d"(b));
    }
  }
}

__device__ void store32_dmma(double* C, const double acc[2][2], double scale, bool accumulate) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = (warp >> 1) * 8 + (lane >> 2), c0 = (warp & 1) * 16 + 2 * (lane & 3);
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double* d = C + r * kLd + c0 + 8 * j + e;
      *d = (accumulate ? *d : 0.0) + scale * acc[j][e];
    }
}


// A (64x64 smem, identity-padded lower) = L L^T in place, X = L^-1; T scratch.  Returns the
// first failing local pivot or -1 (block-uniform).
//   [L00 0; L10 L11]:  L00 = chol(A00), L10 = A10 L00^-T, L11 = chol(A11 - L10 L10^T)
//   [X00 0; X10 X11]:  X00 = L00^-1, X11 = L11^-1, X10 = -X11 L10 X00
__device__ int chol_inv64(double (*A)[kLd], double (*X)[kLd], double (*T)[kLd]) {
  __shared__ int sfail;
  __shared__ __align__(16) double colbuf[2][32];
  __shared__ __align__(16) double ybuf[2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 2) {
    const int f = chol_inv32_2w(&A[0][0], &X[0][0], colbuf, ybuf);
    if (threadIdx.x == 0) sfail = f;
  } else if (warp == 2) {
    for (int c = 0; c < 32; ++c) X[lane][32 + c] = 0.0;
  }
  __syncthreads();
  if (sfail >= 0) return sfail;
  double acc[2][2];
  gemm32_dmma<true>(&A[32][0], &X[0][0], acc);     // L10 = A10 X00^T
  __syncthreads();
  store32_dmma(&A[32][0], acc, 1.0, false);
  __syncthreads();
  gemm32_dmma<true>(&A[32][0], &A[32][0], acc);    // A11 -= L10 L10^T (reads A10, writes A11)
  store32_dmma(&A[32][32], acc, -1.0, true);
  __syncthreads();
  if (warp < 2) {
    const int f = chol_inv32_2w(&A[32][32], &X[32][32], colbuf, ybuf);
    if (threadIdx.x == 0) sfail = f < 0 ? -1 : 32 + f;
  }
  __syncthreads();
  if (sfail >= 0) return sfail;
  gemm32_dmma<false>(&A[32][0], &X[0][0], acc);    // T = L10 X00
  store32_dmma(&T[0][0], acc, 1.0, false);
  __syncthreads();
  gemm32_dmma<false>(&X[32][32], &T[0][0], acc);   // X10 = -X11 T
  store32_dmma(&X[32][0], acc, -1.0, false);
  __syncthreads();
  return -1;
}

// C (64x64, smem) = A (64x64 smem) * B^T (64x64 smem); each thread a 4x4 sub-block.
// C (64x64) = A (64x64 smem) * B^T (64x64 smem) on the fp64 tensor cores (mma.sync m8n8k4 f64).
// Warp w owns rows [16 (w/2), +16) x cols [32 (w%2), +32): 2 x 4 tiles of 8x8.  The thread's 16
// results: acc[i][j] is element (frag_row(i), frag_col(i, j)).
FS_DEVINL int frag_row(int i) { return ((threadIdx.x >> 5) >> 1) * 16 + 8 * (i >> 1) + ((threadIdx.x & 31) >> 2); }
FS_DEVINL int frag_col(int i, int j) {
  return ((threadIdx.x >> 5) & 1) * 32 + 8 * j + 2 * (threadIdx.x & 3) + (i & 1);
}
__device__ void gemm_nt(const double (*A)[kLd], const double (*B)[kLd], double acc[4][4]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32, fr = lane >> 2, fk = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < kNB; k0 += 4) {
    double a[2], b[4];
#pragma unroll
    for (int t = 0; t < 2; ++t) a[t] = A[wr + 8 * t + fr][k0 + fk];
#pragma unroll
    for (int t = 0; t < 4; ++t) b[t] = B[wc + 8 * t + fr][k0 + fk];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int u = 0; u < 4; ++u)
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(acc[2 * t][u]), "+d"(acc[2 * t + 1][u])
                     : "d"(a[t]), "d"(b[u]));
  }
}

// 64x64 tile -> smem: all 16 loads of a thread are issued before its first store (L2
// latency once per tile, not once per element).
constexpr int kPer = kNB * kNB / kThreads;   // 16 elements per thread
__device__ void load_tile(const double* W, int64_t n, int64_t ld, int64_t r0, int64_t c0, double (*T)[kLd]) {
  double v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = u * kThreads + threadIdx.x, r = e >> 6, c = e & 63;
    const int64_t gr = r0 + r, gc = c0 + c;
    v[u] = (gr < n && gc < n) ? W[gr * ld + gc] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = u * kThreads + threadIdx.x;
    T[e >> 6][e & 63] = v[u];
  }
}

// contiguous 64x64 block (an inverted diagonal block) -> smem, batched like load_tile
__device__ void load_block64(const double* __restrict__ src, double (*T)[kLd]) {
  double v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) v[u] = src[u * kThreads + threadIdx.x];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = u * kThreads + threadIdx.x;
    T[e >> 6][e & 63] = v[u];
  }
}

// dst rows [rb, rb+64) x 64 columns <- src (row-major, 64 per row), batched like load_tile
__device__ void copy_panel(double* __restrict__ dst, int64_t ld, const double* __restrict__ src, int64_t rb,
                           int64_t n) {
  double v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = u * kThreads + threadIdx.x;
    const int64_t gr = rb + (e >> 6);
    v[u] = gr < n ? src[gr * kNB + (e & 63)] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = u * kThreads + threadIdx.x;
    const int64_t gr = rb + (e >> 6);
    if (gr < n) dst[gr * ld + (e & 63)] = v[u];
  }
}

__device__ void tile_coords(int t, int& I, int& J) {  // lower tiles in row-major order
  int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  I = i;
  J = t - i * (i + 1) / 2;
}

// Factor diagonal block kk of W (already fully updated) in place and store its inverse in
// Linv[kk] (dense 64x64, identity-padded).  A, X, T: three smem tiles.
#ifdef FS_POTRF_TRACE
__device__ unsigned long long g_potrf_trace[128];
#define POTRF_MARK(i)                                                                              \
  do {                                                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                                     \
      unsigned long long t_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
      g_potrf_trace[(i)] = t_;                                                                     \
    }                                                                                              \
  } while (0)
#else
#define POTRF_MARK(i) \
  do {                \
  } while (0)
#endif

__device__ void factor_diag(double* W, int64_t n, int64_t ld, int kk, int64_t* status, double* Linv,
                            double (*A)[kLd], double (*X)[kLd], double (*T)[kLd], bool preloaded,
                            bool tr = false) {
  const int64_t r0 = (int64_t)kk * kNB;
  const int b = (int)(n - r0 < kNB ? n - r0 : kNB);
  if (tr) POTRF_MARK(85);
  if (!preloaded) load_tile(W, n, ld, r0, r0, A);
  __syncthreads();
  // chol_inv64 reads only the lower triangle (its GEMMs touch A10, A11 and the factors), so only
  // a partial last block needs padding: identity rows r >= b
  if (b < kNB) {
    for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) {
      const int r = e >> 6, c = e & 63;
      if (r >= b && c <= r) A[r][c] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
  }
  if (tr) POTRF_MARK(86);
  const int f = chol_inv64(A, X, T);
  if (tr) POTRF_MARK(87);
  if (f >= 0) {
    if (threadIdx.x == 0) *status = r0 + f + 1;
    return;
  }
  double* li = Linv + (size_t)kk * kNB * kNB;
  for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) {
    const int r = e >> 6, c = e & 63;
    if (r < b && c <= r) W[(r0 + r) * ld + r0 + c] = A[r][c];
    li[e] = X[r][c];
  }
}

// ---------------------------------------------------------------- kernels

__global__ void unpack_lower_kernel(const double* __restrict__ Gp, int64_t n, double add_diag,
                                    double* __restrict__ W, int64_t ldW) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (j >= n) return;
  double v = 0.0;
  if (j <= i) v = Gp[i * (i + 1) / 2 + j] + (i == j ? add_diag : 0.0);
  W[i * ldW + j] = v;
}

constexpr size_t kTileSmem = sizeof(double) * kNB * kLd;

__global__ void __launch_bounds__(kThreads)
potrf_first_kernel(double* W, int64_t n, int64_t ld, double* Linv, int64_t* status) {
  extern __shared__ double dsm[];
  double (*A)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm);
  double (*X)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + kNB * kLd);
  double (*T)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + 2 * kNB * kLd);
  if (*(volatile int64_t*)status != 0) return;
  factor_diag(W, n, ld, 0, status, Linv, A, X, T, false);
}

// out[o] = sum_k M(o, k) x[k] for a 64 x 64 block (M(o, k) = M[o * ld + k], or M[k * ld + o] when
// kTrans), all 256 threads: 4 threads per output, 16 unrolled independent loads each, shuffle
// reduction (fixed order).  x in shared memory; out written by the q == 0 lane (if out != null).
template <bool kTrans>
__device__ double gemv64(const double* __restrict__ M, int64_t ld, const double* x, int rows_valid) {
  const int o = threadIdx.x >> 2, q = threadIdx.x & 3;
  double v[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int k = q * 16 + t;
    v[t] = (kTrans ? k : o) < rows_valid ? (kTrans ? M[(int64_t)k * ld + o] : M[(int64_t)o * ld + k]) : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int t = 0; t < 16; ++t) acc = fma(v[t], x[q * 16 + t], acc);
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  return acc;                                   // valid in the q == 0 lane of each output
}

// Step k, trailing tile `tile` = (I, J), k < J <= I < nb, indexed relative to k+1 (tile 0 is the
// next diagonal block, whose CTA also factors it).
__device__ void step_tile(double* W, int64_t n, int64_t ld, int k, double* Linv, double* panel0, double* panel1,
                          int64_t* status, int tile, double* dsm, double* ut = nullptr, double* tb = nullptr) {
  double (*Lk)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm);              // Linv_kk, later scratch
  double (*XI)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + kNB * kLd);
  double (*XJ)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + 2 * kNB * kLd);
  int I, J;
  tile_coords(tile, I, J);
  I += k + 1;
  J += k + 1;
  const int64_t kc = (int64_t)k * kNB, rI = (int64_t)I * kNB, rJ = (int64_t)J * kNB;
  double* pan_cur = (k & 1) ? panel1 : panel0;     // this step's panel L_{.,k}
  double* pan_prev = (k & 1) ? panel0 : panel1;    // previous step's panel L_{.,k-1}
  // materialise the previous panel L_{.,k-1} into W (nobody reads W column k-1 any more):
  // row block I by the CTA (I, k+1); row block k by the diagonal CTA (k+1, k+1)
  const bool tr = (tile == 0 && k == 5);
  if (tr) POTRF_MARK(80);
  if (J == k + 1 && k >= 1) {
    copy_panel(W + (kc - kNB), ld, pan_prev, rI, n);
    if (I == k + 1) copy_panel(W + (kc - kNB), ld, pan_prev, kc, n);
  }
  if (tr) POTRF_MARK(81);
  {
    // Linv_kk, A_Ik and A_Jk: all 48 loads of a thread in flight before the first store (one L2
    // round trip instead of three)
    const double* li = Linv + (size_t)k * kNB * kNB;
    double vl[kPer], vi[kPer], vj[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = u * kThreads + threadIdx.x, r = e >> 6, c = e & 63;
      vl[u] = li[e];
      vi[u] = (rI + r < n && kc + c < n) ? W[(rI + r) * ld + kc + c] : 0.0;
      vj[u] = (I != J && rJ + r < n && kc + c < n) ? W[(rJ + r) * ld + kc + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = u * kThreads + threadIdx.x, r = e >> 6, c = e & 63;
      Lk[r][c] = vl[u];
      XI[r][c] = vi[u];
      if (I != J) XJ[r][c] = vj[u];
    }
  }
  __syncthreads();
  if (tr) POTRF_MARK(82);
  // X_I = A_Ik Linv_kk^T, X_J = A_Jk Linv_kk^T (the panel TRSM as GEMMs)
  double accI[4][4], accJ[4][4];
  gemm_nt(XI, Lk, accI);
  if (I != J) gemm_nt(XJ, Lk, accJ);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      XI[frag_row(i)][frag_col(i, j)] = accI[i][j];
      if (I != J) XJ[frag_row(i)][frag_col(i, j)] = accJ[i][j];
    }
  __syncthreads();
  if (tr) POTRF_MARK(83);
  if (J == k + 1) {   // store the panel L_Ik
    for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) {
      const int r = e >> 6, c = e & 63;
      const int64_t gr = rI + r;
      if (gr < n) pan_cur[gr * kNB + c] = XI[r][c];
    }
    if (ut) {
      // fused forward substitution (L t = u, right-looking): t_k = Linv_kk ut_k (ut_k is final:
      // its last update came from step k-1), then ut_I -= L_Ik t_k for this CTA's row block
      __shared__ double uk[kNB], tk[kNB];
      if (threadIdx.x < kNB) uk[threadIdx.x] = (kc + threadIdx.x < n) ? ut[kc + threadIdx.x] : 0.0;
      __syncthreads();
      {
        const double acc = gemv64<false>(&Lk[0][0], kLd, uk, kNB);
        const int o = threadIdx.x >> 2;
        if ((threadIdx.x & 3) == 0) {
          tk[o] = acc;
          if (I == k + 1 && kc + o < n) tb[kc + o] = acc;   // the diagonal CTA records t_k
        }
      }
      __syncthreads();
      {
        const double acc = gemv64<false>(&XI[0][0], kLd, tk, kNB);
        const int o = threadIdx.x >> 2;
        if ((threadIdx.x & 3) == 0 && rI + o < n) ut[rI + o] -= acc;
      }
    }
  }
  if (tr) POTRF_MARK(84);
  // A_IJ -= X_I X_J^T (old values loaded up front, the GEMM overlaps their latency)
  double old[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gi = rI + frag_row(i), gj = rJ + frag_col(i, j);
      old[i][j] = (gi < n && gj <= gi) ? W[gi * ld + gj] : 0.0;
    }
  double acc[4][4];
  gemm_nt(XI, (I != J) ? XJ : XI, acc);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gi = rI + frag_row(i), gj = rJ + frag_col(i, j);
      acc[i][j] = old[i][j] - acc[i][j];
      if (gi < n && gj <= gi) W[gi * ld + gj] = acc[i][j];
    }
  if (tr) POTRF_MARK(85);
  if (I == J && I == k + 1) {
    // (block-uniform branch) the updated diagonal tile goes straight into smem for its factor
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) Lk[frag_row(i)][frag_col(i, j)] = acc[i][j];
    factor_diag(W, n, ld, I, status, Linv, Lk, XI, XJ, true, tr);
  }
  if (tr) POTRF_MARK(89);
}

__global__ void __launch_bounds__(kThreads)
potrf_step_kernel(double* W, int64_t n, int64_t ld, int k, double* Linv, double* panel0, double* panel1,
                  int64_t* status) {
  extern __shared__ double dsm[];
  if (*(volatile int64_t*)status != 0) return;
  step_tile(W, n, ld, k, Linv, panel0, panel1, status, blockIdx.x, dsm);
}

// ---- two-phase steps (large n: the step-0 trailing tiles outnumber the CTAs) ----
// The one-phase step recomputes the panel product X_I = A_Ik Linv_kk^T in every tile (I, J) that
// needs it (three 64^3 products per tile).  With many tiles per CTA it pays to form each X_I once:
// phase A writes L_{I,k} = X_I in place into W (each row block by one CTA; CTA 0 forms X_{k+1}
// on its critical path) plus the forward substitution ut_I -= X_I t_k; a grid barrier; phase B
// updates every trailing tile with one product A_IJ -= X_I X_J^T from W's column block k.
__device__ void panel_row_inplace(double* W, int64_t n, int64_t ld, int k, int I, const double* Linv, double* dsm,
                                  double* ut, double* tb, bool record_t) {
  double (*Lk)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm);
  double (*XI)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + kNB * kLd);
  const int64_t kc = (int64_t)k * kNB, rI = (int64_t)I * kNB;
  {
    const double* li = Linv + (size_t)k * kNB * kNB;
    double vl[kPer], vi[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = u * kThreads + threadIdx.x, r = e >> 6, c = e & 63;
      vl[u] = li[e];
      vi[u] = (rI + r < n && kc + c < n) ? W[(rI + r) * ld + kc + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = u * kThreads + threadIdx.x, r = e >> 6, c = e & 63;
      Lk[r][c] = vl[u];
      XI[r][c] = vi[u];
    }
  }
  __syncthreads();
  double acc[4][4];
  gemm_nt(XI, Lk, acc);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      XI[frag_row(i)][frag_col(i, j)] = acc[i][j];
      const int64_t gi = rI + frag_row(i);
      if (gi < n) W[gi * ld + kc + frag_col(i, j)] = acc[i][j];
    }
  __syncthreads();
  if (ut) {   // t_k = Linv_kk ut_k (ut_k final since step k-1), then ut_I -= L_Ik t_k
    __shared__ double uk[kNB], tk[kNB];
    if (threadIdx.x < kNB) uk[threadIdx.x] = (kc + threadIdx.x < n) ? ut[kc + threadIdx.x] : 0.0;
    __syncthreads();
    {
      const double a = gemv64<false>(&Lk[0][0], kLd, uk, kNB);
      const int o = threadIdx.x >> 2;
      if ((threadIdx.x & 3) == 0) {
        tk[o] = a;
        if (record_t && kc + o < n) tb[kc + o] = a;
      }
    }
    __syncthreads();
    if (I < (n + kNB - 1) / kNB) {
      const double a = gemv64<false>(&XI[0][0], kLd, tk, kNB);
      const int o = threadIdx.x >> 2;
      if ((threadIdx.x & 3) == 0 && rI + o < n) ut[rI + o] -= a;
    }
  }
}

// A_IJ -= X_I X_J^T with X_I = L_{I,k}, X_J = L_{J,k} from W's column block k (phase B)
__device__ void update_tile(double* W, int64_t n, int64_t ld, int k, int I, int J, double* dsm) {
  double (*XI)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + kNB * kLd);
  double (*XJ)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + 2 * kNB * kLd);
  const int64_t kc = (int64_t)k * kNB, rI = (int64_t)I * kNB, rJ = (int64_t)J * kNB;
  {
    double vi[kPer], vj[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = u * kThreads + threadIdx.x, r = e >> 6, c = e & 63;
      vi[u] = (rI + r < n) ? W[(rI + r) * ld + kc + c] : 0.0;
      vj[u] = (I != J && rJ + r < n) ? W[(rJ + r) * ld + kc + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = u * kThreads + threadIdx.x, r = e >> 6, c = e & 63;
      XI[r][c] = vi[u];
      if (I != J) XJ[r][c] = vj[u];
    }
  }
  double old[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gi = rI + frag_row(i), gj = rJ + frag_col(i, j);
      old[i][j] = (gi < n && gj <= gi) ? W[gi * ld + gj] : 0.0;
    }
  __syncthreads();
  double acc[4][4];
  gemm_nt(XI, (I != J) ? XJ : XI, acc);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gi = rI + frag_row(i), gj = rJ + frag_col(i, j);
      if (gi < n && gj <= gi) W[gi * ld + gj] = old[i][j] - acc[i][j];
    }
}

// The persistent kernel's step k splits tile 0 = (k+1, k+1) in two:
//  * critical_tile (CTA 0, the step's critical path): X = A_{k+1,k} Linv_kk^T with Linv_kk still in
//    smem from CTA 0's own previous factorisation, the diagonal update A -= X X^T straight into
//    smem, then the factorisation + inversion of block k+1 (kept in smem for step k+1);
//  * aux_tile (the last CTA): everything else tile 0 used to do — copy the previous panel's rows
//    {k, k+1} into W, recompute X, store the panel rows of block k+1, and the fused forward
//    substitution for row block k+1 (t_k = Linv_kk ut_k, ut_{k+1} -= L_{k+1,k} t_k).
// (tools/ubench/potrf_trace.cu: the old tile 0 took 32 us per step, 12 of them off the chain.)
__device__ void critical_tile(double* W, int64_t n, int64_t ld, int k, double* Linv, int64_t* status, double* dsm,
                              double (*P)[kLd], bool store_panel = false) {
  double (*A)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm);
  double (*X)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + kNB * kLd);
  double (*T)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + 2 * kNB * kLd);
  const int I = k + 1;
  const int64_t kc = (int64_t)k * kNB, rI = (int64_t)I * kNB;
  const bool tr = (k == 5);
  if (tr) POTRF_MARK(80);
  load_tile(W, n, ld, rI, kc, X);                  // A_{I,k}
  double old[4][4];                                // the diagonal tile's current lower values
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gi = rI + frag_row(i), gj = rI + frag_col(i, j);
      old[i][j] = (gi < n && gj <= gi) ? W[gi * ld + gj] : 0.0;
    }
  __syncthreads();
  if (tr) POTRF_MARK(81);
  double acc[4][4];
  gemm_nt(X, P, acc);                              // X_I = A_Ik Linv_kk^T
  __syncthreads();
  if (tr) POTRF_MARK(82);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      X[frag_row(i)][frag_col(i, j)] = acc[i][j];
      const int64_t gi = rI + frag_row(i);         // two-phase mode: L_{I,k} = X_I straight into W
      if (store_panel && gi < n) W[gi * ld + kc + frag_col(i, j)] = acc[i][j];
    }
  __syncthreads();
  if (tr) POTRF_MARK(83);
  gemm_nt(X, X, acc);                              // A_II -= X_I X_I^T
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) A[frag_row(i)][frag_col(i, j)] = old[i][j] - acc[i][j];
  if (tr) POTRF_MARK(84);
  factor_diag(W, n, ld, I, status, Linv, A, P, T, true, tr);   // L_II -> W, Linv_II -> Linv and P
  if (tr) POTRF_MARK(88);
  if (tr) POTRF_MARK(89);
}

__device__ void aux_tile(double* W, int64_t n, int64_t ld, int k, const double* Linv, double* panel0,
                         double* panel1, double* dsm, double* ut, double* tb) {
  double (*Lk)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm);
  double (*XI)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + kNB * kLd);
  const int I = k + 1;
  const int64_t kc = (int64_t)k * kNB, rI = (int64_t)I * kNB;
  double* pan_cur = (k & 1) ? panel1 : panel0;
  const double* pan_prev = (k & 1) ? panel0 : panel1;
  if (k >= 1) {                                    // previous panel L_{.,k-1}: rows of blocks k+1, k
    copy_panel(W + (kc - kNB), ld, pan_prev, rI, n);
    copy_panel(W + (kc - kNB), ld, pan_prev, kc, n);
  }
  load_block64(Linv + (size_t)k * kNB * kNB, Lk);
  load_tile(W, n, ld, rI, kc, XI);
  __syncthreads();
  double acc[4][4];
  gemm_nt(XI, Lk, acc);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) XI[frag_row(i)][frag_col(i, j)] = acc[i][j];
  __syncthreads();
  for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) {   // the panel rows L_{I,k}
    const int r = e >> 6, c = e & 63;
    const int64_t gr = rI + r;
    if (gr < n) pan_cur[gr * kNB + c] = XI[r][c];
  }
  if (ut) {
    __shared__ double uk[kNB], tk[kNB];
    if (threadIdx.x < kNB) uk[threadIdx.x] = (kc + threadIdx.x < n) ? ut[kc + threadIdx.x] : 0.0;
    __syncthreads();
    {
      const double a = gemv64<false>(&Lk[0][0], kLd, uk, kNB);
      const int o = threadIdx.x >> 2;
      if ((threadIdx.x & 3) == 0) {
        tk[o] = a;
        if (kc + o < n) tb[kc + o] = a;           // t_k
      }
    }
    __syncthreads();
    {
      const double a = gemv64<false>(&XI[0][0], kLd, tk, kNB);
      const int o = threadIdx.x >> 2;
      if ((threadIdx.x & 3) == 0 && rI + o < n) ut[rI + o] -= a;
    }
  }
}

// grid barrier on a monotonic arrival counter (cooperative launch: all CTAs co-resident; ctl is
// zeroed before the launch): thread 0 adds 1 with release semantics and polls with acquire loads
// until this generation's count (target += gridDim.x per call) — one L2 round trip per CTA
__device__ void grid_barrier(unsigned* count, unsigned& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// The whole factorisation in one persistent cooperative kernel: CTA 0 factors block 0, then
// every step's trailing tiles are spread over the CTAs (tile 0 — the next diagonal block and its
// factorisation, the critical path — always on CTA 0, whose instruction cache stays warm) with
// one grid barrier per step instead of a kernel boundary.  Ends with the last panel's copy.
__global__ void __launch_bounds__(kThreads, 1)
potrf_persistent_kernel(double* W, int64_t n, int64_t ld, double* Linv, double* panel0, double* panel1,
                        int64_t* status, unsigned* ctl, const double* __restrict__ u, double* ut, double* tb,
                        double* __restrict__ z, int skip_bwd) {
  extern __shared__ double dsm[];
  unsigned bar_target = 0;
  double (*P)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + 3 * kNB * kLd);   // CTA 0: Linv_kk
  const int nb = (int)((n + kNB - 1) / kNB);
  if (u)                                                  // working right-hand side of L t = u
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
      ut[e] = u[e];
  POTRF_MARK(0);
  if (blockIdx.x == 0 && *(volatile int64_t*)status == 0) {
    double (*A)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm);
    double (*T)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + 2 * kNB * kLd);
    factor_diag(W, n, ld, 0, status, Linv, A, P, T, false);   // Linv_00 stays in P
  }
  POTRF_MARK(1);
  grid_barrier(ctl, bar_target);
  POTRF_MARK(2);
  int k = 0;
  const int G = gridDim.x;
  // two-phase steps once the first step's trailing tiles reach ~4 per CTA (n >~ 2200; measured:
  // n = 2048 1.04 vs 1.11 ms one- vs two-phase, n = 4096 6.3 -> 5.3 ms, n = 8192 60 -> 29 ms)
  const bool two_phase = (nb - 1) * nb / 2 > 4 * G;
  for (; k + 1 < nb; ++k) {
    if (*(volatile int64_t*)status != 0) break;          // uniform: read after the barrier
    const int t = nb - k - 1, tiles = t * (t + 1) / 2;
    if (two_phase) {
      // phase A: CTA 0 the critical diagonal (X_{k+1} in place), the others the panel rows k+2..
      if (blockIdx.x == 0) {
        __syncthreads();
        critical_tile(W, n, ld, k, Linv, status, dsm, P, true);
      }
      const int first = G > 1 ? (int)blockIdx.x - 1 : 0, stride = G > 1 ? G - 1 : 1;
      if (G == 1 || blockIdx.x >= 1)
        for (int I = k + 2 + first; I < nb; I += stride) {
          __syncthreads();
          panel_row_inplace(W, n, ld, k, I, Linv, dsm, u ? ut : nullptr, tb, I == k + 2);
        }
      if (u && k + 2 >= nb && blockIdx.x == G - 1) {   // no panel rows left: t_k still goes to tb
        __syncthreads();
        __shared__ double uk2[kNB];
        const int64_t kc = (int64_t)k * kNB;
        if (threadIdx.x < kNB) uk2[threadIdx.x] = (kc + threadIdx.x < n) ? ut[kc + threadIdx.x] : 0.0;
        __syncthreads();
        const double a = gemv64<false>(Linv + (size_t)k * kNB * kNB, kNB, uk2, kNB);
        const int o = threadIdx.x >> 2;
        if ((threadIdx.x & 3) == 0 && kc + o < n) tb[kc + o] = a;
      }
      grid_barrier(ctl, bar_target);
      // phase B: every trailing tile but the factored diagonal, one product each; the forward
      // substitution of row block k+1 (its panel rows came from CTA 0)
      for (int tile = 1 + (int)blockIdx.x; tile < tiles; tile += G) {
        __syncthreads();
        int I, J;
        tile_coords(tile, I, J);
        update_tile(W, n, ld, k, I + k + 1, J + k + 1, dsm);
      }
      if (u && blockIdx.x == (G > 1 ? G - 1 : 0)) {
        __syncthreads();
        __shared__ double xk[kNB];
        const int64_t kc = (int64_t)k * kNB, r1 = (int64_t)(k + 1) * kNB;
        if (threadIdx.x < kNB) xk[threadIdx.x] = (kc + threadIdx.x < n) ? tb[kc + threadIdx.x] : 0.0;
        __syncthreads();
        const int valid = (int)(n - r1 < kNB ? n - r1 : kNB);
        const double a = gemv64<false>(W + r1 * ld + kc, ld, xk, valid);   // rows r1.. of L_{.,k}
        const int o = threadIdx.x >> 2;
        if ((threadIdx.x & 3) == 0 && o < valid) ut[r1 + o] -= a;
      }
      grid_barrier(ctl, bar_target);
      continue;
    }
    if (blockIdx.x == 0) {
      __syncthreads();
      critical_tile(W, n, ld, k, Linv, status, dsm, P);
    }
    if (blockIdx.x == G - 1) {
      __syncthreads();
      aux_tile(W, n, ld, k, Linv, panel0, panel1, dsm, u ? ut : nullptr, tb);
    }
    // tiles 1.. over CTAs 1..G-1 (CTA 0 keeps to the critical path when G > 1)
    const int first = G > 1 ? (int)blockIdx.x : (int)blockIdx.x + 1, stride = G > 1 ? G - 1 : 1;
    if (G == 1 || blockIdx.x >= 1)
      for (int tile = first; tile < tiles; tile += stride) {
        __syncthreads();
        step_tile(W, n, ld, k, Linv, panel0, panel1, status, tile, dsm, u ? ut : nullptr, tb);
      }
    if (k < 30) POTRF_MARK(3 + 2 * k);
    grid_barrier(ctl, bar_target);
    if (k < 30) POTRF_MARK(4 + 2 * k);
  }
  POTRF_MARK(70);
  const bool solve = u && *(volatile int64_t*)status == 0;
  if (!two_phase && nb >= 2 && *(volatile int64_t*)status == 0) {      // last panel L_{., nb-2} into W
    const int kk = nb - 2;
    const int64_t kc = (int64_t)kk * kNB;
    const double* panel = (kk & 1) ? panel1 : panel0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (n - kc - kNB) * kNB;
         e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t gr = kc + kNB + e / kNB, c = e % kNB;
      W[gr * ld + kc + c] = panel[gr * kNB + c];
    }
  }
  if (!solve) return;
  __shared__ double zb[kNB], xb[kNB];
  if (blockIdx.x == 0) {
    // last block of the forward solve: t_{nb-1} = Linv ut_{nb-1}
    const int64_t kc = (int64_t)(nb - 1) * kNB;
    if (threadIdx.x < kNB) xb[threadIdx.x] = (kc + threadIdx.x < n) ? ut[kc + threadIdx.x] : 0.0;
    __syncthreads();
    const double acc = gemv64<false>(Linv + (size_t)(nb - 1) * kNB * kNB, kNB, xb, kNB);
    const int o = threadIdx.x >> 2;
    if ((threadIdx.x & 3) == 0 && kc + o < n) tb[kc + o] = acc;
  }
  POTRF_MARK(71);
  if (skip_bwd) return;   // the backward half runs on the TRSV cluster from tb (trsv_backward_cluster)
  grid_barrier(ctl, bar_target);                             // tb = t complete, W holds all of L
  POTRF_MARK(72);
  // backward solve L^T z = t, left-looking per block with release/acquire flags instead of a grid
  // barrier per block: CTA c owns block c (c = blockIdx.x + i*G, taken in decreasing order) and
  // applies tb_c -= L_Bc^T z_B as each z_B (B > c) is published, then z_c = Linv_cc^T tb_c and
  // publishes it.  The L_Bc tile is loaded before waiting for z_B, so a link of the dependency
  // chain costs a flag round trip + a 64-vector load (tools/ubench/potrf_trace.cu: 85 -> ~30 us
  // at n = 1024 against the barrier-per-block version).
  unsigned* zflag = reinterpret_cast<unsigned*>(tb + n);
  const int o = threadIdx.x >> 2, q = threadIdx.x & 3;
  int c_top = (int)blockIdx.x;
  while (c_top + (int)gridDim.x < nb) c_top += gridDim.x;
  for (int c = c_top; c >= 0 && c < nb; c -= gridDim.x) {
    const int64_t rC = (int64_t)c * kNB;
    if (threadIdx.x < kNB) xb[threadIdx.x] = (rC + threadIdx.x < n) ? __ldcg(tb + rC + threadIdx.x) : 0.0;
    for (int B = nb - 1; B > c; --B) {
      const int64_t rB = (int64_t)B * kNB;
      const int valid = (int)(n - rB < kNB ? n - rB : kNB);
      double v[16];                                       // L_Bc^T: element (o, k) = W[rB + k][rC + o]
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int k = q * 16 + t;
        v[t] = k < valid ? W[(rB + k) * ld + rC + o] : 0.0;
      }
      if (threadIdx.x == 0) {
        unsigned f;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(zflag + B) : "memory");
        } while (f == 0);
      }
      __syncthreads();
      if (threadIdx.x < kNB) zb[threadIdx.x] = (rB + threadIdx.x < n) ? __ldcg(z + rB + threadIdx.x) : 0.0;
      __syncthreads();
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < 16; ++t) acc = fma(v[t], zb[q * 16 + t], acc);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (q == 0) xb[o] -= acc;
    }
    __syncthreads();
    const double acc = gemv64<true>(Linv + (size_t)c * kNB * kNB, kNB, xb, kNB);   // Linv_cc^T tb_c
    if (q == 0 && rC + o < n) z[rC + o] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(zflag + c), "r"(1u) : "memory");
    }
  }
  POTRF_MARK(73);
}

__global__ void potrf_tail_kernel(double* W, int64_t n, int64_t ld, int k, const double* panel,
                                  const int64_t* status) {
  // copy the last panel L_{.,k} (rows below block k) into W
  if (*(volatile const int64_t*)status != 0) return;
  const int64_t kc = (int64_t)k * kNB;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (n - kc - kNB) * kNB;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gr = kc + kNB + e / kNB, c = e % kNB;
    W[gr * ld + kc + c] = panel[gr * kNB + c];
  }
}

// Linv[B] = inverse of the diagonal block B of a given lower factor L (for standalone TRSV).
__global__ void __launch_bounds__(kThreads)
invert_diag_blocks_kernel(const double* L, int64_t n, int64_t ld, double* Linv) {
  extern __shared__ double dsm[];
  double (*A)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm);
  double (*X)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + kNB * kLd);
  double (*T)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + 2 * kNB * kLd);
  const int64_t r0 = (int64_t)blockIdx.x * kNB;
  const int b = (int)(n - r0 < kNB ? n - r0 : kNB);
  load_tile(L, n, ld, r0, r0, A);
  __syncthreads();
  for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) {
    const int r = e / kNB, c = e % kNB;
    if (c > r) A[r][c] = 0.0;
    else if (r >= b) A[r][c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  invert_64(A, X, T);
  for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) Linv[(size_t)blockIdx.x * kNB * kNB + e] = X[e / kNB][e % kNB];
}

}  // namespace

cudaError_t invert_diag_blocks(const double* L, int64_t n, int64_t ldL, double* scratch, cudaStream_t st,
                               int* launches) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(invert_diag_blocks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(3 * kTileSmem));
    attr = true;
  }
  const int nb = (int)((n + kNB - 1) / kNB);
  invert_diag_blocks_kernel<<<nb, kThreads, 3 * kTileSmem, st>>>(L, n, ldL, scratch);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

int64_t potrf_scratch_doubles(int64_t n) {
  const int64_t nb = (n + kNB - 1) / kNB;
  return potrf_trsv_flags_offset(n) + nb /* trsv_pair's 2 nb block flags */ + 1 /* blocked: sub status */;
}

int64_t potrf_trsv_flags_offset(int64_t n) {
  const int64_t nb = (n + kNB - 1) / kNB;
  return nb * kNB * kNB /* Linv */ + 2 * n * kNB /* panels */ + 1 /* grid barrier words */ + 2 * n /* solve */ +
         (nb + 1) / 2 /* backward-solve block flags */;
}

cudaError_t unpack_lower(const double* Gp, int64_t n, double add_diag, double* W, int64_t ldW,
                         cudaStream_t st, int* launches) {
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)n);
  unpack_lower_kernel<<<grid, 256, 0, st>>>(Gp, n, add_diag, W, ldW);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- blocked path (large n)
// Right-looking with 256-wide block columns: the diagonal block by the persistent kernel above
// (its four 64-block inverses land in Linv at their global positions), the panel below as a
// GEMM-form TRSM (potrf_panel_kernel), the trailing matrix by the 128 x 128 DMMA tiles of the
// Gram (syrk_dmma_trail, K = 256): the n^3/3 flops run in large tensor-core tiles instead of the
// persistent kernel's 64^3 tile updates with a grid barrier per 64 columns.
constexpr int kNB2 = 256;
constexpr size_t kPanelSmem = 5 * kTileSmem;

// rows [r0, r0 + 64) of the panel below diagonal block [k0, k0 + 64 nbk):
//   X_b = (A_b - sum_{c<b} X_c L_bc^T) Linv_bb^T,  b = 0 .. nbk-1 (4 threads x 4 x 4 DMMA results)
__global__ void __launch_bounds__(kThreads)
potrf_panel_kernel(double* W, int64_t n, int64_t ld, int64_t k0, int nbk, const double* __restrict__ Linv,
                   const int64_t* status) {
  if (*(volatile const int64_t*)status != 0) return;
  extern __shared__ double psm[];
  double (*X[3])[kLd];
  for (int c = 0; c < 3; ++c) X[c] = reinterpret_cast<double (*)[kLd]>(psm + c * kNB * kLd);
  double (*T)[kLd] = reinterpret_cast<double (*)[kLd]>(psm + 3 * kNB * kLd);
  double (*B)[kLd] = reinterpret_cast<double (*)[kLd]>(psm + 4 * kNB * kLd);
  const int64_t r0 = k0 + (int64_t)nbk * kNB + (int64_t)blockIdx.x * kNB;
  for (int b = 0; b < nbk; ++b) {
    const int64_t cb = k0 + (int64_t)b * kNB;
    load_tile(W, n, ld, r0, cb, T);
    double sub[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) sub[i][j] = 0.0;
    for (int c = 0; c < b; ++c) {
      __syncthreads();                          // B free (previous product done)
      load_tile(W, n, ld, cb, k0 + (int64_t)c * kNB, B);   // L_bc
      __syncthreads();
      double acc[4][4];
      gemm_nt(X[c], B, acc);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sub[i][j] += acc[i][j];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) T[frag_row(i)][frag_col(i, j)] -= sub[i][j];
    load_block64(Linv + (size_t)(k0 / kNB + b) * kNB * kNB, B);
    __syncthreads();
    double acc[4][4];
    gemm_nt(T, B, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = frag_row(i), c = frag_col(i, j);
        if (b < 3) X[b][r][c] = acc[i][j];
        if (r0 + r < n) W[(r0 + r) * ld + cb + c] = acc[i][j];
      }
  }
}

// the diagonal block's local status (1-based column) -> the global word, first failure only
__global__ void potrf_status_fixup_kernel(int64_t* status, const int64_t* sub, int64_t k0) {
  const int64_t sv = *(volatile const int64_t*)sub;
  if (*status == 0 && sv != 0) *status = sv + k0;
}

int64_t potrf_blocked_min_n() {
  // measured (tools/large_fit.py): n = 4096 persistent 3.10 vs blocked 3.44 ms; n = 8192 15.7 vs
  // 13.7; n = 16384 107 vs 81
  static const int64_t v = getenv("FS_POTRF_BLOCKED_MINN") ? atoll(getenv("FS_POTRF_BLOCKED_MINN")) : 6144;
  return v;
}

// One-step look-ahead on two streams forked from the caller's: a high-priority stream runs the
// critical path — strip k+1 -= P_k P_k(strip)^T, then the diagonal factor and panel of block
// column k+1 — while a low-priority stream applies the rest of step k's update (columns beyond
// strip k+1), so the latency-bound diagonal/panel kernels hide under the big trailing update.
// The next strip update waits for that rest (it touches the same columns).  Enqueue is
// serialised by a mutex (the streams and events are shared per process).
struct BlockedStreams {
  cudaStream_t hp = nullptr, lp = nullptr;
  static constexpr int kEv = 2 * 160;            // n <= 40960
  cudaEvent_t ev[kEv] = {};
  cudaEvent_t fork = nullptr;
  bool ok = false;
};

BlockedStreams& blocked_streams() {
  static BlockedStreams b;
  static bool init = false;
  if (!init) {
    init = true;
    int lo = 0, hi = 0;
    bool ok = cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess &&
              cudaStreamCreateWithPriority(&b.hp, cudaStreamNonBlocking, hi) == cudaSuccess &&
              cudaStreamCreateWithPriority(&b.lp, cudaStreamNonBlocking, lo) == cudaSuccess &&
              cudaEventCreateWithFlags(&b.fork, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < BlockedStreams::kEv; ++i)
      ok = cudaEventCreateWithFlags(&b.ev[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) cudaGetLastError();
    b.ok = ok;
  }
  return b;
}

cudaError_t potrf_blocked(double* W, int64_t n, int64_t ldW, int64_t* d_status, double* scratch, cudaStream_t st,
                          int* launches) {
  const int64_t nb = (n + kNB - 1) / kNB;
  double* Linv = scratch;
  int64_t* sub = reinterpret_cast<int64_t*>(scratch + potrf_trsv_flags_offset(n) + nb);
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(potrf_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kPanelSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  BlockedStreams& bs = blocked_streams();
  const int64_t steps = (n + kNB2 - 1) / kNB2;
  const bool ahead = bs.ok && 2 * steps <= BlockedStreams::kEv && getenv("FS_POTRF_LOOKAHEAD") == nullptr;
  cudaStream_t hp = ahead ? bs.hp : st, lp = ahead ? bs.lp : st;
  cudaError_t e = cudaSuccess;
  if (ahead) {
    e = cudaEventRecord(bs.fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hp, bs.fork, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(lp, bs.fork, 0);
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(sub, 0, sizeof(int64_t), hp);
  // diagonal block + panel of block column k (on hp)
  auto diag_panel = [&](int64_t k0) -> cudaError_t {
    const int64_t w = std::min<int64_t>(kNB2, n - k0);
    // the diagonal block's working space follows its Linv blocks: it overwrites only Linv
    // blocks of later diagonal blocks (written when those are factored) and the unused panels
    cudaError_t r = potrf_lower(W + k0 * ldW + k0, w, ldW, sub, Linv + (k0 / kNB) * kNB * kNB, hp, launches, nullptr,
                                nullptr, nullptr);
    if (r != cudaSuccess) return r;
    potrf_status_fixup_kernel<<<1, 1, 0, hp>>>(d_status, sub, k0);
    const int64_t nt = n - k0 - w;
    if (nt > 0)
      potrf_panel_kernel<<<(unsigned)((nt + kNB - 1) / kNB), kThreads, kPanelSmem, hp>>>(W, n, ldW, k0, (int)(w / kNB),
                                                                                         Linv, d_status);
    if (launches) *launches += nt > 0 ? 2 : 1;
    return cudaGetLastError();
  };
  if (e == cudaSuccess) e = diag_panel(0);
  for (int64_t s = 0; e == cudaSuccess && (s + 1) * kNB2 < n; ++s) {
    const int64_t k0 = s * kNB2, w = kNB2, r0 = k0 + w, nt = n - r0;   // panel s: rows [r0, n)
    const double* P = W + r0 * ldW + k0;
    const int64_t ws = std::min<int64_t>(kNB2, nt);                     // strip s+1 width
    if (ahead) {
      cudaEvent_t ev_p = bs.ev[2 * s], ev_r = bs.ev[2 * s + 1];
      if ((e = cudaEventRecord(ev_p, hp)) != cudaSuccess) break;        // panel s done
      // rest of step s (columns beyond strip s+1) on lp
      if ((e = cudaStreamWaitEvent(lp, ev_p, 0)) != cudaSuccess) break;
      if (nt > ws && (e = syrk_dmma_trail(P + ws * ldW, nt - ws, w, ldW, W + (r0 + ws) * ldW + r0 + ws, ldW, d_status,
                                          lp, launches)) != cudaSuccess)
        break;
      // strip s+1 on hp, after the previous step's rest (same columns)
      if (s > 0 && (e = cudaStreamWaitEvent(hp, bs.ev[2 * s - 1], 0)) != cudaSuccess) break;
      if ((e = syrk_dmma_trail(P, nt, w, ldW, W + r0 * ldW + r0, ldW, d_status, hp, launches, ws)) != cudaSuccess)
        break;
      if ((e = cudaEventRecord(ev_r, lp)) != cudaSuccess) break;
    } else {
      e = syrk_dmma_trail(P, nt, w, ldW, W + r0 * ldW + r0, ldW, d_status, st, launches);
      if (e != cudaSuccess) break;
    }
    e = diag_panel(r0);
  }
  if (ahead) {                                   // join: the caller's stream waits for both
    cudaError_t e2 = cudaEventRecord(bs.fork, hp);
    if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(st, bs.fork, 0);
    cudaEvent_t last_lp = bs.ev[BlockedStreams::kEv - 1];
    if (e2 == cudaSuccess) e2 = cudaEventRecord(last_lp, lp);
    if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(st, last_lp, 0);
    if (e == cudaSuccess) e = e2;
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

cudaError_t potrf_lower(double* W, int64_t n, int64_t ldW, int64_t* d_status, double* scratch,
                        cudaStream_t st, int* launches, const double* u, double* z, bool* solved) {
  if (solved) *solved = false;
  if (n >= potrf_blocked_min_n() && n > kNB2) return potrf_blocked(W, n, ldW, d_status, scratch, st, launches);
  const int nb = (int)((n + kNB - 1) / kNB);
  double* Linv = scratch;
  double* panel0 = Linv + (int64_t)nb * kNB * kNB;
  double* panel1 = panel0 + n * kNB;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(potrf_first_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(3 * kTileSmem));
    cudaFuncSetAttribute(potrf_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(3 * kTileSmem));
    attr = true;
  }
  // one persistent cooperative kernel when the grid fits (it always does: one CTA per SM)
  {
    static int coop = -1;
    static int grid = 0;
    if (coop < 0) {
      int dev = 0, sms = 0, per_sm = 0, ok = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaFuncSetAttribute(potrf_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4 * kTileSmem));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, potrf_persistent_kernel, kThreads, 4 * kTileSmem);
      coop = (ok && per_sm >= 1) ? 1 : 0;
      grid = sms;
    }
    if (coop == 1) {
      unsigned* ctl = reinterpret_cast<unsigned*>(panel1 + n * kNB);
      cudaError_t e = cudaMemsetAsync(ctl, 0, 2 * sizeof(unsigned), st);
      if (e != cudaSuccess) return e;
      if (u) {                                           // backward-solve block flags (after tb)
        e = cudaMemsetAsync(panel1 + n * kNB + 1 + 2 * n, 0, (size_t)nb * sizeof(unsigned), st);
        if (e != cudaSuccess) return e;
      }
      const int tiles0 = (nb - 1) * nb / 2;
      const int g = std::max(1, std::min(grid, tiles0));
      int64_t nn = n, ldd = ldW;
      double* ut = panel1 + n * kNB + 1;                 // after the barrier words
      double* tb = ut + n;
      // the backward solve: inside the kernel (flag-chained over CTAs, ~48 us at n = 1024) or,
      // when the TRSV cluster fits (n <= 1024), as its backward half (~15 us over DSMEM)
      static const int bwd_env = getenv("FS_POTRF_CLUSTER_BWD") ? atoi(getenv("FS_POTRF_CLUSTER_BWD")) : 1;
      int skip_bwd = (u && bwd_env && trsv_cluster_ok(n)) ? 1 : 0;
      void* args[] = {&W, &nn, &ldd, &Linv, &panel0, &panel1, &d_status, &ctl, &u, &ut, &tb, &z, &skip_bwd};
      e = cudaLaunchCooperativeKernel((const void*)potrf_persistent_kernel, dim3(g), dim3(kThreads), args,
                                      4 * kTileSmem, st);
      if (launches) *launches += 1;
      if (e == cudaSuccess && skip_bwd) e = trsv_backward_cluster(W, n, ldW, Linv, tb, z, d_status, st, launches);
      if (solved && u && e == cudaSuccess) *solved = true;
      return e;
    }
  }
  int count = 0;
  potrf_first_kernel<<<1, kThreads, 3 * kTileSmem, st>>>(W, n, ldW, Linv, d_status);
  ++count;
  for (int k = 0; k + 1 < nb; ++k) {
    const int t = nb - k - 1;   // trailing block count
    potrf_step_kernel<<<t * (t + 1) / 2, kThreads, 3 * kTileSmem, st>>>(W, n, ldW, k, Linv, panel0, panel1,
                                                                          d_status);
    ++count;
  }
  if (nb >= 2) {
    const int k = nb - 2;
    potrf_tail_kernel<<<64, 256, 0, st>>>(W, n, ldW, k, (k & 1) ? panel1 : panel0, d_status);
    ++count;
  }
  if (launches) *launches += count;
  return cudaGetLastError();   // Linv (the TRSV pair's inverted diagonal blocks) comes with the factor
}

}  // namespace fs
