// potrf.cu — fp64 lower Cholesky of the damped Gram matrix W (n x n, row-major), in place.
//
// Replaces solvers.py:74-90 (scipy get_lapack_funcs('potrf') -> LAPACK dpotrf(lower=1,
// clean=1)).  Same failure contract: the first column j whose updated pivot is not strictly
// positive (or is NaN) sets the device status word to j+1 (LAPACK info), which the host maps
// to FactorizationError(pivot=j) (solvers.py:82-87).  The upper triangle is never written
// (fs_unpack_lower leaves it exactly zero: clean=1, test_solvers.py:455).
//
// Blocked right-looking algorithm with 64-wide block columns, ONE launch per block column:
//   step k, CTA (I,J) for k < J <= I:   X_I = A_Ik Linv_kk^T   (TRSM through the inverted
//   diagonal block; X_J likewise), A_IJ -= X_I X_J^T, and
//     * the CTA with J == k+1 stores X_I as the panel L_Ik (double-buffered panel, copied into
//       W by the next step, so no CTA ever overwrites data another CTA of its step still reads)
//     * the CTA with I == J == k+1 factors the freshly updated diagonal block and inverts it
//       (next step's Linv, also kept for the TRSV pair).
// Every kernel first checks the status word, so a breakdown stops the remaining work.
// Deterministic: fixed operation order, no atomics.
#include "common.cuh"
#include "kernels.h"

namespace fs {
namespace {

constexpr int kNB = 64;
constexpr int kThreads = 256;
constexpr int kLd = kNB + 1;   // padded smem row

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

// In-place Cholesky of the identity-padded 64x64 block A (smem, lower) by 256 threads.
// Thread (r = tid/4, q = tid%4) keeps its row's 16 elements A[r][q + 4cc] in REGISTERS for the
// whole factorisation (smem round trips through an aliased array serialise at ~50 cycles each).
// Step j: the pivot column j lives in a double-buffered smem vector col[] written by its owners
// at the end of step j-1, together with 1/d_j computed (one __drcp_rn) by the thread that
// finalised A[j][j]; one barrier per column.  Unscaled update A[r][c] -= A[r][j] A[c][j] / d_j;
// a final pass scales L[r][c] = A[r][c] * rsqrt(d_c).  Sets *fail (first bad pivot or -1).
__device__ void factor_block(double (*A)[kLd], int b, int* fail) {
  __shared__ double col[2][kNB];
  __shared__ double dinv[2];
  __shared__ double dval[kNB];
  const int tid = threadIdx.x, r = tid >> 2, q = tid & 3;
  double a[kNB / 4];
#pragma unroll
  for (int cc = 0; cc < kNB / 4; ++cc) a[cc] = A[r][q + 4 * cc];
  if (q == 0) col[0][r] = A[r][0];
  if (tid == 0) {
    *fail = -1;
    dinv[0] = __drcp_rn(A[0][0]);
  }
#pragma unroll 1
  for (int j = 0; j < b; ++j) {
    __syncthreads();
    const int buf = j & 1;
    const double d = col[buf][j];
    if (!(d > 0.0)) {                  // uniform: every thread reads the same pivot
      if (tid == 0) *fail = j;
      __syncthreads();
      return;
    }
    if (tid == 0) dval[j] = d;
    const double s = (r > j) ? col[buf][r] * dinv[buf] : 0.0;
    double cj[kNB / 4];
#pragma unroll
    for (int cc = 0; cc < kNB / 4; ++cc) cj[cc] = col[buf][q + 4 * cc];
#pragma unroll
    for (int cc = 0; cc < kNB / 4; ++cc) {
      const int c = q + 4 * cc;
      if (r > j && c > j && c <= r) a[cc] = fma(-s, cj[cc], a[cc]);
      // publish column j+1 (final after this update) and its pivot reciprocal; predicated
      // stores with a compile-time register index keep a[] out of local memory
      if (c == j + 1 && j + 1 < b) {
        col[buf ^ 1][r] = a[cc];
        if (r == j + 1) dinv[buf ^ 1] = __drcp_rn(a[cc]);
      }
    }
  }
  __syncthreads();
  // scale: L[r][c] = A[r][c] * rsqrt(d_c) (diagonal: d_c * rsqrt(d_c) = sqrt(d_c))
#pragma unroll
  for (int cc = 0; cc < kNB / 4; ++cc) {
    const int c = q + 4 * cc;
    double v = (c <= r) ? a[cc] : 0.0;
    if (c < b && c <= r) v *= rsqrt(dval[c]);
    if (r >= b || c >= b) v = (r == c) ? 1.0 : 0.0;   // identity padding
    A[r][c] = v;
  }
  __syncthreads();
}

// X <- X L^-T: each of the 64 rows of X solved against the lower 64x64 L (rdiag = 1/L_jj).
// Thread (r, q) handles columns p = q + 4cc of row r.  Step j issues its 32 smem loads up
// front (X[r][.] and L[j][.], all independent), four predicated FMA chains, a 4-lane shuffle
// reduction, and the owner lane stores x_j: one store per step, so nothing serialises on
// smem aliasing.  No block barriers (a row lives in one warp).
__device__ void trsm_rows(const double (*L)[kLd], const double* rdiag, double (*X)[kLd]) {
  const int tid = threadIdx.x, r = tid >> 2, q = tid & 3;
#pragma unroll 1
  for (int j = 0; j < kNB; ++j) {
    double xv[kNB / 4], lj[kNB / 4];
#pragma unroll
    for (int cc = 0; cc < kNB / 4; ++cc) {
      xv[cc] = X[r][q + 4 * cc];
      lj[cc] = L[j][q + 4 * cc];
    }
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int cc = 0; cc < kNB / 4; cc += 4) {
      if (q + 4 * cc < j) s0 = fma(xv[cc], lj[cc], s0);
      if (q + 4 * (cc + 1) < j) s1 = fma(xv[cc + 1], lj[cc + 1], s1);
      if (q + 4 * (cc + 2) < j) s2 = fma(xv[cc + 2], lj[cc + 2], s2);
      if (q + 4 * (cc + 3) < j) s3 = fma(xv[cc + 3], lj[cc + 3], s3);
    }
    double sum = (s0 + s1) + (s2 + s3);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (q == (j & 3)) X[r][j] = (X[r][j] - sum) * rdiag[j];
    __syncwarp();
  }
}

// C (64x64, smem) = A (64x64 smem) * B^T (64x64 smem); each thread a 4x4 sub-block.
__device__ void gemm_nt(const double (*A)[kLd], const double (*B)[kLd], double acc[4][4]) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
#pragma unroll 8
  for (int p = 0; p < kNB; ++p) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = A[ty + 16 * i][p];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = B[tx + 16 * j][p];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
  }
}

__device__ void load_tile(const double* W, int64_t n, int64_t ld, int64_t r0, int64_t c0, double (*T)[kLd]) {
  for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) {
    const int r = e / kNB, c = e % kNB;
    const int64_t gr = r0 + r, gc = c0 + c;
    T[r][c] = (gr < n && gc < n) ? W[gr * ld + gc] : 0.0;
  }
}

__device__ void tile_coords(int t, int& I, int& J) {  // lower tiles in row-major order
  int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  I = i;
  J = t - i * (i + 1) / 2;
}

// Factor diagonal block kk of W (already fully updated) in place.
__device__ void factor_diag(double* W, int64_t n, int64_t ld, int kk, int64_t* status, double (*A)[kLd], int* fail) {
  const int64_t r0 = (int64_t)kk * kNB;
  const int b = (int)(n - r0 < kNB ? n - r0 : kNB);
  load_tile(W, n, ld, r0, r0, A);
  __syncthreads();
  for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) {   // identity padding, lower only
    const int r = e >> 6, c = e & 63;
    if (c > r) A[r][c] = 0.0;
    else if (r >= b) A[r][c] = (r == c) ? 1.0 : 0.0;
  }
  factor_block(A, b, fail);
  if (*fail >= 0) {
    if (threadIdx.x == 0) *status = r0 + *fail + 1;
    return;
  }
  for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) {
    const int r = e >> 6, c = e & 63;
    if (r < b && c <= r) W[(r0 + r) * ld + r0 + c] = A[r][c];
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
potrf_first_kernel(double* W, int64_t n, int64_t ld, int64_t* status) {
  extern __shared__ double dsm[];
  double (*A)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm);
  __shared__ int fail;
  if (*(volatile int64_t*)status != 0) return;
  factor_diag(W, n, ld, 0, status, A, &fail);
}

// Step k: tiles (I, J) of the trailing matrix, k < J <= I < nb, indexed relative to k+1.
__global__ void __launch_bounds__(kThreads)
potrf_step_kernel(double* W, int64_t n, int64_t ld, int k, double* panel0, double* panel1, int64_t* status) {
  extern __shared__ double dsm[];
  double (*Lk)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm);              // L_kk, later scratch
  double (*XI)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + kNB * kLd);
  double (*XJ)[kLd] = reinterpret_cast<double (*)[kLd]>(dsm + 2 * kNB * kLd);
  __shared__ double rdiag[kNB];
  __shared__ int fail;
  if (*(volatile int64_t*)status != 0) return;
  int I, J;
  tile_coords(blockIdx.x, I, J);
  I += k + 1;
  J += k + 1;
  const int64_t kc = (int64_t)k * kNB, rI = (int64_t)I * kNB, rJ = (int64_t)J * kNB;
  double* pan_cur = (k & 1) ? panel1 : panel0;     // this step's panel L_{.,k}
  double* pan_prev = (k & 1) ? panel0 : panel1;    // previous step's panel L_{.,k-1}
  // materialise the previous panel L_{.,k-1} into W (nobody reads W column k-1 any more):
  // row block I by the CTA (I, k+1); row block k by the diagonal CTA (k+1, k+1)
  if (J == k + 1 && k >= 1) {
    for (int pass = 0; pass < (I == k + 1 ? 2 : 1); ++pass) {
      const int64_t rb = pass == 0 ? rI : kc;
      for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) {
        const int r = e >> 6, c = e & 63;
        const int64_t gr = rb + r;
        if (gr < n) W[gr * ld + (kc - kNB) + c] = pan_prev[gr * kNB + c];
      }
    }
  }
  load_tile(W, n, ld, kc, kc, Lk);                 // L_kk (factored by the previous step)
  load_tile(W, n, ld, rI, kc, XI);                 // A_Ik
  if (I != J) load_tile(W, n, ld, rJ, kc, XJ);     // A_Jk
  __syncthreads();
  if (threadIdx.x < kNB) {
    const int j = threadIdx.x;
    const double d = Lk[j][j];
    rdiag[j] = (kc + j < n) ? 1.0 / d : 1.0;
    if (kc + j >= n) Lk[j][j] = 1.0;
  }
  __syncthreads();
  trsm_rows(Lk, rdiag, XI);                        // X_I = A_Ik L_kk^-T
  if (I != J) trsm_rows(Lk, rdiag, XJ);
  __syncthreads();
  if (J == k + 1) {   // store the panel L_Ik
    for (int e = threadIdx.x; e < kNB * kNB; e += kThreads) {
      const int r = e >> 6, c = e & 63;
      const int64_t gr = rI + r;
      if (gr < n) pan_cur[gr * kNB + c] = XI[r][c];
    }
  }
  // A_IJ -= X_I X_J^T
  double acc[4][4];
  gemm_nt(XI, (I != J) ? XJ : XI, acc);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gi = rI + ty + 16 * i, gj = rJ + tx + 16 * j;
      if (gi < n && gj <= gi) W[gi * ld + gj] -= acc[i][j];
    }
  if (I == J && I == k + 1) {
    __syncthreads();   // (block-uniform branch) this CTA's tile update is complete and visible
    factor_diag(W, n, ld, I, status, Lk, &fail);
  }
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
  return nb * kNB * kNB /* Linv */ + 2 * n * kNB /* panels */;
}

cudaError_t unpack_lower(const double* Gp, int64_t n, double add_diag, double* W, int64_t ldW,
                         cudaStream_t st, int* launches) {
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)n);
  unpack_lower_kernel<<<grid, 256, 0, st>>>(Gp, n, add_diag, W, ldW);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t potrf_lower(double* W, int64_t n, int64_t ldW, int64_t* d_status, double* scratch,
                        cudaStream_t st, int* launches) {
  const int nb = (int)((n + kNB - 1) / kNB);
  double* Linv = scratch;
  double* panel0 = Linv + (int64_t)nb * kNB * kNB;
  double* panel1 = panel0 + n * kNB;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(potrf_first_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kTileSmem));
    cudaFuncSetAttribute(potrf_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(3 * kTileSmem));
    attr = true;
  }
  int count = 0;
  potrf_first_kernel<<<1, kThreads, kTileSmem, st>>>(W, n, ldW, d_status);
  ++count;
  for (int k = 0; k + 1 < nb; ++k) {
    const int t = nb - k - 1;   // trailing block count
    potrf_step_kernel<<<t * (t + 1) / 2, kThreads, 3 * kTileSmem, st>>>(W, n, ldW, k, panel0, panel1, d_status);
    ++count;
  }
  if (nb >= 2) {
    const int k = nb - 2;
    potrf_tail_kernel<<<64, 256, 0, st>>>(W, n, ldW, k, (k & 1) ? panel1 : panel0, d_status);
    ++count;
  }
  if (launches) *launches += count;
  // inverted diagonal blocks for the TRSV pair (all blocks in parallel, off the factor's path)
  return invert_diag_blocks(W, n, ldW, Linv, st, launches);
}

}  // namespace fs
