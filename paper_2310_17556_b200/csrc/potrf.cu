// potrf.cu — fp64 lower Cholesky of the damped Gram matrix W (n x n, row-major).
//
// Replaces solvers.py:74-90 (scipy get_lapack_funcs('potrf') -> LAPACK dpotrf(lower=1,
// clean=1)).  Same failure contract: the first column j whose updated pivot is not
// strictly positive (or is NaN) sets the device status word to j+1 (LAPACK info),
// which the host maps to FactorizationError(pivot=j) (solvers.py:82-87).  The upper
// triangle is left exactly zero (clean=1; test_solvers.py:455).
//
// Blocked right-looking algorithm, panel width 64: diag factor (1 CTA, panel in SMEM)
// -> panel TRSM (one thread per row, row in registers) -> trailing SYRK update (64x64
// fp64 tiles).  Every kernel first checks the status word so a breakdown stops the
// remaining work.  Deterministic (fixed operation order, no atomics).
#include "common.cuh"
#include "kernels.h"

namespace fs {
namespace {

constexpr int kNB = 64;

__global__ void unpack_lower_kernel(const double* __restrict__ Gp, int64_t n, double add_diag,
                                    double* __restrict__ W, int64_t ldW) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (j >= n) return;
  double v = 0.0;
  if (j <= i) v = Gp[i * (i + 1) / 2 + j] + (i == j ? add_diag : 0.0);
  W[i * ldW + j] = v;
}

__global__ void __launch_bounds__(256)
potrf_diag_kernel(double* __restrict__ W, int64_t ldW, int64_t k0, int b, int64_t* status) {
  __shared__ double A[kNB][kNB + 1];
  __shared__ int fail;
  if (*(volatile int64_t*)status != 0) return;
  const int tid = threadIdx.x;
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int r = e / b, c = e % b;
    A[r][c] = (c <= r) ? W[(k0 + r) * ldW + k0 + c] : 0.0;
  }
  if (tid == 0) fail = 0;
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    if (tid == 0) {
      const double d = A[j][j];
      if (!(d > 0.0)) {          // catches d <= 0 and NaN, like dpotrf
        fail = 1;
        *status = k0 + j + 1;
      } else {
        A[j][j] = sqrt(d);
      }
    }
    __syncthreads();
    if (fail) return;
    const double djj = A[j][j];
    for (int i = j + 1 + tid; i < b; i += blockDim.x) A[i][j] /= djj;
    __syncthreads();
    // trailing update of the block: A[i][k] -= A[i][j] A[k][j], j < k <= i
    const int rem = b - j - 1;
    for (int e = tid; e < rem * rem; e += blockDim.x) {
      const int i = j + 1 + e / rem, k = j + 1 + e % rem;
      if (k <= i) A[i][k] = fma(-A[i][j], A[k][j], A[i][k]);
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int r = e / b, c = e % b;
    if (c <= r) W[(k0 + r) * ldW + k0 + c] = A[r][c];
  }
}

// L21[i, :] = A21[i, :] * L11^-T, one thread per row, row held in registers.
__global__ void __launch_bounds__(64)
potrf_panel_kernel(double* __restrict__ W, int64_t n, int64_t ldW, int64_t k0, int b,
                   const int64_t* status) {
  __shared__ double L[kNB][kNB + 1];
  if (*(volatile const int64_t*)status != 0) return;
  for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
    const int r = e / kNB, c = e % kNB;
    double v;
    if (r < b && c < b) v = (c <= r) ? W[(k0 + r) * ldW + k0 + c] : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    L[r][c] = v;
  }
  __syncthreads();
  const int64_t i = k0 + b + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* row = W + i * ldW + k0;
  double x[kNB];
#pragma unroll
  for (int j = 0; j < kNB; ++j) x[j] = (j < b) ? row[j] : 0.0;
#pragma unroll
  for (int j = 0; j < kNB; ++j) {
    double s = x[j];
#pragma unroll
    for (int p = 0; p < j; ++p) s = fma(-x[p], L[j][p], s);
    x[j] = s / L[j][j];
  }
#pragma unroll
  for (int j = 0; j < kNB; ++j)
    if (j < b) row[j] = x[j];
}

// A22 -= L21 L21^T on lower 64x64 tiles of the trailing matrix.
__global__ void __launch_bounds__(256)
potrf_update_kernel(double* __restrict__ W, int64_t n, int64_t ldW, int64_t k0, int b,
                    const int64_t* status) {
  constexpr int T = 64, BK = 16;
  __shared__ double As[BK][T + 1];
  __shared__ double Bs[BK][T + 1];
  if (*(volatile const int64_t*)status != 0) return;
  const int64_t t = blockIdx.x;
  int I = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((int64_t)(I + 1) * (I + 2) / 2 <= t) ++I;
  while ((int64_t)I * (I + 1) / 2 > t) --I;
  const int J = (int)(t - (int64_t)I * (I + 1) / 2);
  const int64_t base = k0 + b;
  const int64_t r0 = base + (int64_t)I * T, c0 = base + (int64_t)J * T;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double acc[4][4] = {};
  for (int p0 = 0; p0 < b; p0 += BK) {
    __syncthreads();
    for (int e = tid; e < T * BK; e += 256) {
      const int r = e / BK, p = e % BK;
      const int64_t ga = r0 + r, gb = c0 + r;
      As[p][r] = (ga < n && p0 + p < b) ? W[ga * ldW + k0 + p0 + p] : 0.0;
      Bs[p][r] = (gb < n && p0 + p < b) ? W[gb * ldW + k0 + p0 + p] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < BK; ++p) {
      double a[4], c[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = As[p][ty + 16 * q]; c[q] = Bs[p][tx + 16 * q]; }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[q][s] = fma(a[q], c[s], acc[q][s]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int64_t gi = r0 + ty + 16 * q, gj = c0 + tx + 16 * s;
      if (gi < n && gj <= gi) W[gi * ldW + gj] -= acc[q][s];
    }
}

}  // namespace

cudaError_t unpack_lower(const double* Gp, int64_t n, double add_diag, double* W, int64_t ldW,
                         cudaStream_t st, int* launches) {
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)n);
  unpack_lower_kernel<<<grid, 256, 0, st>>>(Gp, n, add_diag, W, ldW);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t potrf_lower(double* W, int64_t n, int64_t ldW, int64_t* d_status, cudaStream_t st,
                        int* launches) {
  int count = 0;
  for (int64_t k0 = 0; k0 < n; k0 += kNB) {
    const int b = (int)std::min<int64_t>(kNB, n - k0);
    potrf_diag_kernel<<<1, 256, 0, st>>>(W, ldW, k0, b, d_status);
    ++count;
    const int64_t rest = n - k0 - b;
    if (rest > 0) {
      potrf_panel_kernel<<<(unsigned)((rest + 63) / 64), 64, 0, st>>>(W, n, ldW, k0, b, d_status);
      const int64_t nt = (rest + 63) / 64;
      potrf_update_kernel<<<(unsigned)(nt * (nt + 1) / 2), 256, 0, st>>>(W, n, ldW, k0, b, d_status);
      count += 2;
    }
  }
  if (launches) *launches += count;
  return cudaGetLastError();
}

}  // namespace fs
