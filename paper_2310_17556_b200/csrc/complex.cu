// complex.cu — complex score matrices reduced to the real path.
//
// solve_realpart (solvers.py:216-240): C = [Re S; Im S] (2n x m, sr.py:61-70), C^T C = Re[S^H S].
// solve_chol_hermitian (solvers.py:209-213): the real representation
//   rho(S) = [[Re S, -Im S], [Im S, Re S]] (2n x 2m)  with  rho(S)^T rho(S) = rho(S^H S),
// so (S^H S + lam I) x = v  <=>  (rho^T rho + lam I) [Re x; Im x] = [Re v; Im v], solved by the
// plain real route (tensor-core Gram of the 2n rows, fp64 potrf, ...).  One streaming pass
// de-interleaves the (re, im) pairs into the aligned real layout.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace fs {
namespace {

template <typename T>
__global__ void embed_kernel(const T* __restrict__ S, int64_t n, int64_t m, int64_t ldS, int kind, T* __restrict__ out,
                             int64_t ldo) {
  // grid-stride over (row i < n, column j < m); S holds (re, im) pairs, ldS in complex elements
  const int64_t total = n * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / m, j = e - i * m;
    const T re = S[2 * (i * ldS + j)], im = S[2 * (i * ldS + j) + 1];
    if (kind == 0) {
      out[i * ldo + j] = re;
      out[(n + i) * ldo + j] = im;
    } else {
      out[i * ldo + j] = re;
      out[i * ldo + m + j] = -im;
      out[(n + i) * ldo + j] = im;
      out[(n + i) * ldo + m + j] = re;
    }
  }
}

// Packed-lower index of the symmetric 2n x 2n Gram of C = [Re S; Im S].
__device__ __forceinline__ int64_t pidx(int64_t a, int64_t b) {
  return a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a;
}

// W = S S^H + lam I (n x n, interleaved complex, row ld ldW) from the packed Gram G2 of C:
//   Re W_ij = G2(i, j) + G2(n+i, n+j)    (Re S Re S^T + Im S Im S^T)
//   Im W_ij = G2(n+i, j) - G2(i, n+j)    (Im S Re S^T - Re S Im S^T)
// Entry (j, i) reads the same two G2 entries, so W is exactly Hermitian and Im W_ii = 0
// exactly (core.py:286-289 symmetrises, then adds lam on the diagonal).
__global__ void hermitian_gram_kernel(const double* __restrict__ G2, int64_t n, double lam, double* __restrict__ W,
                                      int64_t ldW) {
  const int64_t total = n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    const int64_t a = i >= j ? i : j, b = i >= j ? j : i;   // compute the lower entry (a, b)
    const double re = G2[pidx(a, b)] + G2[pidx(n + a, n + b)];
    const double im = G2[pidx(n + a, b)] - G2[pidx(a, n + b)];
    W[2 * (i * ldW + j)] = i == j ? re + lam : re;
    W[2 * (i * ldW + j) + 1] = i == j ? 0.0 : (i > j ? im : -im);
  }
}

// Packed lower rho(G) = [[Re G, -Im G], [Im G, Re G]] (2n x 2n) for G = S S^H, from the packed
// Gram G2 of C = [Re S; Im S]; rho(G) is symmetric and has every eigenvalue of G twice.
__global__ void rho_gram_kernel(const double* __restrict__ G2, int64_t n, double* __restrict__ R) {
  const int64_t N = 2 * n, total = N * (N + 1) / 2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = (int64_t)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
    while ((a + 1) * (a + 2) / 2 <= e) ++a;
    while (a * (a + 1) / 2 > e) --a;
    const int64_t b = e - a * (a + 1) / 2;            // a >= b
    const int64_t i = a % n, j = b % n;
    const bool lo_a = a >= n, lo_b = b >= n;
    double val;
    if (lo_a == lo_b) {                               // Re G_ij (diagonal blocks)
      val = G2[pidx(i, j)] + G2[pidx(n + i, n + j)];
    } else {                                          // a in the lower block row, b in the left: Im G_ij
      val = G2[pidx(n + i, j)] - G2[pidx(i, n + j)];
    }
    R[e] = val;
  }
}

// Complex eigenvectors of G from the real eigenvectors of rho(G) (Y: 2n x 2n row-major, column k
// <-> w2[k], descending).  Column k maps to u_k = Y[:n, k] + i Y[n:, k], an eigenvector of G; each
// eigenvalue's real eigenspace is closed under multiplication by i, so a cluster of 2d equal
// eigenvalues spans d complex directions.  One CTA walks the candidates in order and keeps u_k
// when its component orthogonal (complex inner product) to the vectors already kept in the same
// cluster (eigenvalues within tol) has norm > 1/2; n vectors are kept.  U: n x n interleaved
// complex (column j <-> w[j]).
__global__ void herm_extract_kernel(const double* __restrict__ Y, const double* __restrict__ w2, int n, double tol,
                                    double* __restrict__ U, double* __restrict__ w, int* __restrict__ kept,
                                    double* __restrict__ scratch) {
  __shared__ double red[2][32];
  __shared__ int s_take;
  const int N = 2 * n;
  int nk = 0;          // kept so far
  int cluster0 = 0;    // index into the kept list where the current cluster starts
  double* cr = scratch;          // candidate, real part (n)
  double* ci = scratch + n;      // imaginary part
  auto block_sum2 = [&](double a, double b, double& ra, double& rb) {
    a = warp_sum(a);
    b = warp_sum(b);
    if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = a; red[1][threadIdx.x >> 5] = b; }
    __syncthreads();
    double sa = 0.0, sb = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { sa += red[0][q]; sb += red[1][q]; }
    __syncthreads();
    ra = sa;
    rb = sb;
  };
  for (int k = 0; k < N && nk < n; ++k) {
    if (k > 0 && !(fabs(w2[k] - w2[k - 1]) <= tol)) cluster0 = nk;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      cr[i] = Y[(int64_t)i * N + k];
      ci[i] = Y[(int64_t)(n + i) * N + k];
    }
    __syncthreads();
    for (int j = cluster0; j < nk; ++j) {             // remove components along kept u_j: c -= (u_j^H c) u_j
      double pr = 0.0, pi = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double ur = U[2 * ((int64_t)i * n + j)], ui = U[2 * ((int64_t)i * n + j) + 1];
        pr += ur * cr[i] + ui * ci[i];
        pi += ur * ci[i] - ui * cr[i];
      }
      block_sum2(pr, pi, pr, pi);
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double ur = U[2 * ((int64_t)i * n + j)], ui = U[2 * ((int64_t)i * n + j) + 1];
        cr[i] -= pr * ur - pi * ui;
        ci[i] -= pr * ui + pi * ur;
      }
      __syncthreads();
    }
    double nr = 0.0, dummy = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) nr += cr[i] * cr[i] + ci[i] * ci[i];
    block_sum2(nr, 0.0, nr, dummy);
    if (threadIdx.x == 0) s_take = nr > 0.25 ? 1 : 0;
    __syncthreads();
    if (s_take) {
      const double inv = 1.0 / sqrt(nr);
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        U[2 * ((int64_t)i * n + nk)] = cr[i] * inv;
        U[2 * ((int64_t)i * n + nk) + 1] = ci[i] * inv;
      }
      if (threadIdx.x == 0) w[nk] = w2[k];
      ++nk;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *kept = nk;
}

}  // namespace

cudaError_t rho_gram(const double* G2, int64_t n, double* R, int num_sms, cudaStream_t st, int* launches) {
  const int64_t total = 2 * n * (2 * n + 1);
  const unsigned grid = (unsigned)std::min<int64_t>((total / 2 + 255) / 256, (int64_t)num_sms * 8);
  rho_gram_kernel<<<grid, 256, 0, st>>>(G2, n, R);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t herm_extract(const double* Y, const double* w2, int64_t n, double tol, double* U, double* w, int* kept,
                         double* scratch, cudaStream_t st, int* launches) {
  herm_extract_kernel<<<1, 1024, 0, st>>>(Y, w2, (int)n, tol, U, w, kept, scratch);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t hermitian_gram(const double* G2, int64_t n, double lam, double* W, int64_t ldW, int num_sms,
                           cudaStream_t st, int* launches) {
  const int64_t total = n * n;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms * 8);
  hermitian_gram_kernel<<<grid, 256, 0, st>>>(G2, n, lam, W, ldW);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t embed_complex(bool f64, const void* S, int64_t n, int64_t m, int64_t ldS, int kind, void* out, int64_t ldo,
                          int num_sms, cudaStream_t st, int* launches) {
  const unsigned grid = (unsigned)(num_sms * 8);
  if (f64) embed_kernel<double><<<grid, 256, 0, st>>>((const double*)S, n, m, ldS, kind, (double*)out, ldo);
  else embed_kernel<float><<<grid, 256, 0, st>>>((const float*)S, n, m, ldS, kind, (float*)out, ldo);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace fs
