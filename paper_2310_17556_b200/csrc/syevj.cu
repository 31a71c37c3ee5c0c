// syevj.cu — symmetric eigendecomposition of the n x n Gram matrix (fp64), parallel Jacobi.
//
// Replaces solvers.py:261 (np.linalg.eigh -> LAPACK dsyevd) on the eigh comparison route
// (SURVEY §8a9/§8f-2): A = U diag(w) U^T with w sorted descending (the reference reverses
// eigh's ascending order, solvers.py:265-266).
//
// Two-sided cyclic Jacobi with the round-robin (tournament) ordering: a sweep is n-1 rounds,
// each round rotates n/2 disjoint index pairs at once.  Every element of A belongs to exactly
// one 2x2 block (row pair k1, column pair k2), whose new value J_k1^T B J_k2 depends only on
// that block's old values, so a round is ONE fully parallel pass (A double-buffered: the
// rotations of a round are computed from the old copy while the new one is written), followed by
// one grid-wide barrier.  One persistent cooperative kernel runs all sweeps; each CTA owns a
// stripe of row pairs (and the matching rows of U^T, updated in place).  The sweep stops when
// the off-diagonal Frobenius norm falls below tol * ||A||_F (fixed-order reduction:
// deterministic).  Rotations follow Golub & Van Loan sym.schur2 (|t| <= 1, the stable root).
// A single-CTA bitonic sort orders the eigenpairs.
#include "common.cuh"
#include "kernels.h"

namespace fs {
namespace {

constexpr int kJThreads = 512;

struct Rot {
  double c, s;
};

FS_DEVINL void pair_of_round(int r, int k, int np1, int& p, int& q) {
  // players 0..np1 (np1 = n-1); position 0 of the top row is fixed at player np1
  p = (k == 0) ? np1 : (r + k) % np1;
  q = (r - k + np1) % np1;
}

FS_DEVINL Rot schur2(double app, double aqq, double apq) {
  Rot R{1.0, 0.0};
  if (apq != 0.0) {
    const double tau = (aqq - app) / (2.0 * apq);
    const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
    R.c = 1.0 / sqrt(1.0 + t * t);
    R.s = t * R.c;
  }
  return R;
}

// sense-reversing grid barrier (the launch is cooperative: all CTAs are co-resident)
FS_DEVINL void grid_barrier(unsigned* count, volatile unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// A0/A1: n x n (n even), A0 holds the input; Ut: n x n, U^T (row i = eigenvector i at the end).
// partial: gridDim.x doubles; ctl: [count, gen]; info: [sweeps, final A index]
__global__ void __launch_bounds__(kJThreads, 1)
jacobi_kernel(double* __restrict__ A0, double* __restrict__ A1, double* __restrict__ Ut, int n, int max_sweeps,
              double tol, double* __restrict__ partial, unsigned* ctl, int* info, double* __restrict__ wraw) {
  extern __shared__ Rot rot[];           // n/2 rotations of the current round
  __shared__ double red[kJThreads / 32];
  const int half = n / 2, np1 = n - 1;
  double* Aold = A0;
  double* Anew = A1;
  // ||A||_F^2 (fixed order: per-CTA partials, then CTA-ordered sum by every CTA)
  auto frob_off = [&](const double* A, bool off_only) -> double {
    double s = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * kJThreads + threadIdx.x; e < (int64_t)n * n;
         e += (int64_t)gridDim.x * kJThreads) {
      const int i = (int)(e / n), j = (int)(e % n);
      if (!off_only || i != j) s += A[e] * A[e];
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kJThreads / 32; ++w) t += red[w];
      partial[blockIdx.x] = t;
    }
    grid_barrier(ctl, ctl + 1);
    double tot = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) tot += partial[b];
    grid_barrier(ctl, ctl + 1);          // partial[] may be overwritten afterwards
    return tot;
  };
  const double fro2 = frob_off(Aold, false);
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    const double off2 = frob_off(Aold, true);
    if (!(off2 > tol * tol * fro2)) break;
    for (int r = 0; r < np1; ++r) {
      // rotations of this round from the old copy (every CTA computes all of them)
      for (int k = threadIdx.x; k < half; k += kJThreads) {
        int p, q;
        pair_of_round(r, k, np1, p, q);
        rot[k] = schur2(Aold[(int64_t)p * n + p], Aold[(int64_t)q * n + q], Aold[(int64_t)p * n + q]);
      }
      __syncthreads();
      // this CTA's row pairs: 2x2 blocks (k1, k2) of A, and rows p1, q1 of U^T
      for (int k1 = blockIdx.x; k1 < half; k1 += gridDim.x) {
        int p1, q1;
        pair_of_round(r, k1, np1, p1, q1);
        const Rot R1 = rot[k1];
        const double* op = Aold + (int64_t)p1 * n;
        const double* oq = Aold + (int64_t)q1 * n;
        double* np_ = Anew + (int64_t)p1 * n;
        double* nq_ = Anew + (int64_t)q1 * n;
        for (int k2 = threadIdx.x; k2 < half; k2 += kJThreads) {
          int p2, q2;
          pair_of_round(r, k2, np1, p2, q2);
          const Rot R2 = rot[k2];
          const double bpp = op[p2], bpq = op[q2], bqp = oq[p2], bqq = oq[q2];
          // rows: J1^T B
          const double rpp = R1.c * bpp - R1.s * bqp, rpq = R1.c * bpq - R1.s * bqq;
          const double rqp = R1.s * bpp + R1.c * bqp, rqq = R1.s * bpq + R1.c * bqq;
          // columns: (J1^T B) J2
          np_[p2] = R2.c * rpp - R2.s * rpq;
          np_[q2] = R2.s * rpp + R2.c * rpq;
          nq_[p2] = R2.c * rqp - R2.s * rqq;
          nq_[q2] = R2.s * rqp + R2.c * rqq;
        }
        // U^T <- J1^T U^T on rows p1, q1 (owned by this CTA alone)
        double* up = Ut + (int64_t)p1 * n;
        double* uq = Ut + (int64_t)q1 * n;
        for (int j = threadIdx.x; j < n; j += kJThreads) {
          const double a = up[j], b = uq[j];
          up[j] = R1.c * a - R1.s * b;
          uq[j] = R1.s * a + R1.c * b;
        }
      }
      grid_barrier(ctl, ctl + 1);
      double* t = Aold; Aold = Anew; Anew = t;
    }
  }
  for (int i = blockIdx.x * kJThreads + threadIdx.x; i < n; i += gridDim.x * kJThreads) wraw[i] = Aold[(int64_t)i * n + i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    info[0] = sweep;
    info[1] = sweep < max_sweeps ? 0 : 1;   // 1: not converged within max_sweeps
  }
}

// eigenvalues (diag of the converged A), sorted descending with their indices; n_sort = pow2 >= n
__global__ void sort_desc_kernel(const double* __restrict__ wraw, int n_real, int n_sort, double* __restrict__ w,
                                 int* __restrict__ idx) {
  extern __shared__ unsigned char sm_raw[];
  double* key = reinterpret_cast<double*>(sm_raw);
  int* id = reinterpret_cast<int*>(key + n_sort);
  for (int i = threadIdx.x; i < n_sort; i += blockDim.x) {
    key[i] = i < n_real ? wraw[i] : -INFINITY;   // padding sorts last
    id[i] = i;
  }
  __syncthreads();
  for (int size = 2; size <= n_sort; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n_sort; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
          // descending blocks: larger first; ties broken by index for determinism
          const bool gt = key[i] > key[j] || (key[i] == key[j] && id[i] < id[j]);
          if (desc != gt) {
            const double tk = key[i]; key[i] = key[j]; key[j] = tk;
            const int ti = id[i]; id[i] = id[j]; id[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n_real; i += blockDim.x) {
    w[i] = key[i];
    idx[i] = id[i];
  }
}

// U (n_real x n_real, row-major, column j = eigenvector of w[j]) from U^T rows in sorted order
__global__ void gather_u_kernel(const double* __restrict__ Ut, int n, int n_real, const int* __restrict__ idx,
                                double* __restrict__ U, int64_t ldu) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n_real * n_real) return;
  const int i = (int)(e / n_real), j = (int)(e % n_real);
  U[i * ldu + j] = Ut[(int64_t)idx[j] * n + i];
}

// full symmetric matrix from the packed lower Gram (exactly symmetric, as solvers.py:259's
// 0.5 (G + G^T) makes it), zero padding row/column
__global__ void init_eig_kernel(const double* __restrict__ Gp, int n_real, int n, double* __restrict__ A0,
                                double* __restrict__ Ut) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * n) return;
  const int64_t i = e / n, j = e % n;
  const int64_t hi = i > j ? i : j, lo = i > j ? j : i;
  A0[e] = (i < n_real && j < n_real) ? Gp[hi * (hi + 1) / 2 + lo] : 0.0;
  Ut[e] = (i == j) ? 1.0 : 0.0;
}

// z = U_r diag(1 / (w_j + lam)) U_r^T u over the r leading eigenpairs (the eigh route's
// x = V (s^2+lam)^-1 V^T v + (v - V V^T v)/lam == (v - S^T z)/lam with z = -lam * that; here
// the sign is folded: z is returned as (G + lam I)^-1 u restricted to the kept subspace)
__global__ void eig_apply_t_kernel(const double* __restrict__ U, int64_t ldu, int n, int r, const double* __restrict__ u,
                                   const double* __restrict__ w, double lam, double* __restrict__ t) {
  // one warp per eigenvector j: t_j = (U[:, j] . u) / (max(w_j, 0) + lam)
  const int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= r) return;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s = fma(U[(int64_t)i * ldu + j], u[i], s);
  s = warp_sum(s);
  if (lane == 0) t[j] = s / (fmax(w[j], 0.0) + lam);
}
__global__ void eig_apply_z_kernel(const double* __restrict__ U, int64_t ldu, int n, int r, const double* __restrict__ t,
                                   double* __restrict__ z) {
  // one warp per row i: z_i = U[i, :r] . t
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n) return;
  double s = 0.0;
  for (int j = lane; j < r; j += 32) s = fma(U[(int64_t)i * ldu + j], t[j], s);
  s = warp_sum(s);
  if (lane == 0) z[i] = s;
}

}  // namespace

size_t syevj_workspace_bytes(int64_t n, int num_sms) {
  const int64_t np = (n + 1) & ~(int64_t)1;
  return (size_t)3 * np * np * sizeof(double) + (size_t)num_sms * sizeof(double) + (size_t)np * (sizeof(double) + 4) +
         64;
}

int64_t syevj_max_n() { return 8192; }

cudaError_t eig_apply(const double* U, int64_t ldu, int64_t n, int64_t r, const double* u, const double* w, double lam,
                      double* t, double* z, cudaStream_t st, int* launches) {
  if (r > 0) eig_apply_t_kernel<<<(unsigned)((r + 7) / 8), 256, 0, st>>>(U, ldu, (int)n, (int)r, u, w, lam, t);
  eig_apply_z_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(U, ldu, (int)n, (int)r, t, z);
  if (launches) *launches += r > 0 ? 2 : 1;
  return cudaGetLastError();
}

cudaError_t syevj(const double* Gp, int64_t n, double* w, double* U, int64_t ldu, int max_sweeps, double tol,
                  void* ws, int num_sms, int* d_info, cudaStream_t st, int* launches) {
  if (n < 1 || n > syevj_max_n()) return cudaErrorInvalidValue;
  const int np = (int)((n + 1) & ~(int64_t)1);
  double* A0 = reinterpret_cast<double*>(ws);
  double* A1 = A0 + (size_t)np * np;
  double* Ut = A1 + (size_t)np * np;
  double* partial = Ut + (size_t)np * np;
  double* wraw = partial + num_sms;
  int* idx = reinterpret_cast<int*>(wraw + np);
  unsigned* ctl = reinterpret_cast<unsigned*>(idx + np);
  cudaError_t e = cudaMemsetAsync(ctl, 0, 2 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  const int64_t tot = (int64_t)np * np;
  init_eig_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Gp, (int)n, np, A0, Ut);
  const size_t smem = (size_t)(np / 2) * sizeof(Rot);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(sort_desc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 8192);
    attr = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_kernel, kJThreads, smem);
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int npi = np;
  void* args[] = {&A0, &A1, &Ut, &npi, &max_sweeps, &tol, &partial, &ctl, &d_info, &wraw};
  e = cudaLaunchCooperativeKernel((const void*)jacobi_kernel, dim3(num_sms), dim3(kJThreads), args, smem, st);
  if (e != cudaSuccess) return e;
  int n_sort = 1;
  while (n_sort < np) n_sort <<= 1;
  sort_desc_kernel<<<1, 1024, (size_t)n_sort * 12, st>>>(wraw, (int)n, n_sort, w, idx);
  gather_u_kernel<<<(unsigned)((n * n + 255) / 256), 256, 0, st>>>(Ut, np, (int)n, idx, U, ldu);
  if (launches) *launches += 4;
  return cudaGetLastError();
}

}  // namespace fs
