// svd.cu — the kernels of the direct-SVD comparison route ("svda").
//
// The reference's thin_svd_direct calls np.linalg.svd -> LAPACK dgesdd on S (solvers.py:280-291).
// The B200 route never touches an n x m matrix except through the Gram SYRK and fs_apply_rows:
//   shifted CholeskyQR3 of S^T (Fukaya et al. 2020):  S = L Q^T with Q^T Q = I, L lower n x n
//     G = S S^T + s I, L1 = chol(G), Q1^T = L1^-1 S, then twice L_k = chol(Q^T Q), Q^T <- L_k^-1 Q^T
//   one-sided Jacobi SVD of the n x n triangular factor: L = W diag(sigma) Z^T
//   => S = W diag(sigma) (Q Z)^T:  U = W, V^T = Z^T Q^T.
// This file holds the two n x n pieces: the triangular inverse (for Q^T = L^-1 Q^T on the tensor
// cores) and the one-sided (Hestenes) Jacobi SVD, which works on L's columns directly so the
// condition number is not squared (a Gram eigendecomposition would lose every sigma below
// sqrt(u) sigma_max).
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace fs {
namespace {

// ---- triangular inverse: Xt[j][:] = (L^-1 e_j)^T, i.e. row j of Xt = column j of L^-1 ----
// One warp per column j: forward substitution x_i = (delta_ij - sum_{j<=k<i} L_ik x_k) / L_ii,
// the dot product over a contiguous stretch of L's row i (lanes stride k, warp-sum).
__global__ void tri_inverse_kernel(const double* __restrict__ L, int64_t n, int64_t ldL, double* __restrict__ Xt) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += warps) {
    double* x = Xt + j * n;
    for (int64_t i = lane; i < j; i += 32) x[i] = 0.0;
    for (int64_t i = j; i < n; ++i) {
      const double* l = L + i * ldL;
      double s = 0.0;
      for (int64_t k = j + lane; k < i; k += 32) s = fma(l[k], x[k], s);
      s = warp_sum(s);
      if (lane == 0) x[i] = ((i == j ? 1.0 : 0.0) - s) / l[i];
      __syncwarp();
    }
  }
}

__global__ void transpose_kernel(const double* __restrict__ in, int64_t rows, int64_t cols, int64_t ldi,
                                 double* __restrict__ out, int64_t ldo) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (r < rows && c < cols) ? in[r * ldi + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = c0 + k, c = r0 + threadIdx.x;   // out[r][c] = in[c][r]
    if (r < cols && c < rows) out[r * ldo + c] = tile[threadIdx.x][k];
  }
}

// ---- one-sided Jacobi SVD ----
constexpr int kSThreads = 512;

FS_DEVINL void round_pair(int r, int k, int np1, int& p, int& q) {
  p = (k == 0) ? np1 : (r + k) % np1;
  q = (r - k + np1) % np1;
}

// grid barrier on a monotonic arrival counter (cooperative launch; ctl zeroed before it): thread
// 0 adds 1 with release semantics and polls with acquire loads for this generation's count
FS_DEVINL void grid_sync(unsigned* count, unsigned& target) {
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

// B: np x np (rows = columns of the input A; padding rows zero), Vt: np x np (identity at the
// start).  Each round rotates the np/2 disjoint row pairs (p, q) of the round-robin schedule, one
// TEAM of tw warps per pair (tw = 1, 2, 4 or 8 so that the teams cover the pairs): each warp
// forms its segment's alpha = |b_p|^2, beta = |b_q|^2, gamma = b_p . b_q, the team adds the
// segments in fixed order through shared memory (one named barrier), and when |gamma| > tol
// sqrt(alpha beta) every warp applies the Rutishauser rotation to its segment of rows p, q of B
// and of Vt.  (One warp per pair left a round L2-latency bound: 32 dependent load steps per lane;
// four warps per pair at n = 1024 give 8, with 128 instead of 32 CTAs.)  A sweep with no rotation
// ends the iteration.  ctl: [count, gen, rotations(sweep parity 0/1)]; info: [sweeps, not
// converged].
__global__ void __launch_bounds__(kSThreads, 1)
jacobi_svd_kernel(double* __restrict__ B, double* __restrict__ Vt, int np, int max_sweeps, double tol, unsigned* ctl,
                  int* info, int tw) {
  __shared__ double part[2][kSThreads / 32][3];          // [round parity][warp][a, b, g]
  const int half = np / 2, np1 = np - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int teams_total = gridDim.x * (kSThreads / 32) / tw;
  const int team = (blockIdx.x * (kSThreads / 32) + warp) / tw, w_in = warp % tw;
  const int team0 = warp - w_in;                         // the team's first warp in this CTA
  unsigned* rotations = ctl + 2;
  unsigned bar_target = 0;
  int sweep = 0, par = 0;
  bool converged = false;
  for (; sweep < max_sweeps && !converged; ++sweep) {
    unsigned* cnt = rotations + (sweep & 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) rotations[(sweep + 1) & 1] = 0u;   // next sweep's counter
    for (int r = 0; r < np1; ++r) {
      for (int k = team; k < half; k += teams_total) {
        int p, q;
        round_pair(r, k, np1, p, q);
        double* bp = B + (int64_t)p * np;
        double* bq = B + (int64_t)q * np;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = w_in * 32 + lane; i < np; i += 32 * tw) {
          const double x = bp[i], y = bq[i];
          a = fma(x, x, a);
          b = fma(y, y, b);
          g = fma(x, y, g);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        if (tw > 1) {
          if (lane == 0) { part[par][warp][0] = a; part[par][warp][1] = b; part[par][warp][2] = g; }
          asm volatile("bar.sync %0, %1;" ::"r"(1 + team0 / tw), "r"(32 * tw) : "memory");
          a = b = g = 0.0;
          for (int w = 0; w < tw; ++w) {                 // fixed order: identical in every warp
            a += part[par][team0 + w][0];
            b += part[par][team0 + w][1];
            g += part[par][team0 + w][2];
          }
          par ^= 1;   // the next pair's partials go to the other buffer (no second barrier)
        }
        if (fabs(g) > tol * sqrt(a * b) && g != 0.0) {
          const double zeta = (b - a) / (2.0 * g);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int i = w_in * 32 + lane; i < np; i += 32 * tw) {
            const double x = bp[i], y = bq[i];
            bp[i] = c * x - s * y;
            bq[i] = s * x + c * y;
          }
          double* vp = Vt + (int64_t)p * np;
          double* vq = Vt + (int64_t)q * np;
          for (int i = w_in * 32 + lane; i < np; i += 32 * tw) {
            const double x = vp[i], y = vq[i];
            vp[i] = c * x - s * y;
            vq[i] = s * x + c * y;
          }
          if (lane == 0 && w_in == 0) atomicAdd(cnt, 1u);
        }
      }
      grid_sync(ctl, bar_target);
    }
    converged = *(volatile unsigned*)cnt == 0u;
    grid_sync(ctl, bar_target);   // everyone read the counter before it is reset two sweeps on
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    info[0] = sweep;
    info[1] = converged ? 0 : 1;
  }
}

// sigma_i = |row i of B| (one warp per row)
__global__ void row_norms_kernel(const double* __restrict__ B, int np, int n, double* __restrict__ sig) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n) return;
  double s = 0.0;
  for (int k = lane; k < np; k += 32) s = fma(B[(int64_t)i * np + k], B[(int64_t)i * np + k], s);
  s = warp_sum(s);
  if (lane == 0) sig[i] = sqrt(s);
}

// descending sort of n keys with indices (bitonic, one CTA; n_sort = pow2 >= n)
__global__ void sort_desc_idx_kernel(const double* __restrict__ keys, int n, int n_sort, double* __restrict__ out,
                                     int* __restrict__ idx) {
  extern __shared__ unsigned char sm_raw[];
  double* key = reinterpret_cast<double*>(sm_raw);
  int* id = reinterpret_cast<int*>(key + n_sort);
  for (int i = threadIdx.x; i < n_sort; i += blockDim.x) {
    key[i] = i < n ? keys[i] : -INFINITY;
    id[i] = i;
  }
  __syncthreads();
  for (int size = 2; size <= n_sort; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n_sort; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
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
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    out[i] = key[i];
    idx[i] = id[i];
  }
}

// sorted factors: U[:, j] = B[idx_j, :n] / sigma_j (n x n, row-major, ldu), Zt[j, :] = Vt[idx_j, :n]
__global__ void gather_svd_kernel(const double* __restrict__ B, const double* __restrict__ Vt, int np, int n,
                                  const int* __restrict__ idx, const double* __restrict__ sig, double* __restrict__ U,
                                  int64_t ldu, double* __restrict__ Zt, int64_t ldz) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * n) return;
  const int a = (int)(e / n), b = (int)(e % n);
  // U[a][b] = B[idx_b][a] / sig_b ; Zt[a][b] = Vt[idx_a][b]
  const double sb = sig[b];
  U[a * ldu + b] = sb > 0.0 ? B[(int64_t)idx[b] * np + a] / sb : 0.0;
  Zt[a * ldz + b] = Vt[(int64_t)idx[a] * np + b];
}

__global__ void init_svd_kernel(const double* __restrict__ A, int64_t n, int64_t lda, int np, double* __restrict__ B,
                                double* __restrict__ Vt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)np * np) return;
  const int64_t i = e / np, j = e % np;
  // B = A^T (row i of B = column i of A), zero padding
  B[e] = (i < n && j < n) ? A[j * lda + i] : 0.0;
  Vt[e] = (i == j) ? 1.0 : 0.0;
}

}  // namespace

cudaError_t tri_inverse(const double* L, int64_t n, int64_t ldL, double* Linv, int64_t ldo, double* scratch,
                        int num_sms, cudaStream_t st, int* launches) {
  if (n < 1) return cudaErrorInvalidValue;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 7) / 8, (int64_t)num_sms * 4);
  tri_inverse_kernel<<<blocks, 256, 0, st>>>(L, n, ldL, scratch);
  dim3 tb(32, 8), tg((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  transpose_kernel<<<tg, tb, 0, st>>>(scratch, n, n, n, Linv, ldo);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

size_t jacobi_svd_workspace_bytes(int64_t n) {
  const int64_t np = (n + 1) & ~(int64_t)1;
  return (size_t)2 * np * np * sizeof(double) + (size_t)np * (sizeof(double) + sizeof(int)) + 64;
}

cudaError_t jacobi_svd(const double* A, int64_t n, int64_t lda, double* sigma, double* U, int64_t ldu, double* Zt,
                       int64_t ldz, int max_sweeps, double tol, void* ws, int num_sms, int* d_info, cudaStream_t st,
                       int* launches) {
  if (n < 1 || n > 16384) return cudaErrorInvalidValue;
  const int np = (int)((n + 1) & ~(int64_t)1);
  double* B = reinterpret_cast<double*>(ws);
  double* Vt = B + (size_t)np * np;
  double* sraw = Vt + (size_t)np * np;
  int* idx = reinterpret_cast<int*>(sraw + np);
  unsigned* ctl = reinterpret_cast<unsigned*>(idx + np);
  cudaError_t e = cudaMemsetAsync(ctl, 0, 4 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  const int64_t tot = (int64_t)np * np;
  init_svd_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A, n, lda, np, B, Vt);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_svd_kernel, kSThreads, 0);
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  // warps per pair: the largest of 8, 4, 2, 1 whose teams still fit on the SMs (each pair gets a
  // team; a small n keeps few CTAs, which makes the grid barrier cheaper)
  const int wpc = kSThreads / 32;
  int tw = 8;
  while (tw > 1 && (int64_t)(np / 2) * tw > (int64_t)num_sms * wpc) tw >>= 1;
  const int want = std::max(1, std::min(num_sms, (int)(((int64_t)(np / 2) * tw + wpc - 1) / wpc)));
  int npi = np;
  void* args[] = {&B, &Vt, &npi, &max_sweeps, &tol, &ctl, &d_info, &tw};
  e = cudaLaunchCooperativeKernel((const void*)jacobi_svd_kernel, dim3(want), dim3(kSThreads), args, 0, st);
  if (e != cudaSuccess) return e;
  row_norms_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(B, np, (int)n, sraw);
  int n_sort = 1;
  while (n_sort < n) n_sort <<= 1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sort_desc_idx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
    attr = true;
  }
  sort_desc_idx_kernel<<<1, 1024, (size_t)n_sort * 12, st>>>(sraw, (int)n, n_sort, sigma, idx);
  gather_svd_kernel<<<(unsigned)((n * n + 255) / 256), 256, 0, st>>>(B, Vt, np, (int)n, idx, sigma, U, ldu, Zt, ldz);
  if (launches) *launches += 5;
  return cudaGetLastError();
}

}  // namespace fs
