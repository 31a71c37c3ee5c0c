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
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace fs {
namespace {

constexpr int kJThreads = 512;

FS_DEVINL unsigned long long ptx_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct Rot {
  double c, s;
};

FS_DEVINL void pair_of_round(int r, int k, int np1, int& p, int& q) {
  // players 0..np1 (np1 = n-1); position 0 of the top row is fixed at player np1.  0 <= r, k <
  // np1, so both sums wrap at most once: compare-and-subtract instead of an integer modulo (the
  // block kernel's inner sweep evaluates this five times per thread and round)
  const int a = r + k, b = r - k + np1;
  p = (k == 0) ? np1 : (a >= np1 ? a - np1 : a);
  q = b >= np1 ? b - np1 : b;
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

// The same rotation with the hardware reciprocal / reciprocal-sqrt approximations + Newton
// steps (~1 ulp) instead of the library's IEEE division and square root, whose special-case
// paths made the rotation the longest link of the block kernel's inner round.  Off-diagonals in
// the denormal range count as converged; a huge tau takes the asymptote t = 1 / (2 tau).
FS_DEVINL double rcp_fast(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}
FS_DEVINL double rsqrt_fast(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double h = 0.5 * d * y * y;
  y = y * (1.5 - h);
  h = 0.5 * d * y * y;
  return y * (1.5 - h);
}
FS_DEVINL Rot schur2_fast(double app, double aqq, double apq) {
  Rot R{1.0, 0.0};
  if (fabs(apq) > 1e-290) {
    const double tau = (aqq - app) * rcp_fast(2.0 * apq);
    const double at = fabs(tau);
    double t;
    if (at > 1e150) {
      t = 0.5 * rcp_fast(at);
    } else {
      const double x = fma(tau, tau, 1.0);
      t = rcp_fast(at + x * rsqrt_fast(x));    // x rsqrt(x) = sqrt(1 + tau^2)
    }
    if (!(tau >= 0.0)) t = -t;
    R.c = rsqrt_fast(fma(t, t, 1.0));
    R.s = t * R.c;
  }
  return R;
}

// grid barrier on a monotonic arrival counter (the launch is cooperative: all CTAs are
// co-resident): each CTA's thread 0 adds 1 with release semantics and waits, with acquire loads,
// for the count of this barrier's generation (target += gridDim.x per call; ctl is zeroed before
// the launch).  One L2 round trip per CTA instead of the sense-reversing barrier's atomic +
// generation flip + re-read (~3.2 -> ~2 us per barrier with 148 CTAs).
FS_DEVINL void grid_barrier(unsigned* count, unsigned& target) {
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

// A0/A1: n x n (n even), A0 holds the input; Ut: n x n, U^T (row i = eigenvector i at the end).
// partial: gridDim.x doubles; ctl: [count, gen]; info: [sweeps, final A index]
__global__ void __launch_bounds__(kJThreads, 1)
jacobi_kernel(double* __restrict__ A0, double* __restrict__ A1, double* __restrict__ Ut, int n, int max_sweeps,
              double tol, double* __restrict__ partial, unsigned* ctl, int* info, double* __restrict__ wraw) {
  extern __shared__ Rot rot[];           // n/2 rotations of the current round
  __shared__ double red[kJThreads / 32];
  unsigned bar_target = 0;
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
    grid_barrier(ctl, bar_target);
    double tot = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) tot += partial[b];
    grid_barrier(ctl, bar_target);          // partial[] may be overwritten afterwards
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
      grid_barrier(ctl, bar_target);
      double* t = Aold; Aold = Anew; Anew = t;
    }
  }
  for (int i = blockIdx.x * kJThreads + threadIdx.x; i < n; i += gridDim.x * kJThreads) wraw[i] = Aold[(int64_t)i * n + i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    info[0] = sweep;
    info[1] = sweep < max_sweeps ? 0 : 1;   // 1: not converged within max_sweeps
  }
}

// ---------------------------------------------------------------- block Jacobi (n >= 128)
// The scalar kernel above is latency-bound: n-1 rounds per sweep, each a full pass over A plus a
// grid barrier (~10 us at n = 1024: 11 sweeps = 110 ms).  The block version pairs 32-row blocks
// (round-robin over 2q = np/32 blocks, q pairs per round, 2q-1 rounds per sweep):
//   phase A  one CTA per pair: the 64 x 64 super-block [I J] x [I J] gets one inner cyclic Jacobi
//            sweep in shared memory (63 rounds of 32 disjoint rotations), accumulating V (64 x 64,
//            orthogonal); V^T goes to global memory
//   phase B  every 64 x 64 block (P1, P2 >= ... lower) of A: A'_{P1P2} = V1^T A_{P1P2} V2 (two DMMA
//            64^3 products, written to both triangles of the other buffer: exactly symmetric), and
//            every 64 x 64 block of U: U_{c,P2} <- U_{c,P2} V2 (in place)
// with a grid barrier after each phase.  Same rotations as scalar cyclic Jacobi, applied as
// tensor-core block products: the n^3 work per sweep runs on DMMA and a sweep costs 2q-1 rounds of
// (one inner sweep + two barriers) instead of np-1 fully serialised rounds.
constexpr int kBB = 32;                 // block rows
constexpr int kSB = 2 * kBB;            // super-block (pair) size
constexpr int kBP = kSB + 4;            // smem pitch of the DMMA tiles (conflict-free fragments, as potrf)
constexpr int kMP = kSB + 1;            // smem pitch of the inner-sweep matrices
constexpr int kBThreads = 256;
constexpr size_t kBSmemA = (size_t)3 * kSB * kMP * sizeof(double);           // M, M', V
constexpr size_t kBSmemB = (size_t)6 * kSB * kBP * sizeof(double);           // X, Vt1, Vt2, T + U's X, V
constexpr size_t kBSmem = kBSmemA > kBSmemB ? kBSmemA : kBSmemB;

// super-block row r (0..63) of pair (I, J) -> matrix row
FS_DEVINL int sb_row(int I, int J, int r) { return r < kBB ? I * kBB + r : J * kBB + r - kBB; }

// C (64 x 64, 4 x 4 per thread) = A B^T, both 64 x 64 row-major in smem (pitch kBP), fp64 tensor
// cores (mma.sync m8n8k4): warp w owns rows [16 (w/2), +16) x cols [32 (w%2), +32)
FS_DEVINL int bfrag_row(int i) { return ((threadIdx.x >> 5) >> 1) * 16 + 8 * (i >> 1) + ((threadIdx.x & 31) >> 2); }
FS_DEVINL int bfrag_col(int i, int j) { return ((threadIdx.x >> 5) & 1) * 32 + 8 * j + 2 * (threadIdx.x & 3) + (i & 1); }
FS_DEVINL void bgemm_nt(const double* A, const double* B, double acc[4][4]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32, fr = lane >> 2, fk = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < kSB; k0 += 4) {
    double a[2], b[4];
#pragma unroll
    for (int t = 0; t < 2; ++t) a[t] = A[(wr + 8 * t + fr) * kBP + k0 + fk];
#pragma unroll
    for (int t = 0; t < 4; ++t) b[t] = B[(wc + 8 * t + fr) * kBP + k0 + fk];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int u = 0; u < 4; ++u)
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
            : "+d"(acc[2 * t][u]), "+d"(acc[2 * t + 1][u])
            : "d"(a[t]), "d"(b[u]));
  }
}

// rows of pair P1 x columns of pair P2 of an np x np matrix -> smem (pitch kBP); transposed: the
// element (r, c) is stored at [c][r]
FS_DEVINL void load_pair_block(const double* __restrict__ M, int np, int I1, int J1, int I2, int J2, double* dst,
                               bool transposed) {
  for (int e = threadIdx.x; e < kSB * kSB; e += kBThreads) {
    const int r = e >> 6, c = e & 63;
    const double val = M[(int64_t)sb_row(I1, J1, r) * np + sb_row(I2, J2, c)];
    if (transposed) dst[c * kBP + r] = val;
    else dst[r * kBP + c] = val;
  }
}

// FS_SYEVJ_DBG: CTA 0's %globaltimer split of the rounds (phase A, barrier, phase B, barrier), ns
__device__ unsigned long long g_bj_time[4];


__global__ void __launch_bounds__(kBThreads, 1)
bjacobi_kernel(double* __restrict__ A0, double* __restrict__ A1, double* __restrict__ U, double* __restrict__ Vt,
               int np, int max_sweeps, double tol, double* __restrict__ partial, unsigned* ctl, int* info,
               double* __restrict__ wraw, int dbg) {
  extern __shared__ double bsm[];
  __shared__ double red[kBThreads / 32];
  unsigned bar_target = 0;
  unsigned long long tA = 0, tB1 = 0, tB = 0, tB2 = 0, t0 = 0, t1 = 0;
  auto now = [&]() -> unsigned long long { return dbg ? ptx_globaltimer() : 0ull; };
  const int nblk = np / kBB, q = nblk / 2, rounds = nblk - 1;
  double* Aold = A0;
  double* Anew = A1;
  auto frob = [&](const double* A, bool off_only) -> double {
    double s = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * kBThreads + threadIdx.x; e < (int64_t)np * np;
         e += (int64_t)gridDim.x * kBThreads) {
      const int i = (int)(e / np), j = (int)(e % np);
      if (!off_only || i != j) s += A[e] * A[e];
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kBThreads / 32; ++w) t += red[w];
      partial[blockIdx.x] = t;
    }
    grid_barrier(ctl, bar_target);
    double tot = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) tot += partial[b];
    grid_barrier(ctl, bar_target);
    return tot;
  };
  // U <- U V for every (64-row chunk c, pair P2) block of a round's rotations Vp (in place:
  // each block by one CTA), tasks spread over CTAs first, first + stride, ...
  auto u_update = [&](const double* Vp, int rr, int t0, int t1, int first, int stride) {
    if (first < 0) return;
    double* X = bsm + 4 * kSB * kBP;                 // past phase A's buffers (kBSmem holds both)
    double* V2t = X + kSB * kBP;
    for (int ut = t0 + first; ut < t1; ut += stride) {
      const int c = ut / q, P2 = ut % q;
      int I2, J2;
      pair_of_round(rr, P2, rounds, I2, J2);
      for (int e = threadIdx.x; e < kSB * kSB; e += kBThreads) {
        const int a = e >> 6, b = e & 63;
        X[a * kBP + b] = U[(int64_t)(c * kSB + a) * np + sb_row(I2, J2, b)];
        V2t[a * kBP + b] = Vp[(size_t)P2 * kSB * kSB + e];
      }
      __syncthreads();
      double acc[4][4];
      bgemm_nt(X, V2t, acc);                         // U' = U V2
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          U[(int64_t)(c * kSB + bfrag_row(i)) * np + sb_row(I2, J2, bfrag_col(i, j))] = acc[i][j];
      __syncthreads();
    }
  };
  int nround = 0, prev_r = 0;                        // rounds done (all sweeps), the last one's index
  // a round's U blocks [0, ndefer) are applied during the NEXT round's phase A by the CTAs the
  // inner sweeps leave idle (ten each at most: about one inner sweep's time), the rest in its phase B
  const int spare = (int)gridDim.x - q;
  const int ndefer = spare > 0 ? min(q * q, 10 * spare) : q * q;
  const double fro2 = frob(Aold, false);
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    const double off2 = frob(Aold, true);
    if (!(off2 > tol * tol * fro2)) break;
    for (int r = 0; r < rounds; ++r) {
      t0 = now();
      // ---------------- phase A: inner sweep of each pair's super-block; meanwhile the other
      // CTAs apply the PREVIOUS round's rotations to U (U feeds nothing inside the iteration) ----
      double* Vr = Vt + (size_t)(nround & 1) * q * kSB * kSB;             // this round's V^T
      const double* Vp = Vt + (size_t)((nround & 1) ^ 1) * q * kSB * kSB; // the previous round's
      if (nround > 0 && (int)gridDim.x > q) u_update(Vp, prev_r, 0, ndefer, (int)blockIdx.x - q, (int)gridDim.x - q);
      for (int P = blockIdx.x; P < q; P += gridDim.x) {
        int I, J;
        pair_of_round(r, P, rounds, I, J);
        double* M = bsm;
        double* M2 = bsm + kSB * kMP;
        double* V = bsm + 2 * kSB * kMP;
        const bool full = r == 0;
        for (int e = threadIdx.x; e < kSB * kSB; e += kBThreads) {
          const int a = e >> 6, b = e & 63;
          M[a * kMP + b] = Aold[(int64_t)sb_row(I, J, a) * np + sb_row(I, J, b)];
          if (full) V[a * kMP + b] = a == b ? 1.0 : 0.0;
        }
        __syncthreads();
        // every warp computes all 32 rotations of an inner round (lane k: pair k) and takes the
        // ones it needs by shuffle: one CTA barrier per inner round.  The first round of a sweep
        // runs the full cyclic sweep of the super-block (63 rounds: pairs inside I, inside J and
        // across); later rounds only the 1024 cross pairs (I_k, J_{(k+t) mod 32}), 32 rounds —
        // every index pair is still rotated at least once per outer sweep, as in cyclic Jacobi,
        // and the inner sweeps (the latency-bound phase) take half the rounds
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        auto inner_pair = [&](int ir, int k, int& p, int& qq) {
          if (full) pair_of_round(ir, k, kSB - 1, p, qq);
          else { p = k; qq = kBB + ((k + ir) & (kBB - 1)); }
        };
        // cross rounds: V in registers.  Lane k holds, for rows warp + 8 i, column k (the I half,
        // fixed) and column 32 + ((k + ir) mod 32) (the J half: its pair partner this round); after
        // the round the J column moves one lane down (shuffle), so V never touches shared memory
        // until the 32 rounds bring every J column back to lane k
        constexpr int kNV = kSB / (kBThreads / 32);
        double vI[kNV], vJ[kNV];
#pragma unroll
        for (int i = 0; i < kNV; ++i) {
          const int row = warp + (kBThreads / 32) * i;
          vI[i] = row == lane ? 1.0 : 0.0;
          vJ[i] = row == kBB + lane ? 1.0 : 0.0;
        }
        for (int ir = 0; ir < (full ? kSB - 1 : kBB); ++ir) {
          int pk, qk;
          inner_pair(ir, lane, pk, qk);
          const Rot Rk = schur2_fast(M[pk * kMP + pk], M[qk * kMP + qk], M[pk * kMP + qk]);
          // M' = J^T M J by 2 x 2 blocks (k1 = warp + 8 i, k2 = lane), and V <- V J (columns pk,
          // qk of rows warp + 8 i; each (row, pair) by one thread).  All shared loads of the round
          // are issued before any store: M / M2 swap every round and V is updated in place, so the
          // compiler cannot move a load above a store itself (each load -> FMA -> store chain
          // otherwise waits out the shared-memory latency in turn)
          constexpr int kNI = kBB / (kBThreads / 32);
          int p1[kNI], q1[kNI];
          double bpp[kNI], bpq[kNI], bqp[kNI], bqq[kNI], r1c[kNI], r1s[kNI], va[kNV], vb[kNV];
#pragma unroll
          for (int i = 0; i < kNI; ++i) {
            const int k1 = warp + (kBThreads / 32) * i;
            inner_pair(ir, k1, p1[i], q1[i]);
            bpp[i] = M[p1[i] * kMP + pk];
            bpq[i] = M[p1[i] * kMP + qk];
            bqp[i] = M[q1[i] * kMP + pk];
            bqq[i] = M[q1[i] * kMP + qk];
          }
          if (full) {
#pragma unroll
            for (int i = 0; i < kNV; ++i) {
              const int row = warp + (kBThreads / 32) * i;
              va[i] = V[row * kMP + pk];
              vb[i] = V[row * kMP + qk];
            }
          }
#pragma unroll
          for (int i = 0; i < kNI; ++i) {
            const int k1 = warp + (kBThreads / 32) * i;
            r1c[i] = __shfl_sync(0xffffffffu, Rk.c, k1);
            r1s[i] = __shfl_sync(0xffffffffu, Rk.s, k1);
          }
#pragma unroll
          for (int i = 0; i < kNI; ++i) {
            const double rpp = r1c[i] * bpp[i] - r1s[i] * bqp[i], rpq = r1c[i] * bpq[i] - r1s[i] * bqq[i];
            const double rqp = r1s[i] * bpp[i] + r1c[i] * bqp[i], rqq = r1s[i] * bpq[i] + r1c[i] * bqq[i];
            M2[p1[i] * kMP + pk] = Rk.c * rpp - Rk.s * rpq;
            M2[p1[i] * kMP + qk] = Rk.s * rpp + Rk.c * rpq;
            M2[q1[i] * kMP + pk] = Rk.c * rqp - Rk.s * rqq;
            M2[q1[i] * kMP + qk] = Rk.s * rqp + Rk.c * rqq;
          }
          if (full) {
#pragma unroll
            for (int i = 0; i < kNV; ++i) {
              const int row = warp + (kBThreads / 32) * i;
              V[row * kMP + pk] = Rk.c * va[i] - Rk.s * vb[i];
              V[row * kMP + qk] = Rk.s * va[i] + Rk.c * vb[i];
            }
          } else {
#pragma unroll
            for (int i = 0; i < kNV; ++i) {
              const double a = vI[i], b = vJ[i];
              vI[i] = Rk.c * a - Rk.s * b;
              vJ[i] = __shfl_sync(0xffffffffu, Rk.s * a + Rk.c * b, (lane + 1) & 31);
            }
          }
          __syncthreads();
          double* tmp = M; M = M2; M2 = tmp;
        }
        if (!full) {   // the register V (every J column back at lane k) -> shared
#pragma unroll
          for (int i = 0; i < kNV; ++i) {
            const int row = warp + (kBThreads / 32) * i;
            V[row * kMP + lane] = vI[i];
            V[row * kMP + kBB + lane] = vJ[i];
          }
          __syncthreads();
        }
        // V^T to global: Vt[P][i][j] = V[j][i]
        double* vt = Vr + (size_t)P * kSB * kSB;
        for (int e = threadIdx.x; e < kSB * kSB; e += kBThreads) vt[e] = V[(e & 63) * kMP + (e >> 6)];
        __syncthreads();
      }
      if (nround > 0 && (int)gridDim.x <= q) u_update(Vp, prev_r, 0, ndefer, (int)blockIdx.x, (int)gridDim.x);
      t1 = now(); tA += t1 - t0; t0 = t1;
      grid_barrier(ctl, bar_target);
      t1 = now(); tB1 += t1 - t0; t0 = t1;
      // ---------------- phase B: A' = J^T A J (lower pair blocks, mirrored) ----------------
      const int atasks = q * (q + 1) / 2;
      for (int task = blockIdx.x; task < atasks; task += gridDim.x) {
        double* X = bsm;
        double* V1t = bsm + kSB * kBP;
        double* V2t = bsm + 2 * kSB * kBP;
        double* T = bsm + 3 * kSB * kBP;
        double acc[4][4];
        if (task < atasks) {
          int P1 = (int)((sqrt(8.0 * (double)task + 1.0) - 1.0) * 0.5);
          while ((P1 + 1) * (P1 + 2) / 2 <= task) ++P1;
          while (P1 * (P1 + 1) / 2 > task) --P1;
          const int P2 = task - P1 * (P1 + 1) / 2;
          int I1, J1, I2, J2;
          pair_of_round(r, P1, rounds, I1, J1);
          pair_of_round(r, P2, rounds, I2, J2);
          // X^T (columns of P2 as rows) so that T = V1^T X is one A B^T product: T[i][j] =
          // sum_k V1t[i][k] Xt[j][k]
          load_pair_block(Aold, np, I1, J1, I2, J2, X, true);
          const double* v1 = Vr + (size_t)P1 * kSB * kSB;
          const double* v2 = Vr + (size_t)P2 * kSB * kSB;
          for (int e = threadIdx.x; e < kSB * kSB; e += kBThreads) {
            V1t[(e >> 6) * kBP + (e & 63)] = v1[e];
            // V2 itself (rows [k][j] = V2t[j][k]): stored so that T V2 = A B^T with B[j][k] = V2[k][j]
            V2t[(e >> 6) * kBP + (e & 63)] = v2[e];
          }
          __syncthreads();
          bgemm_nt(V1t, X, acc);                    // T = V1^T X
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) T[bfrag_row(i) * kBP + bfrag_col(i, j)] = acc[i][j];
          __syncthreads();
          bgemm_nt(T, V2t, acc);                    // A' = T V2
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int gr = sb_row(I1, J1, bfrag_row(i)), gc = sb_row(I2, J2, bfrag_col(i, j));
              Anew[(int64_t)gr * np + gc] = acc[i][j];
              if (P1 != P2) Anew[(int64_t)gc * np + gr] = acc[i][j];
            }
        }
        __syncthreads();
      }
      // the rest of this round's U blocks (after the A tasks: same CTAs, next free slots)
      u_update(Vr, r, ndefer, q * q, ((int)blockIdx.x + atasks) % (int)gridDim.x, (int)gridDim.x);
      t1 = now(); tB += t1 - t0; t0 = t1;
      grid_barrier(ctl, bar_target);
      t1 = now(); tB2 += t1 - t0;
      double* t = Aold; Aold = Anew; Anew = t;
      prev_r = r;
      ++nround;
    }
  }
  if (nround > 0) {                                   // the last round's rotations
    u_update(Vt + (size_t)((nround & 1) ^ 1) * q * kSB * kSB, prev_r, 0, ndefer, (int)blockIdx.x, (int)gridDim.x);
    grid_barrier(ctl, bar_target);
  }
  if (dbg && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == (unsigned)q)) {
    const int o = blockIdx.x == 0 ? 0 : 2;
    if (o == 0) { g_bj_time[0] = tA; g_bj_time[1] = tB1 + tB2; g_bj_time[2] = tB; }
    else g_bj_time[3] = tA;
  }
  for (int i = blockIdx.x * kBThreads + threadIdx.x; i < np; i += gridDim.x * kBThreads)
    wraw[i] = Aold[(int64_t)i * np + i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    info[0] = sweep;
    info[1] = sweep < max_sweeps ? 0 : 1;
  }
}

// U (n_real x n_real) from the block kernel's U (columns = eigenvectors) in sorted order
__global__ void gather_ucol_kernel(const double* __restrict__ Ub, int np, int n_real, const int* __restrict__ idx,
                                   double* __restrict__ U, int64_t ldu) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n_real * n_real) return;
  const int i = (int)(e / n_real), j = (int)(e % n_real);
  U[i * ldu + j] = Ub[(int64_t)i * np + idx[j]];
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
  const int64_t np = (n + kSB - 1) / kSB * kSB;   // covers the scalar kernel's even padding too
  return (size_t)3 * np * np * sizeof(double) + (size_t)2 * np * kSB * sizeof(double) /* Vt x 2 */ +
         (size_t)num_sms * sizeof(double) + (size_t)np * (sizeof(double) + 4) + 64;
}

bool syevj_block(int64_t n) {
  static const int env = getenv("FS_SYEVJ_BLOCK") ? atoi(getenv("FS_SYEVJ_BLOCK")) : 1;
  return env != 0 && n >= 2 * kSB;
}

int64_t syevj_max_n() { return 16384; }   // the one-CTA sort: 12 B x 16384 of shared memory

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
  if (syevj_block(n)) {
    const int np = (int)((n + kSB - 1) / kSB * kSB);
    double* A0 = reinterpret_cast<double*>(ws);
    double* A1 = A0 + (size_t)np * np;
    double* Ub = A1 + (size_t)np * np;
    double* Vt = Ub + (size_t)np * np;
    double* partial = Vt + (size_t)2 * np * kSB;
    double* wraw = partial + num_sms;
    int* idx = reinterpret_cast<int*>(wraw + np);
    unsigned* ctl = reinterpret_cast<unsigned*>(idx + np);
    cudaError_t e = cudaMemsetAsync(ctl, 0, 2 * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    const int64_t tot = (int64_t)np * np;
    init_eig_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Gp, (int)n, np, A0, Ub);   // U = I
    static bool battr = false;
    if (!battr) {
      cudaFuncSetAttribute(bjacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBSmem);
      cudaFuncSetAttribute(sort_desc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
      battr = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bjacobi_kernel, kBThreads, kBSmem);
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int npi = np;
    static const int dbg = getenv("FS_SYEVJ_DBG") ? atoi(getenv("FS_SYEVJ_DBG")) : 0;
    int dbgi = dbg;
    void* args[] = {&A0, &A1, &Ub, &Vt, &npi, &max_sweeps, &tol, &partial, &ctl, &d_info, &wraw, &dbgi};
    e = cudaLaunchCooperativeKernel((const void*)bjacobi_kernel, dim3(num_sms), dim3(kBThreads), args, kBSmem, st);
    if (e != cudaSuccess) return e;
    int n_sort = 1;
    while (n_sort < np) n_sort <<= 1;
    sort_desc_kernel<<<1, 1024, (size_t)n_sort * 12, st>>>(wraw, (int)n, n_sort, w, idx);
    gather_ucol_kernel<<<(unsigned)((n * n + 255) / 256), 256, 0, st>>>(Ub, np, (int)n, idx, U, ldu);
    if (launches) *launches += 4;
    if (dbg) {
      unsigned long long h[4] = {};
      cudaStreamSynchronize(st);
      cudaMemcpyFromSymbol(h, g_bj_time, sizeof h);
      fprintf(stderr, "bjacobi CTA 0: phase A %.2f ms, barriers %.2f ms, phase B %.2f ms; CTA q (U work) %.2f ms\n",
              h[0] * 1e-6, h[1] * 1e-6, h[2] * 1e-6, h[3] * 1e-6);
    }
    return cudaGetLastError();
  }
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
    cudaFuncSetAttribute(sort_desc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
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
