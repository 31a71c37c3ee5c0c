// trsv.cu — z <- L^-T (L^-1 z) with the lower Cholesky factor (fp64).
//
// Replaces solvers.py:111 (solve_triangular(L, t1, lower=True, trans='N')) and
// solvers.py:114 (trans='T') — the two LAPACK dtrtrs calls of _chol_apply.
// Blocked substitution over 64-row blocks using the inverted diagonal blocks Linv_BB that
// potrf already produced: each block step is an off-diagonal GEMV (coalesced row reads of L,
// L2-resident) followed by a 64x64 GEMV with Linv_BB — no dependent global-load chains.
// One CTA of 1024 threads; deterministic (fixed reduction order).
#include <stdio.h>
#include <stdlib.h>

#include <string.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

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

// Flag-chained variant: CTA B owns 64-row block B.  Forward: t_B = z_B - sum_{C<B} L_BC z'_C,
// each term applied as soon as CTA C publishes z'_C (release/acquire flag), then
// z'_B = Linv_BB t_B.  Backward: t_B = z'_B - sum_{C>B} L_CB^T z_C as the z_C are published,
// z_B = Linv_BB^T t_B.  The off-diagonal products of all blocks run in parallel; the critical
// path is one 64 x 64 GEMV + a flag hop per block and direction (the single-CTA kernel above
// streams all of L through one SM twice: 258 us at n = 1024).  Fixed accumulation order
// (C ascending / descending per thread): deterministic, identical z on every call.
constexpr int kFT = 256;                       // threads per CTA (8 warps)
constexpr int kFW = kFT / 32;

// The 8 rows' warp sums as a reduce-scatter butterfly: xor 16 / 8 / 4 each halve the values a
// lane carries (it keeps the half its partner sends), xor 2 / 1 finish the single value.  9
// fp64 shuffles per warp instead of 40 (the shuffle unit, not the latency, bounded the
// interleaved sums: ~0.7 us per block on the TRSV's critical path).  Lane l ends with the sum of
// row 4 ((l >> 4) & 1) + 2 ((l >> 3) & 1) + ((l >> 2) & 1).
FS_DEVINL double reduce_scatter8(const double (&v)[8], int lane) {
  const bool b4 = lane & 16, b2 = lane & 8, b1 = lane & 4;
  double h[4], q[2];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double send = b4 ? v[j] : v[j + 4], keep = b4 ? v[j + 4] : v[j];
    h[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double send = b2 ? h[j] : h[j + 2], keep = b2 ? h[j + 2] : h[j];
    q[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double r = (b1 ? q[1] : q[0]) + __shfl_xor_sync(0xffffffffu, b1 ? q[0] : q[1], 4);
  r += __shfl_xor_sync(0xffffffffu, r, 2);
  r += __shfl_xor_sync(0xffffffffu, r, 1);
  return r;
}


FS_DEVINL int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FS_DEVINL void st_rel(int* p, int v) { asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
FS_DEVINL void wait_flag(const int* p) {
  if (threadIdx.x == 0 && ld_acq(p) == 0) {
    // a peer that never publishes is a bug: trap after ~20 s instead of hanging the device
    const uint64_t t0 = fs::ptx::globaltimer();
    while (ld_acq(p) == 0) {
      __nanosleep(20);
      if (fs::ptx::globaltimer() - t0 > 20000000000ull) __trap();
    }
  }
  __syncthreads();
}

constexpr int kSP = kNB + 1;                   // smem pitch (doubles) of the preloaded 64 x 64 blocks

// z = Linv^T t (column c, rows c+q, c+q+4, ...): all 16 shared loads issued before the FMA chain
// (a data-dependent trip count kept each FMA waiting on its own loads; backward link 0.7 -> 0.5
// us).  The FMA order is the loop's: bit-identical.  (The forward z' = Linv t keeps its loop:
// unrolled, its 16 row loads per thread doubled the conflicting shared-memory traffic.)
FS_DEVINL double lcol_dot(const double* LI, const double* t, int c, int q) {
  double lv[16], tv[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int r = min(c + q + 4 * k, kNB - 1);
    lv[k] = LI[r * kSP + c];
    tv[k] = t[r];
  }
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (c + q + 4 * k < kNB) sum = fma(lv[k], tv[k], sum);
  return sum;
}

constexpr size_t kFlagSmem = 3 * (size_t)kNB * kSP * sizeof(double);

__global__ void __launch_bounds__(kFT, 1)
trsv_pair_flag_kernel(const double* __restrict__ L, int64_t n, int64_t ld, const double* __restrict__ Linv,
                      double* __restrict__ z, const int64_t* status, int* __restrict__ fflag, int* __restrict__ bflag) {
  extern __shared__ double fsm[];
  double* LI = fsm;                            // Linv_BB
  double* LP = LI + kNB * kSP;                 // L_{B,B-1}: the forward step on the critical path
  double* LN = LP + kNB * kSP;                 // L_{B+1,B}: the backward step on the critical path
  __shared__ double t[kNB], zin[kNB], ub[kNB];
  __shared__ double part[kFW][kNB];
  if (status && *(volatile const int64_t*)status != 0) return;   // uniform: every CTA returns
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (int)((n + kNB - 1) / kNB);
  const int B = blockIdx.x;
  const int64_t r0 = (int64_t)B * kNB;
  const int b = (int)(n - r0 < kNB ? n - r0 : kNB);
  const int bn = B + 1 < nb ? (int)(n - r0 - kNB < kNB ? n - r0 - kNB : kNB) : 0;   // rows of block B + 1
  // the blocks the two critical-path steps need do not depend on z: load them before any wait
  for (int e = threadIdx.x; e < kNB * kNB; e += kFT) {
    const int r = e >> 6, c = e & 63;
    LI[r * kSP + c] = Linv[(size_t)B * kNB * kNB + e];
    LP[r * kSP + c] = (B > 0 && r < b) ? L[(r0 + r) * ld + r0 - kNB + c] : 0.0;
    LN[r * kSP + c] = (r < bn && c < b) ? L[(r0 + kNB + r) * ld + r0 + c] : 0.0;
  }
  if (threadIdx.x < kNB) ub[threadIdx.x] = threadIdx.x < b ? z[r0 + threadIdx.x] : 0.0;   // u_B, off the chain
  __syncthreads();
  // ---------------- forward: rows r = warp + 8 i of block B, columns lane, lane + 32 ----------------
  double acc[kNB / kFW];
#pragma unroll
  for (int i = 0; i < kNB / kFW; ++i) acc[i] = 0.0;
  // off the critical path: the L_BC rows of the next published block are loaded (registers)
  // before waiting for its flag, so the L2 latency overlaps the wait
  double lrow[kNB / kFW][2];
  auto load_rows = [&](int C, double (&dst)[kNB / kFW][2]) {
#pragma unroll
    for (int i = 0; i < kNB / kFW; ++i) {
      const int r = warp + kFW * i;
      const double* row = L + (r0 + r) * ld + (int64_t)C * kNB;
      dst[i][0] = r < b ? row[lane] : 0.0;
      dst[i][1] = r < b ? row[lane + 32] : 0.0;
    }
  };
  if (B >= 2) load_rows(0, lrow);
  for (int C = 0; C < B - 1; ++C) {
    double nrow[kNB / kFW][2];
    if (C + 1 < B - 1) load_rows(C + 1, nrow);
    wait_flag(fflag + C);
    const int64_t c0 = (int64_t)C * kNB;
    const double z0 = z[c0 + lane], z1 = z[c0 + lane + 32];
#pragma unroll
    for (int i = 0; i < kNB / kFW; ++i) {
      acc[i] = fma(lrow[i][0], z0, acc[i]);
      acc[i] = fma(lrow[i][1], z1, acc[i]);
    }
    if (C + 1 < B - 1) {
#pragma unroll
      for (int i = 0; i < kNB / kFW; ++i) { lrow[i][0] = nrow[i][0]; lrow[i][1] = nrow[i][1]; }
    }
  }
  if (B > 0) {                                 // C = B - 1 from shared memory
    wait_flag(fflag + B - 1);
    if (threadIdx.x < kNB) zin[threadIdx.x] = z[r0 - kNB + threadIdx.x];
    __syncthreads();
    const double z0 = zin[lane], z1 = zin[lane + 32];
#pragma unroll
    for (int i = 0; i < kNB / kFW; ++i) {
      const int r = warp + kFW * i;
      acc[i] = fma(LP[r * kSP + lane], z0, acc[i]);
      acc[i] = fma(LP[r * kSP + lane + 32], z1, acc[i]);
    }
  }
  static_assert(kNB / kFW == 8, "the butterfly reduces 8 rows per warp");
  {
    const double sum = reduce_scatter8(acc, lane);
    const int r = warp + kFW * (4 * ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1) + ((lane >> 2) & 1));
    if ((lane & 3) == 0) t[r] = (r < b) ? ub[r] - sum : 0.0;
  }
  __syncthreads();
  {                                            // z'_B = Linv_BB t  (4 threads per row)
    const int r = threadIdx.x >> 2, q = threadIdx.x & 3;
    double sum = 0.0;
    for (int c = q; c <= r; c += 4) sum = fma(LI[r * kSP + c], t[c], sum);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (q == 0 && r < b) z[r0 + r] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_rel(fflag + B, 1);
  }
  // ---------------- backward: columns lane, lane + 32 of block B, rows of block C by warp ----------------
  double a0 = 0.0, a1 = 0.0;
  for (int C = nb - 1; C > B + 1; --C) {
    wait_flag(bflag + C);
    const int64_t c0 = (int64_t)C * kNB;
    const int bc = (int)(n - c0 < kNB ? n - c0 : kNB);
    for (int r = warp; r < bc; r += kFW) {
      const double zi = z[c0 + r];
      const double* row = L + (c0 + r) * ld + r0;
      if (lane < b) a0 = fma(row[lane], zi, a0);
      if (lane + 32 < b) a1 = fma(row[lane + 32], zi, a1);
    }
  }
  if (B + 1 < nb) {                            // C = B + 1 from shared memory
    wait_flag(bflag + B + 1);
    if (threadIdx.x < kNB) zin[threadIdx.x] = threadIdx.x < bn ? z[r0 + kNB + threadIdx.x] : 0.0;
    __syncthreads();
    for (int r = warp; r < bn; r += kFW) {
      const double zi = zin[r];
      a0 = fma(LN[r * kSP + lane], zi, a0);
      a1 = fma(LN[r * kSP + lane + 32], zi, a1);
    }
  }
  part[warp][lane] = a0;
  part[warp][lane + 32] = a1;
  __syncthreads();
  if (threadIdx.x < kNB) {
    const int c = threadIdx.x;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < kFW; ++w) sum += part[w][c];
    t[c] = (c < b) ? z[r0 + c] - sum : 0.0;
  }
  __syncthreads();
  {                                            // z_B = Linv_BB^T t
    const int c = threadIdx.x >> 2, q = threadIdx.x & 3;
    double sum = lcol_dot(LI, t, c, q);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (q == 0 && c < b) z[r0 + c] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_rel(bflag + B, 1);
  }
}

// Cluster variant (nb <= 16 blocks, one CTA per block, one thread-block cluster): the same
// substitution order, but every published block of z travels CTA-to-CTA through distributed
// shared memory — st.async of the 64 values into each consumer's buffer with that consumer's
// mbarrier completing on the bytes — instead of a global store, a release flag and an acquire
// poll on the other side.  A hop (receive, two 64 x 64 smem GEMVs, push) drops to ~1 us.
constexpr int kCMaxNb = 16;
constexpr size_t kClusterSmem = 3 * (size_t)kNB * kSP * sizeof(double) + 2 * (size_t)kCMaxNb * kNB * sizeof(double);

FS_DEVINL void st_async_f64(uint32_t addr, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(addr), "d"(v),
               "r"(bar) : "memory");
}

__device__ unsigned long long g_trsv_t[kCMaxNb][4];   // FS_TRSV_DBG: per block fwd arrive/push, bwd arrive/push

__global__ void __launch_bounds__(kFT, 1)
trsv_pair_cluster_kernel(const double* __restrict__ L, int64_t n, int64_t ld, const double* __restrict__ Linv,
                         double* __restrict__ z, const int64_t* status, int dbg, const double* __restrict__ tfwd) {
  // tfwd != nullptr: backward solve only, L^T z = tfwd (the forward half already ran inside potrf)
  extern __shared__ double csm[];
  double* LI = csm;
  double* LP = LI + kNB * kSP;
  double* LN = LP + kNB * kSP;
  double* zf = LN + kNB * kSP;                 // [kCMaxNb][64] published z' blocks (forward)
  double* zb = zf + kCMaxNb * kNB;             // [kCMaxNb][64] published z blocks (backward)
  __shared__ __align__(8) uint64_t fbar[kCMaxNb], bbar[kCMaxNb];
  __shared__ double t[kNB], ub[kNB];
  __shared__ double part[kFW][kNB];
  const bool stop = status && *(volatile const int64_t*)status != 0;   // uniform over the cluster
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (int)((n + kNB - 1) / kNB);
  const int B = (int)fs::ptx::cluster_ctarank();
  const int64_t r0 = (int64_t)B * kNB;
  const int b = (int)(n - r0 < kNB ? n - r0 : kNB);
  const int bn = B + 1 < nb ? (int)(n - r0 - kNB < kNB ? n - r0 - kNB : kNB) : 0;
  if (threadIdx.x == 0) {
    for (int c = 0; c < nb; ++c) {
      fs::ptx::mbar_init(&fbar[c], 1);
      fs::ptx::mbar_init(&bbar[c], 1);
    }
    fs::ptx::fence_mbar_init();
    // each barrier completes once: on the 64 values of the block it names (one local arrival
    // carries the expected bytes, so a peer's bytes may land before it)
    for (int c = 0; c < B; ++c) fs::ptx::mbar_arrive_expect_tx(&fbar[c], kNB * 8);
    for (int c = B + 1; c < nb; ++c) fs::ptx::mbar_arrive_expect_tx(&bbar[c], kNB * 8);
  }
  for (int e = threadIdx.x; e < kNB * kNB; e += kFT) {
    const int r = e >> 6, c = e & 63;
    LI[r * kSP + c] = Linv[(size_t)B * kNB * kNB + e];
    LP[r * kSP + c] = (B > 0 && r < b && !tfwd) ? L[(r0 + r) * ld + r0 - kNB + c] : 0.0;   // forward only
    LN[r * kSP + c] = (r < bn && c < b) ? L[(r0 + kNB + r) * ld + r0 + c] : 0.0;
  }
  if (threadIdx.x < kNB) ub[threadIdx.x] = threadIdx.x < b ? z[r0 + threadIdx.x] : 0.0;   // u_B, off the chain
  fs::ptx::cluster_sync();                      // barriers armed everywhere before any push
  auto push = [&](double* buf, uint64_t* bars, int slot, int dst, double val, int c) {
    const uint32_t a = fs::ptx::mapa(fs::ptx::smem_u32(buf + slot * kNB + c), (uint32_t)dst);
    const uint32_t br = fs::ptx::mapa(fs::ptx::smem_u32(&bars[slot]), (uint32_t)dst);
    st_async_f64(a, val, br);
  };
  if (!stop && tfwd) {
    if (threadIdx.x < kNB) zf[B * kNB + threadIdx.x] = threadIdx.x < b ? tfwd[r0 + threadIdx.x] : 0.0;
    __syncthreads();
  }
  if (!stop && !tfwd) {
    // ---------------- forward ----------------
    double acc[kNB / kFW];
#pragma unroll
    for (int i = 0; i < kNB / kFW; ++i) acc[i] = 0.0;
    // off the critical path: the L_BC rows of the next block C are loaded (registers) before
    // waiting for z'_C, so the L2 latency overlaps the wait; C = B-1 comes from shared memory
    double lrow[kNB / kFW][2];
    auto load_rows = [&](int C, double (&dst)[kNB / kFW][2]) {
#pragma unroll
      for (int i = 0; i < kNB / kFW; ++i) {
        const int r = warp + kFW * i;
        const double* row = L + (r0 + r) * ld + (int64_t)C * kNB;
        dst[i][0] = r < b ? row[lane] : 0.0;
        dst[i][1] = r < b ? row[lane + 32] : 0.0;
      }
    };
    if (B >= 2) load_rows(0, lrow);
    for (int C = 0; C < B - 1; ++C) {
      double nrow[kNB / kFW][2];
      if (C + 1 < B - 1) load_rows(C + 1, nrow);
      fs::ptx::mbar_wait(&fbar[C], 0);
      const double z0 = zf[C * kNB + lane], z1 = zf[C * kNB + lane + 32];
#pragma unroll
      for (int i = 0; i < kNB / kFW; ++i) {
        acc[i] = fma(lrow[i][0], z0, acc[i]);
        acc[i] = fma(lrow[i][1], z1, acc[i]);
      }
      if (C + 1 < B - 1) {
#pragma unroll
        for (int i = 0; i < kNB / kFW; ++i) { lrow[i][0] = nrow[i][0]; lrow[i][1] = nrow[i][1]; }
      }
    }
    if (B > 0) {                                // C = B - 1: the critical block, from shared memory
      fs::ptx::mbar_wait(&fbar[B - 1], 0);
      const double z0 = zf[(B - 1) * kNB + lane], z1 = zf[(B - 1) * kNB + lane + 32];
#pragma unroll
      for (int i = 0; i < kNB / kFW; ++i) {
        const int r = warp + kFW * i;
        acc[i] = fma(LP[r * kSP + lane], z0, acc[i]);
        acc[i] = fma(LP[r * kSP + lane + 32], z1, acc[i]);
      }
    }
    if (dbg && threadIdx.x == 0) g_trsv_t[B][0] = fs::ptx::globaltimer();
    {
      const double sum = reduce_scatter8(acc, lane);
      const int r = warp + kFW * (4 * ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1) + ((lane >> 2) & 1));
      if ((lane & 3) == 0) t[r] = (r < b) ? ub[r] - sum : 0.0;
    }
    __syncthreads();
    {                                           // z'_B = Linv_BB t, kept locally and pushed to B+1..
      const int r = threadIdx.x >> 2, q = threadIdx.x & 3;
      double sum = 0.0;
      for (int c = q; c <= r; c += 4) sum = fma(LI[r * kSP + c], t[c], sum);
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      if (q == 0) {
        const double zr = r < b ? sum : 0.0;
        zf[B * kNB + r] = zr;
        for (int d = B + 1; d < nb; ++d) push(zf, fbar, B, d, zr, r);
      }
    }
    __syncthreads();
    if (dbg && threadIdx.x == 0) g_trsv_t[B][1] = fs::ptx::globaltimer();
  }
  if (!stop) {
    // ---------------- backward ----------------
    double a0 = 0.0, a1 = 0.0;
    for (int C = nb - 1; C > B; --C) {
      fs::ptx::mbar_wait(&bbar[C], 0);
      const int64_t c0 = (int64_t)C * kNB;
      const int bc = (int)(n - c0 < kNB ? n - c0 : kNB);
      if (C == B + 1) {
        for (int r = warp; r < bn; r += kFW) {
          const double zi = zb[C * kNB + r];
          a0 = fma(LN[r * kSP + lane], zi, a0);
          a1 = fma(LN[r * kSP + lane + 32], zi, a1);
        }
      } else {
        for (int r = warp; r < bc; r += kFW) {
          const double zi = zb[C * kNB + r];
          const double* row = L + (c0 + r) * ld + r0;
          if (lane < b) a0 = fma(row[lane], zi, a0);
          if (lane + 32 < b) a1 = fma(row[lane + 32], zi, a1);
        }
      }
    }
    if (dbg && threadIdx.x == 0) g_trsv_t[B][2] = fs::ptx::globaltimer();
    part[warp][lane] = a0;
    part[warp][lane + 32] = a1;
    __syncthreads();
    if (threadIdx.x < kNB) {
      const int c = threadIdx.x;
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < kFW; ++w) sum += part[w][c];
      t[c] = (c < b) ? zf[B * kNB + c] - sum : 0.0;
    }
    __syncthreads();
    {                                           // z_B = Linv_BB^T t -> z, pushed to 0..B-1
      const int c = threadIdx.x >> 2, q = threadIdx.x & 3;
      double sum = lcol_dot(LI, t, c, q);
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      if (q == 0) {
        if (c < b) z[r0 + c] = sum;
        const double zc = c < b ? sum : 0.0;
        for (int d = 0; d < B; ++d) push(zb, bbar, B, d, zc, c);
      }
    }
    if (dbg && threadIdx.x == 0) g_trsv_t[B][3] = fs::ptx::globaltimer();
  }
  fs::ptx::cluster_sync();                      // no CTA leaves while a peer may still push to it
}


}  // namespace
bool trsv_cluster_ok(int64_t n);
namespace {

// The pair on one thread-block cluster of nb CTAs (nb <= 16; non-portable above 8), or
// cudaErrorNotSupported when that cluster cannot be used (the caller falls back).  tfwd: the
// backward half only, from the forward result tfwd.
cudaError_t launch_cluster(const double* L, int64_t n, int64_t ldL, const double* Linv, double* z,
                           const int64_t* d_status, cudaStream_t st, int* launches, const double* tfwd) {
  if (!trsv_cluster_ok(n)) return cudaErrorNotSupported;   // attributes + schedulability, cached per nb
  const int64_t nb = (n + kNB - 1) / kNB;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3((unsigned)nb);
  cfg.blockDim = dim3(kFT);
  cfg.dynamicSmemBytes = kClusterSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)nb;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static const int dbg = getenv("FS_TRSV_DBG") ? atoi(getenv("FS_TRSV_DBG")) : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, trsv_pair_cluster_kernel, L, n, ldL, Linv, z, d_status, dbg, tfwd);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cudaErrorNotSupported;
  }
  if (launches) *launches += 1;
  if (dbg) {
    unsigned long long h[kCMaxNb][4] = {};
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_trsv_t, sizeof h);
    const unsigned long long t0 = h[0][0];
    for (int B = 0; B < (int)nb; ++B)
      fprintf(stderr, "trsv block %2d: fwd ready %6.2f pushed %6.2f | bwd ready %6.2f pushed %6.2f us\n", B,
              (h[B][0] - t0) * 1e-3, (h[B][1] - t0) * 1e-3, (h[B][2] - t0) * 1e-3, (h[B][3] - t0) * 1e-3);
  }
  return cudaGetLastError();
}

}  // namespace

// Whether the cluster kernel can run the pair (or its backward half) for this n: nb in [2, 16],
// the attributes set and a cluster of nb CTAs schedulable.  Cached per nb.
bool trsv_cluster_ok(int64_t n) {
  static const int cl_env = getenv("FS_TRSV_CLUSTER") ? atoi(getenv("FS_TRSV_CLUSTER")) : 1;
  static int ok[kCMaxNb + 1] = {};                 // 0 unknown, 1 yes, -1 no
  const int64_t nb = (n + kNB - 1) / kNB;
  if (!cl_env || nb < 2 || nb > kCMaxNb) return false;
  if (ok[nb] == 0) {
    bool good = cudaFuncSetAttribute(trsv_pair_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kClusterSmem) == cudaSuccess &&
                cudaFuncSetAttribute(trsv_pair_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                    cudaSuccess;
    if (good) {
      cudaLaunchConfig_t cfg;
      memset(&cfg, 0, sizeof cfg);
      cfg.gridDim = dim3((unsigned)nb);
      cfg.blockDim = dim3(kFT);
      cfg.dynamicSmemBytes = kClusterSmem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)nb;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int clusters = 0;
      good = cudaOccupancyMaxActiveClusters(&clusters, trsv_pair_cluster_kernel, &cfg) == cudaSuccess && clusters >= 1;
    }
    cudaGetLastError();
    ok[nb] = good ? 1 : -1;
  }
  return ok[nb] == 1;
}

// The backward half on the cluster from the forward result t (potrf's fused forward solve):
// z = L^-T t.  Call only when trsv_cluster_ok(n).
cudaError_t trsv_backward_cluster(const double* L, int64_t n, int64_t ldL, const double* Linv, const double* t,
                                  double* z, const int64_t* d_status, cudaStream_t st, int* launches) {
  if (!trsv_cluster_ok(n)) return cudaErrorNotSupported;
  return launch_cluster(L, n, ldL, Linv, z, d_status, st, launches, t);
}

cudaError_t trsv_pair(const double* L, int64_t n, int64_t ldL, const double* Linv, double* z,
                      const int64_t* d_status, cudaStream_t st, int* launches) {
  const int64_t nb = (n + kNB - 1) / kNB;
  static const int env = getenv("FS_TRSV_FLAGS") ? atoi(getenv("FS_TRSV_FLAGS")) : 1;
  static const int cl_env = getenv("FS_TRSV_CLUSTER") ? atoi(getenv("FS_TRSV_CLUSTER")) : 1;
  if (env && cl_env) {
    const cudaError_t e = launch_cluster(L, n, ldL, Linv, z, d_status, st, launches, nullptr);
    if (e != cudaErrorNotSupported) return e;
  }
  // every block's CTA must be resident while earlier ones spin on its flags: nb <= (CTAs per SM)
  // x SMs (2 per SM: ~100 KB of shared memory each; n <= 18944 on 148 SMs).  Linv is the potrf
  // scratch, the flags sit at its end.
  static int resident = -1;
  if (resident < 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(trsv_pair_flag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFlagSmem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trsv_pair_flag_kernel, kFT, kFlagSmem) != cudaSuccess)
      per_sm = 0;
    cudaGetLastError();
    resident = per_sm * sms;
  }
  if (env && nb >= 2 && nb <= resident) {
    int* flags = reinterpret_cast<int*>(const_cast<double*>(Linv) + potrf_trsv_flags_offset(n));
    cudaError_t e = cudaMemsetAsync(flags, 0, 2 * nb * sizeof(int), st);
    if (e != cudaSuccess) return e;
    static bool attr = false;
    if (!attr) {
      e = cudaFuncSetAttribute(trsv_pair_flag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFlagSmem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    trsv_pair_flag_kernel<<<(unsigned)nb, kFT, kFlagSmem, st>>>(L, n, ldL, Linv, z, d_status, flags, flags + nb);
  } else {
    trsv_pair_kernel<<<1, kThreads, 0, st>>>(L, n, ldL, Linv, z, d_status);
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace fs
