// syrk_dmma.cu — exact-product fp64 Gram G = S S^T + λI on the fp64 tensor cores (DMMA).
//
// Replaces core.py:284-289 (numpy A @ A.T -> OpenBLAS dsyrk, symmetrize, += lam) for
// FS_PREC_FP64: every product s_ik * s_jk is an IEEE fp64 FMA (fp32 scores are widened
// exactly), i.e. the reference's own arithmetic — executed as mma.sync.m8n8k4.f64, the
// fp64 tensor-core instruction (tcgen05 has no fp64 kind on sm_100a).
//
// 128 x 128 lower tiles of G, 256 threads = 8 warps of 64 x 32 (8 x 4 MMA tiles of 8 x 8: 64
// fp64 accumulator registers per thread).  K advances in 32-column stages, double-buffered
// through shared memory: the next stage's global loads are issued into registers before the
// current stage's MMAs and stored after them.  Shared rows are 36 doubles apart, so the eight
// 32-byte fragment rows a warp reads hit distinct bank groups (two wavefronts, the minimum).
// Split-K over P CTAs per tile (contiguous column ranges) with a fixed-order fp64 reduction of
// the partial tiles: deterministic.  The roofline is the fp64 tensor rate; the loads are a few
// bytes per clock per SM.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>

namespace fs {
namespace {

constexpr int kT = 128;                 // tile edge
constexpr int kK = 32;                  // K columns per stage
constexpr int kLd = kK + 4;             // smem row pitch (doubles)
constexpr int kThreads = 256;
constexpr int kStageDoubles = 2 * kT * kLd;   // A and B
constexpr size_t kSmemBytes = 2 * kStageDoubles * sizeof(double);   // 147 KB

FS_DEVINL void tile_ij(int t, int& I, int& J) {   // lower tiles, row-major
  int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  I = i;
  J = t - i * (i + 1) / 2;
}

FS_DEVINL void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// One 32-column stage: 8 k-steps of the warp's 8 x 4 grid of m8n8k4 fp64 MMAs.  T = float: the
// stage holds the fp32 scores as they are and each fragment is widened on its way to the
// registers (exact) — half the shared-memory bytes of an fp64 stage.  Row pitch LD elements (36:
// the eight fragment rows of a load hit distinct banks in both widths).
template <typename T = double, int LD = kLd>
FS_DEVINL void stage_mma(double (&acc)[8][4][2], const T* A, const T* B, int wr, int wc, int fr, int fk) {
#pragma unroll
  for (int ks = 0; ks < kK; ks += 4) {
    double af[8], bf[4];
#pragma unroll
    for (int a = 0; a < 8; ++a) af[a] = (double)A[(wr + 8 * a + fr) * LD + ks + fk];
#pragma unroll
    for (int b = 0; b < 4; ++b) bf[b] = (double)B[(wc + 8 * b + fr) * LD + ks + fk];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma(acc[a][b], af[a], bf[b]);
  }
}

// Tile epilogue: packed lower G (+ lam on the diagonal) when the tile has one split, else the
// partial tile into the split-K workspace (row-major 128 x 128 per block).
FS_DEVINL void store_tile(const double (&acc)[8][4][2], int64_t rA, int64_t rB, int64_t n, double lam, double* ws,
                          double* Gp, int direct, int wr, int wc, int fr, int lane, int64_t ldc = 0) {
  // accumulator fragment (m8n8 f64): thread holds rows fr, columns 2*(lane&3) + {0,1}
  const int cc = 2 * (lane & 3);
  if (ldc > 0) {
    // trailing update of a blocked Cholesky: C (row-major, pitch ldc, lower) -= the tile
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t gi = rA + wr + 8 * a + fr, gj = rB + wc + 8 * b + cc + e;
          if (gi < n && gj <= gi) Gp[gi * ldc + gj] -= acc[a][b][e];
        }
  } else if (direct) {
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t gi = rA + wr + 8 * a + fr, gj = rB + wc + 8 * b + cc + e;
          if (gi < n && gj <= gi) Gp[gi * (gi + 1) / 2 + gj] = acc[a][b][e] + (gi == gj ? lam : 0.0);
        }
  } else {
    double* out = ws + (size_t)blockIdx.x * kT * kT;
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        *reinterpret_cast<double2*>(out + (wr + 8 * a + fr) * kT + wc + 8 * b + cc) =
            make_double2(acc[a][b][0], acc[a][b][1]);
  }
}

// Two-level accumulation.  One fp64 register chain over a 250k-column split accumulates ~sqrt(250k)
// ulps of rounding (4.8e-14 of the diagonal at 1024 x 1e6, 100x numpy's dgemm — enough to
// lift the solve's first-pass residual over the 1e-10 refinement threshold).  Every kFlush stages
// (2048 columns) each thread adds its registers into a private slot of the CTA's 128 x 128
// workspace tile (L2-resident; the split-K partial's own slot) and restarts them from zero, so
// the long chain runs over ~120 block sums instead of 250k products (error 8e-16 of the diagonal,
// numpy's level; Gram +4%, every 32 stages +8.5%).  All warps flush at the same stage (staggering
// them stalls every stage's barrier instead: 38 -> 52 ms).
constexpr int kFlush = 64;

FS_DEVINL void red_add_f64(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

FS_DEVINL void flush_acc(double (&acc)[8][4][2], double* buf, bool first, int wr, int wc, int fr, int lane) {
  const int cc = 2 * (lane & 3);
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      double* q = buf + (wr + 8 * a + fr) * kT + wc + 8 * b + cc;
      if (first) {
        *reinterpret_cast<double2*>(q) = make_double2(0.0 + acc[a][b][0], 0.0 + acc[a][b][1]);
      } else {
        // the add happens at L2 (no load round trip on the critical stage); one writer per
        // element, program order: the same fl(old + acc) as a read-modify-write
        red_add_f64(q, acc[a][b][0]);
        red_add_f64(q + 1, acc[a][b][1]);
      }
      acc[a][b][0] = acc[a][b][1] = 0.0;
    }
}

FS_DEVINL void unflush_acc(double (&acc)[8][4][2], const double* buf, int wr, int wc, int fr, int lane) {
  const int cc = 2 * (lane & 3);
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const double2 o = __ldcg(reinterpret_cast<const double2*>(buf + (wr + 8 * a + fr) * kT + wc + 8 * b + cc));
      acc[a][b][0] = o.x + acc[a][b][0];
      acc[a][b][1] = o.y + acc[a][b][1];
    }
}

// Stage loader: rows [r0, r0+128) x cols [k0, k0+32) of S -> 16 doubles per thread in registers.
// Thread t covers row (t >> 1) and 16 consecutive columns ((t & 1) * 16 ...).
template <typename T>
struct Loader {
  double v[16];
  FS_DEVINL void load(const T* __restrict__ S, int64_t n, int64_t kend, int64_t ldS, int64_t r0, int64_t k0,
                      bool vec) {
    const int r = threadIdx.x >> 1, c = (threadIdx.x & 1) * 16;
    const int64_t gr = r0 + r, gc = k0 + c;
    if (gr < n && vec && gc + 16 <= kend) {
      const T* p = S + gr * ldS + gc;
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
      for (int e = 0; e < 16; ++e) v[e] = (gr < n && gc + e < kend) ? (double)__ldg(S + gr * ldS + gc + e) : 0.0;
    }
  }
  FS_DEVINL void store(double* __restrict__ dst) const {
    const int r = threadIdx.x >> 1, c = (threadIdx.x & 1) * 16;
    double2* d = reinterpret_cast<double2*>(dst + r * kLd + c);
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = make_double2(v[2 * q], v[2 * q + 1]);
  }
};

template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
syrk_dmma_kernel(const T* __restrict__ S, int64_t n, int64_t m, int64_t ldS, int64_t kchunk, int P, double lam,
                 double* __restrict__ ws, double* __restrict__ Gp, int direct, int vec, int flush, int64_t ldc = 0,
                 const int64_t* status = nullptr, int jmax = 0) {
  if (status && *(volatile const int64_t*)status != 0) return;
  extern __shared__ __align__(16) double dsm[];
  int I, J;
  if (jmax > 0) {
    I = blockIdx.x / jmax;
    J = blockIdx.x % jmax;
    if (J > I) return;
  } else {
    tile_ij(blockIdx.x / P, I, J);
  }
  const int split = blockIdx.x % P;
  const bool diag = I == J;
  const int64_t kbeg = (int64_t)split * kchunk;
  const int64_t kend = std::min<int64_t>(m, kbeg + kchunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 2) * 64, wc = (warp & 3) * 32;   // warp tile origin (rows of A, rows of B)
  const int fr = lane >> 2, fk = lane & 3;                 // fragment row / k within an 8 x 4 slab
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  Loader<T> la, lb;
  const int64_t rA = (int64_t)I * kT, rB = (int64_t)J * kT;
  int buf = 0;
  if (kbeg < kend) {
    la.load(S, n, kend, ldS, rA, kbeg, vec);
    if (!diag) lb.load(S, n, kend, ldS, rB, kbeg, vec);
    la.store(dsm);
    if (!diag) lb.store(dsm + kT * kLd);
  }
  __syncthreads();
  double* fbuf = ws + (size_t)blockIdx.x * kT * kT;
  int since = 0;
  bool flushed = false;
  for (int64_t k0 = kbeg; k0 < kend; k0 += kK) {
    const bool more = k0 + kK < kend;
    if (more) {                                           // next stage -> registers
      la.load(S, n, kend, ldS, rA, k0 + kK, vec);
      if (!diag) lb.load(S, n, kend, ldS, rB, k0 + kK, vec);
    }
    const double* A = dsm + buf * kStageDoubles;
    stage_mma(acc, A, diag ? A : A + kT * kLd, wr, wc, fr, fk);
    if (more) {
      double* nxt = dsm + (buf ^ 1) * kStageDoubles;
      la.store(nxt);
      if (!diag) lb.store(nxt + kT * kLd);
    }
    __syncthreads();
    buf ^= 1;
    if (flush && ++since == kFlush && more) {
      flush_acc(acc, fbuf, !flushed, wr, wc, fr, lane);
      flushed = true;
      since = 0;
    }
  }
  if (flushed) unflush_acc(acc, fbuf, wr, wc, fr, lane);
  store_tile(acc, rA, rB, n, lam, ws, Gp, direct, wr, wc, fr, lane, ldc);
}

// Scores with 16-byte aligned rows: global -> shared with cp.async (no register staging, no
// store pass after the MMAs).  fp64: three stages in flight (3 x 72 KB); fp32: four (4 x 36 KB),
// the fp32 values staged as they are and widened per fragment.  Thread t copies the 16-byte pieces
// of its rows (8 per operand and stage in fp64, 4 in fp32); pieces past the last row or column
// are zero-filled (src-size).
template <typename T> struct Async;
template <> struct Async<double> { static constexpr int kStages = 3, kPieces = 16, kPerPiece = 2; };
template <> struct Async<float> { static constexpr int kStages = 4, kPieces = 8, kPerPiece = 4; };
template <typename T> constexpr int async_stage_elems() { return 2 * kT * kLd; }
template <typename T> constexpr size_t async_smem_bytes() {
  return (size_t)Async<T>::kStages * async_stage_elems<T>() * sizeof(T);   // 221 KB fp64, 147 KB fp32
}
constexpr size_t kAsyncSmemBytes = async_smem_bytes<double>();

FS_DEVINL void cp16(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

template <typename T>
FS_DEVINL void issue_stage(T* dst, const T* __restrict__ S, int64_t n, int64_t kend, int64_t ldS, int64_t r0,
                           int64_t k0) {
  constexpr int kPieces = Async<T>::kPieces, kPer = Async<T>::kPerPiece;
#pragma unroll
  for (int q = 0; q < kT * kPieces / kThreads; ++q) {
    const int piece = threadIdx.x + q * kThreads;       // 128 rows x kPieces pieces
    const int r = piece / kPieces, c = (piece % kPieces) * kPer;
    const int64_t gr = r0 + r, gc = k0 + c;
    const int64_t left = kend - gc;
    const int bytes = gr < n ? (int)(left >= kPer ? 16 : left > 0 ? left * (int64_t)sizeof(T) : 0) : 0;
    cp16(dst + r * kLd + c, bytes ? S + gr * ldS + gc : S, bytes);
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
syrk_dmma_async_kernel(const T* __restrict__ S, int64_t n, int64_t m, int64_t ldS, int64_t kchunk, int P,
                       double lam, double* __restrict__ ws, double* __restrict__ Gp, int direct, int flush,
                       int64_t ldc = 0, const int64_t* status = nullptr, int jmax = 0) {
  if (status && *(volatile const int64_t*)status != 0) return;
  constexpr int kAsyncStages = Async<T>::kStages;
  constexpr int kStageElems = async_stage_elems<T>();
  extern __shared__ __align__(16) unsigned char dsm_raw[];
  T* dsm = reinterpret_cast<T*>(dsm_raw);
  int I, J;
  if (jmax > 0) {            // column strip: tiles (I, J) with J < jmax, grid jmax x row tiles
    I = blockIdx.x / jmax;
    J = blockIdx.x % jmax;
    if (J > I) return;
  } else {
    tile_ij(blockIdx.x / P, I, J);
  }
  const int split = blockIdx.x % P;
  const bool diag = I == J;
  const int64_t kbeg = (int64_t)split * kchunk;
  const int64_t kend = m < kbeg + kchunk ? m : kbeg + kchunk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 2) * 64, wc = (warp & 3) * 32;
  const int fr = lane >> 2, fk = lane & 3;
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int64_t rA = (int64_t)I * kT, rB = (int64_t)J * kT;
  if (ldc > 0 && threadIdx.x < kT && rA + threadIdx.x < n) {
    // trailing update: pull this tile's rows of C into L2 while the MMAs run, so the closing
    // read-modify-write hits L2 (C is far larger than L2 at the sizes this path serves)
    const double* crow = Gp + (rA + threadIdx.x) * ldc + rB;
    const int64_t cols = std::min<int64_t>(kT, rA + threadIdx.x - rB + 1);
    if (cols > 0) {
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(crow) & ~(uintptr_t)15;
      const uintptr_t a1 = (reinterpret_cast<uintptr_t>(crow + cols) + 15) & ~(uintptr_t)15;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
    }
  }
  const int nst = kbeg < kend ? (int)((kend - kbeg + kK - 1) / kK) : 0;
  auto issue = [&](int st) {
    if (st < nst) {
      T* d = dsm + (st % kAsyncStages) * kStageElems;
      issue_stage<T>(d, S, n, kend, ldS, rA, kbeg + (int64_t)st * kK);
      if (!diag) issue_stage<T>(d + kT * kLd, S, n, kend, ldS, rB, kbeg + (int64_t)st * kK);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");   // empty groups keep the count uniform
  };
#pragma unroll
  for (int q = 0; q < kAsyncStages - 1; ++q) issue(q);
  int buf = 0;
  double* fbuf = ws + (size_t)blockIdx.x * kT * kT;
  int since = 0;
  bool flushed = false;
  for (int st = 0; st < nst; ++st) {
    // stage st landed (this thread's pieces): kAsyncStages - 2 younger groups may stay in flight
    asm volatile("cp.async.wait_group %0;" ::"n"(kAsyncStages - 2) : "memory");
    __syncthreads();                                       // ... everyone's; stage st-1 fully consumed
    issue(st + kAsyncStages - 1);                          // refills the buffer stage st-1 used
    const T* A = dsm + buf * kStageElems;
    stage_mma<T>(acc, A, diag ? A : A + kT * kLd, wr, wc, fr, fk);
    buf = buf == kAsyncStages - 1 ? 0 : buf + 1;
    if (flush && ++since == kFlush && st + 1 < nst) {
      flush_acc(acc, fbuf, !flushed, wr, wc, fr, lane);
      flushed = true;
      since = 0;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (flushed) unflush_acc(acc, fbuf, wr, wc, fr, lane);
  store_tile(acc, rA, rB, n, lam, ws, Gp, direct, wr, wc, fr, lane, ldc);
}

// Fixed-order sum of the P split-K partials of a tile.  Block (tile, part): kRedParts slices of
// the tile's elements, so a one-tile problem still spreads its reduction over many SMs (64 x 4096
// fp64: 112 -> ~5 us with the split count P = 32).
constexpr int kRedParts = 16;
__global__ void syrk_dmma_reduce(const double* __restrict__ ws, int P, int64_t n, double lam, double* __restrict__ Gp) {
  const int tile = blockIdx.x / kRedParts, part = blockIdx.x % kRedParts;
  int I, J;
  tile_ij(tile, I, J);
  constexpr int kPer = kT * kT / kRedParts;
  for (int e = part * kPer + threadIdx.x; e < (part + 1) * kPer; e += blockDim.x) {
    const int r = e / kT, c = e % kT;
    const int64_t gi = (int64_t)I * kT + r, gj = (int64_t)J * kT + c;
    if (gi >= n || gj > gi) continue;
    double s = 0.0;
    for (int q = 0; q < P; ++q) s += ws[((size_t)tile * P + q) * kT * kT + e];
    Gp[gi * (gi + 1) / 2 + gj] = s + (gi == gj ? lam : 0.0);
  }
}

struct DPlan {
  int tiles, P;
  int64_t kchunk;
};

// Fraction of the SM-slots of the last full round that P-way split tiles keep busy.
double round_fill(int tiles, int P, int num_sms) {
  const int64_t units = (int64_t)tiles * P, rounds = (units + num_sms - 1) / num_sms;
  return (double)units / (double)(rounds * num_sms);
}

// cap: bytes of split-K partial / flush tiles available (SIZE_MAX: the unconstrained plan)
DPlan dplan(int64_t n, int64_t m, int num_sms, size_t cap) {
  DPlan p;
  const int nb = (int)((n + kT - 1) / kT);
  p.tiles = nb * (nb + 1) / 2;
  const int64_t kblocks = (m + kK - 1) / kK;
  if (p.tiles < num_sms) {
    p.P = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms / p.tiles, kblocks / 4));
  } else {
    // more tiles than SMs: split K when it fills the last round better (n = 4096: 528 tiles are
    // 3.57 rounds -> 5-way splits fill 17.8 of 18), within the workspace the context holds and
    // keeping >= 16 stages per unit
    p.P = 1;
    double best = round_fill(p.tiles, 1, num_sms);
    for (int P = 2; P <= 8; ++P) {
      if (kblocks / P < 16 || (size_t)p.tiles * P * kT * kT * sizeof(double) > cap) break;
      const double f = round_fill(p.tiles, P, num_sms);
      if (f > best + 0.03) { best = f; p.P = P; }
    }
  }
  p.kchunk = ((kblocks + p.P - 1) / p.P) * kK;
  p.P = (int)((m + p.kchunk - 1) / p.kchunk);
  return p;
}

// FS_DMMA_ASYNC=0 selects the register-staged loader for fp64 scores too (A/B switch).
bool dmma_async() {
  static const bool on = [] {
    const char* e = getenv("FS_DMMA_ASYNC");
    return !(e && e[0] == '0');
  }();
  return on;
}

// FS_DMMA_FLUSH=0 turns the two-level accumulation off (single register chain; A/B switch).
bool dmma_flush() {
  static const bool on = [] {
    const char* e = getenv("FS_DMMA_FLUSH");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

// One 128 x 128 fp64 tile per CTA of the grid: the split-K partial and, with or without a split,
// the CTA's flush slot of the two-level accumulation.  A context sized for (n_max, m_max) holds
// the unconstrained plan of that problem (or one tile per SM, whichever is larger); every smaller
// problem's plan then fits, because dplan caps its split count by the bytes actually held.
size_t syrk_dmma_workspace_bytes(int64_t n, int64_t m, int num_sms) {
  const DPlan p = dplan(n, m, num_sms, SIZE_MAX);
  return (size_t)std::max<int64_t>(num_sms, (int64_t)p.tiles * p.P) * kT * kT * sizeof(double);
}

size_t syrk_dmma_plan_bytes(int64_t n, int64_t m, int num_sms) {
  const DPlan p = dplan(n, m, num_sms, SIZE_MAX);
  return (size_t)p.tiles * p.P * kT * kT * sizeof(double);
}

int syrk_dmma_splits(int64_t n, int64_t m, int num_sms, size_t ws_bytes) { return dplan(n, m, num_sms, ws_bytes).P; }

cudaError_t syrk_dmma(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS, double lam, double* Gp,
                      double* ws, size_t ws_bytes, int num_sms, cudaStream_t st, int* launches) {
  DPlan p = dplan(n, m, num_sms, ws_bytes);
  const int direct = p.P == 1 ? 1 : 0;
  const int vec = ((reinterpret_cast<uintptr_t>(S) | (uintptr_t)(ldS * (s_f64 ? 8 : 4))) & 15) == 0 ? 1 : 0;
  const unsigned grid = (unsigned)(p.tiles * p.P);
  if (!direct && (!ws || (size_t)grid * kT * kT * sizeof(double) > ws_bytes)) return cudaErrorInvalidValue;
  // the flush slots are the split-K partial tiles' own: one 128 x 128 fp64 tile per CTA
  const int flush = ws && (size_t)grid * kT * kT * sizeof(double) <= ws_bytes && dmma_flush() ? 1 : 0;
  if (s_f64 && vec && dmma_async()) {
    cudaFuncSetAttribute(syrk_dmma_async_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kAsyncSmemBytes);
    syrk_dmma_async_kernel<double><<<grid, kThreads, kAsyncSmemBytes, st>>>((const double*)S, n, m, ldS, p.kchunk,
                                                                             p.P, lam, ws, Gp, direct, flush);
  } else if (!s_f64 && vec && dmma_async()) {
    constexpr size_t smem32 = async_smem_bytes<float>();
    cudaFuncSetAttribute(syrk_dmma_async_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem32);
    syrk_dmma_async_kernel<float><<<grid, kThreads, smem32, st>>>((const float*)S, n, m, ldS, p.kchunk, p.P, lam, ws,
                                                                  Gp, direct, flush);
  } else if (s_f64) {
    cudaFuncSetAttribute(syrk_dmma_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    syrk_dmma_kernel<double><<<grid, kThreads, kSmemBytes, st>>>((const double*)S, n, m, ldS, p.kchunk, p.P, lam, ws,
                                                                 Gp, direct, vec, flush);
  } else {
    cudaFuncSetAttribute(syrk_dmma_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    syrk_dmma_kernel<float><<<grid, kThreads, kSmemBytes, st>>>((const float*)S, n, m, ldS, p.kchunk, p.P, lam, ws,
                                                                Gp, direct, vec, flush);
  }
  if (launches) *launches += 1;
  if (!direct) {
    syrk_dmma_reduce<<<p.tiles * kRedParts, 256, 0, st>>>(ws, p.P, n, lam, Gp);
    if (launches) *launches += 1;
  }
  return cudaGetLastError();
}

// Trailing update of a blocked Cholesky: C (nt x nt lower, row-major pitch ldc) -= P P^T with P
// the nt x K panel (row-major, pitch ldP) — the same 128 x 128 DMMA tiles as the Gram, no split,
// subtracted in place.  Skipped entirely once *status is set.
cudaError_t syrk_dmma_trail(const double* P, int64_t nt, int64_t K, int64_t ldP, double* C, int64_t ldc,
                            const int64_t* status, cudaStream_t st, int* launches, int64_t cols) {
  if (nt <= 0 || K <= 0) return cudaSuccess;
  const int64_t T = (nt + kT - 1) / kT;
  // cols > 0: only the first `cols` columns of C (a strip of whole 128-column tiles)
  const int jmax = cols > 0 ? (int)std::min<int64_t>(T, (cols + kT - 1) / kT) : 0;
  const unsigned grid = jmax > 0 ? (unsigned)(T * jmax) : (unsigned)(T * (T + 1) / 2);
  const bool vec = ((reinterpret_cast<uintptr_t>(P) | (uintptr_t)(ldP * 8)) & 15) == 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(syrk_dmma_async_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kAsyncSmemBytes);
    cudaFuncSetAttribute(syrk_dmma_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    attr = true;
  }
  if (vec)
    syrk_dmma_async_kernel<double><<<grid, kThreads, kAsyncSmemBytes, st>>>(P, nt, K, ldP, K, 1, 0.0, nullptr, C, 1, 0,
                                                                             ldc, status, jmax);
  else
    syrk_dmma_kernel<double><<<grid, kThreads, kSmemBytes, st>>>(P, nt, K, ldP, K, 1, 0.0, nullptr, C, 1, 0, 0, ldc,
                                                                 status, jmax);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace fs
