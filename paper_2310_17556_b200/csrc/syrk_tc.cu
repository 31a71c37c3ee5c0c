// syrk_tc.cu — Gram W = S S^T (+λI) for fp32 scores on the 5th-gen tensor cores, CTA pairs.
//
// Replaces core.py:284 (numpy A @ A.T -> OpenBLAS dsyrk) for FS_PREC_TF32X3.
//
// Precision mode "3xTF32": every fp32 element x is split into hi = trunc_tf32(x) (the tensor
// core truncates raw fp32 operands to tf32 itself, tools/probe_tf32.py) and lo = x - hi (exact
// in fp32, written by the converter warps), and each K-step issues three
// tcgen05.mma.kind::tf32:  lo*hi^T + hi*lo^T + hi*hi^T.  The dropped lo*lo^T term is
// <= 2^-20 relative; off the diagonal it is sign-random, on the diagonal a ~3e-7 bias.
// The tensor core's fp32 accumulation truncates (round-toward-zero-like; measured ~2^-25
// relative per MMA into one accumulator), so the TMEM accumulator is drained every
// kDrainBlocks K-blocks (24 MMAs) into round-to-nearest fp32 register sums, which are
// flushed into fp64 every kFlushChunks drains.  Deterministic: fixed chunk boundaries and a
// fixed-order fp64 reduction over split-K partials.
//
// Work decomposition: 128-row blocks; a PAIR TILE is rows {2p, 2p+1} x cols {2q, 2q+1}
// (q <= p), computed by a cluster of two CTAs with tcgen05.mma.cta_group::2 (M=256, N=256):
// CTA c holds A = row block 2p+c and the B half = row block 2q+c in its own smem and owns the
// 128 x 256 accumulator of its row block in its own TMEM.  On diagonal pair tiles A == B, so
// each CTA loads a single box.  Per K-column every CTA loads 2 boxes (1 on the diagonal) instead
// of the 3 of a single-CTA 128x256 tile, and the tensor core reads half of B from each SM.
// Split-K over P clusters per pair tile, contiguous K ranges (S streamed ~once from HBM).
//
// Roles per CTA (512 threads, setmaxnreg-rebalanced):
//   warp 0      producer: 1-D bulk copies of its own pre-swizzled 16 KB S_t tiles (tiles.cuh),
//               own barrier, + L2 bulk prefetch kPfDist K-blocks ahead
//   warp 1      TMEM allocator (cta_group::2, both CTAs); MMA issuer in the leader CTA only
//   warps 4-7   converters: raw -> lo ring (integer mask + FADD); release-arrive on the LEADER's
//               conv barrier (mapa), so the leader's MMA sees both CTAs' operands converted
//   warps 8-15  epilogue: tcgen05.ld own TMEM -> fp32 RN sums -> fp64 partials; release-arrive
//               on the leader's tempty barrier
// MMA completion is tcgen05.commit.cta_group::2 ... multicast::cluster to both CTAs.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"
#include "tiles.cuh"

namespace fs {
namespace {

constexpr int kBlk = 128;                 // rows per block / per CTA operand box
constexpr int kN = 256;                   // MMA N (two B halves of 128 rows)
constexpr int kBK = kTileCols;            // fp32 columns per K-block (128 B rows, SWIZZLE_128B)
constexpr int kRowBytes = 4 * kBK;
constexpr int kRaw = 4;                   // raw ring (TMA destination, read by MMA as hi)
constexpr int kLo = 3;                    // lo ring (>= 3: the lo slot loop MMA->converter->MMA must not throttle)
constexpr int kBoxBytes = kBlk * kRowBytes;   // 16 KB
constexpr int kStageBytes = 2 * kBoxBytes;    // A box + B box
constexpr int kThreads = 512;
constexpr int kTmemCols = 2 * kN;         // double-buffered fp32 accumulator
constexpr int kDrainBlocks = 2;           // 2 x 32 columns = 24 MMAs per drained chunk
constexpr int kFlushChunks = 128;        // fp32 register sums -> fp64 every 128 drains (64: Gram error
                                          // 6.3e-7 vs 6.6e-7 of the diagonal, +0.06 ms; tools/flush_accuracy.py)
constexpr int kPfDist = 8;                // K-blocks between an L2 prefetch and its bulk load
constexpr int kRegsProducer = 56, kRegsConverter = 80, kRegsEpilogue = 184;
constexpr int kRegsProducerRing = 48, kRegsConverterRing = 88;   // ring: the converters load 8 float4 per batch
constexpr uint32_t kIdesc = ptx::idesc_tf32(2 * kBlk, kN);
// F16X2 (tiles.cuh): a stage holds the hi+lo tiles of the A and B row blocks (4 x 16 KB), no
// converter ring; kind::f16 MMAs (K = 16) on 64-column K-blocks
// F16X2 direct (kDirect): the SYRK reads fp32 S itself (2-D TMA, 64-column x 128-row boxes of
// 256-byte rows) into a ring of kXS raw slots, and its converter warps write the hi/lo planes
// into the same 2-stage operand ring the pre-tiled mode fills by bulk copy — no S_t16 round trip
// through HBM (the 4.1 GB write + read that cost the retile pass 1.3 ms).
constexpr int kXS = 3;                          // raw fp32 box slots (direct mode)
constexpr int kXBytes = kBlk * kTile16Cols * 4; // one 128 x 64 fp32 box: 32 KB
template <bool kF16, bool kDirect = false> constexpr int raw_stages() { return kDirect ? 2 : kF16 ? 3 : kRaw; }
template <bool kF16> constexpr int lo_stages() { return kF16 ? 0 : kLo; }
template <bool kF16> constexpr int stage_bytes() { return kF16 ? 4 * kBoxBytes : kStageBytes; }
// F16X2 ring (kRing): the SYRK's converter warps split fp32 S themselves, but each (K-block, row
// block) tile ONCE for the whole grid, into an L2-resident ring of pre-swizzled hi/lo tiles that
// every consuming CTA then bulk-copies exactly as in the pre-tiled mode (see syrk_f16_ring).
constexpr int kRingMaxNb = 24;                  // row blocks (n <= 3072): the per-CTA u partials
constexpr int kRingRowsPerBatch = 4;           // converter rows per load batch (8 spills at 88 registers)
constexpr int kRingMaxDepth = 16;               // K-blocks per group's ring
constexpr int kRingMaxSlots = 74 * kRingMaxDepth;   // P * R counters (P <= clusters <= 74)
constexpr size_t kRingBytes = (size_t)48 << 20; // ring budget (L2 is 126 MB)
template <bool kF16, bool kDirect = false, bool kRing = false> constexpr size_t smem_bytes() {
  return (size_t)(raw_stages<kF16, kDirect>() * stage_bytes<kF16>() + lo_stages<kF16>() * kStageBytes) +
         (kDirect ? (size_t)kXS * kXBytes + 128 * 8 : 0) + (kRing ? (size_t)kRingMaxNb * kBlk * 8 : 0) + 1024 +
         (kDirect ? 256 : 512);
}
struct RingArgs {          // F16X2 ring mode inputs
  const float* S;          // fp32 scores (row-major, ldS)
  int64_t ldS, m;
  const float* v;          // u = S v partials (or null)
  const float* scale;      // per-row power-of-two scales
  int* flags;              // |= 1 non-finite input, |= 2 fp16 overflow
  uint8_t* ring;           // [P][R][nbt] hi+lo tile pairs (32 KB each)
  int* ready;              // [P][R] tiles converted into the slot (monotonic over rounds)
  int* freed;              // [P][R] CTAs whose copy of the slot landed (monotonic)
  double* upart;           // [P][2 tiles][n] per-CTA u partials
  int R;                   // ring depth in K-blocks
};
struct DirectArgs {        // F16X2 direct mode inputs
  const float* v;          // u = S v partials for the diagonal pair tiles' units (or null)
  const float* scale;      // per-row power-of-two scales
  int* flags;              // |= 1 non-finite input, |= 2 fp16 overflow
  double* upart;           // [split][n] partial u
  int64_t m;               // columns of S (v's length)
};
constexpr uint32_t kIdescF16 = ptx::idesc_f16(2 * kBlk, kN);

constexpr int kMaxSplitLarge = 8;                        // split-K factor cap when tiles >= clusters
constexpr size_t kMaxSplitWsBytes = (size_t)2 << 30;      // ... and its fp64 partials (2 GB)

struct Plan {
  int nb, np, tile0, tiles, P, clusters, KB, KC, D, kb_base;
  bool direct;
};

// Per-tile split counts (split mode): tile t owns units [base[t], base[t+1]), each a contiguous
// K range of kc[t] K-blocks.  nt == 0: uniform P / KC (direct mode or the plain split).
constexpr int kMaxMapTiles = 80;
struct UnitMap {
  int nt;
  int base[kMaxMapTiles + 1];
  int kc[kMaxMapTiles];
};

// Uniform split, unit order: tile-major (u = t * P + q) while every unit has its own cluster —
// measured faster at the headline (10 tiles x 7 splits: 2.76 vs 3.05 ms split-major) — and
// split-major (u = q * tiles + t, signalled by a negative P) when the clusters run several units
// each: the clusters of a round then walk the same K range of every tile, so tiles sharing a row
// block share it in L2 (n = 8192: 205.6 vs 214.8 ms tile-major).
FS_DEVINL int unit_split(const UnitMap& um, int u, int P, int tiles, int t) {
  return um.nt ? u - um.base[t] : P < 0 ? u / tiles : u % P;
}
FS_DEVINL void unit_decode(const UnitMap& um, int u, int P, int KC, int KB, int tiles, int& t, int& kb0, int& nk) {
  int q;
  if (um.nt == 0) {
    t = P < 0 ? u % tiles : u / P;
    q = P < 0 ? u / tiles : u % P;
    kb0 = q * KC;
    nk = min(KC, KB - kb0);
    return;
  }
  t = 0;
  while (t + 1 < um.nt && um.base[t + 1] <= u) ++t;
  q = u - um.base[t];
  kb0 = q * um.kc[t];
  nk = min(um.kc[t], KB - kb0);
}

FS_DEVINL void pair_of(int t, int& p, int& q) {  // lower pair tiles (p >= q), row-major
  int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  p = i;
  q = t - i * (i + 1) / 2;
}

// lo = x - trunc_tf32(x) (exact in fp32), itself rounded to nearest tf32 (add half an ulp of
// the kept 10-bit mantissa, then mask) so that the tensor core's own truncation of the lo
// operand cannot bias the hi*lo terms.  Integer ops only (no cvt).
FS_DEVINL float tf32_lo(uint32_t xb) {
  const float lo = __uint_as_float(xb) - __uint_as_float(xb & 0xFFFFE000u);
  return __uint_as_float((__float_as_uint(lo) + 0x1000u) & 0xFFFFE000u);
}

FS_DEVINL float fmax3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// FS_SYRK_DBG bit 256: the leader's MMA thread records cycles spent waiting for operands / for
// a free TMEM buffer, and the total (one row per cluster), printed by the host after the launch
__device__ unsigned long long g_syrk_wait[74 * 4];
__device__ unsigned long long g_conv_wait[74 * 4];   // FS_SYRK_DBG bit 512: converter warp 0 of the leader


struct Ring {  // stage index + mbarrier phase of a circular buffer
  int s = 0;
  uint32_t ph = 0;
  FS_DEVINL void next(int depth) { if (++s == depth) { s = 0; ph ^= 1; } }
};

template <bool kF16, bool kDirect = false, bool kRing = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
syrk_tc_kernel(const uint8_t* __restrict__ St, int64_t n, int nbt, int tile0, int tiles, int P, int KB, int KC, int D,
               double* __restrict__ accbuf, double* __restrict__ Gp, double lam, int direct, int dbg, int kb_base,
               int accum, const double* __restrict__ inv_scale, const __grid_constant__ CUtensorMap tmap, int sym,
               const __grid_constant__ UnitMap um, int units, const DirectArgs da, const RingArgs ra) {
  constexpr int kRawS = raw_stages<kF16, kDirect>();
  constexpr int kLoS = lo_stages<kF16>();
  constexpr int kSB = stage_bytes<kF16>();
  constexpr int kBlkBytes = kF16 ? 2 * kBoxBytes : kBoxBytes;   // one row block's K-block (hi+lo for F16X2)
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by offset, so the compiler keeps the shared window (LDS/STS, not generic)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* raw = smem;
  uint8_t* lo = smem + (size_t)kRawS * kSB;
  uint8_t* xraw = smem + (size_t)kRawS * kSB + (size_t)kLoS * kStageBytes;   // direct: fp32 box slots
  double* xu = reinterpret_cast<double*>(xraw + (kDirect ? (size_t)kXS * kXBytes : 0));   // [128]
  double* xur = xu + (kDirect ? 128 : 0);                                                 // ring: [nbt][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xur + (kRing ? kRingMaxNb * kBlk : 0));
  uint64_t* full = bars;                 // local TMA -> local converters / relay   [kRawS]
  uint64_t* conv = full + kRawS;         // both CTAs' converters -> leader MMA     [kRawS]
  uint64_t* empty = conv + kRawS;        // MMA (multicast) -> each producer        [kRawS]
  uint64_t* lo_free = empty + kRawS;     // MMA (multicast) -> each converter group [kLoS]
  uint64_t* tfull = lo_free + kLoS;      // MMA (multicast) -> each epilogue        [2]
  uint64_t* tempty = tfull + 2;          // both CTAs' epilogues -> leader MMA      [2]
  uint64_t* xfull = tempty + 2;          // direct: TMA -> converters                [kXS]
  uint64_t* xempty = xfull + kXS;        // direct: converters -> producer           [kXS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xempty + kXS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = ptx::cluster_ctarank();   // 0 = leader
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRawS; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&conv[s], 2);                 // one elected arrive per CTA
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kLoS; ++s) ptx::mbar_init(&lo_free[s], 1);
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 2);                // one elected arrive per CTA
    }
    if (kDirect)
      for (int s = 0; s < kXS; ++s) {
        ptx::mbar_init(&xfull[s], 1);
        ptx::mbar_init(&xempty[s], 1);
      }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc2<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();                   // barriers initialised and TMEM allocated in both CTAs
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int wg = warp >> 2;

  if (wg == 0) {
    if constexpr (kRing) ptx::setmaxnreg_dec<kRegsProducerRing>();
    else ptx::setmaxnreg_dec<kRegsProducer>();
    if (kRing && warp == 0 && lane == 0) {
      // ====== ring producer: wait until the group's converters filled the slot, then the same
      //        1-D bulk copies of pre-swizzled tiles as the pre-tiled mode ======
      Ring rr;
      const int u = cluster;                      // ring mode: one unit per cluster
      if (u < units) {
        int t, kb0, nk;
        unit_decode(um, u, P, KC, KB, tiles, t, kb0, nk);
        const int q = unit_split(um, u, P, tiles, t);
        int pp, qq; pair_of(tile0 + t, pp, qq);
        const int blkA = 2 * pp + (int)crank, blkB = 2 * qq + (int)crank;
        const bool diag = pp == qq;
        const uint32_t bytes = (diag ? 1 : 2) * kBlkBytes;
        const uint8_t* ringq = ra.ring + (size_t)q * ra.R * nbt * kBlkBytes;
        const int* rdy = ra.ready + q * ra.R;
        int slot = 0, round = 0;
        for (int k = 0; k < nk; ++k) {
          ptx::mbar_wait(&empty[rr.s], rr.ph ^ 1);
          ptx::wait_ge(rdy + slot, nbt * (round + 1));
          ptx::fence_proxy_async_global();
          uint8_t* st = raw + (size_t)rr.s * kSB;
          ptx::mbar_arrive_expect_tx(&full[rr.s], bytes);
          ptx::bulk_load(st, ringq + ((size_t)slot * nbt + blkA) * kBlkBytes, kBlkBytes, &full[rr.s]);
          if (!diag) ptx::bulk_load(st + kBlkBytes, ringq + ((size_t)slot * nbt + blkB) * kBlkBytes, kBlkBytes, &full[rr.s]);
          rr.next(kRawS);
          if (++slot == ra.R) { slot = 0; ++round; }
        }
      }
    } else if (kRing && warp == 2 && lane == 0) {
      // ====== ring relay: own copy landed -> leader's conv barrier, and the slot is free for the
      //        group's converters as far as this CTA is concerned ======
      Ring rr;
      const uint32_t conv0 = ptx::mapa(ptx::smem_u32(conv), 0);
      const int u = cluster;
      if (u < units) {
        int t, kb0, nk;
        unit_decode(um, u, P, KC, KB, tiles, t, kb0, nk);
        int* fre = ra.freed + unit_split(um, u, P, tiles, t) * ra.R;
        int slot = 0;
        for (int k = 0; k < nk; ++k) {
          ptx::mbar_wait(&full[rr.s], rr.ph);
          ptx::mbar_arrive_cluster(conv0 + rr.s * 8);
          ptx::red_release_gpu_add(fre + slot, 1);
          rr.next(kRawS);
          if (++slot == ra.R) slot = 0;
        }
      }
    } else if (kDirect && warp == 0 && lane == 0) {
      // ============ direct producer: fp32 boxes of S (own row blocks) -> raw slots ============
      ptx::tma_prefetch_desc(&tmap);
      Ring xr;
      for (int u = cluster; u < units; u += nclusters) {
        int t, kb0, nk;
        unit_decode(um, u, P, KC, KB, tiles, t, kb0, nk);
        int pp, qq; pair_of(tile0 + t, pp, qq);
        const int rowA = (2 * pp + (int)crank) * kBlk, rowB = (2 * qq + (int)crank) * kBlk;
        const bool diag = pp == qq;
        for (int k = 0; k < nk; ++k) {
          const int col = (kb_base + kb0 + k) * kTile16Cols;
          for (int b = 0; b < (diag ? 1 : 2); ++b) {
            ptx::mbar_wait(&xempty[xr.s], xr.ph ^ 1);
            ptx::mbar_arrive_expect_tx(&xfull[xr.s], kXBytes);
            ptx::tma_load_2d(xraw + (size_t)xr.s * kXBytes, &tmap, &xfull[xr.s], col, b ? rowB : rowA);
            xr.next(kXS);
          }
        }
      }
    } else if (!kDirect && !kRing && warp == 0 && lane == 0) {
      // ============ bulk-copy producer (each CTA: its own pre-swizzled S_t tiles) ============
      Ring rr;
      for (int u = cluster; u < units; u += nclusters) {
        int t, kb0, nk;
        unit_decode(um, u, P, KC, KB, tiles, t, kb0, nk);
        int pp, qq; pair_of(tile0 + t, pp, qq);
        const int blkA = 2 * pp + (int)crank, blkB = 2 * qq + (int)crank;
        const bool diag = pp == qq;                       // A == B: one tile
        const uint32_t bytes = (diag ? 1 : 2) * kBlkBytes;
        for (int k = 0; k < nk; ++k) {
          const size_t krow = (size_t)(kb_base + kb0 + k) * nbt;
          // L2 bulk prefetch kPfDist K-blocks ahead: off by default (measured neutral for TF32X3 and
          // ~5% slower for F16X2, tools/syrk_ablate.sh); FS_SYRK_DBG bit 64 re-enables it
          if ((dbg & 64) && k + kPfDist < nk) {
            const size_t pk = (size_t)(kb_base + kb0 + k + kPfDist) * nbt;
            ptx::bulk_prefetch_l2(St + (pk + blkA) * kBlkBytes, kBlkBytes);
            if (!diag) ptx::bulk_prefetch_l2(St + (pk + blkB) * kBlkBytes, kBlkBytes);
          }
          ptx::mbar_wait(&empty[rr.s], rr.ph ^ 1);
          uint8_t* st = raw + (size_t)rr.s * kSB;
          // each CTA's own bulk copies complete on its own full barrier; the converter warps
          // (TF32X3: lo; F16X2: the hi/2 plane of diagonal tiles, or a plain relay) then arrive
          // on the leader's conv barrier
          if (dbg & 1) { ptx::mbar_arrive(&full[rr.s]); rr.next(kRawS); continue; }
          ptx::mbar_arrive_expect_tx(&full[rr.s], bytes);
          ptx::bulk_load(st, St + (krow + blkA) * kBlkBytes, kBlkBytes, &full[rr.s]);
          if (!diag) ptx::bulk_load(st + kBlkBytes, St + (krow + blkB) * kBlkBytes, kBlkBytes, &full[rr.s]);
          rr.next(kRawS);
        }
      }
    } else if (warp == 1 && lane == 0 && crank == 0) {
      // ======================= MMA issuer (leader CTA) =======================
      Ring rr, lr;
      uint32_t chunk = 0;
      long long w_data = 0, w_tmem = 0;
      const long long t_start = clock64();
      uint64_t g_start;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
      for (int u = cluster; u < units; u += nclusters) {
        int t, kb0, nk;
        unit_decode(um, u, P, KC, KB, tiles, t, kb0, nk);
        int pp, qq; pair_of(tile0 + t, pp, qq);
        const int b_off = (pp == qq) ? 0 : kBlkBytes;
        uint32_t dacc = 0;
        for (int k = 0; k < nk; ++k) {
          const int kin = k % D;
          if (kin == 0) {
            const uint32_t b = chunk & 1;
            const long long t0 = (dbg & 256) ? clock64() : 0;
            ptx::mbar_wait(&tempty[b], ((chunk >> 1) & 1) ^ 1);
            if (dbg & 256) w_tmem += clock64() - t0;
            ptx::tc_fence_after();
            dacc = tmem + b * kN;
          }
          const long long t1 = (dbg & 256) ? clock64() : 0;
          ptx::mbar_wait(&conv[rr.s], rr.ph);
          if (dbg & 256) w_data += clock64() - t1;
          ptx::tc_fence_after();
          const uint32_t rs = ptx::smem_u32(raw + (size_t)rr.s * kSB);
          // hi operands: the raw stage (TF32X3: the fp32 tile, truncated by the tensor core) or
          // the hi plane (F16X2); lo operands: the converter ring or the lo plane
          const uint32_t ha = rs, hb = rs + b_off;
          const uint32_t la = kF16 ? rs + kBoxBytes : ptx::smem_u32(lo + (size_t)lr.s * kStageBytes);
          const uint32_t lb = kF16 ? rs + b_off + kBoxBytes : la + b_off;
          // small correction products first (while this chunk's accumulator is still small, the
          // tensor core's truncating accumulation loses least), then the four hi*hi products
          if (kF16 && sym && pp == qq && !(dbg & 4)) {
            // diagonal pair tile: D = lo h^T + (hi/2) h^T, symmetrised in the reduce
            // (D + D^T = h h^T + lo h^T + h lo^T): 8 MMAs per K-block instead of 12
            const uint32_t h2 = rs + 2 * kBoxBytes;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t off = kk * 32;
              ptx::mma2_f16(dacc, ptx::desc_kmajor<kRowBytes>(la + off), ptx::desc_kmajor<kRowBytes>(hb + off),
                            kIdescF16, (kin > 0 || kk > 0) ? 1u : 0u);
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t off = kk * 32;
              ptx::mma2_f16(dacc, ptx::desc_kmajor<kRowBytes>(h2 + off), ptx::desc_kmajor<kRowBytes>(hb + off),
                            kIdescF16, 1u);
            }
          } else if (!(dbg & 4)) {
#pragma unroll
            for (int kk = 0; kk < ((dbg & 128) ? 0 : 4); ++kk) {
              const uint32_t off = kk * 32;   // 8 tf32 / 16 fp16 = 32 bytes of K per MMA
              if constexpr (kF16) {
                ptx::mma2_f16(dacc, ptx::desc_kmajor<kRowBytes>(la + off), ptx::desc_kmajor<kRowBytes>(hb + off),
                              kIdescF16, (kin > 0 || kk > 0) ? 1u : 0u);
                ptx::mma2_f16(dacc, ptx::desc_kmajor<kRowBytes>(ha + off), ptx::desc_kmajor<kRowBytes>(lb + off),
                              kIdescF16, 1u);
              } else {
                ptx::mma2_tf32(dacc, ptx::desc_kmajor<kRowBytes>(la + off), ptx::desc_kmajor<kRowBytes>(hb + off),
                               kIdesc, (kin > 0 || kk > 0) ? 1u : 0u);
                ptx::mma2_tf32(dacc, ptx::desc_kmajor<kRowBytes>(ha + off), ptx::desc_kmajor<kRowBytes>(lb + off),
                               kIdesc, 1u);
              }
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t off = kk * 32;
              if constexpr (kF16)
                ptx::mma2_f16(dacc, ptx::desc_kmajor<kRowBytes>(ha + off), ptx::desc_kmajor<kRowBytes>(hb + off),
                              kIdescF16, 1u);
              else
                ptx::mma2_tf32(dacc, ptx::desc_kmajor<kRowBytes>(ha + off), ptx::desc_kmajor<kRowBytes>(hb + off),
                               kIdesc, 1u);
            }
          }
          ptx::mma2_commit_mc(&empty[rr.s], 0x3);
          if constexpr (!kF16) ptx::mma2_commit_mc(&lo_free[lr.s], 0x3);
          if (kin == D - 1 || k == nk - 1) {
            ptx::mma2_commit_mc(&tfull[chunk & 1], 0x3);
            ++chunk;
          }
          rr.next(kRawS);
          if constexpr (!kF16) lr.next(kLo);
        }
      }
      if ((dbg & 256) && cluster < 74) {
        g_syrk_wait[cluster * 4 + 0] = w_data;
        g_syrk_wait[cluster * 4 + 1] = w_tmem;
        g_syrk_wait[cluster * 4 + 2] = clock64() - t_start;
        uint64_t g_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
        g_syrk_wait[cluster * 4 + 3] = g_end - g_start;
      }
    }
  } else if (wg == 1 && kDirect) {
    // ====== F16X2 direct converters: fp32 box -> hi/lo fp16 planes (the retile16 arithmetic:
    //        hi = fp16_rn(x s), lo = fp16_rn(x s - hi)) in the SWIZZLE_128B operand image; on
    //        diagonal pair tiles also u = S v for this CTA's row block over the unit's K range ======
    ptx::setmaxnreg_dec<kRegsConverter>();
    const int ct = threadIdx.x - 128, cw = ct >> 5;
    const int half16 = lane >> 4, cq = lane & 15, cj = cq >> 1, ch = cq & 1;
    const uint32_t conv0 = ptx::mapa(ptx::smem_u32(conv), 0);
    Ring cr, xr;
    float amax = 0.f, xmax = 0.f;
    long long cw_empty = 0, cw_full = 0, cw_work = 0, cw_bar = 0;
    const long long cw_t0 = clock64();
    for (int u = cluster; u < units; u += nclusters) {
      int t, kb0, nk;
      unit_decode(um, u, P, KC, KB, tiles, t, kb0, nk);
      int pp, qq; pair_of(tile0 + t, pp, qq);
      const bool diag = pp == qq;
      const int64_t rowA = (int64_t)(2 * pp + (int)crank) * kBlk, rowB = (int64_t)(2 * qq + (int)crank) * kBlk;
      const bool want_u = diag && da.v != nullptr;
      if (want_u) xu[ct] = 0.0;
      // lane l holds the scale of row (step l/2 of this warp, half l%2) for the A and B boxes;
      // a step fetches its row's scale with one shuffle
      float scA, scB;
      {
        const int r = ((lane >> 1) * 4 + cw) * 2 + (lane & 1);
        scA = rowA + r < n ? __ldg(da.scale + rowA + r) : 1.f;
        scB = rowB + r < n ? __ldg(da.scale + rowB + r) : 1.f;
      }
      ptx::named_bar_sync(1, 128);
      for (int k = 0; k < nk; ++k) {
        const int64_t col0 = (int64_t)(kb_base + kb0 + k) * kTile16Cols + 4 * cq;
        float4 vv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (want_u) {
          const float* vp = da.v + col0;
          vv.x = col0 < da.m ? vp[0] : 0.f;
          vv.y = col0 + 1 < da.m ? vp[1] : 0.f;
          vv.z = col0 + 2 < da.m ? vp[2] : 0.f;
          vv.w = col0 + 3 < da.m ? vp[3] : 0.f;
        }
        long long c0 = (dbg & 512) ? clock64() : 0;
        ptx::mbar_wait(&empty[cr.s], cr.ph ^ 1);               // operand stage free (MMA done)
        if (dbg & 512) { const long long c1 = clock64(); cw_empty += c1 - c0; c0 = c1; }
        uint8_t* stg = raw + (size_t)cr.s * kSB;
        for (int b = 0; b < (diag ? 1 : 2); ++b) {
          if (dbg & 512) c0 = clock64();
          ptx::mbar_wait(&xfull[xr.s], xr.ph);
          if (dbg & 512) { const long long c1 = clock64(); cw_full += c1 - c0; c0 = c1; }
          const uint8_t* src = xraw + (size_t)xr.s * kXBytes;
          uint8_t* hi = stg + b * 2 * kBoxBytes;
          const float scb = b ? scB : scA;
          const bool ub = want_u && b == 0;
          // row r = ((g + q) * 4 + cw) * 2 + half16 with g a multiple of 8: r & 7 is per-thread
          // constant, so is the swizzled column offset
          const int swz = ((cj ^ ((cw * 2 + half16) & 7)) << 4) + ch * 8;
#pragma unroll 1
          for (int g = 0; g < kBlk / 8; g += 8) {
            // all eight shared loads of the group first (latency once per group, not per step)
            float4 x[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int r = ((g + q) * 4 + cw) * 2 + half16;
              x[q] = *reinterpret_cast<const float4*>(src + r * (kTile16Cols * 4) + cq * 16);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int step = g + q;
              const int r = (step * 4 + cw) * 2 + half16;
              const float sc = __shfl_sync(0xffffffffu, scb, step * 2 + half16);
              // packed fp32x2 arithmetic (FMUL2/FFMA2): the same IEEE results as the scalar ops
              const float2 s2 = make_float2(sc, sc), m1 = make_float2(-1.f, -1.f);
              const float2 y01 = __fmul2_rn(make_float2(x[q].x, x[q].y), s2);
              const float2 y23 = __fmul2_rn(make_float2(x[q].z, x[q].w), s2);
              const __half2 h01 = __float22half2_rn(y01), h23 = __float22half2_rn(y23);
              const float2 r01 = __ffma2_rn(__half22float2(h01), m1, y01);   // y - hi, exact
              const float2 r23 = __ffma2_rn(__half22float2(h23), m1, y23);
              const __half2 l01 = __float22half2_rn(r01), l23 = __float22half2_rn(r23);
              // NaN-propagating maxima: |x| (non-finite input) and |x s| (>= 65520: fp16 overflow)
              amax = fmax3_nan(amax, fabsf(y01.x), fabsf(y01.y));
              amax = fmax3_nan(amax, fabsf(y23.x), fabsf(y23.y));
              xmax = fmax3_nan(xmax, fabsf(x[q].x), fabsf(x[q].y));
              xmax = fmax3_nan(xmax, fabsf(x[q].z), fabsf(x[q].w));
              const int off = r * 128 + swz;
              uint2 hv, lv;
              hv.x = *reinterpret_cast<const uint32_t*>(&h01); hv.y = *reinterpret_cast<const uint32_t*>(&h23);
              lv.x = *reinterpret_cast<const uint32_t*>(&l01); lv.y = *reinterpret_cast<const uint32_t*>(&l23);
              *reinterpret_cast<uint2*>(hi + off) = hv;
              *reinterpret_cast<uint2*>(hi + kBoxBytes + off) = lv;
            }
            if (ub) {
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float p = fmaf(x[q].w, vv.w, fmaf(x[q].z, vv.z, fmaf(x[q].y, vv.y, x[q].x * vv.x)));
                p += __shfl_xor_sync(0xffffffffu, p, 1);
                p += __shfl_xor_sync(0xffffffffu, p, 2);
                p += __shfl_xor_sync(0xffffffffu, p, 4);
                p += __shfl_xor_sync(0xffffffffu, p, 8);
                if (cq == 0) xu[((g + q) * 4 + cw) * 2 + half16] += (double)p;
              }
            }
          }
          if (dbg & 512) { const long long c1 = clock64(); cw_work += c1 - c0; c0 = c1; }
          ptx::named_bar_sync(1, 128);                         // every read of the raw slot done
          if (dbg & 512) { const long long c1 = clock64(); cw_bar += c1 - c0; c0 = c1; }
          if (ct == 0) ptx::mbar_arrive(&xempty[xr.s]);
          xr.next(kXS);
        }
        ptx::fence_async_smem();                               // generic writes -> async proxy
        ptx::named_bar_sync(1, 128);
        if (ct == 0) ptx::mbar_arrive_cluster(conv0 + cr.s * 8);
        cr.next(kRawS);
      }
      if (want_u) {
        ptx::named_bar_sync(1, 128);
        const int64_t row = rowA + ct;
        if (row < n) da.upart[(int64_t)unit_split(um, u, P, tiles, t) * n + row] = xu[ct];
      }
    }
    if ((dbg & 512) && ct == 0 && crank == 0 && cluster < 74) {
      g_conv_wait[cluster * 4 + 0] = cw_empty;
      g_conv_wait[cluster * 4 + 1] = cw_full;
      g_conv_wait[cluster * 4 + 2] = cw_work;
      g_conv_wait[cluster * 4 + 3] = clock64() - cw_t0;
      (void)cw_bar;
    }
    // the retile16 rules: non-finite input; isinf(fp16_rn(x s)) <=> |x s| >= 65520
    const bool bad = !isfinite(xmax), ovf = !bad && amax >= 65520.f;
    const unsigned bb = __ballot_sync(0xffffffffu, bad), bo = __ballot_sync(0xffffffffu, ovf);
    if (lane == 0 && (bb | bo)) atomicOr(da.flags, (bb ? 1 : 0) | (bo ? 2 : 0));
  } else if (wg == 1 && kRing) {
    // ====== ring converters: the group's CTAs split its (K-block, row block) tiles round-robin
    //        (item k * nbt + rb -> CTA (2 t + crank) of the 2 * tiles in the group) and write the
    //        hi/lo planes (the retile16 arithmetic) into slot k % R of the group's L2-resident
    //        ring; u = S v partials per row in shared memory (fp64, fixed order) ======
    ptx::setmaxnreg_dec<kRegsConverterRing>();
    const int ct = threadIdx.x - 128, cw = ct >> 5;
    const int j = lane & 7, rl = lane >> 3;       // 16-byte chunk of the tile row, row in a 4-row group
    for (int e = ct; e < nbt * kBlk; e += 128) xur[e] = 0.0;
    bool bad = false, ovf = false;
    const int u = cluster;
    int q = 0, g = 0;
    const int G = 2 * tiles;
    ptx::named_bar_sync(1, 128);
    if (u < units) {
      int t, kb0, nk;
      unit_decode(um, u, P, KC, KB, tiles, t, kb0, nk);
      q = unit_split(um, u, P, tiles, t);
      g = 2 * t + (int)crank;
      uint8_t* ringq = ra.ring + (size_t)q * ra.R * nbt * kBlkBytes;
      int* rdy = ra.ready + q * ra.R;
      const int* fre = ra.freed + q * ra.R;
      const uint64_t pol_first = ptx::policy_evict_first(), pol_last = ptx::policy_evict_last();
      const bool vec = ((reinterpret_cast<uintptr_t>(ra.S) | (uintptr_t)(ra.ldS * 4)) & 15) == 0;
      const int64_t total = (int64_t)nk * nbt;
      // this thread's L2 prefetch of one 256-byte row piece of an upcoming tile
      auto prefetch = [&](int64_t idx) {
        if (idx >= total) return;
        const int k = (int)(idx / nbt), rb = (int)(idx % nbt);
        const int64_t row = (int64_t)rb * kBlk + ct, col = (int64_t)(kb_base + kb0 + k) * kTile16Cols;
        if (row < n && vec && col + kTile16Cols <= ra.m)
          ptx::bulk_prefetch_l2_hint(ra.S + row * ra.ldS + col, kTile16Cols * 4, pol_first);
      };
      int64_t it = (int64_t)g;
      prefetch(it);
      prefetch(it + G);
      long long c_wait = 0, c_conv = 0, c_pub = 0;
      const long long c_t0 = clock64();
      for (; it < total; it += G) {
        prefetch(it + 2 * G);
        const int k = (int)(it / nbt), rb = (int)(it % nbt);
        const int slot = k % ra.R, round = k / ra.R;
        long long c0 = (dbg & 512) ? clock64() : 0;
        if (round > 0 && ct == 0) ptx::wait_ge(fre + slot, G * round);   // every CTA copied round - 1 out
        ptx::named_bar_sync(1, 128);
        if (dbg & 512) { const long long c1 = clock64(); c_wait += c1 - c0; c0 = c1; }
        uint8_t* tile = ringq + ((size_t)slot * nbt + rb) * kBlkBytes;
        const int64_t c = (int64_t)(kb_base + kb0 + k) * kTile16Cols + j * 8;   // this lane's 8 columns
        const bool fullc = vec && c + 8 <= ra.m;
        float4 w0 = make_float4(0.f, 0.f, 0.f, 0.f), w1 = w0;
        if (ra.v) {
          if (fullc) {
            w0 = __ldg(reinterpret_cast<const float4*>(ra.v + c));
            w1 = __ldg(reinterpret_cast<const float4*>(ra.v + c) + 1);
          } else {
            float a[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) a[e] = (c + e < ra.m) ? __ldg(ra.v + c + e) : 0.f;
            w0 = make_float4(a[0], a[1], a[2], a[3]);
            w1 = make_float4(a[4], a[5], a[6], a[7]);
          }
        }
        constexpr int kRB = kRingRowsPerBatch;           // rows per thread per batch (all loads first)
#pragma unroll 1
        for (int h = 0; h < ((dbg & 2048) ? 0 : 8 / kRB); ++h) {   // dbg 2048: publish without converting
          float4 buf[kRB][2];
#pragma unroll
          for (int b = 0; b < kRB; ++b) {
            const int r = ((h * kRB + b) * 4 + cw) * 4 + rl;
            const int64_t i = (int64_t)rb * kBlk + r;
            const float* row = ra.S + i * ra.ldS + c;
            if (i < n && fullc) {
              buf[b][0] = ptx::ld_hint_f4(reinterpret_cast<const float4*>(row), pol_first);
              buf[b][1] = ptx::ld_hint_f4(reinterpret_cast<const float4*>(row) + 1, pol_first);
            } else {
              float a[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) a[e] = (i < n && c + e < ra.m) ? __ldg(row + e) : 0.f;
              buf[b][0] = make_float4(a[0], a[1], a[2], a[3]);
              buf[b][1] = make_float4(a[4], a[5], a[6], a[7]);
            }
          }
#pragma unroll
          for (int b = 0; b < kRB; ++b) {
            const int r = ((h * kRB + b) * 4 + cw) * 4 + rl;
            const int64_t i = (int64_t)rb * kBlk + r;
            const float sc = i < n ? __ldg(ra.scale + i) : 1.f;
            const float xs[8] = {buf[b][0].x, buf[b][0].y, buf[b][0].z, buf[b][0].w,
                                 buf[b][1].x, buf[b][1].y, buf[b][1].z, buf[b][1].w};
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              bad |= !isfinite(xs[e]) || !isfinite(xs[e + 1]);
              const float y0 = xs[e] * sc, y1 = xs[e + 1] * sc;
              const __half2 h = __floats2half2_rn(y0, y1);
              const float2 hf = __half22float2(h);
              ovf |= isinf(hf.x) || isinf(hf.y);
              const __half2 l = __floats2half2_rn(y0 - hf.x, y1 - hf.y);
              hw[e / 2] = *reinterpret_cast<const uint32_t*>(&h);
              lw[e / 2] = *reinterpret_cast<const uint32_t*>(&l);
            }
            const int off = r * 128 + ((j ^ (r & 7)) << 4);
            ptx::st_evict_last(tile + off, make_uint4(hw[0], hw[1], hw[2], hw[3]), pol_last);
            ptx::st_evict_last(tile + kBoxBytes + off, make_uint4(lw[0], lw[1], lw[2], lw[3]), pol_last);
            if (ra.v) {
              float p = 0.f;
              p = fmaf(xs[0], w0.x, p); p = fmaf(xs[1], w0.y, p); p = fmaf(xs[2], w0.z, p); p = fmaf(xs[3], w0.w, p);
              p = fmaf(xs[4], w1.x, p); p = fmaf(xs[5], w1.y, p); p = fmaf(xs[6], w1.z, p); p = fmaf(xs[7], w1.w, p);
              p += __shfl_xor_sync(0xffffffffu, p, 1);   // the row's 8 lanes (64 columns)
              p += __shfl_xor_sync(0xffffffffu, p, 2);
              p += __shfl_xor_sync(0xffffffffu, p, 4);
              if (j == 0) xur[rb * kBlk + r] += (double)p;
            }
          }
        }
        if (dbg & 512) { const long long c1 = clock64(); c_conv += c1 - c0; c0 = c1; }
        if (!(dbg & 1024)) ptx::fence_proxy_async_global();   // generic writes -> the consumers' bulk copies
        ptx::named_bar_sync(1, 128);
        if (ct == 0) ptx::red_release_gpu_add(rdy + slot, 1);
        if (dbg & 512) { const long long c1 = clock64(); c_pub += c1 - c0; }
      }
      if ((dbg & 512) && ct == 0 && cluster < 74 && crank == 0) {
        g_conv_wait[cluster * 4 + 0] = c_wait;
        g_conv_wait[cluster * 4 + 1] = c_conv;
        g_conv_wait[cluster * 4 + 2] = c_pub;
        g_conv_wait[cluster * 4 + 3] = clock64() - c_t0;
      }
    }
    const unsigned bb = __ballot_sync(0xffffffffu, bad), bo = __ballot_sync(0xffffffffu, ovf);
    if (lane == 0 && (bb | bo)) atomicOr(ra.flags, (bb ? 1 : 0) | (bo ? 2 : 0));
    if (ra.v && u < units) {
      ptx::named_bar_sync(1, 128);
      double* up = ra.upart + ((size_t)q * G + g) * n;
      for (int e = ct; e < n; e += 128) up[e] = xur[e];
    }
  } else if (wg == 1 && kF16) {
    // ====== F16X2 relay: own TMA completion -> leader's conv barrier; on diagonal pair tiles
    //        (symmetric mode) the hi/2 plane is written into the stage's free half first ======
    ptx::setmaxnreg_dec<kRegsConverter>();
    const int ct = threadIdx.x - 128;
    const uint32_t conv0 = ptx::mapa(ptx::smem_u32(conv), 0);
    Ring rr;
    for (int u = cluster; u < units; u += nclusters) {
      int t, kb0, nk;
      unit_decode(um, u, P, KC, KB, tiles, t, kb0, nk);
      int pp, qq; pair_of(tile0 + t, pp, qq);
      const bool half_plane = sym && pp == qq;
      for (int k = 0; k < nk; ++k) {
        ptx::mbar_wait(&full[rr.s], rr.ph);
        if (half_plane) {
          const uint4* h4 = reinterpret_cast<const uint4*>(raw + (size_t)rr.s * kSB);          // hi tile
          uint4* d4 = reinterpret_cast<uint4*>(raw + (size_t)rr.s * kSB + 2 * kBoxBytes);        // free half
          const __half2 half2v = __floats2half2_rn(0.5f, 0.5f);
#pragma unroll 8
          for (int i = ct; i < kBoxBytes / 16; i += 128) {
            uint4 x = h4[i];
            __half2* hx = reinterpret_cast<__half2*>(&x);
#pragma unroll
            for (int e = 0; e < 4; ++e) hx[e] = __hmul2(hx[e], half2v);   // exact (power of two)
            d4[i] = x;
          }
          ptx::fence_async_smem();
          ptx::named_bar_sync(1, 128);
        }
        if (ct == 0) ptx::mbar_arrive_cluster(conv0 + rr.s * 8);
        rr.next(kRawS);
      }
    }
  } else if (wg == 1) {
    // ======================= converters (each CTA: its own smem) =======================
    ptx::setmaxnreg_dec<kRegsConverter>();
    const int ct = threadIdx.x - 128;
    const uint32_t conv0 = ptx::mapa(ptx::smem_u32(conv), 0);   // leader's conv[0]
    Ring rr, lr;
    for (int u = cluster; u < units; u += nclusters) {
      int t, kb0, nk;
      unit_decode(um, u, P, KC, KB, tiles, t, kb0, nk);
      int pp, qq; pair_of(tile0 + t, pp, qq);
      const int nvec = ((pp == qq) ? 1 : 2) * (kBoxBytes / 16);
      for (int k = 0; k < nk; ++k) {
        ptx::mbar_wait(&full[rr.s], rr.ph);
        ptx::mbar_wait(&lo_free[lr.s], lr.ph ^ 1);
        if (!(dbg & 2)) {
          // the tensor core truncates fp32 operands to tf32 (measured: tools/probe_tf32.py), so the
          // raw tile already IS hi = trunc(x); only lo = x - trunc(x) (exact in fp32) is written
          const uint4* r4 = reinterpret_cast<const uint4*>(raw + (size_t)rr.s * kSB);
          float4* l4 = reinterpret_cast<float4*>(lo + (size_t)lr.s * kStageBytes);
#pragma unroll 8
          for (int i = ct; i < nvec; i += 128) {
            const uint4 x = r4[i];
            float4 l;
            l.x = tf32_lo(x.x); l.y = tf32_lo(x.y); l.z = tf32_lo(x.z); l.w = tf32_lo(x.w);
            l4[i] = l;
          }
          ptx::fence_async_smem();
        }
        ptx::named_bar_sync(1, 128);                 // all converter writes of this stage done
        if (ct == 0) ptx::mbar_arrive_cluster(conv0 + rr.s * 8);
        rr.next(kRawS);
        lr.next(kLo);
      }
    }
  } else {
    // ======================= epilogue (8 warps, own TMEM) =======================
    ptx::setmaxnreg_inc<kRegsEpilogue>();
    const int sub = warp & 3, half = (warp - 8) >> 2;
    const int r = 32 * sub + lane;                       // row within this CTA's 128-row block
    const uint32_t lane_base = (uint32_t)(32 * sub) << 16;
    const uint32_t tempty0 = ptx::mapa(ptx::smem_u32(tempty), 0);
    float acc[kN / 2];
    uint32_t chunk = 0;
    for (int u = cluster; u < units; u += nclusters) {
      int t, kb0, nk;
      unit_decode(um, u, P, KC, KB, tiles, t, kb0, nk);
      int pp, qq; pair_of(tile0 + t, pp, qq);
      const int nch = (nk + D - 1) / D;
      const size_t slot = direct ? (size_t)blockIdx.x : ((size_t)u * 2 + crank);
      double* __restrict__ sc = accbuf + slot * kBlk * kN + (size_t)half * (kN / 2) * kBlk + r;  // [c][r]
      bool first_flush = true;
      for (int j = 0; j < nch; ++j) {
        const uint32_t b = chunk & 1;
        ptx::mbar_wait(&tfull[b], (chunk >> 1) & 1);
        ptx::tc_fence_after();
        const bool fresh = (j % kFlushChunks) == 0;
#pragma unroll
        for (int cb = 0; cb < (dbg & 16 ? 0 : kN / 64); ++cb) {
          uint32_t v[32];
          ptx::tmem_ld_32x32b_x32(tmem + lane_base + b * kN + half * (kN / 2) + cb * 32, v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float x = __uint_as_float(v[e]);
            acc[cb * 32 + e] = fresh ? x : acc[cb * 32 + e] + x;
          }
        }
        ptx::tc_fence_before();
        ptx::named_bar_sync(2, 256);                 // all epilogue TMEM reads of this chunk done
        if (threadIdx.x == 256) ptx::mbar_arrive_cluster(tempty0 + b * 8);
        ++chunk;
        if (!(dbg & 8) && ((j + 1) % kFlushChunks == 0 || j == nch - 1)) {
          // the fp64 partial tiles (36 MB at the headline) are re-read and rewritten every 64
          // drains: kept in L2 (evict_last) so the flushes stop costing DRAM traffic
          const uint64_t pol = (dbg & 4096) ? 0ull : ptx::policy_evict_last();
          if (first_flush || (dbg & 8192)) {
            // dbg 8192: the earlier read-modify-write flush (load latency on this thread)
#pragma unroll
            for (int g = 0; g < kN / 2; g += 16) {
              double old[16];
              if (!first_flush) {
#pragma unroll
                for (int e = 0; e < 16; ++e)
                  old[e] = pol ? ptx::ld_hint_f64(sc + (size_t)(g + e) * kBlk, pol) : sc[(size_t)(g + e) * kBlk];
              }
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const double val = (first_flush ? 0.0 : old[e]) + (double)acc[g + e];
                if (pol) ptx::st_hint_f64(sc + (size_t)(g + e) * kBlk, val, pol);
                else sc[(size_t)(g + e) * kBlk] = val;
              }
            }
          } else {
            // later flushes: fp64 adds performed at L2 (red, no return value), so the epilogue
            // goes straight back to draining TMEM; each slot element has this one writer, whose
            // adds land in program order: the same fl(old + acc) sequence as a read-modify-write
#pragma unroll
            for (int e = 0; e < kN / 2; ++e) {   // fully unrolled: acc stays in registers
              if (pol) ptx::red_add_hint_f64(sc + (size_t)e * kBlk, (double)acc[e], pol);
              else ptx::red_add_f64(sc + (size_t)e * kBlk, (double)acc[e]);
            }
          }
          first_flush = false;
        }
      }
      if (direct) {
        const int64_t gi = (int64_t)(2 * pp + crank) * kBlk + r;
        if (gi < n) {
          for (int e = 0; e < kN / 2; ++e) {
            const int c = half * (kN / 2) + e;
            const int64_t gj = (int64_t)(2 * qq) * kBlk + c;
            if (gj > gi) break;
            double* g = Gp + gi * (gi + 1) / 2 + gj;
            double val = __ldcg(sc + (size_t)e * kBlk);   // L2: where the flush's adds were performed
            if (kF16) val *= inv_scale[gi] * inv_scale[gj];       // exact: powers of two
            *g = (accum ? *g : 0.0) + val + (gi == gj ? lam : 0.0);
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();                   // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) ptx::tmem_dealloc2<kTmemCols>(tmem);
}

// Fixed-order sum of the P split-K partial tiles -> packed lower Gram (+λ on the diagonal).
// Block (t, c): pair tile t, CTA half c (row block 2p+c).
constexpr int kRedSplit = 16;   // blocks per (pair tile, CTA half): 2048 elements each
__global__ void syrk_tc_reduce(const double* __restrict__ ws, int tile0, int tiles, int P, int64_t n, double lam,
                               double* __restrict__ Gp, int accum, const double* __restrict__ inv_scale, int sym,
                               const __grid_constant__ UnitMap um) {
  const int tc = blockIdx.x / kRedSplit, part = blockIdx.x % kRedSplit;
  int pp, qq;
  pair_of(tile0 + (tc >> 1), pp, qq);
  const int c = tc & 1;
  constexpr int kPer = kBlk * kN / kRedSplit;
  for (int e = part * kPer + threadIdx.x; e < (part + 1) * kPer; e += blockDim.x) {
    const int col = e / kBlk, r = e % kBlk;
    const int64_t gi = (int64_t)(2 * pp + c) * kBlk + r, gj = (int64_t)(2 * qq) * kBlk + col;
    if (gi >= n || gj > gi) continue;
    const int tt = tc >> 1;
    const int nu = um.nt ? um.base[tt + 1] - um.base[tt] : (P < 0 ? -P : P);
    // unit of split q: map mode base[t] + q; uniform tile-major t * P + q, split-major (P < 0)
    // q * tiles + t
    auto unit = [&](int q) -> size_t {
      return um.nt ? (size_t)um.base[tt] + q : P < 0 ? (size_t)q * tiles + tt : (size_t)tt * P + q;
    };
    double s = 0.0;
    for (int q = 0; q < nu; ++q) s += ws[(unit(q) * 2 + c) * kBlk * kN + e];
    if (sym && pp == qq) {
      // symmetric mode on a diagonal pair tile: G = D + D^T; D(j, i) sits in the half of row j
      const int jl = (int)(gj - (int64_t)(2 * qq) * kBlk), il = c * kBlk + r;   // pair-local indices
      const int c2 = jl / kBlk, r2 = jl % kBlk;
      for (int q = 0; q < nu; ++q) s += ws[(unit(q) * 2 + c2) * kBlk * kN + (size_t)il * kBlk + r2];
    }
    if (inv_scale) s *= inv_scale[gi] * inv_scale[gj];
    double* g = Gp + gi * (gi + 1) / 2 + gj;
    *g = (accum ? *g : 0.0) + s + (gi == gj ? lam : 0.0);
  }
}

void pair_of_host(int t, int& p, int& q) {
  int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  p = i;
  q = t - i * (i + 1) / 2;
}

Plan make_plan(int64_t n, int64_t m, int num_sms, int prow0 = 0, int prow1 = -1, int kb_begin = 0, int kb_end = -1,
               int bk = kBK) {
  Plan p;
  p.nb = (int)((n + kBlk - 1) / kBlk);
  p.np = (p.nb + 1) / 2;
  if (prow1 < 0 || prow1 > p.np) prow1 = p.np;
  p.tile0 = prow0 * (prow0 + 1) / 2;
  p.tiles = prow1 * (prow1 + 1) / 2 - p.tile0;
  p.KB = (int)((m + bk - 1) / bk);
  if (kb_end < 0 || kb_end > p.KB) kb_end = p.KB;
  p.kb_base = kb_begin;
  p.KB = kb_end - kb_begin;
  const int max_clusters = num_sms / 2;
  if (p.tiles >= max_clusters) {
    // whole pair tiles per unit leave a partial last round (n = 8192: 528 tiles on 74 clusters =
    // 7.14 rounds run as 8); split-K units of 1/P tile even it out when the workspace allows:
    // minimise ceil(tiles P / clusters) / P
    // (a split costs L2 sharing and a reduce pass: only worth it when it removes > 8% of the
    // rounds — n = 4096, 136 tiles: direct 41.2 ms, 7 splits 43.0 ms)
    p.P = 1;
    const double direct_rounds = std::ceil((double)p.tiles / max_clusters);
    double best = direct_rounds;
    for (int P = 2; P <= kMaxSplitLarge && p.KB / P >= 8; ++P) {
      if ((size_t)2 * p.tiles * P * kBlk * kN * sizeof(double) > kMaxSplitWsBytes) break;
      const double t = std::ceil((double)p.tiles * P / max_clusters) / P;
      if (t < best - 1e-9) { best = t; p.P = P; }
    }
    static const int large_split = getenv("FS_SYRK_LARGE_SPLIT") ? atoi(getenv("FS_SYRK_LARGE_SPLIT")) : 1;
    if (best > 0.92 * direct_rounds || !large_split) p.P = 1;
  } else {
    p.P = std::max(1, std::min(max_clusters / p.tiles, p.KB / 8));
  }
  p.KC = (p.KB + p.P - 1) / p.P;          // K-blocks per split, contiguous in m
  p.P = (p.KB + p.KC - 1) / p.KC;          // every split non-empty
  p.clusters = std::min(p.tiles * p.P, max_clusters);
  p.D = getenv("FS_SYRK_DRAIN") ? atoi(getenv("FS_SYRK_DRAIN")) : kDrainBlocks;
  p.direct = p.P == 1;
  return p;
}

}  // namespace

size_t syrk_tc_plan_bytes(int64_t n, int64_t m, int num_sms) {
  Plan p = make_plan(n, m, num_sms);
  return (size_t)(p.direct ? 2 * p.clusters : 2 * p.tiles * p.P) * kBlk * kN * sizeof(double);
}

bool syrk_tc_supported(const void* S, int64_t ldS) {
  return (reinterpret_cast<uintptr_t>(S) % 16 == 0) && ((ldS * 4) % 16 == 0);
}

size_t syrk_tc_workspace_bytes(int64_t n, int64_t m, int num_sms) {
  // one fp64 128x256 partial per CTA of a split-K unit, or per resident CTA (direct mode).  Units
  // <= clusters while the pair tiles are fewer than the clusters; with more tiles make_plan may
  // split each tile up to kMaxSplitLarge ways within kMaxSplitWsBytes — sized here for the
  // largest n the context serves, which covers every smaller (n, m).
  (void)m;
  const int64_t nb = (n + kBlk - 1) / kBlk, np = (nb + 1) / 2, tiles = np * (np + 1) / 2;
  size_t slots = (size_t)num_sms;
  if (tiles >= num_sms / 2)
    slots = std::max(slots, std::min((size_t)2 * tiles * kMaxSplitLarge,
                                     kMaxSplitWsBytes / ((size_t)kBlk * kN * sizeof(double))));
  return slots * kBlk * kN * sizeof(double);
}

namespace {
// S_t16 viewed as a 2-D fp16 tensor of 128-byte rows: box = one (K-block, row block) hi+lo pair
// (256 rows), no swizzle (the tiles are stored in the swizzled smem image already).
cudaError_t st16_tensor_map(CUtensorMap* map, const uint8_t* St16, int64_t n, int64_t m) {
  const uint64_t rows = (uint64_t)tiles_nb(n) * tiles16_kb(m) * 2 * kTileRows;
  return make_tensor_map_2d(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, St16, kTile16Cols, rows, kTile16Cols * 2,
                            kTile16Cols, 2 * kTileRows);
}

// u[i] (+)= sum over the diagonal tiles' splits of the direct mode's partial u (fixed order)
__global__ void reduce_upart_kernel(const double* __restrict__ upart, int nsplit, int64_t n, double* __restrict__ u,
                                    int accum) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int q = 0; q < nsplit; ++q) s += upart[(int64_t)q * n + i];
  u[i] = (accum ? u[i] : 0.0) + s;
}

template <bool kF16, bool kDirect = false>
cudaError_t syrk_launch(const uint8_t* St, int64_t n, int64_t m, double lam, double* G_packed, double* ws, int num_sms,
                        cudaStream_t st, int* launches, int prow0, int prow1, int kb_begin, int kb_end, int accum,
                        const double* inv_scale, const float* S32 = nullptr, int64_t ldS = 0,
                        DirectArgs da = DirectArgs{}, double* u = nullptr) {
  Plan p = make_plan(n, m, num_sms, prow0, prow1, kb_begin, kb_end, kF16 ? kTile16Cols : kBK);
  if (p.tiles <= 0 || p.KB <= 0) return cudaSuccess;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(syrk_tc_kernel<kF16, kDirect>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_bytes<kF16, kDirect>());
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  static const int dbg = getenv("FS_SYRK_DBG") ? atoi(getenv("FS_SYRK_DBG")) : 0;  // ablation experiments only
  // symmetric diagonal-tile mode (F16X2, split-K partials through the reduce kernel): diagonal
  // pair tiles cost 8 MMAs per K-block instead of 12, so they get proportionally fewer splits
  // measured: 10% fewer SM cycles but a 9% lower clock (the re-split K windows cost DRAM reads and
  // power) and a longer reduce: net slower at the headline, so off unless FS_SYRK_SYM=1
  static const int sym_env = getenv("FS_SYRK_SYM") ? atoi(getenv("FS_SYRK_SYM")) : 0;
  const int sym = (kF16 && !kDirect && !p.direct && sym_env && p.tiles <= kMaxMapTiles) ? 1 : 0;
  UnitMap um;
  memset(&um, 0, sizeof um);
  int units = p.tiles * p.P, clusters = p.clusters;
  if (sym) {
    int n_d = 0;
    for (int t = 0; t < p.tiles; ++t) {
      int a, b;
      pair_of_host(p.tile0 + t, a, b);
      n_d += (a == b);
    }
    const int n_o = p.tiles - n_d, maxc = num_sms / 2;
    // minimise max(3 / P_o, 2 / P_d) subject to n_o P_o + n_d P_d <= maxc, >= 8 K-blocks per unit
    int best_o = p.P, best_d = p.P;
    double best = 1e30;
    for (int po = 1; po <= maxc; ++po)
      for (int pd = 1; pd <= maxc; ++pd) {
        if (n_o * po + n_d * pd > maxc || (n_o && p.KB / po < 8) || (n_d && p.KB / pd < 8)) continue;
        const double span = std::max(n_o ? 3.0 / po : 0.0, n_d ? 2.0 / pd : 0.0);
        if (span < best - 1e-12) { best = span; best_o = po; best_d = pd; }
      }
    um.nt = p.tiles;
    int acc = 0;
    for (int t = 0; t < p.tiles; ++t) {
      int a, b;
      pair_of_host(p.tile0 + t, a, b);
      const int pt = (a == b) ? best_d : best_o;
      const int kc = (p.KB + pt - 1) / pt;
      um.base[t] = acc;
      um.kc[t] = kc;
      acc += (p.KB + kc - 1) / kc;                         // every unit non-empty
    }
    um.base[p.tiles] = acc;
    units = acc;
    clusters = std::min(units, maxc);
  }
  // split-major unit order (signalled by a negative P) when clusters run several units each
  const int p_arg = (p.P > 1 && p.tiles * p.P > p.clusters) ? -p.P : p.P;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof tmap);
  if (kDirect) {
    // fp32 S: 64-column x 128-row boxes (256-byte rows, no swizzle; rows >= n / cols >= m read as 0)
    cudaError_t e = make_tensor_map_2d(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, S32, (uint64_t)m, (uint64_t)n,
                                       (uint64_t)ldS * 4, kTile16Cols, kBlk);
    if (e != cudaSuccess) return e;
  } else if (kF16) {
    cudaError_t e = st16_tensor_map(&tmap, St, n, m);
    if (e != cudaSuccess) return e;
  }
  syrk_tc_kernel<kF16, kDirect><<<2 * clusters, kThreads, smem_bytes<kF16, kDirect>(), st>>>(
      St, n, (int)tiles_nb(n), p.tile0, p.tiles, p_arg, p.KB, p.KC, p.D, ws, G_packed, lam, p.direct ? 1 : 0, dbg,
      p.kb_base, accum, inv_scale, tmap, sym, um, units, da, RingArgs{});
  if (launches) *launches += 1;
  if (dbg & 256) {
    unsigned long long h[74 * 4] = {};
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_syrk_wait, sizeof h);
    double wd = 0, wt = 0, tot = 0, ns = 0;
    int c = 0;
    for (int i = 0; i < 74; ++i)
      if (h[i * 4 + 3]) { wd += h[i * 4]; wt += h[i * 4 + 1]; tot += h[i * 4 + 2]; ns += h[i * 4 + 3]; ++c; }
    if (c) fprintf(stderr, "syrk mma thread: wait operands %.0f%%, wait tmem %.0f%%, %.0f kcycles in %.3f ms -> %.0f MHz (%d clusters)\n",
                   100 * wd / tot, 100 * wt / tot, tot / c / 1e3, ns / c / 1e6, tot / ns * 1e3, c);
  }
  if ((dbg & 512) && kDirect) {
    unsigned long long h[74 * 4] = {};
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_conv_wait, sizeof h);
    double we = 0, wf = 0, ww = 0, tot = 0;
    for (int i = 0; i < 74; ++i)
      if (h[i * 4 + 3]) { we += h[i * 4]; wf += h[i * 4 + 1]; ww += h[i * 4 + 2]; tot += h[i * 4 + 3]; }
    if (tot > 0)
      fprintf(stderr, "syrk converter warp: wait stage %.0f%%, wait fp32 box %.0f%%, convert %.0f%%, rest %.0f%%\n",
              100 * we / tot, 100 * wf / tot, 100 * ww / tot, 100 * (tot - we - wf - ww) / tot);
  }
  if (!p.direct) {
    syrk_tc_reduce<<<2 * p.tiles * kRedSplit, 256, 0, st>>>(ws, p.tile0, p.tiles, p_arg, n, lam, G_packed, accum,
                                                            inv_scale, sym, um);
    if (launches) *launches += 1;
  }
  if (kDirect && da.v && u) {   // the diagonal pair tiles' units (uniform split P) hold u's partials
    reduce_upart_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(da.upart, p.P, n, u, accum);
    if (launches) *launches += 1;
  }
  return cudaGetLastError();
}
// Clusters of the ring kernel that can be resident at once (its CTAs wait on one another's
// conversions, so the whole grid must be co-resident); 0 on failure.
int ring_max_clusters() {
  static int cached = -1;
  if (cached >= 0) return cached;
  cudaError_t e = cudaFuncSetAttribute(syrk_tc_kernel<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_bytes<true, false, true>());
  int nc = 0;
  if (e == cudaSuccess) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(2 * 74);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem_bytes<true, false, true>();
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    e = cudaOccupancyMaxActiveClusters(&nc, syrk_tc_kernel<true, false, true>, &cfg);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    nc = 0;
  }
  cached = nc;
  return nc;
}

// Ring geometry for (n, m, K-range): plan with clusters capped at the co-resident count, one unit
// per cluster (tile-major), ring depth R from the bytes available.  R = 0: the shape does not
// qualify (too many pair tiles or row blocks, or too little ring memory).
struct RingPlan {
  Plan p;
  int R;
};
RingPlan ring_plan(int64_t n, int64_t m, int num_sms, int kb_begin, int kb_end, size_t ring_bytes) {
  RingPlan rp;
  rp.R = 0;
  const int mc = std::min(ring_max_clusters(), num_sms / 2);
  rp.p = make_plan(n, m, 2 * std::max(mc, 1), 0, -1, kb_begin, kb_end, kTile16Cols);
  const Plan& p = rp.p;
  const int nbt = (int)tiles_nb(n);
  if (mc < 1 || p.tiles > mc || p.tiles * p.P > mc || nbt > kRingMaxNb || p.KB <= 0) return rp;
  const size_t per_round = (size_t)p.P * nbt * 2 * kBoxBytes;   // one K-block of every group
  rp.R = (int)std::min<size_t>(kRingMaxDepth, ring_bytes / per_round);
  if (rp.R < 4) rp.R = 0;
  return rp;
}
}  // namespace

size_t syrk_ring_bytes() { return kRingBytes; }
size_t syrk_ring_upart_doubles(int64_t n) { return (size_t)148 * (size_t)std::min<int64_t>(n, kRingMaxNb * kBlk); }

bool syrk_ring_ok(int64_t n, int64_t m, int num_sms) {
  static const int env = getenv("FS_F16_RING") ? atoi(getenv("FS_F16_RING")) : 0;   // off: converter-bound (DESIGN K1)
  if (!env) return false;
  return ring_plan(n, m, num_sms, 0, -1, kRingBytes).R > 0;
}

cudaError_t syrk_f16_ring(const float* S, int64_t ldS, int64_t n, int64_t m, const float* scale,
                          const double* inv_scale, const float* v, int* flags, double* upart, double* u, double lam,
                          double* G_packed, double* ws, uint8_t* ring, int* counters, int num_sms, cudaStream_t st,
                          int* launches, int kb_begin, int kb_end, int accum) {
  if (!syrk_tc_supported(S, ldS)) return cudaErrorNotSupported;
  RingPlan rp = ring_plan(n, m, num_sms, kb_begin, kb_end, kRingBytes);
  if (rp.R == 0) return cudaErrorNotSupported;
  const Plan& p = rp.p;
  if (p.tiles <= 0 || p.KB <= 0) return cudaSuccess;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(syrk_tc_kernel<true, false, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_bytes<true, false, true>());
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  static const int dbg = getenv("FS_SYRK_DBG") ? atoi(getenv("FS_SYRK_DBG")) : 0;
  int* ready = counters;
  int* freed = counters + kRingMaxSlots;
  cudaError_t e = cudaMemsetAsync(counters, 0, 2 * kRingMaxSlots * sizeof(int), st);
  if (e != cudaSuccess) return e;
  UnitMap um;
  memset(&um, 0, sizeof um);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof tmap);
  RingArgs ra{S, ldS, m, v, scale, flags, ring, ready, freed, upart, rp.R};
  const int units = p.tiles * p.P;   // one per cluster, tile-major (P > 0)
  syrk_tc_kernel<true, false, true><<<2 * units, kThreads, smem_bytes<true, false, true>(), st>>>(
      nullptr, n, (int)tiles_nb(n), p.tile0, p.tiles, p.P, p.KB, p.KC, p.D, ws, G_packed, lam, p.direct ? 1 : 0, dbg,
      p.kb_base, accum, inv_scale, tmap, 0, um, units, DirectArgs{}, ra);
  if (launches) *launches += 1;
  if (dbg & 256) {
    unsigned long long h[74 * 4] = {};
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_syrk_wait, sizeof h);
    double wd = 0, wt = 0, tot = 0, ns = 0;
    int c = 0;
    for (int i = 0; i < 74; ++i)
      if (h[i * 4 + 3]) { wd += h[i * 4]; wt += h[i * 4 + 1]; tot += h[i * 4 + 2]; ns += h[i * 4 + 3]; ++c; }
    if (c) fprintf(stderr, "ring syrk mma thread: wait operands %.0f%%, wait tmem %.0f%%, %.0f kcycles in %.3f ms -> %.0f MHz (%d clusters, R=%d)\n",
                   100 * wd / tot, 100 * wt / tot, tot / c / 1e3, ns / c / 1e6, tot / ns * 1e3, c, rp.R);
  }
  if (dbg & 512) {
    unsigned long long h[74 * 4] = {};
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_conv_wait, sizeof h);
    double w = 0, c = 0, pb = 0, tot = 0;
    for (int i = 0; i < 74; ++i)
      if (h[i * 4 + 3]) { w += h[i * 4]; c += h[i * 4 + 1]; pb += h[i * 4 + 2]; tot += h[i * 4 + 3]; }
    if (tot > 0)
      fprintf(stderr, "ring converters (thread 0 of each leader): wait freed %.0f%%, load+convert+store %.0f%%, fence+publish %.0f%%, rest %.0f%%\n",
              100 * w / tot, 100 * c / tot, 100 * pb / tot, 100 * (tot - w - c - pb) / tot);
  }
  if (!p.direct) {
    syrk_tc_reduce<<<2 * p.tiles * kRedSplit, 256, 0, st>>>(ws, p.tile0, p.tiles, p.P, n, lam, G_packed, accum,
                                                            inv_scale, 0, um);
    if (launches) *launches += 1;
  }
  if (v && u) {
    reduce_upart_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(upart, p.P * 2 * p.tiles, n, u, accum);
    if (launches) *launches += 1;
  }
  return cudaGetLastError();
}

cudaError_t syrk_tc(const uint8_t* St, int64_t n, int64_t m, double lam, double* G_packed, double* ws, int num_sms,
                    cudaStream_t st, int* launches, int prow0, int prow1, int kb_begin, int kb_end, int accum) {
  return syrk_launch<false>(St, n, m, lam, G_packed, ws, num_sms, st, launches, prow0, prow1, kb_begin, kb_end, accum,
                            nullptr);
}

cudaError_t syrk_f16_direct(const float* S, int64_t ldS, int64_t n, int64_t m, const float* scale,
                            const double* inv_scale, const float* v, int* flags, double* upart, double* u, double lam,
                            double* G_packed, double* ws, int num_sms, cudaStream_t st, int* launches, int kb_begin,
                            int kb_end, int accum) {
  if (!syrk_tc_supported(S, ldS)) return cudaErrorNotSupported;
  DirectArgs da{v, scale, flags, upart, m};
  return syrk_launch<true, true>(nullptr, n, m, lam, G_packed, ws, num_sms, st, launches, 0, -1, kb_begin, kb_end,
                                 accum, inv_scale, S, ldS, da, u);
}

cudaError_t syrk_f16(const uint8_t* St16, int64_t n, int64_t m, const double* inv_scale, double lam, double* G_packed,
                     double* ws, int num_sms, cudaStream_t st, int* launches, int kb_begin, int kb_end, int accum) {
  return syrk_launch<true>(St16, n, m, lam, G_packed, ws, num_sms, st, launches, 0, -1, kb_begin, kb_end, accum,
                           inv_scale);
}

}  // namespace fs
