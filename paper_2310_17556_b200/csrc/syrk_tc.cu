// syrk_tc.cu — Gram W = S S^T (+λI) for fp32 scores on the 5th-gen tensor cores.
//
// Replaces core.py:284 (numpy A @ A.T -> OpenBLAS dsyrk) for FS_PREC_TF32X3.
//
// Precision mode "3xTF32": every fp32 element x is split on the fly into
//   hi = rna_tf32(x)  (11 significant bits, exact in tf32)   lo = x - hi  (exact in fp32)
// and each K-step issues three tcgen05.mma.kind::tf32:  hi*hi^T + hi*lo^T + lo*hi^T
// (the dropped lo*lo^T term is <= 2^-22 relative and unbiased in sign off the diagonal).
// The tensor core's fp32 accumulation truncates (round-toward-zero-like; measured ~2^-25
// relative per MMA into one accumulator), so the TMEM accumulator is drained every
// kDrainBlocks K-blocks (24 MMAs) into round-to-nearest fp32 register sums, which are
// flushed into fp64 every kFlushChunks drains.  Deterministic: fixed chunk boundaries and a
// fixed-order fp64 reduction over split-K partials.
//
// Layout / pipeline (one CTA per SM, 512 threads, setmaxnreg-rebalanced):
//   warp 0      TMA producer: S boxes (128 rows x kBK fp32, swizzled) -> raw ring
//               + L2 bulk prefetch of 1 KB row spans 32 K-blocks ahead (DRAM sees long bursts)
//   warp 1      TMEM allocator + single-thread MMA issuer (M=128, N=256, K=8 per MMA)
//   warps 4-7   converters: raw -> hi in place, lo -> lo ring, fence.proxy.async
//   warps 8-15  epilogue: tcgen05.ld (32x32b) -> fp32 RN sums -> fp64 partial tile (L2)
// Work decomposition: lower block tiles (I, J0..J0+1) of 128-row blocks; split-K over
// P CTAs per tile, each a contiguous K range, so the CTAs of all tiles with the same split
// index walk the same columns of S together (S read ~once from HBM, reused from L2).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace fs {
namespace {

constexpr int kNB = 2;                    // 128-row blocks per B tile -> N = 256
constexpr int kM = 128;
constexpr int kN = 128 * kNB;
#ifndef FS_SYRK_BK
#define FS_SYRK_BK 32
#endif
constexpr int kBK = FS_SYRK_BK;           // fp32 columns per K-block (rows of 4*kBK bytes, swizzled)
constexpr int kRowBytes = 4 * kBK;
constexpr int kRaw = kBK == 16 ? 6 : 3;   // raw (TMA destination, hi in place) ring depth
constexpr int kLo = kBK == 16 ? 2 : 1;    // lo ring depth
constexpr int kBoxBytes = 128 * kBK * 4;  // one 128-row box = 8 KB
constexpr int kStageBytes = (kNB + 1) * kBoxBytes;
constexpr int kThreads = 512;
constexpr int kTmemCols = 2 * kN;         // double-buffered fp32 accumulator
constexpr int kDrainBlocks = 64 / kBK;     // 4 x 16 or 2 x 32 columns: 24 MMAs per drain
constexpr int kFlushChunks = 64;
constexpr int kPfSpan = 1024 / kRowBytes; // K-blocks per L2 prefetch span (1 KB per row)
constexpr int kPfAhead = 2;               // spans prefetched ahead of the TMA loads
constexpr int kRegsProducer = 56, kRegsConverter = 64, kRegsEpilogue = 192;
constexpr uint32_t kIdesc = ptx::idesc_tf32(kM, kN);
constexpr size_t kSmemBytes = (size_t)(kRaw + kLo) * kStageBytes + 1024 + 512;

struct Plan {
  int nb, tiles, P, grid, KB, KC, D;
  bool direct;
};

FS_DEVINL void tile_of(int t, int nb, int& I, int& J0) {
  int acc = 0;
  for (int i = 0; i < nb; ++i) {
    const int cnt = i / kNB + 1;
    if (t < acc + cnt) { I = i; J0 = (t - acc) * kNB; return; }
    acc += cnt;
  }
  I = nb - 1; J0 = 0;
}

struct Ring {  // stage index + mbarrier phase of a circular buffer
  int s = 0;
  uint32_t ph = 0;
  FS_DEVINL void next(int depth) { if (++s == depth) { s = 0; ph ^= 1; } }
};

__global__ void __launch_bounds__(kThreads, 1)
syrk_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap pmap, int64_t n,
               int nb, int tiles, int P, int KB, int KC, int D, double* __restrict__ accbuf,
               double* __restrict__ Gp, double lam, int direct, int dbg) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* raw = smem;
  uint8_t* lo = smem + (size_t)kRaw * kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)(kRaw + kLo) * kStageBytes);
  uint64_t* full = bars;                 // TMA -> converters        [kRaw]
  uint64_t* conv = full + kRaw;          // converters -> MMA        [kRaw]
  uint64_t* empty = conv + kRaw;         // MMA -> TMA (raw free)    [kRaw]
  uint64_t* lo_free = empty + kRaw;      // MMA -> converters        [kLo]
  uint64_t* tfull = lo_free + kLo;       // MMA -> epilogue          [2]
  uint64_t* tempty = tfull + 2;          // epilogue -> MMA          [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRaw; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&conv[s], 128);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kLo; ++s) ptx::mbar_init(&lo_free[s], 1);
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 256);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tmap);
    ptx::tma_prefetch_desc(&pmap);
  }
  if (warp == 1) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int units = tiles * P;
  const int wg = warp >> 2;

  if (wg == 0) {
    ptx::setmaxnreg_dec<kRegsProducer>();
    if (warp == 0 && lane == 0) {
      // ======================= TMA producer =======================
      Ring rr;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int t = u / P, q = u % P;
        int I, J0; tile_of(t, nb, I, J0);
        const bool a_in_b = I >= J0 && I < J0 + kNB;
        const uint32_t bytes = (kNB + (a_in_b ? 0 : 1)) * kBoxBytes;
        const int kb0 = q * KC, nk = min(KC, KB - kb0);   // contiguous K range of this split
        for (int k = 0; k < nk; ++k) {
          if (!(dbg & 32) && k % kPfSpan == 0) {
            // keep kPfAhead spans of every operand row block in flight to L2
            for (int a = (k == 0 ? 0 : kPfAhead); a <= kPfAhead; ++a) {
              const int pk = k + a * kPfSpan;
              if (pk >= nk) break;
              const int pcol = (kb0 + pk) * kBK;
#pragma unroll
              for (int j = 0; j < kNB; ++j) ptx::tma_prefetch_l2_2d(&pmap, pcol, (J0 + j) * 128);
              if (!a_in_b) ptx::tma_prefetch_l2_2d(&pmap, pcol, I * 128);
            }
          }
          ptx::mbar_wait(&empty[rr.s], rr.ph ^ 1);
          if (dbg & 1) { ptx::mbar_arrive(&full[rr.s]); rr.next(kRaw); continue; }
          ptx::mbar_arrive_expect_tx(&full[rr.s], bytes);
          uint8_t* st = raw + (size_t)rr.s * kStageBytes;
          const int col = (kb0 + k) * kBK;
#pragma unroll
          for (int j = 0; j < kNB; ++j) ptx::tma_load_2d(st + j * kBoxBytes, &tmap, &full[rr.s], col, (J0 + j) * 128);
          if (!a_in_b) ptx::tma_load_2d(st + kNB * kBoxBytes, &tmap, &full[rr.s], col, I * 128);
          rr.next(kRaw);
        }
      }
    } else if (warp == 1 && lane == 0) {
      // ======================= MMA issuer =======================
      Ring rr, lr;
      uint32_t chunk = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int t = u / P, q = u % P;
        int I, J0; tile_of(t, nb, I, J0);
        const bool a_in_b = I >= J0 && I < J0 + kNB;
        const int a_off = a_in_b ? (I - J0) * kBoxBytes : kNB * kBoxBytes;
        const int kb0 = q * KC, nk = min(KC, KB - kb0);
        uint32_t dacc = 0;
        for (int k = 0; k < nk; ++k) {
          const int kin = k % D;
          if (kin == 0) {
            const uint32_t b = chunk & 1;
            ptx::mbar_wait(&tempty[b], ((chunk >> 1) & 1) ^ 1);
            ptx::tc_fence_after();
            dacc = tmem + b * kN;
          }
          ptx::mbar_wait(&conv[rr.s], rr.ph);
          ptx::tc_fence_after();
          const uint32_t rs = ptx::smem_u32(raw + (size_t)rr.s * kStageBytes);
          const uint32_t ls = ptx::smem_u32(lo + (size_t)lr.s * kStageBytes);
#pragma unroll
          for (int kk = 0; kk < (dbg & 4 ? 0 : kBK / 8); ++kk) {
            const uint32_t off = kk * 32;
            const uint64_t a_hi = ptx::desc_kmajor<kRowBytes>(rs + a_off + off);
            const uint64_t a_lo = ptx::desc_kmajor<kRowBytes>(ls + a_off + off);
            const uint64_t b_hi = ptx::desc_kmajor<kRowBytes>(rs + off);
            const uint64_t b_lo = ptx::desc_kmajor<kRowBytes>(ls + off);
            ptx::mma_tf32(dacc, a_lo, b_hi, kIdesc, (kin > 0 || kk > 0) ? 1u : 0u);
            ptx::mma_tf32(dacc, a_hi, b_lo, kIdesc, 1u);
            ptx::mma_tf32(dacc, a_hi, b_hi, kIdesc, 1u);
          }
          ptx::mma_commit(&empty[rr.s]);
          ptx::mma_commit(&lo_free[lr.s]);
          if (kin == D - 1 || k == nk - 1) {
            ptx::mma_commit(&tfull[chunk & 1]);
            ++chunk;
          }
          rr.next(kRaw);
          lr.next(kLo);
        }
      }
    }
  } else if (wg == 1) {
    // ======================= converters =======================
    ptx::setmaxnreg_dec<kRegsConverter>();
    const int ct = threadIdx.x - 128;
    Ring rr, lr;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int t = u / P, q = u % P;
      int I, J0; tile_of(t, nb, I, J0);
      const bool a_in_b = I >= J0 && I < J0 + kNB;
      const int nvec = (kNB + (a_in_b ? 0 : 1)) * (kBoxBytes / 16);
      const int kb0 = q * KC, nk = min(KC, KB - kb0);
      for (int k = 0; k < nk; ++k) {
        ptx::mbar_wait(&full[rr.s], rr.ph);
        ptx::mbar_wait(&lo_free[lr.s], lr.ph ^ 1);
        if (!(dbg & 2)) {
          float4* r4 = reinterpret_cast<float4*>(raw + (size_t)rr.s * kStageBytes);
          float4* l4 = reinterpret_cast<float4*>(lo + (size_t)lr.s * kStageBytes);
#pragma unroll 4
          for (int i = ct; i < nvec; i += 128) {
            const float4 x = r4[i];
            float4 h, l;
            h.x = ptx::tf32_rna(x.x); h.y = ptx::tf32_rna(x.y); h.z = ptx::tf32_rna(x.z); h.w = ptx::tf32_rna(x.w);
            l.x = x.x - h.x; l.y = x.y - h.y; l.z = x.z - h.z; l.w = x.w - h.w;
            r4[i] = h;
            l4[i] = l;
          }
          ptx::fence_async_smem();
        }
        ptx::mbar_arrive(&conv[rr.s]);
        rr.next(kRaw);
        lr.next(kLo);
      }
    }
  } else {
    // ======================= epilogue (8 warps) =======================
    ptx::setmaxnreg_inc<kRegsEpilogue>();
    // warp -> TMEM lane quarter (warp & 3) and column half ((warp - 8) >> 2); thread -> one row
    const int sub = warp & 3, half = (warp - 8) >> 2;
    const int r = 32 * sub + lane;
    const uint32_t lane_base = (uint32_t)(32 * sub) << 16;
    float acc[kN / 2];
    uint32_t chunk = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int t = u / P, q = u % P;
      int I, J0; tile_of(t, nb, I, J0);
      const int kb0 = q * KC, nk = min(KC, KB - kb0);
      const int nch = (nk + D - 1) / D;
      double* __restrict__ sc = (direct ? accbuf + (size_t)blockIdx.x * kM * kN : accbuf + (size_t)u * kM * kN) +
                                (size_t)half * (kN / 2) * kM + r;   // column-major [c][r], this thread's row
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
        ptx::mbar_arrive(&tempty[b]);
        ++chunk;
        if (!(dbg & 8) && ((j + 1) % kFlushChunks == 0 || j == nch - 1)) {
          // fp64 flush, 16 independent loads in flight per group
#pragma unroll
          for (int g = 0; g < kN / 2; g += 16) {
            double old[16];
            if (!first_flush) {
#pragma unroll
              for (int e = 0; e < 16; ++e) old[e] = sc[(size_t)(g + e) * kM];
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) sc[(size_t)(g + e) * kM] = (first_flush ? 0.0 : old[e]) + (double)acc[g + e];
          }
          first_flush = false;
        }
      }
      if (direct) {
        const int64_t gi = (int64_t)I * 128 + r;
        if (gi < n) {
          for (int e = 0; e < kN / 2; ++e) {
            const int c = half * (kN / 2) + e;
            const int64_t gj = (int64_t)J0 * 128 + c;
            if (gj > gi) break;
            Gp[gi * (gi + 1) / 2 + gj] = sc[(size_t)e * kM] + (gi == gj ? lam : 0.0);
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc<kTmemCols>(tmem);
}

// Fixed-order sum of the P split-K partial tiles -> packed lower Gram (+λ on the diagonal).
__global__ void syrk_tc_reduce(const double* __restrict__ ws, int nb, int P, int64_t n, double lam,
                               double* __restrict__ Gp) {
  int I, J0;
  tile_of(blockIdx.x, nb, I, J0);
  for (int e = threadIdx.x; e < kM * kN; e += blockDim.x) {
    const int c = e / kM, r = e % kM;
    const int64_t gi = (int64_t)I * 128 + r, gj = (int64_t)J0 * 128 + c;
    if (gi >= n || gj > gi) continue;
    double s = 0.0;
    for (int q = 0; q < P; ++q) s += ws[((size_t)blockIdx.x * P + q) * kM * kN + e];
    Gp[gi * (gi + 1) / 2 + gj] = s + (gi == gj ? lam : 0.0);
  }
}

Plan make_plan(int64_t n, int64_t m, int num_sms) {
  Plan p;
  p.nb = (int)((n + 127) / 128);
  p.tiles = 0;
  for (int i = 0; i < p.nb; ++i) p.tiles += i / kNB + 1;
  p.KB = (int)((m + kBK - 1) / kBK);
  p.P = p.tiles >= num_sms ? 1 : std::max(1, std::min(num_sms / p.tiles, p.KB / 16));  // >= 16 K-blocks per unit
  p.KC = (p.KB + p.P - 1) / p.P;          // K-blocks per split, contiguous in m
  p.P = (p.KB + p.KC - 1) / p.KC;          // every split non-empty
  const int units = p.tiles * p.P;
  p.grid = std::min(units, num_sms);
  p.D = kDrainBlocks;
  p.direct = p.P == 1;
  return p;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

}  // namespace

size_t syrk_tc_plan_bytes(int64_t n, int64_t m, int num_sms) {
  Plan p = make_plan(n, m, num_sms);
  return (size_t)(p.direct ? p.grid : p.tiles * p.P) * kM * kN * sizeof(double);
}

bool syrk_tc_supported(const void* S, int64_t ldS) {
  return (reinterpret_cast<uintptr_t>(S) % 16 == 0) && ((ldS * 4) % 16 == 0);
}

size_t syrk_tc_workspace_bytes(int64_t n, int64_t m, int num_sms) {
  // one fp64 partial tile per unit (split-K) or per resident CTA (direct): never more than
  // num_sms slots for ANY (n, m), so a context sized once serves every smaller problem
  (void)n; (void)m;
  return (size_t)num_sms * kM * kN * sizeof(double);
}

cudaError_t syrk_tc(const float* S, int64_t n, int64_t m, int64_t ldS, double lam, double* G_packed, double* ws,
                    int num_sms, cudaStream_t st, int* launches) {
  EncodeTiledFn encode = get_encode();
  if (!encode) return cudaErrorNotSupported;
  Plan p = make_plan(n, m, num_sms);
  CUtensorMap tmap, pmap;
  const cuuint64_t gdim[2] = {(cuuint64_t)m, (cuuint64_t)n};
  const cuuint64_t gstride[1] = {(cuuint64_t)ldS * 4};
  const cuuint32_t box[2] = {(cuuint32_t)kBK, 128u};
  const cuuint32_t pbox[2] = {(cuuint32_t)(kBK * kPfSpan), 128u};   // 1 KB x 128 rows prefetch box
  const cuuint32_t estride[2] = {1u, 1u};
  CUresult cr = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(S), gdim, gstride, box, estride,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, kBK == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  cr = encode(&pmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(S), gdim, gstride, pbox, estride,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(syrk_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  static const int dbg = getenv("FS_SYRK_DBG") ? atoi(getenv("FS_SYRK_DBG")) : 0;  // ablation experiments only
  syrk_tc_kernel<<<p.grid, kThreads, kSmemBytes, st>>>(tmap, pmap, n, p.nb, p.tiles, p.P, p.KB, p.KC, p.D, ws,
                                                       G_packed, lam, p.direct ? 1 : 0, dbg);
  if (launches) *launches += 1;
  if (!p.direct) {
    syrk_tc_reduce<<<p.tiles, 256, 0, st>>>(ws, p.nb, p.P, n, lam, G_packed);
    if (launches) *launches += 1;
  }
  return cudaGetLastError();
}

}  // namespace fs
