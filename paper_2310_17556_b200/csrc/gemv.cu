// gemv.cu — HBM-bound streaming passes over the score matrix S (n x m, row-major).
//
//   gemv_rows        u = S w            (solvers.py:110 "A @ b", core.py:297 "A @ x")
//   gemv_cols_solve  x = (v - S^T z)/λ  (solvers.py:122-126, fused epilogue; refinement :188)
//   residual_cols    r = S^T y + λx - v, ||r||², ||v||²   (core.py:297, :319-321)
//
// Roofline: each pass reads S once (n·m·s bytes) plus O(m) vectors; the kernels are
// sized to keep ~32–64 KB of loads in flight per SM (Little's law at ~6.5 TB/s) and
// use 16-byte L1::no_allocate / L2::evict_first loads.  All reductions are fixed-order
// (per-chunk partials reduced in chunk order) so results are bit-reproducible.
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"
#include "tiles.cuh"

#include <algorithm>
#include <stdlib.h>
#include <string.h>

namespace fs {
namespace {

constexpr int kRowThreads = 256;   // 8 warps
constexpr int kRowUnroll = 8;      // vectors per lane per row
constexpr int kColThreads = 256;

template <typename TS> struct VecOf;
template <> struct VecOf<float> { using V = float4; static constexpr int N = 4; };
template <> struct VecOf<double> { using V = double2; static constexpr int N = 2; };

template <typename T> FS_DEVINL void vec_to_array(const float4& v, T* a) { a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w; }
template <typename T> FS_DEVINL void vec_to_array(const double2& v, T* a) { a[0] = v.x; a[1] = v.y; }

// fp32 -> fp64, exact, on the integer + fp64 pipes instead of the XU pipe (F2F.F64.F32 paced the
// fused x + y pass: ncu XU 63% busy).  Arithmetic shift right by 3 puts sign | exponent | mantissa
// where an fp64 with exponent field e (bias 1023) wants them, the mask clears the sign copies, the
// low word takes the last 3 mantissa bits; the double read is x * 2^-896 (denormal x included),
// the multiply by 2^896 is exact.  fp32 inf/NaN (rejected by input validation) map to finite values.
FS_DEVINL double f2d_alu(float x) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t hi = ((uint32_t)((int32_t)u >> 3)) & 0x8FFFFFFFu;
  return __hiloint2double((int)hi, (int)(u << 29)) * 0x1p896;
}
// element e of a 4-float vector: 3 of 4 through the integer pipe, 1 through the XU pipe (balances
// the two; the fp64 pipe takes the extra DMULs)
template <typename T> FS_DEVINL double to_f64_mix(T x, int e) { return (double)x; }
template <> FS_DEVINL double to_f64_mix<float>(float x, int e) { return (e & 3) == 3 ? (double)x : f2d_alu(x); }

template <typename TS>
constexpr int row_chunk_cols() { return kWarp * VecOf<TS>::N * kRowUnroll; }

// One CTA = one column chunk of width CW; warp w handles rows w, w+8, ...
// Products: fp32 x fp32 are formed in fp32 and summed per lane (32 terms) before the
// fp64 warp reduction; any fp64 operand forces exact fp64 products.
template <typename TS, typename TW, bool kVec>
__global__ void __launch_bounds__(kRowThreads)
gemv_rows_kernel(const TS* __restrict__ S, int64_t n, int64_t m, int64_t ldS,
                 const TW* __restrict__ w, double* __restrict__ partials) {
  using VT = typename VecOf<TS>::V;
  constexpr int VN = VecOf<TS>::N;
  constexpr int CW = row_chunk_cols<TS>();
  constexpr bool kF32 = sizeof(TS) == 4 && sizeof(TW) == 4;
  using Acc = typename std::conditional<kF32, float, double>::type;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * CW;
  Acc wr[kRowUnroll][VN];
#pragma unroll
  for (int u = 0; u < kRowUnroll; ++u)
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      int64_t c = c0 + (int64_t)(u * kWarp + lane) * VN + e;
      wr[u][e] = c < m ? (Acc)w[c] : (Acc)0;
    }
  const bool full = c0 + CW <= m;
  for (int64_t i = warp; i < n; i += kRowThreads / kWarp) {
    const TS* row = S + i * ldS + c0;
    Acc acc = 0;
    if (kVec && full) {
      VT buf[kRowUnroll];
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u)
        buf[u] = ld_stream(reinterpret_cast<const VT*>(row + (u * kWarp + lane) * VN));
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        TS a[VN];
        vec_to_array(buf[u], a);
#pragma unroll
        for (int e = 0; e < VN; ++e) acc = fma((Acc)a[e], wr[u][e], acc);
      }
    } else {
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u)
#pragma unroll
        for (int e = 0; e < VN; ++e) {
          int64_t c = (int64_t)(u * kWarp + lane) * VN + e;
          if (c0 + c < m) acc = fma((Acc)ld_stream(row + c), wr[u][e], acc);
        }
    }
    double s = warp_sum((double)acc);
    if (lane == 0) partials[(int64_t)blockIdx.x * n + i] = s;
  }
}

// fp32 u = S w that also writes the tiled copy S_t (tiles.cuh) of the CTA's column chunk:
// each lane's float4 is exactly one 16-byte chunk of one tile row, so every warp store is
// four full 128-byte tile rows.  Columns in [m, KB*32) and rows in [n, nb*128) are zeroed.
__global__ void __launch_bounds__(kRowThreads, 2)
gemv_rows_retile_kernel(const float* __restrict__ S, int64_t n, int64_t m, int64_t ldS,
                        const float* __restrict__ w, double* __restrict__ partials, uint8_t* __restrict__ St,
                        int has_w, int vec_ok, int64_t r0, int64_t r1, int64_t rz, int* __restrict__ nonfinite,
                        int64_t cb0) {
  constexpr int VN = 4;
  constexpr int CW = row_chunk_cols<float>();            // 1024 columns = 32 K-blocks
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t cb = cb0 + blockIdx.x;                   // global column chunk
  const int64_t c0 = cb * CW;
  const int64_t nb = tiles_nb(n), KB = tiles_kb(m);
  // the chunk's weights live in smem (registers go to the loads in flight: 2 CTAs per SM)
  __shared__ float4 wsm[CW / VN];
  for (int t = threadIdx.x; t < CW / VN; t += kRowThreads) {
    float a[VN];
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      const int64_t c = c0 + (int64_t)t * VN + e;
      a[e] = (has_w && c < m) ? w[c] : 0.f;
    }
    wsm[t] = make_float4(a[0], a[1], a[2], a[3]);
  }
  __syncthreads();
  const bool full = vec_ok && c0 + CW <= m;
  const int chunk = lane & 7;
  // rows [r0, r1) are read from S; rows [r1, rz) are zero padding of the tiled copy
  bool bad = false;
  for (int64_t i = r0 + warp; i < rz; i += kRowThreads / kWarp) {
    float4 buf[kRowUnroll];
    if (i < r1) {
      const float* row = S + i * ldS + c0;
      if (full) {
#pragma unroll
        for (int u = 0; u < kRowUnroll; ++u) buf[u] = ld_stream(reinterpret_cast<const float4*>(row + (u * kWarp + lane) * VN));
      } else {
#pragma unroll
        for (int u = 0; u < kRowUnroll; ++u) {
          float a[VN];
#pragma unroll
          for (int e = 0; e < VN; ++e) {
            const int64_t c = (int64_t)(u * kWarp + lane) * VN + e;
            a[e] = (c0 + c < m) ? __ldg(row + c) : 0.f;
          }
          buf[u] = make_float4(a[0], a[1], a[2], a[3]);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) buf[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) {
      const int64_t kb = (c0 >> 5) + u * 4 + (lane >> 3);
      if (kb < KB) *reinterpret_cast<float4*>(St + tile_chunk_offset(nb, kb, i, chunk)) = buf[u];
      bad |= !(isfinite(buf[u].x) && isfinite(buf[u].y) && isfinite(buf[u].z) && isfinite(buf[u].w));
    }
    if (i < r1 && has_w) {
      float acc = 0.f;
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        const float4 wv = wsm[u * kWarp + lane];
        acc = fmaf(buf[u].x, wv.x, acc); acc = fmaf(buf[u].y, wv.y, acc);
        acc = fmaf(buf[u].z, wv.z, acc); acc = fmaf(buf[u].w, wv.w, acc);
      }
      const double s = warp_sum((double)acc);
      if (lane == 0) partials[cb * n + i] = s;
    }
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(nonfinite, 1);
}

// out[i] = sum_{c=0..C-1} partials[c*n + i], fixed order: block = 32 rows; warp w sums the
// chunks c = w, w+8, ... (coalesced 256-byte rows), then the 8 warp sums in warp order.
constexpr int kRedRows = 32, kRedWarps = 8;
__global__ void __launch_bounds__(kRedRows * kRedWarps)
reduce_chunks_kernel(const double* __restrict__ partials, int64_t chunks, int64_t n, int64_t stride,
                     double* __restrict__ out) {
  __shared__ double part[kRedWarps][kRedRows];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * kRedRows + lane;
  double s0 = 0.0, s1 = 0.0;
  if (i < n) {
    int64_t c = w;
    for (; c + kRedWarps < chunks; c += 2 * kRedWarps) {
      s0 += partials[c * stride + i];
      s1 += partials[(c + kRedWarps) * stride + i];
    }
    if (c < chunks) s0 += partials[c * stride + i];
  }
  part[w][lane] = s0 + s1;
  __syncthreads();
  if (w == 0 && i < n) {
    double s = 0.0;
    for (int k = 0; k < kRedWarps; ++k) s += part[k][lane];
    out[i] = s;
  }
}

// One thread owns VN consecutive columns and walks all n rows.
template <typename TS, typename TV, bool kVec>
__global__ void __launch_bounds__(kColThreads)
gemv_cols_solve_kernel(const TS* __restrict__ S, int64_t n, int64_t m, int64_t ldS,
                       const double* __restrict__ z, const TV* __restrict__ v, double lam,
                       int accumulate, double* __restrict__ x) {
  using VT = typename VecOf<TS>::V;
  constexpr int VN = VecOf<TS>::N;
  constexpr int kZ = 2048;
  constexpr int kInner = 16;  // fp32 partial sums span 16 rows before folding into fp64
  // fp32 S with an fp32 right-hand side multiplies in fp32 (z rounded once); an fp64 right-hand
  // side (fp64 precision mode) makes every product and sum exact fp64
  using Zt = typename std::conditional<sizeof(TS) == 8 || sizeof(TV) == 8, double, float>::type;
  __shared__ Zt zs[kZ];
  const int64_t col = ((int64_t)blockIdx.x * kColThreads + threadIdx.x) * VN;
  double acc[VN];
#pragma unroll
  for (int e = 0; e < VN; ++e) acc[e] = 0.0;
  const bool full = kVec && (col + VN <= m);
  for (int64_t r0 = 0; r0 < n; r0 += kZ) {
    const int rows = (int)(n - r0 < kZ ? n - r0 : kZ);
    __syncthreads();
    for (int t = threadIdx.x; t < rows; t += kColThreads) zs[t] = (Zt)z[r0 + t];
    __syncthreads();
    if (col >= m) continue;
    const TS* base = S + r0 * ldS + col;
    for (int i0 = 0; i0 < rows; i0 += kInner) {
      Zt part[VN];
#pragma unroll
      for (int e = 0; e < VN; ++e) part[e] = 0;
      const int cnt = min(kInner, rows - i0);
      if (full && cnt == kInner) {
        VT buf[kInner];
#pragma unroll
        for (int k = 0; k < kInner; ++k)
          buf[k] = ld_stream(reinterpret_cast<const VT*>(base + (int64_t)(i0 + k) * ldS));
#pragma unroll
        for (int k = 0; k < kInner; ++k) {
          TS a[VN];
          vec_to_array(buf[k], a);
#pragma unroll
          for (int e = 0; e < VN; ++e) part[e] = fma(zs[i0 + k], (Zt)a[e], part[e]);
        }
      } else {
        for (int k = 0; k < cnt; ++k)
#pragma unroll
          for (int e = 0; e < VN; ++e)
            if (col + e < m) part[e] = fma(zs[i0 + k], (Zt)ld_stream(base + (int64_t)(i0 + k) * ldS + e), part[e]);
      }
#pragma unroll
      for (int e = 0; e < VN; ++e) acc[e] += (double)part[e];
    }
  }
  if (col >= m) return;
#pragma unroll
  for (int e = 0; e < VN; ++e) {
    const int64_t c = col + e;
    if (c < m) {
      double xv = ((double)v[c] - acc[e]) / lam;  // true IEEE division (x = v/λ exactly for S = 0)
      if (accumulate) xv = x[c] + xv;
      x[c] = xv;
    }
  }
}

// Fused x = (v - S^T z)/λ (optionally x += ...) and the residual's first product y = S x.
// Persistent CTAs (one per SM; 512 threads = 16 column groups of two 16-byte vectors x 32 row
// groups) walk column panels of 512-byte row segments (fp32: 128 columns).  Per panel:
//   (1) x: each thread sums its rows' z-weighted vectors (Zt partial sums of 8 rows, fp64
//       across them); the row groups are added in fixed order (warp xor, then warps) -> x;
//   (2) y: the panel is read again (L2 hit) and S[i, panel] . x[panel] (exact fp64 products)
//       is added to a per-CTA smem accumulator yacc[column group][row] (one owner per slot).
// At the end each CTA writes sum_cg yacc[cg][.] as its y partial; reduce_chunks adds the CTA
// partials in order.  S leaves HBM once instead of twice (gemv_cols_solve + gemv_rows).
constexpr int kCYThreads = 512;
constexpr int kCYCG = 16;                      // column groups: 256-byte fp32 row segments
constexpr int kCYRG = kCYThreads / kCYCG;      // 32 row groups
constexpr int kCYWarps = kCYThreads / kWarp;   // 16 (2 row groups each)
constexpr int kCYU = 8;                        // rows per unrolled batch (per thread)
constexpr int kCYV = 2;                        // adjacent 16-byte vectors per thread and row

template <typename TS> constexpr int cy_cols() { return kCYCG * kCYV * VecOf<TS>::N; }

// yacc row stride: n rounded to 16 plus one (the 16 column groups of a row on distinct banks)
__host__ __device__ inline int64_t cy_pitch(int64_t n) { return ((n + 15) & ~(int64_t)15) + 1; }

template <typename TS>
size_t cy_smem_bytes(int64_t n) {
  return (size_t)kCYCG * cy_pitch(n) * sizeof(double) + (size_t)kCYWarps * cy_cols<TS>() * sizeof(double) +
         cy_cols<TS>() * sizeof(double) + (size_t)n * sizeof(double);
}

template <typename TS, typename TV>
__global__ void __launch_bounds__(kCYThreads, 1)
cols_solve_y_kernel(const TS* __restrict__ S, int64_t n, int64_t m, int64_t ldS, const double* __restrict__ z,
                    const TV* __restrict__ v, double lam, int accumulate, double* __restrict__ x,
                    double* __restrict__ ypart, int y_only, const __grid_constant__ CUtensorMap pmap, int use_pf) {
  using VT = typename VecOf<TS>::V;
  constexpr int VN1 = VecOf<TS>::N;
  constexpr int VN = VN1 * kCYV;                // columns per thread
  constexpr int CW = cy_cols<TS>();
  using Zt = typename std::conditional<sizeof(TV) == 8, double, float>::type;
  extern __shared__ double cy_sm[];
  const int64_t P = cy_pitch(n);
  double* yacc = cy_sm;                                   // [kCYCG][P]
  double* red = yacc + (size_t)kCYCG * P;                 // [kCYWarps][CW]
  double* xs = red + kCYWarps * CW;                       // [CW]
  double* zs = xs + CW;                                   // [n]
  const int cg = threadIdx.x % kCYCG, rg = threadIdx.x / kCYCG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (!y_only)
    for (int64_t i = threadIdx.x; i < n; i += kCYThreads) zs[i] = z[i];
  for (int64_t i = threadIdx.x; i < (int64_t)kCYCG * P; i += kCYThreads) yacc[i] = 0.0;
  const int64_t panels = (m + CW - 1) / CW;
  // TMA L2 prefetch of a whole panel: n/256 box requests issued by one thread
  auto prefetch = [&](int64_t q) {
    if (!use_pf || threadIdx.x != 0 || q >= panels) return;
    for (int64_t r = 0; r < n; r += 256)
      asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(&pmap), "r"((int)(q * CW)),
                   "r"((int)r)
                   : "memory");
  };
  prefetch(blockIdx.x);
  __syncthreads();
  for (int64_t q = blockIdx.x; q < panels; q += gridDim.x) {
    prefetch(q + gridDim.x);            // the next panel streams into L2 while this one is computed
    const int64_t col = q * CW + cg * VN;
    const bool full = col + VN <= m;
    if (y_only) {
      if (threadIdx.x < CW) {
        const int64_t c = q * CW + threadIdx.x;
        xs[threadIdx.x] = c < m ? x[c] : 0.0;
      }
    } else {
      // ---- (1) x for the panel ----
      double acc[VN];
#pragma unroll
      for (int e = 0; e < VN; ++e) acc[e] = 0.0;
      if (col < m) {
        for (int64_t i0 = rg; i0 < n; i0 += (int64_t)kCYRG * kCYU) {
          Zt part[VN];
#pragma unroll
          for (int e = 0; e < VN; ++e) part[e] = 0;
          if (full && i0 + (int64_t)kCYRG * (kCYU - 1) < n) {
            VT buf[kCYU][kCYV];
#pragma unroll
            for (int u = 0; u < kCYU; ++u)
#pragma unroll
              for (int w = 0; w < kCYV; ++w)
                buf[u][w] = __ldg(reinterpret_cast<const VT*>(S + (i0 + kCYRG * u) * ldS + col + w * VN1));
#pragma unroll
            for (int u = 0; u < kCYU; ++u) {
              TS a[VN];
#pragma unroll
              for (int w = 0; w < kCYV; ++w) vec_to_array(buf[u][w], a + w * VN1);
#pragma unroll
              for (int e = 0; e < VN; ++e) part[e] = fma((Zt)zs[i0 + kCYRG * u], (Zt)a[e], part[e]);
            }
          } else {
            for (int u = 0; u < kCYU; ++u) {
              const int64_t i = i0 + kCYRG * u;
              if (i >= n) break;
#pragma unroll
              for (int e = 0; e < VN; ++e)
                if (col + e < m) part[e] = fma((Zt)zs[i], (Zt)__ldg(S + i * ldS + col + e), part[e]);
            }
          }
#pragma unroll
          for (int e = 0; e < VN; ++e) acc[e] += (double)part[e];
        }
      }
#pragma unroll
      for (int e = 0; e < VN; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 16);   // the warp's 2 row groups
      if (lane < kCYCG) {
#pragma unroll
        for (int e = 0; e < VN; ++e) red[warp * CW + cg * VN + e] = acc[e];
      }
      __syncthreads();
      if (threadIdx.x < CW) {
        const int t = threadIdx.x;
        double sum = 0.0;
#pragma unroll
        for (int g = 0; g < kCYWarps; ++g) sum += red[g * CW + t];
        const int64_t c = q * CW + t;
        double xv = 0.0;
        if (c < m) {
          xv = ((double)v[c] - sum) / lam;   // true IEEE division, as gemv_cols_solve
          if (accumulate) xv = x[c] + xv;
          x[c] = xv;
        }
        xs[t] = xv;
      }
    }
    __syncthreads();
    // ---- (2) y += S[:, panel] x[panel] (exact fp64 products; the panel is re-read from L2) ----
    if (col < m) {
      double xv[VN];
#pragma unroll
      for (int e = 0; e < VN; ++e) xv[e] = xs[cg * VN + e];
      double* ya = yacc + (size_t)cg * P;
      for (int64_t i0 = rg; i0 < n; i0 += (int64_t)kCYRG * kCYU) {
        if (full && i0 + (int64_t)kCYRG * (kCYU - 1) < n) {
          VT buf[kCYU][kCYV];
#pragma unroll
          for (int u = 0; u < kCYU; ++u)
#pragma unroll
            for (int w = 0; w < kCYV; ++w)
              buf[u][w] = ld_stream(reinterpret_cast<const VT*>(S + (i0 + kCYRG * u) * ldS + col + w * VN1));
#pragma unroll
          for (int u = 0; u < kCYU; ++u) {
            TS a[VN];
#pragma unroll
            for (int w = 0; w < kCYV; ++w) vec_to_array(buf[u][w], a + w * VN1);
            double p = 0.0;
#pragma unroll
            for (int e = 0; e < VN; ++e) p = fma((double)a[e], xv[e], p);
            ya[i0 + kCYRG * u] += p;
          }
        } else {
          for (int u = 0; u < kCYU; ++u) {
            const int64_t i = i0 + kCYRG * u;
            if (i >= n) break;
            double p = 0.0;
#pragma unroll
            for (int e = 0; e < VN; ++e)
              if (col + e < m) p = fma((double)__ldg(S + i * ldS + col + e), xv[e], p);
            ya[i] += p;
          }
        }
      }
    }
    __syncthreads();   // xs / red reuse by the next panel
  }
  for (int64_t i = threadIdx.x; i < n; i += kCYThreads) {
    double sum = 0.0;
#pragma unroll
    for (int g = 0; g < kCYCG; ++g) sum += yacc[(size_t)g * P + i];
    ypart[(int64_t)blockIdx.x * n + i] = sum;
  }
}

// Cluster variant for n <= 4576 (4-CTA clusters up to n = 1144, the headline n = 1024; 8 and 16 above).  The TMA engine moves ~one box row
// per 8 SM clocks, so 128-byte-wide boxes cap a full strided read of S at ~4.6 TB/s while
// 256-byte rows reach ~6.6 TB/s (tools/ubench/tma_seg.cu).  A panel is therefore 256 bytes of
// columns (64 fp32 / 32 fp64), split by ROWS over a cluster of CL CTAs: CTA r streams rows
// [r*NCH*30, (r+1)*NCH*30) of each panel as NCH 30-row TMA boxes (rows past n arrive as zeros)
// into one slot-set of a ring, completing on the set's single mbarrier.  x needs the column sums
// over all n rows: each CTA reduces its rows and pushes its partial column sums into every peer's
// exchange buffer with st.async (the data and the peer's mbarrier complete_tx travel together);
// every CTA adds the CL partials in rank order, so x is identical everywhere.  Software
// pipeline, one CTA barrier per panel: iteration j
//   warps 2-3  (after the push below) x of panel j-1 from the exchange, pushed an iteration ago
//   all warps  x-phase of panel j: partial column sums
//   -- barrier --
//   warps 0-1  sum the per-warp partials of panel j, push them to the cluster
//   all warps  y += S_{panel j-1} x_{j-1} from the still-resident set, release the set
// S is read from HBM exactly once.
// CTAs per cluster (row split): 4 up to n = 1144, 8 up to n = 2288, 16 (non-portable) up to 4576
// 15 consumer warps + 1 producer warp: 4 warps per SM sub-partition, so up to 128 registers per
// thread (a 17th warp would cap every thread at 96)
constexpr int kCLCW = 15;                        // consumer warps
constexpr int kCLCons = kCLCW * kWarp;
constexpr int kCLThreads = kCLCons + kWarp;
// 26 rows per chunk (TMA box outer dimension) = 13 row pairs: at most two per x-group and per
// y-group warp (with 30 rows one x warp carried three pairs and paced the whole pass), and small
// enough that three 10-chunk slot-sets fit beside the fixed buffers for every cluster size
constexpr int kCLRows = 26;
constexpr int kCLChunk = kCLRows * 256;          // 6.5 KB per chunk slot (128-byte aligned)
constexpr int kCLMaxV = 11;                      // chunks per CTA and panel -> 286 rows per CTA
constexpr int kCLMaxRows4 = 4 * kCLRows * kCLMaxV;   // n <= 1144 with 4-CTA clusters
constexpr int kCLMaxRows8 = 8 * kCLRows * kCLMaxV;   // n <= 2288 with 8-CTA clusters
constexpr int kCLMaxRows16 = 16 * kCLRows * kCLMaxV;  // n <= 4576 with 16-CTA (non-portable) clusters
constexpr int kCLG = 3;                          // chunks per batch of shared loads (y group)
constexpr int kCLXW = 7;                         // x-group warps (partial sums, exchange, x)
// exchange buffers: x of panel j-1 is formed after panel j's push, so a peer may push panels
// j+1 and j+2 before this CTA consumes j-1 (it cannot push j+3: that needs this CTA's push j+1)
// exchange buffers: a peer's push of panel q needs its slot-set of q - R free, i.e. this CTA's push
// of q - R, which needs this CTA's own y group past q - 2R — so the x partials of panel p (read
// when this CTA's y group forms x of p) are safe from a peer's push of p + K for K >= 2R.  K per
// cluster size; the slot-set count R is capped at (K - 1) / 2.
__host__ __device__ constexpr int cl_xb(int CL) { return CL >= 16 ? 5 : 9; }
constexpr int kCLYW = kCLCW - kCLXW;             // y-group warps (8)
constexpr int kCLXThreads = kCLXW * kWarp;
constexpr int kCLSets = 8;                       // max panel slot-sets in the ring
__host__ __device__ constexpr size_t cl_fixed(int CL) {
  return 2 * kCLXW * 64 * 8 + cl_xb(CL) * (CL + 1) * 64 * 8 + 2 * 64 * 8 + (2 * kCLSets + cl_xb(CL)) * 8;
}
// as many chunk slots as fit beside the fixed buffers in 227 KB (33 / 32 / 30 for CL = 4 / 8 / 16)
__host__ __device__ constexpr int cl_slots(int CL) {
  return (int)((227 * 1024 - 1024 - cl_fixed(CL)) / kCLChunk) < 33 ? (int)((227 * 1024 - 1024 - cl_fixed(CL)) / kCLChunk)
                                                                    : 33;
}
__host__ __device__ constexpr size_t cl_smem(int CL) { return 1024 + (size_t)cl_slots(CL) * kCLChunk + cl_fixed(CL); }

// chunks per CTA: the template instance (3, 6, 8, 10 or 11) covering ceil(n / (CL * 26))
inline int cl_nch(int64_t n, int CL) {
  const int c = (int)((n + CL * kCLRows - 1) / (CL * kCLRows));
  return c <= 3 ? 3 : c <= 6 ? 6 : c <= 8 ? 8 : c <= 10 ? 10 : 11;
}

// remote (DSMEM) store that completes 8 transaction bytes on the receiving CTA's mbarrier: the
// data and its signal travel together, no cluster-scope fence (a release.cluster arrive compiles
// to MEMBAR.GPU and cost more than a whole panel)
FS_DEVINL void st_async_f64(uint32_t addr, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(addr), "d"(v),
               "r"(bar) : "memory");
}
FS_DEVINL void bar_arrive_n(int id, int count) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory"); }

template <typename TS, typename TV, int NCH, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kCLThreads, 1)
cols_solve_y_cl_kernel(const __grid_constant__ CUtensorMap smap, int64_t n, int64_t m, const double* __restrict__ z,
                       const TV* __restrict__ v, double lam, int accumulate, double* __restrict__ x,
                       double* __restrict__ ypart, int y_only) {
  constexpr int VN1 = 16 / (int)sizeof(TS);       // columns per 16-byte vector
  constexpr int CW = 16 * VN1;                    // columns per panel (256 bytes)
  constexpr int kSlots = cl_slots(CL);
  constexpr int kCLXB = cl_xb(CL);                // exchange buffers
  constexpr int R0 = kSlots / NCH < kCLSets ? kSlots / NCH : kCLSets;
  constexpr int R = R0 < (kCLXB - 1) / 2 ? R0 : (kCLXB - 1) / 2;   // slot-sets
  constexpr int RPC = NCH * kCLRows;              // rows per CTA
  constexpr int RP = kCLRows / 2;                 // row pairs per chunk (one warp-wide load each)
  constexpr uint32_t kSetBytes = NCH * kCLChunk;
  constexpr int PA = (RP + kCLXW - 1) / kCLXW;    // row pairs per x-group warp (3)
  constexpr int PB = (RP + kCLYW - 1) / kCLYW;    // row pairs per y-group warp (2)
  static_assert(R >= 2, "panel j's x-phase runs beside panel j-1's y-phase");
  using VT = typename VecOf<TS>::V;
  using Zt = typename std::conditional<sizeof(TV) == 8, double, float>::type;
  extern __shared__ __align__(1024) unsigned char cl_raw[];
  unsigned char* ring = cl_raw + ((1024u - (ptx::smem_u32(cl_raw) & 1023u)) & 1023u);   // [R][NCH][7.5 KB]
  double* red = (double*)(ring + (size_t)kSlots * kCLChunk);       // [2][x warps][64]
  double* xch = red + 2 * kCLXW * 64;                              // [kCLXB][CL][64] partial column sums
  double* xo = xch + kCLXB * CL * 64;                              // [kCLXB][64] old x (accumulate; from rank 0)
  double* xs = xo + kCLXB * 64;                                    // [2][64]
  uint64_t* full = (uint64_t*)(xs + 2 * 64);                       // [sets]
  uint64_t* empty = full + kCLSets;                                // [sets]
  uint64_t* xbar = empty + kCLSets;                                // [kCLXB]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)ptx::cluster_ctarank();
  const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int64_t row0 = (int64_t)rank * RPC;
  const int64_t panels = (m + CW - 1) / CW;
  const int64_t np = panels > cid ? (panels - 1 - cid) / ncl + 1 : 0;
  if (tid == 0) {
    for (int s = 0; s < R; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], kCLYW); }
    for (int b = 0; b < kCLXB; ++b) ptx::mbar_init(&xbar[b], 1);
    ptx::fence_mbar_init();
  }
  ptx::cluster_sync();                             // peers' exchange barriers exist before use
  const int vq = lane & 15, half = lane >> 4;
  const int off = half * 256 + vq * 16;            // within a row pair
  if (warp == kCLCW) {
    // ---------------- producer: one slot-set (NCH boxes, one mbarrier) per panel ----------------
    if (lane == 0) {
      ptx::tma_prefetch_desc(&smap);
      int set = 0;
      uint32_t use = 0;                            // completed passes over the ring
      for (int64_t j = 0; j < np; ++j) {
        if (use > 0) ptx::mbar_wait(&empty[set], (use - 1) & 1);
        const int32_t col = (int32_t)((cid + j * ncl) * CW);
        ptx::mbar_arrive_expect_tx(&full[set], kSetBytes);
#pragma unroll
        for (int k = 0; k < NCH; ++k)
          ptx::tma_load_2d(ring + (size_t)(set * NCH + k) * kCLChunk, &smap, &full[set], col,
                           (int32_t)(row0 + k * kCLRows));
        if (++set == R) { set = 0; ++use; }
      }
    }
    __syncwarp();
  } else if (warp < kCLXW) {
    // ---------------- x group: partial column sums of panel j, pushed to the cluster ----------------
    // (never waits on the exchange: the y group forms x, so the exchange latency overlaps the
    // next panels' partial sums)
    // warp a owns row pairs a, a + 7, a + 14 of every chunk
    Zt zr[NCH][PA];
#pragma unroll
    for (int k = 0; k < NCH; ++k)
#pragma unroll
      for (int p = 0; p < PA; ++p) {
        const int rp = warp + p * kCLXW;
        const int64_t row = row0 + k * kCLRows + 2 * rp + half;
        zr[k][p] = (!y_only && rp < RP && row < n) ? (Zt)z[row] : (Zt)0;
      }
    int setx = 0;
    uint32_t phx = 0;
    // accumulate: the old x of the panel is pushed with rank 0's partials; it is loaded one panel
    // ahead so the global-load latency stays off the exchange (the y group waits for that push)
    const bool xo_push = accumulate && rank == 0 && tid < CW && !y_only;
    double xold_next = 0.0;
    if (xo_push && np > 0) {
      const int64_t c = cid * CW + tid;
      xold_next = c < m ? x[c] : 0.0;
    }
    for (int64_t j = 0; j < np && !y_only; ++j) {
      const int rb = (int)(j & 1);
      Zt acc[VN1];
#pragma unroll
      for (int e = 0; e < VN1; ++e) acc[e] = 0;
      ptx::mbar_wait(&full[setx], phx);
      const unsigned char* src = ring + (size_t)setx * kSetBytes + off;
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        VT bv[PA];
#pragma unroll
        for (int p = 0; p < PA; ++p)
          if (warp + p * kCLXW < RP) bv[p] = *reinterpret_cast<const VT*>(src + k * kCLChunk + (warp + p * kCLXW) * 512);
#pragma unroll
        for (int p = 0; p < PA; ++p) {
          if (warp + p * kCLXW < RP) {
            TS a[VN1];
            vec_to_array(bv[p], a);
#pragma unroll
            for (int e = 0; e < VN1; ++e) {
              if constexpr (sizeof(Zt) == 8) acc[e] = fma(to_f64_mix(a[e], e), zr[k][p], acc[e]);
              else acc[e] = fma((Zt)a[e], zr[k][p], acc[e]);
            }
          }
        }
      }
      double* rw = red + rb * kCLXW * 64 + warp * 64;
#pragma unroll
      for (int e = 0; e < VN1; ++e) {
        double d = (double)acc[e];
        d += __shfl_xor_sync(0xffffffffu, d, 16);
        if (lane < 16) rw[vq * VN1 + e] = d;
      }
      ptx::named_bar_sync(1, kCLXThreads);         // red[rb] holds panel j's per-warp partials
      if (tid < CW) {                              // warps 0-1 push them to every CTA
        double part = 0.0;
#pragma unroll
        for (int w = 0; w < kCLXW; ++w) part += red[(rb * kCLXW + w) * 64 + tid];
        // the local barrier expects all CL partial vectors (a peer's complete_tx may land
        // before this expect_tx: the phase cannot complete until this one arrival is made)
        const int xb = (int)(j % kCLXB);
        if (tid == 0) ptx::mbar_arrive_expect_tx(&xbar[xb], (CL + (accumulate ? 1 : 0)) * CW * 8);
        const uint32_t mine = ptx::smem_u32(xch + (xb * CL + rank) * 64 + tid);
        const uint32_t bar = ptx::smem_u32(&xbar[xb]);
#pragma unroll
        for (int r = 0; r < CL; ++r) st_async_f64(ptx::mapa(mine, r), part, ptx::mapa(bar, r));
        if (xo_push) {
          const double xold = xold_next;
          if (j + 1 < np) {
            const int64_t cn = (cid + (j + 1) * ncl) * CW + tid;
            xold_next = cn < m ? x[cn] : 0.0;
          }
          const uint32_t xa = ptx::smem_u32(xo + xb * 64 + tid);
#pragma unroll
          for (int r = 0; r < CL; ++r) st_async_f64(ptx::mapa(xa, r), xold, ptx::mapa(bar, r));
        }
      }
      if (++setx == R) { setx = 0; phx ^= 1; }
    }
  } else {
    // ---------------- y group: x of panel p from the exchange, then y += S_panel x_panel ----------------
    const int wb = warp - kCLXW;                   // warp b owns row pairs b, b + 8 of every chunk
    const int ty = tid - kCLXThreads;              // 0 .. 255; ty < 64 forms x of column ty
    const bool xw = ty < CW;
    double vnext = 0.0;                            // v (or x, y-only) one panel ahead
    if (xw && np > 0) {
      const int64_t c = cid * CW + ty;
      vnext = c < m ? (y_only ? x[c] : (double)v[c]) : 0.0;
    }
    double yreg[NCH][PB];
#pragma unroll
    for (int k = 0; k < NCH; ++k)
#pragma unroll
      for (int p = 0; p < PB; ++p) yreg[k][p] = 0.0;
    int sety = 0;
    uint32_t phy = 0;
    for (int64_t p = 0; p < np; ++p) {
      const int b = (int)(p & 1);
      if (xw) {
        const int64_t c = (cid + p * ncl) * CW + ty;
        const double vc = vnext;
        if (p + 1 < np) {
          const int64_t cn = c + ncl * CW;
          vnext = cn < m ? (y_only ? x[cn] : (double)v[cn]) : 0.0;
        }
        double xv = 0.0;
        if (y_only) {
          xv = vc;
        } else {
          const int xb = (int)(p % kCLXB);
          ptx::mbar_wait(&xbar[xb], (uint32_t)((p / kCLXB) & 1));
          double sum = 0.0;
#pragma unroll
          for (int r = 0; r < CL; ++r) sum += xch[(xb * CL + r) * 64 + ty];
          if (c < m) {
            xv = (vc - sum) / lam;     // true division: x = v / lam exactly when S = 0 (solvers.py:124-126)
            // accumulate: the old x travels with rank 0's partials (read there before the push,
            // so no rank can see rank 0's overwrite of x[c])
            if (accumulate) xv = xo[xb * 64 + ty] + xv;
            if (rank == 0) x[c] = xv;
          }
        }
        xs[b * 64 + ty] = xv;
      }
      ptx::named_bar_sync(2, kCLYW * kWarp);       // xs[b] holds x of panel p (xs[b] of p-2 fully read)
      double xv[VN1];
#pragma unroll
      for (int e = 0; e < VN1; ++e) xv[e] = xs[b * 64 + vq * VN1 + e];
      ptx::mbar_wait(&full[sety], phy);            // (already complete: makes the TMA data visible here)
      const unsigned char* src = ring + (size_t)sety * kSetBytes + off;
#pragma unroll
      for (int k0 = 0; k0 < NCH; k0 += kCLG) {
        VT bv[kCLG][PB];
#pragma unroll
        for (int k = 0; k < kCLG; ++k)
#pragma unroll
          for (int q = 0; q < PB; ++q)
            if (k0 + k < NCH && wb + q * kCLYW < RP)
              bv[k][q] = *reinterpret_cast<const VT*>(src + (k0 + k) * kCLChunk + (wb + q * kCLYW) * 512);
#pragma unroll
        for (int k = 0; k < kCLG; ++k)
#pragma unroll
          for (int q = 0; q < PB; ++q)
            if (k0 + k < NCH && wb + q * kCLYW < RP) {
              TS a[VN1];
              vec_to_array(bv[k][q], a);
#pragma unroll
              for (int e = 0; e < VN1; ++e) yreg[k0 + k][q] = fma(to_f64_mix(a[e], e), xv[e], yreg[k0 + k][q]);
            }
      }
      __syncwarp();                                // the whole warp has consumed the slot-set
      if (lane == 0) ptx::mbar_arrive(&empty[sety]);
      if (++sety == R) { sety = 0; phy ^= 1; }
    }
#pragma unroll
    for (int k = 0; k < NCH; ++k)
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        double t = yreg[k][q];
        t += __shfl_xor_sync(0xffffffffu, t, 1);
        t += __shfl_xor_sync(0xffffffffu, t, 2);
        t += __shfl_xor_sync(0xffffffffu, t, 4);
        t += __shfl_xor_sync(0xffffffffu, t, 8);
        const int rp = wb + q * kCLYW;
        const int64_t row = row0 + k * kCLRows + 2 * rp + half;
        if (rp < RP && vq == 0 && row < n) ypart[cid * n + row] = t;
      }
  }
  ptx::cluster_sync();                             // no CTA leaves while a peer may still signal it
}

template <typename TS, typename TV, int CL>
cudaError_t launch_cols_solve_y_cl(int nch, unsigned grid, cudaStream_t st, const CUtensorMap& smap, int64_t n,
                                   int64_t m, const double* z, const TV* v, double lam, int acc, double* x,
                                   double* ypart, int y_only) {
  auto pick = [&](auto kfn) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cl_smem(CL));
    if (CL > 8) cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    kfn<<<grid, kCLThreads, cl_smem(CL), st>>>(smap, n, m, z, v, lam, acc, x, ypart, y_only);
  };
  switch (nch) {
    case 3: pick(cols_solve_y_cl_kernel<TS, TV, 3, CL>); break;
    case 6: pick(cols_solve_y_cl_kernel<TS, TV, 6, CL>); break;
    case 8: pick(cols_solve_y_cl_kernel<TS, TV, 8, CL>); break;
    case 10: pick(cols_solve_y_cl_kernel<TS, TV, 10, CL>); break;
    default: pick(cols_solve_y_cl_kernel<TS, TV, 11, CL>); break;
  }
  return cudaGetLastError();
}

// most clusters of CL CTAs (one per SM, cl_smem) the GPU runs at once; cached per CL
template <typename TS, int CL>
int cl_max_active(int num_sms) {
  static int max_cl = 0;
  if (!max_cl) {
    auto probe = cols_solve_y_cl_kernel<TS, float, 10, CL>;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cl_smem(CL));
    if (CL > 8) cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(CL * 32));
    cfg.blockDim = dim3(kCLThreads);
    cfg.dynamicSmemBytes = cl_smem(CL);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = CL;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, (void*)probe, &cfg) != cudaSuccess || mc < 1) {
      cudaGetLastError();
      mc = CL > 8 ? -1 : num_sms / CL;              // non-portable size not schedulable: unused
    }
    max_cl = mc;
  }
  return max_cl;
}

// the cluster pass for CL-CTA clusters (S read once); ypart gets one row per cluster
template <typename TS, int CL>
cudaError_t cols_solve_y_cl_t(const CUtensorMap& smap, int64_t n, int64_t m, const double* z, const void* v,
                              bool v_f64, double lam, bool accumulate, double* x, double* ypart, int64_t ypart_rows,
                              double* y, int num_sms, cudaStream_t st, int* launches, int y_only) {
  constexpr int64_t CW = 256 / (int64_t)sizeof(TS);
  const int64_t panels = (m + CW - 1) / CW;
  // same capacity bound as the panel kernel's grid
  const int64_t cap = (m + row_chunk_cols<double>() - 1) / row_chunk_cols<double>();
  const int64_t ncl = std::min<int64_t>(std::min<int64_t>(cl_max_active<TS, CL>(num_sms), num_sms / CL),
                                        std::min(panels, cap));
  if (ypart_rows < ncl) return cudaErrorInvalidValue;
  const unsigned grid = (unsigned)(ncl * CL);
  const int nch = cl_nch(n, CL);
  cudaError_t e = v_f64 ? launch_cols_solve_y_cl<TS, double, CL>(nch, grid, st, smap, n, m, z, (const double*)v, lam,
                                                                 accumulate ? 1 : 0, x, ypart, y_only)
                        : launch_cols_solve_y_cl<TS, float, CL>(nch, grid, st, smap, n, m, z, (const float*)v, lam,
                                                                accumulate ? 1 : 0, x, ypart, y_only);
  if (e != cudaSuccess) return e;
  reduce_chunks_kernel<<<(unsigned)((n + kRedRows - 1) / kRedRows), kRedRows * kRedWarps, 0, st>>>(ypart, ncl, n, n, y);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

// r = S^T y + λx - v with exact fp64 products; per-block ||r||², ||v||² partials.
template <typename TS, typename TV, bool kVec>
__global__ void __launch_bounds__(kColThreads)
residual_cols_kernel(const TS* __restrict__ S, int64_t n, int64_t m, int64_t ldS,
                     const double* __restrict__ y, const double* __restrict__ x,
                     const TV* __restrict__ v, double lam, double* __restrict__ r,
                     double* __restrict__ block_sums) {
  using VT = typename VecOf<TS>::V;
  constexpr int VN = VecOf<TS>::N;
  constexpr int kZ = 2048;
  constexpr int kInner = 16;
  __shared__ double ys[kZ];
  __shared__ double red[2][kColThreads / kWarp];
  const int64_t col = ((int64_t)blockIdx.x * kColThreads + threadIdx.x) * VN;
  double acc[VN];
#pragma unroll
  for (int e = 0; e < VN; ++e) acc[e] = 0.0;
  const bool full = kVec && (col + VN <= m);
  for (int64_t r0 = 0; r0 < n; r0 += kZ) {
    const int rows = (int)(n - r0 < kZ ? n - r0 : kZ);
    __syncthreads();
    for (int t = threadIdx.x; t < rows; t += kColThreads) ys[t] = y[r0 + t];
    __syncthreads();
    if (col >= m) continue;
    const TS* base = S + r0 * ldS + col;
    for (int i0 = 0; i0 < rows; i0 += kInner) {
      const int cnt = min(kInner, rows - i0);
      if (full && cnt == kInner) {
        VT buf[kInner];
#pragma unroll
        for (int k = 0; k < kInner; ++k)
          buf[k] = ld_stream(reinterpret_cast<const VT*>(base + (int64_t)(i0 + k) * ldS));
#pragma unroll
        for (int k = 0; k < kInner; ++k) {
          TS a[VN];
          vec_to_array(buf[k], a);
#pragma unroll
          for (int e = 0; e < VN; ++e) acc[e] = fma(ys[i0 + k], (double)a[e], acc[e]);
        }
      } else {
        for (int k = 0; k < cnt; ++k)
#pragma unroll
          for (int e = 0; e < VN; ++e)
            if (col + e < m) acc[e] = fma(ys[i0 + k], (double)ld_stream(base + (int64_t)(i0 + k) * ldS + e), acc[e]);
      }
    }
  }
  double rr = 0.0, vv = 0.0;
  if (col < m) {
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      const int64_t c = col + e;
      if (c < m) {
        const double vc = (double)v[c];
        const double rc = (acc[e] + lam * x[c]) - vc;  // ((A@x)@A + lam*x) - v, core.py:297/:319
        if (r) r[c] = rc;
        rr += rc * rc;
        vv += vc * vc;
      }
    }
  }
  rr = warp_sum(rr);
  vv = warp_sum(vv);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { red[0][warp] = rr; red[1][warp] = vv; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kColThreads / kWarp; ++w) { a += red[0][w]; b += red[1][w]; }
    block_sums[2 * blockIdx.x] = a;
    block_sums[2 * blockIdx.x + 1] = b;
  }
}

__global__ void reduce_pairs_kernel(const double* __restrict__ block_sums, int64_t blocks,
                                    double* __restrict__ sums) {
  // one warp, fixed order: lane l sums blocks l, l+32, ...; then a fixed shuffle tree
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < blocks; i += 32) {
    a += block_sums[2 * i];
    b += block_sums[2 * i + 1];
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if (threadIdx.x == 0) { sums[0] = a; sums[1] = b; }
}

// flag |= 1 if any of the rows x cols entries (leading dimension ld) is not finite.  2-D grid:
// blockIdx.y strides rows, x-threads stride the row's columns (coalesced, no 64-bit division);
// 4 loads in flight per thread.
template <typename T>
__global__ void check_finite_kernel(const T* __restrict__ a, int64_t rows, int64_t cols, int64_t ld,
                                    int* __restrict__ flag, unsigned* __restrict__ rowmax) {
  // rowmax (optional): per-row max |a| as float bits (non-negative floats order like unsigned ints),
  // one atomicMax per block and row after a block reduction
  __shared__ float red[32];
  bool bad = false;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const T* row = a + r * ld;
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float mx = 0.f;
    for (; c + 3 * step < cols; c += 4 * step) {
      const T x0 = ld_stream(row + c), x1 = ld_stream(row + c + step), x2 = ld_stream(row + c + 2 * step),
              x3 = ld_stream(row + c + 3 * step);
      bad |= !(isfinite(x0) && isfinite(x1) && isfinite(x2) && isfinite(x3));
      if (rowmax) mx = fmaxf(fmaxf(fmaxf(mx, fabsf((float)x0)), fabsf((float)x1)), fmaxf(fabsf((float)x2), fabsf((float)x3)));
    }
    for (; c < cols; c += step) {
      const T x = ld_stream(row + c);
      bad |= !isfinite(x);
      if (rowmax) mx = fmaxf(mx, fabsf((float)x));
    }
    if (rowmax) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
      __syncthreads();
      if (threadIdx.x == 0) {
        float b = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b = fmaxf(b, red[w]);
        if (b > 0.f) atomicMax(rowmax + r, __float_as_uint(b));
      }
      __syncthreads();
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// The same check (and row maxima) for wide rows: one block per (row, 8192-element column chunk),
// every thread's 32 elements loaded as independent 16-byte vectors before any use (128 bytes in
// flight per thread), one block reduction and atomicMax per (row, chunk).  The strided kernel
// above walks all rows inside each block with 16 bytes in flight and two barriers per row: 2.9 ms
// for a 1024 x 1e6 fp32 matrix, against ~0.65 ms at the copy bandwidth here.
constexpr int kCFChunk = 8192;
template <typename T>
__global__ void __launch_bounds__(256)
check_finite_rows_kernel(const T* __restrict__ a, int64_t rows, int64_t cols, int64_t ld, int* __restrict__ flag,
                         unsigned* __restrict__ rowmax) {
  using VT = typename VecOf<T>::V;
  constexpr int VN = VecOf<T>::N;
  constexpr int kPer = kCFChunk / 256 / VN;      // vectors per thread
  __shared__ float red[8];
  bool bad = false;
  const int64_t c0 = (int64_t)blockIdx.x * kCFChunk;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const T* row = a + r * ld;
    float mx = 0.f;
    if (c0 + kCFChunk <= cols && (reinterpret_cast<uintptr_t>(row + c0) & 15) == 0) {
      VT v[kPer];
#pragma unroll
      for (int k = 0; k < kPer; ++k) v[k] = ld_stream(reinterpret_cast<const VT*>(row + c0) + k * 256 + threadIdx.x);
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        T e[VN];
        vec_to_array(v[k], e);
#pragma unroll
        for (int i = 0; i < VN; ++i) {
          bad |= !isfinite(e[i]);
          mx = fmaxf(mx, fabsf((float)e[i]));
        }
      }
    } else {
      const int64_t c1 = c0 + kCFChunk < cols ? c0 + kCFChunk : cols;
      for (int64_t c = c0 + threadIdx.x; c < c1; c += 256) {
        const T x = ld_stream(row + c);
        bad |= !isfinite(x);
        mx = fmaxf(mx, fabsf((float)x));
      }
    }
    if (rowmax) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
      __syncthreads();
      if (threadIdx.x == 0) {
        float b = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) b = fmaxf(b, red[w]);
        if (b > 0.f) atomicMax(rowmax + r, __float_as_uint(b));
      }
      __syncthreads();
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// F16X2 row scales from exact row maxima: 2^k with max |S_i| 2^k in [2^14, 2^15), so no element
// of the row can overflow fp16 (max 65504) and elements down to 2^-18 of the row maximum keep a
// normal lo plane (all 22 bits).
__global__ void scales_from_max_kernel(const float* __restrict__ absmax, int64_t n, float* __restrict__ scale,
                                       double* __restrict__ inv_scale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float mx = absmax[i];
  int k = 0;
  if (mx > 0.f && isfinite(mx)) {
    int e;
    frexpf(mx, &e);                     // mx in [2^(e-1), 2^e)
    k = 15 - e;                         // mx * 2^k in [2^14, 2^15)
    k = k > 120 ? 120 : (k < -120 ? -120 : k);
  }
  scale[i] = ldexpf(1.f, k);
  inv_scale[i] = ldexp(1.0, -k);
}

__global__ void widen_kernel(const float* __restrict__ in, int64_t m, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = (double)in[i];
}

inline bool aligned16(const void* p, int64_t ld, int es) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ((ld * es) % 16 == 0);
}

template <typename TS>
cudaError_t gemv_rows_t(const TS* S, int64_t n, int64_t m, int64_t ldS, const void* w, bool w_f64,
                        double* partials, double* u, cudaStream_t st, int* launches) {
  constexpr int CW = row_chunk_cols<TS>();
  const int64_t chunks = (m + CW - 1) / CW;
  const bool vec = aligned16(S, ldS, sizeof(TS));
  dim3 grid((unsigned)chunks);
  if (w_f64) {
    if (vec) gemv_rows_kernel<TS, double, true><<<grid, kRowThreads, 0, st>>>(S, n, m, ldS, (const double*)w, partials);
    else gemv_rows_kernel<TS, double, false><<<grid, kRowThreads, 0, st>>>(S, n, m, ldS, (const double*)w, partials);
  } else {
    if (vec) gemv_rows_kernel<TS, float, true><<<grid, kRowThreads, 0, st>>>(S, n, m, ldS, (const float*)w, partials);
    else gemv_rows_kernel<TS, float, false><<<grid, kRowThreads, 0, st>>>(S, n, m, ldS, (const float*)w, partials);
  }
  reduce_chunks_kernel<<<(unsigned)((n + kRedRows - 1) / kRedRows), kRedRows * kRedWarps, 0, st>>>(partials, chunks, n, n,
                                                                                                 u);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

template <typename TS>
cudaError_t gemv_cols_t(const TS* S, int64_t n, int64_t m, int64_t ldS, const double* z,
                        const void* v, bool v_f64, double lam, bool accumulate, double* x,
                        cudaStream_t st, int* launches) {
  constexpr int VN = VecOf<TS>::N;
  const int64_t blocks = (m + (int64_t)kColThreads * VN - 1) / ((int64_t)kColThreads * VN);
  const bool vec = aligned16(S, ldS, sizeof(TS));
  dim3 grid((unsigned)blocks);
  const int acc = accumulate ? 1 : 0;
#define FS_COLS(TV, VEC) gemv_cols_solve_kernel<TS, TV, VEC><<<grid, kColThreads, 0, st>>>(S, n, m, ldS, z, (const TV*)v, lam, acc, x)
  if (v_f64) { if (vec) FS_COLS(double, true); else FS_COLS(double, false); }
  else { if (vec) FS_COLS(float, true); else FS_COLS(float, false); }
#undef FS_COLS
  if (launches) *launches += 1;
  return cudaGetLastError();
}

template <typename TS>
cudaError_t cols_solve_y_t(const TS* S, int64_t n, int64_t m, int64_t ldS, const double* z, const void* v,
                           bool v_f64, double lam, bool accumulate, double* x, double* ypart, int64_t ypart_rows,
                           double* y, int num_sms, cudaStream_t st, int* launches, int y_only = 0) {
  // one support rule and one grid size for the fused pass and the y-only pass, so that a
  // recomputed y = S x is bit-identical to the solve's (test_solvers.py:109-114)
  if (!aligned16(S, ldS, sizeof(TS))) return cudaErrorNotSupported;
  // n <= 4576: the cluster kernel (S read from HBM once, in 256-byte TMA rows); 4-CTA clusters up
  // to n = 1144, 8-CTA to 2288, 16-CTA (non-portable, when schedulable) above
  static const int cl_env = getenv("FS_CY_CL") ? atoi(getenv("FS_CY_CL")) : 1;
  static const int cl_min = getenv("FS_CY_CLMIN") ? atoi(getenv("FS_CY_CLMIN")) : 4;   // experiments: force 8 / 16
  if (cl_env && n <= kCLMaxRows16 && (n <= kCLMaxRows8 || cl_max_active<TS, 16>(num_sms) >= 4)) {
    CUtensorMap smap;
    memset(&smap, 0, sizeof smap);
    if (make_tensor_map_2d(&smap, sizeof(TS) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           S, (uint64_t)m, (uint64_t)n, (uint64_t)ldS * sizeof(TS), 256 / sizeof(TS), kCLRows) ==
        cudaSuccess)
      return n <= kCLMaxRows4 && cl_min <= 4
                 ? cols_solve_y_cl_t<TS, 4>(smap, n, m, z, v, v_f64, lam, accumulate, x, ypart, ypart_rows, y, num_sms,
                                            st, launches, y_only)
             : n <= kCLMaxRows8 && cl_min <= 8
                 ? cols_solve_y_cl_t<TS, 8>(smap, n, m, z, v, v_f64, lam, accumulate, x, ypart, ypart_rows, y, num_sms,
                                            st, launches, y_only)
                 : cols_solve_y_cl_t<TS, 16>(smap, n, m, z, v, v_f64, lam, accumulate, x, ypart, ypart_rows, y,
                                             num_sms, st, launches, y_only);
  }
  const size_t smem = cy_smem_bytes<TS>(n);
  if (smem > 200 * 1024) return cudaErrorNotSupported;
  const int64_t panels = (m + cy_cols<TS>() - 1) / cy_cols<TS>();
  const int64_t cap = (m + row_chunk_cols<double>() - 1) / row_chunk_cols<double>();
  int64_t G = std::min<int64_t>((int64_t)num_sms, std::min(panels, cap));
  if (ypart_rows < G) return cudaErrorInvalidValue;
  const int acc = accumulate ? 1 : 0;
  CUtensorMap pmap;
  memset(&pmap, 0, sizeof pmap);
  // TMA L2 prefetch of the next panel: measured slower (1.0 -> 1.38 ms with 512-B panels: the two
  // panels per SM overflow L2; 1.15 ms with 256-B panels), so off unless FS_CY_PF=1
  static const int pf_env = getenv("FS_CY_PF") ? atoi(getenv("FS_CY_PF")) : 0;
  int use_pf = pf_env;
  if (use_pf)
    use_pf = make_tensor_map_2d(&pmap, sizeof(TS) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                S, (uint64_t)m, (uint64_t)n, (uint64_t)ldS * sizeof(TS), cy_cols<TS>(), 256) ==
                     cudaSuccess
                 ? 1
                 : 0;
  if (v_f64) {
    auto kfn = cols_solve_y_kernel<TS, double>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kfn<<<(unsigned)G, kCYThreads, smem, st>>>(S, n, m, ldS, z, (const double*)v, lam, acc, x, ypart, y_only, pmap,
                                               use_pf);
  } else {
    auto kfn = cols_solve_y_kernel<TS, float>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kfn<<<(unsigned)G, kCYThreads, smem, st>>>(S, n, m, ldS, z, (const float*)v, lam, acc, x, ypart, y_only, pmap,
                                               use_pf);
  }
  reduce_chunks_kernel<<<(unsigned)((n + kRedRows - 1) / kRedRows), kRedRows * kRedWarps, 0, st>>>(ypart, G, n, n, y);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

template <typename TS>
cudaError_t residual_cols_t(const TS* S, int64_t n, int64_t m, int64_t ldS, const double* y,
                            const double* x, const void* v, bool v_f64, double lam, double* r,
                            double* block_sums, double* sums, cudaStream_t st, int* launches) {
  constexpr int VN = VecOf<TS>::N;
  const int64_t blocks = (m + (int64_t)kColThreads * VN - 1) / ((int64_t)kColThreads * VN);
  const bool vec = aligned16(S, ldS, sizeof(TS));
  dim3 grid((unsigned)blocks);
#define FS_RES(TV, VEC) residual_cols_kernel<TS, TV, VEC><<<grid, kColThreads, 0, st>>>(S, n, m, ldS, y, x, (const TV*)v, lam, r, block_sums)
  if (v_f64) { if (vec) FS_RES(double, true); else FS_RES(double, false); }
  else { if (vec) FS_RES(float, true); else FS_RES(float, false); }
#undef FS_RES
  reduce_pairs_kernel<<<1, 32, 0, st>>>(block_sums, blocks, sums);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

// ---- F16X2 split (tiles.cuh) ----
// Row scales from a sample of each row (its first kScaleSample columns): s_i = 2^k with the
// sample maximum scaled into [2^6, 2^7), leaving 2^9 of headroom below the fp16 maximum for the
// rest of the row; an element that still overflows sets bit 1 of the flag word and the caller
// recomputes the Gram with TF32X3.  Power-of-two scales are exact in both directions.
constexpr int kScaleSample = 4096;
__global__ void row_scale_kernel(const float* __restrict__ S, int64_t n, int64_t cols, int64_t ldS,
                                 float* __restrict__ scale, double* __restrict__ inv_scale) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x / kWarp) + (threadIdx.x >> 5);
  if (i >= n) return;
  float mx = 0.f;
  for (int64_t c = lane; c < cols; c += kWarp) mx = fmaxf(mx, fabsf(S[i * ldS + c]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int k = 0;
  if (mx > 0.f && isfinite(mx)) {
    int e;
    frexpf(mx, &e);                     // mx in [2^(e-1), 2^e)
    k = 7 - e;                          // mx * 2^k in [2^6, 2^7)
    k = k > 100 ? 100 : (k < -100 ? -100 : k);
  }
  if (lane == 0) {
    scale[i] = ldexpf(1.f, k);
    inv_scale[i] = ldexp(1.0, -k);
  }
}

// Column range [c0, c1) of all rows (c0 a multiple of 1024): the F16X2 planes of S_t16 (tiles.cuh)
// and the u = S w partials of the 1024-column chunks.  CTA = (128-row block, 1024-column chunk =
// 16 K-blocks);
// warp w owns K-blocks w and w+8.  A warp instruction covers 4 consecutive tile rows of one
// K-block (lane -> row 4g + lane/8, 16-byte chunk lane%8), so each store writes 512 contiguous
// bytes of a tile (a row-per-warp mapping scatters 128-byte rows over 4 tiles: 1.60 vs 1.33 ms
// for the pass at the headline).  u partials: per-warp per-row sums in shared memory, added in warp order.
constexpr int kRTRows = 128;
constexpr int kRTThreads = 256;
constexpr int kRTGroup = 4;                       // 4-row groups per unrolled batch (16 rows)
__global__ void __launch_bounds__(kRTThreads, 3)
retile16_tiles_kernel(const float* __restrict__ S, int64_t n, int64_t m, int64_t ldS, const float* __restrict__ w,
                      double* __restrict__ partials, uint8_t* __restrict__ St, const float* __restrict__ scale,
                      int has_w, int vec_ok, int* __restrict__ flags, int64_t cb0, int64_t ncb) {
  constexpr int CW = 1024;
  __shared__ float usm[kRTThreads / 32][kRTRows];
  __shared__ float ssm[kRTRows];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nb = tiles_nb(n), KB = tiles16_kb(m);
  const int64_t cb = cb0 + blockIdx.x % ncb;
  const int64_t rb = blockIdx.x / ncb;
  for (int t = threadIdx.x; t < kRTRows; t += kRTThreads) {
    const int64_t i = rb * kRTRows + t;
    ssm[t] = i < n ? scale[i] : 1.f;
  }
  for (int t = threadIdx.x; t < (kRTThreads / 32) * kRTRows; t += kRTThreads) (&usm[0][0])[t] = 0.f;
  __syncthreads();
  const int j = lane & 7, rl = lane >> 3;        // chunk in the tile row, row within the 4-row group
  bool bad = false, ovf = false;
  for (int q = 0; q < 2; ++q) {
    const int64_t kb = cb * (CW / 64) + warp + 8 * q;
    if (kb >= KB) continue;
    const int64_t c = kb * 64 + j * 8;            // this lane's 8 columns
    float4 w0 = make_float4(0.f, 0.f, 0.f, 0.f), w1 = w0;
    if (has_w) {
      if (c + 8 <= m) {
        w0 = __ldg(reinterpret_cast<const float4*>(w + c));
        w1 = __ldg(reinterpret_cast<const float4*>(w + c) + 1);
      } else {
        float a[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] = (c + e < m) ? __ldg(w + c + e) : 0.f;
        w0 = make_float4(a[0], a[1], a[2], a[3]);
        w1 = make_float4(a[4], a[5], a[6], a[7]);
      }
    }
    uint8_t* tile = St + ((size_t)kb * nb + rb) * 2 * kTileBytes;     // hi tile, lo tile follows
    const bool fullc = vec_ok && c + 8 <= m;
    for (int g0 = 0; g0 < kRTRows / 4; g0 += kRTGroup) {
      float4 buf[kRTGroup][2];
#pragma unroll
      for (int u = 0; u < kRTGroup; ++u) {
        const int r = (g0 + u) * 4 + rl;
        const int64_t i = rb * kRTRows + r;
        const float* row = S + i * ldS + c;
        if (i < n && fullc) {
          buf[u][0] = ld_stream(reinterpret_cast<const float4*>(row));
          buf[u][1] = ld_stream(reinterpret_cast<const float4*>(row) + 1);
        } else {
          float a[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) a[e] = (i < n && c + e < m) ? __ldg(row + e) : 0.f;
          buf[u][0] = make_float4(a[0], a[1], a[2], a[3]);
          buf[u][1] = make_float4(a[4], a[5], a[6], a[7]);
        }
      }
#pragma unroll
      for (int u = 0; u < kRTGroup; ++u) {
        const int r = (g0 + u) * 4 + rl;
        const float sc = ssm[r];
        const float xs[8] = {buf[u][0].x, buf[u][0].y, buf[u][0].z, buf[u][0].w,
                             buf[u][1].x, buf[u][1].y, buf[u][1].z, buf[u][1].w};
        __align__(16) __half hi[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          bad |= !isfinite(xs[e]);
          const float y = xs[e] * sc;
          hi[e] = __float2half_rn(y);
          const float hf = __half2float(hi[e]);
          ovf |= isinf(hf);
          lo[e] = __float2half_rn(y - hf);
        }
        const int off = r * 128 + ((j ^ (r & 7)) << 4);
        *reinterpret_cast<uint4*>(tile + off) = *reinterpret_cast<const uint4*>(hi);
        *reinterpret_cast<uint4*>(tile + kTileBytes + off) = *reinterpret_cast<const uint4*>(lo);
        if (has_w) {
          float p = 0.f;
          p = fmaf(xs[0], w0.x, p); p = fmaf(xs[1], w0.y, p); p = fmaf(xs[2], w0.z, p); p = fmaf(xs[3], w0.w, p);
          p = fmaf(xs[4], w1.x, p); p = fmaf(xs[5], w1.y, p); p = fmaf(xs[6], w1.z, p); p = fmaf(xs[7], w1.w, p);
          p += __shfl_xor_sync(0xffffffffu, p, 1);     // the row's 8 lanes (64 columns)
          p += __shfl_xor_sync(0xffffffffu, p, 2);
          p += __shfl_xor_sync(0xffffffffu, p, 4);
          if (j == 0) usm[warp][r] += p;
        }
      }
    }
  }
  if (flags) {
    const unsigned bb = __ballot_sync(0xffffffffu, bad), bo = __ballot_sync(0xffffffffu, ovf);
    if (lane == 0 && (bb | bo)) atomicOr(flags, (bb ? 1 : 0) | (bo ? 2 : 0));
  }
  if (has_w) {
    __syncthreads();
    for (int t = threadIdx.x; t < kRTRows; t += kRTThreads) {
      const int64_t i = rb * kRTRows + t;
      double sum = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < kRTThreads / 32; ++w2) sum += (double)usm[w2][t];
      if (i < n) partials[cb * n + i] = sum;
    }
  }
}

__global__ void flag_bit_kernel(const int* __restrict__ flags, int bit, double* __restrict__ out) {
  *out = (*flags & bit) ? 1.0 : 0.0;
}

}  // namespace

cudaError_t flag_bit_to_double(const int* flags, int bit, double* out, cudaStream_t st, int* launches) {
  flag_bit_kernel<<<1, 1, 0, st>>>(flags, bit, out);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t check_finite(const void* a, bool is64, int64_t rows, int64_t cols, int64_t ld, int* flag, int num_sms,
                         cudaStream_t st, int* launches, unsigned* rowmax) {
  if (cols >= kCFChunk) {   // wide rows: one block per (row, column chunk)
    const int64_t gx = (cols + kCFChunk - 1) / kCFChunk;
    const dim3 grid((unsigned)gx, (unsigned)std::min<int64_t>(rows, 65535));
    if (is64) check_finite_rows_kernel<double><<<grid, 256, 0, st>>>((const double*)a, rows, cols, ld, flag, rowmax);
    else check_finite_rows_kernel<float><<<grid, 256, 0, st>>>((const float*)a, rows, cols, ld, flag, rowmax);
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  // ~num_sms * 8 blocks: x covers the columns (<= 1024 per block row), y the rows
  const int64_t want = (int64_t)num_sms * 8;
  const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((cols + 1023) / 1024, want));
  const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(rows, 65535), want / gx));
  const dim3 grid((unsigned)gx, (unsigned)gy);
  if (is64) check_finite_kernel<double><<<grid, 256, 0, st>>>((const double*)a, rows, cols, ld, flag, rowmax);
  else check_finite_kernel<float><<<grid, 256, 0, st>>>((const float*)a, rows, cols, ld, flag, rowmax);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t scales_from_max(const float* absmax, int64_t n, float* scale, double* inv_scale, cudaStream_t st,
                            int* launches) {
  scales_from_max_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(absmax, n, scale, inv_scale);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t widen_f32(const float* in, int64_t m, double* out, cudaStream_t st, int* launches) {
  widen_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(in, m, out);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t gemv_rows_retile(const float* S, int64_t n, int64_t m, int64_t ldS, const float* w, double* partials,
                             double* u, uint8_t* St, cudaStream_t st, int* launches, int64_t r0, int64_t r1,
                             int* nonfinite) {
  constexpr int CW = row_chunk_cols<float>();
  const int64_t chunks = (m + CW - 1) / CW;
  const int vec_ok = aligned16(S, ldS, 4) ? 1 : 0;
  if (r1 < 0) r1 = n;
  const int64_t rz = (r1 == n) ? tiles_nb(n) * kTileRows : r1;   // the last rows also zero the padding
  gemv_rows_retile_kernel<<<(unsigned)chunks, kRowThreads, 0, st>>>(S, n, m, ldS, w, partials, St, w != nullptr,
                                                                     vec_ok, r0, r1, rz, nonfinite, 0);
  if (launches) *launches += 1;
  if (w && r1 > r0) {
    reduce_chunks_kernel<<<(unsigned)((r1 - r0 + kRedRows - 1) / kRedRows), kRedRows * kRedWarps, 0, st>>>(
        partials + r0, chunks, r1 - r0, n, u + r0);
    if (launches) *launches += 1;
  }
  return cudaGetLastError();
}

cudaError_t retile_cols(const float* S, int64_t n, int64_t m, int64_t ldS, const float* w, double* partials,
                        uint8_t* St, int64_t c0, int64_t c1, int* nonfinite, cudaStream_t st, int* launches) {
  constexpr int CW = row_chunk_cols<float>();
  if (c0 % CW) return cudaErrorInvalidValue;
  const int64_t cb0 = c0 / CW, cb1 = (c1 + CW - 1) / CW;
  if (cb1 <= cb0) return cudaSuccess;
  const int vec_ok = aligned16(S, ldS, 4) ? 1 : 0;
  gemv_rows_retile_kernel<<<(unsigned)(cb1 - cb0), kRowThreads, 0, st>>>(
      S, n, m, ldS, w, partials, St, w != nullptr, vec_ok, 0, n, tiles_nb(n) * kTileRows, nonfinite, cb0);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t row_scales(const float* S, int64_t n, int64_t m, int64_t ldS, float* scale, double* inv_scale,
                       cudaStream_t st, int* launches, int64_t sample_cols) {
  int64_t cols = m < kScaleSample ? m : kScaleSample;
  if (sample_cols > 0 && sample_cols < cols) cols = sample_cols;
  row_scale_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(S, n, cols, ldS, scale, inv_scale);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t retile16_cols(const float* S, int64_t n, int64_t m, int64_t ldS, const float* w, double* partials,
                          uint8_t* St, const float* scale, int64_t c0, int64_t c1, int* flags, cudaStream_t st,
                          int* launches) {
  constexpr int CW = 1024;
  if (c0 % CW) return cudaErrorInvalidValue;
  const int64_t cb0 = c0 / CW, cb1 = (c1 + CW - 1) / CW;
  if (cb1 <= cb0) return cudaSuccess;
  const int vec_ok = aligned16(S, ldS, 4) ? 1 : 0;
  const int64_t ncb = cb1 - cb0;
  retile16_tiles_kernel<<<(unsigned)(ncb * tiles_nb(n)), kRTThreads, 0, st>>>(S, n, m, ldS, w, partials, St, scale,
                                                                                w != nullptr, vec_ok, flags, cb0, ncb);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t reduce_row_partials(const double* partials, int64_t n, int64_t m, double* u, cudaStream_t st,
                                int* launches) {
  constexpr int CW = row_chunk_cols<float>();
  const int64_t chunks = (m + CW - 1) / CW;
  reduce_chunks_kernel<<<(unsigned)((n + kRedRows - 1) / kRedRows), kRedRows * kRedWarps, 0, st>>>(partials, chunks, n,
                                                                                                 n, u);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

int64_t gemv_rows_chunk_cols() { return row_chunk_cols<float>(); }

int64_t gemv_rows_chunks(int64_t m, bool s_is_f64) {
  const int64_t cw = s_is_f64 ? row_chunk_cols<double>() : row_chunk_cols<float>();
  return (m + cw - 1) / cw;
}

int64_t residual_cols_blocks(int64_t m, bool s_is_f64) {
  const int64_t w = (int64_t)kColThreads * (s_is_f64 ? 2 : 4);
  return (m + w - 1) / w;
}

cudaError_t gemv_rows(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS, const void* w,
                      bool w_f64, double* partials, double* u, cudaStream_t st, int* launches) {
  if (s_f64) return gemv_rows_t<double>((const double*)S, n, m, ldS, w, w_f64, partials, u, st, launches);
  return gemv_rows_t<float>((const float*)S, n, m, ldS, w, w_f64, partials, u, st, launches);
}

cudaError_t gemv_cols_solve(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS,
                            const double* z, const void* v, bool v_f64, double lam, bool accumulate,
                            double* x, cudaStream_t st, int* launches) {
  if (s_f64) return gemv_cols_t<double>((const double*)S, n, m, ldS, z, v, v_f64, lam, accumulate, x, st, launches);
  return gemv_cols_t<float>((const float*)S, n, m, ldS, z, v, v_f64, lam, accumulate, x, st, launches);
}

cudaError_t gemv_cols_solve_y(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS, const double* z,
                              const void* v, bool v_f64, double lam, bool accumulate, double* x, double* ypart,
                              int64_t ypart_rows, double* y, int num_sms, cudaStream_t st, int* launches) {
  if (s_f64)
    return cols_solve_y_t<double>((const double*)S, n, m, ldS, z, v, v_f64, lam, accumulate, x, ypart, ypart_rows, y,
                                  num_sms, st, launches);
  return cols_solve_y_t<float>((const float*)S, n, m, ldS, z, v, v_f64, lam, accumulate, x, ypart, ypart_rows, y,
                               num_sms, st, launches);
}

cudaError_t gemv_rows_panel(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS, const double* x,
                            double* ypart, int64_t ypart_rows, double* y, int num_sms, cudaStream_t st,
                            int* launches) {
  if (s_f64)
    return cols_solve_y_t<double>((const double*)S, n, m, ldS, nullptr, x, true, 1.0, false, const_cast<double*>(x),
                                  ypart, ypart_rows, y, num_sms, st, launches, 1);
  return cols_solve_y_t<float>((const float*)S, n, m, ldS, nullptr, x, true, 1.0, false, const_cast<double*>(x), ypart,
                               ypart_rows, y, num_sms, st, launches, 1);
}

cudaError_t residual_cols(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS,
                          const double* y, const double* x, const void* v, bool v_f64, double lam,
                          double* r, double* block_sums, double* sums, cudaStream_t st,
                          int* launches) {
  if (s_f64) return residual_cols_t<double>((const double*)S, n, m, ldS, y, x, v, v_f64, lam, r, block_sums, sums, st, launches);
  return residual_cols_t<float>((const float*)S, n, m, ldS, y, x, v, v_f64, lam, r, block_sums, sums, st, launches);
}

}  // namespace fs
