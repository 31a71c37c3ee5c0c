// syrk_simt.cu — exact-product fp64 Gram  G = S S^T + λI (lower triangle, packed).
//
// Replaces core.py:284-289 (numpy A @ A.T -> OpenBLAS dsyrk, symmetrize, += lam).
// This is the FS_PREC_FP64 mode: every product s_ik * s_jk is formed and summed in
// fp64 (fp32 inputs are widened exactly), i.e. the reference's own arithmetic.
// 64x64 lower tiles, 256 threads (4x4 outputs each), split-K over m with a
// fixed-order reduction of the per-split partial tiles (deterministic).
#include "common.cuh"
#include "kernels.h"

namespace fs {
namespace {

constexpr int kTile = 64;
constexpr int kBK = 16;
constexpr int kThreads = 256;

FS_DEVINL void tile_coords(int64_t t, int& I, int& J) {
  int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((int64_t)(i + 1) * (i + 2) / 2 <= t) ++i;
  while ((int64_t)i * (i + 1) / 2 > t) --i;
  I = i;
  J = (int)(t - (int64_t)i * (i + 1) / 2);
}

template <typename T>
FS_DEVINL void load_slab(const T* __restrict__ S, int64_t n, int64_t m, int64_t ldS, int row0,
                         int64_t k0, double (*dst)[kTile + 1], int tid) {
  // 64 rows x 16 cols; thread -> (row = tid/4, 4 consecutive cols)
  const int r = tid >> 2, c = (tid & 3) * 4;
  const int64_t gr = row0 + r;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t gc = k0 + c + e;
    double val = 0.0;
    if (gr < n && gc < m) val = (double)__ldg(S + gr * ldS + gc);
    dst[c + e][r] = val;
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
syrk_simt_kernel(const T* __restrict__ S, int64_t n, int64_t m, int64_t ldS, int64_t kchunk,
                 double lam, double* __restrict__ ws, double* __restrict__ Gp, int direct) {
  __shared__ double As[kBK][kTile + 1];
  __shared__ double Bs[kBK][kTile + 1];
  int I, J;
  tile_coords(blockIdx.x, I, J);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t kbeg = (int64_t)blockIdx.y * kchunk;
  const int64_t kend = (m < kbeg + kchunk) ? m : kbeg + kchunk;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const bool diag = (I == J);
  for (int64_t k0 = kbeg; k0 < kend; k0 += kBK) {
    __syncthreads();
    load_slab(S, n, kend, ldS, I * kTile, k0, As, tid);
    if (!diag) load_slab(S, n, kend, ldS, J * kTile, k0, Bs, tid);
    __syncthreads();
    double (*B)[kTile + 1] = diag ? As : Bs;
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = B[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
  }
  if (direct) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t gi = (int64_t)I * kTile + ty + 16 * i, gj = (int64_t)J * kTile + tx + 16 * j;
        if (gi < n && gj <= gi) Gp[gi * (gi + 1) / 2 + gj] = acc[i][j] + (gi == gj ? lam : 0.0);
      }
  } else {
    double* out = ws + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (kTile * kTile);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) out[(ty + 16 * i) * kTile + tx + 16 * j] = acc[i][j];
  }
}

__global__ void syrk_simt_reduce(const double* __restrict__ ws, int64_t tiles, int splits,
                                 int64_t n, double lam, double* __restrict__ Gp) {
  int I, J;
  tile_coords(blockIdx.x, I, J);
  for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
    const int r = e / kTile, c = e % kTile;
    const int64_t gi = (int64_t)I * kTile + r, gj = (int64_t)J * kTile + c;
    if (gi >= n || gj > gi) continue;
    double s = 0.0;
    for (int p = 0; p < splits; ++p) s += ws[((int64_t)p * tiles + blockIdx.x) * (kTile * kTile) + e];
    Gp[gi * (gi + 1) / 2 + gj] = s + (gi == gj ? lam : 0.0);
  }
}

void plan(int64_t n, int64_t m, int num_sms, int64_t& tiles, int& splits, int64_t& kchunk) {
  const int64_t nb = (n + kTile - 1) / kTile;
  tiles = nb * (nb + 1) / 2;
  int64_t want = (4LL * num_sms + tiles - 1) / tiles;       // ~4 CTAs per SM
  const int64_t max_by_k = (m + 255) / 256;                 // >= 256 columns per split
  splits = (int)std::max<int64_t>(1, std::min<int64_t>(want, max_by_k));
  kchunk = (m + splits - 1) / splits;
  kchunk = (kchunk + kBK - 1) / kBK * kBK;
  splits = (int)((m + kchunk - 1) / kchunk);
}

}  // namespace

size_t syrk_simt_plan_bytes(int64_t n, int64_t m, int num_sms) {
  int64_t tiles, kchunk;
  int splits;
  plan(n, m, num_sms, tiles, splits, kchunk);
  return splits > 1 ? (size_t)splits * tiles * kTile * kTile * sizeof(double) : 0;
}

size_t syrk_simt_workspace_bytes(int64_t n, int64_t m, int num_sms) {
  // splits > 1 only when tiles < 4*num_sms, and then splits*tiles <= 4*num_sms + tiles
  // < 8*num_sms: a bound that holds for every (n, m), so one context serves smaller problems
  (void)n; (void)m;
  return (size_t)8 * num_sms * kTile * kTile * sizeof(double);
}

cudaError_t syrk_simt(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS, double lam,
                      double* G_packed, double* ws, int num_sms, cudaStream_t st, int* launches) {
  int64_t tiles, kchunk;
  int splits;
  plan(n, m, num_sms, tiles, splits, kchunk);
  dim3 grid((unsigned)tiles, (unsigned)splits);
  const int direct = splits == 1;
  if (s_f64)
    syrk_simt_kernel<double><<<grid, kThreads, 0, st>>>((const double*)S, n, m, ldS, kchunk, lam, ws, G_packed, direct);
  else
    syrk_simt_kernel<float><<<grid, kThreads, 0, st>>>((const float*)S, n, m, ldS, kchunk, lam, ws, G_packed, direct);
  if (launches) *launches += 1;
  if (!direct) {
    syrk_simt_reduce<<<(unsigned)tiles, 256, 0, st>>>(ws, tiles, splits, n, lam, G_packed);
    if (launches) *launches += 1;
  }
  return cudaGetLastError();
}

}  // namespace fs
