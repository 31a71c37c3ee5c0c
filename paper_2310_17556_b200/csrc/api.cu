// api.cu — the extern "C" boundary declared in include/fs.h.
//
// The one-shot fs_chol_solve is the drop-in for _solve_chol_impl (solvers.py:151-194):
//   gram (core.py:270-290) -> potrf (solvers.py:74-90) -> _chol_apply (solvers.py:101-127)
//   -> first-pass residual (solvers.py:160-170) -> optional one-step refinement (:183-194).
// Stream-ordered; one host synchronisation at the end to read the pivot/status word and
// the residual norms.  Multi-rank: the caller's allreduce sums [G_packed | u], y and the
// norm pair; everything else is rank-local (column-sharded S, v, x).
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/fs.h"
#include "kernels.h"
#include "tiles.cuh"

struct fs_ctx {
  int device = 0;
  int num_sms = 148;
  int64_t n_max = 0, m_max = 0;
  double* d_packed = nullptr;   // n(n+1)/2 packed Gram | n u   (the all-reduce buffer)
  double* d_W = nullptr;        // n x n, becomes L in place
  double* d_z = nullptr;        // n
  double* d_y = nullptr;        // n
  double* d_zacc = nullptr;     // n: accumulated z of the z-space refinement
  double* d_partials = nullptr; // row-GEMV chunk partials
  double* d_block_sums = nullptr;
  double* d_sums = nullptr;     // 4
  double* d_r = nullptr;        // m (residual vector, refinement right-hand side)
  double* d_v64 = nullptr;      // m (fp64 copy of an fp32 v in fp64 precision mode)
  double* d_syrk_ws = nullptr;
  size_t syrk_bytes = 0;
  double* d_potrf = nullptr;    // inverted diagonal blocks (Linv) + double-buffered panels
  int64_t* d_status = nullptr;
  int64_t* h_status = nullptr;  // pinned
  double* h_sums = nullptr;     // pinned
  size_t ws_bytes = 0;
  int64_t launches = 0;
  std::string err;
  // multi-rank failure protocol (see solve_tail): first local failure of the current solve, an
  // empty (zero-column) shard, and whether this rank's own input was non-finite
  int poison_rc = 0;
  std::string poison_msg;
  bool empty_shard = false;
  bool local_nonfinite = false;
  uint8_t* d_St = nullptr;      // tiled copy of S for the tensor-core Gram (lazy, tiles.cuh)
  size_t St_bytes = 0;
  // F16X2 ring SYRK (lazy): the L2-resident tile ring, its ready/freed counters, u partials
  // z-space refinement's correction solve: 0 = the Cholesky factor in d_W (TRSV pair), 1 = the
  // eigh route's kept eigenpairs (d_U, d_w, eig_rank)
  int z_solver = 0;
  int64_t eig_rank = 0;
  uint8_t* d_ring = nullptr;
  int* d_ring_cnt = nullptr;
  double* d_ring_upart = nullptr;
  // eigh comparison route (lazy): Jacobi workspace, U (n_max^2), w, scratch, info
  void* d_eig = nullptr;
  double* d_U = nullptr;
  double* d_w = nullptr;
  double* d_t = nullptr;
  int* d_info = nullptr;
  int* h_info = nullptr;        // pinned [2]
  double* h_w = nullptr;        // pinned n_max
  void* d_svd = nullptr;        // direct-SVD route (lazy): Jacobi SVD workspace / tri-inverse scratch
  size_t svd_bytes = 0;
  float* d_scale = nullptr;     // F16X2 row scales (n_max)
  double* d_inv_scale = nullptr;
  int* d_ovf = nullptr;         // F16X2 retile flags (bit 1: fp16 overflow)
  // F16X2 exact row scales: a caller-supplied row max |S_i| (fs_set_row_absmax, used by the next
  // solve / Gram), or this context's own pass over S after an overflow of the sampled scales
  const float* hint_absmax = nullptr;
  int64_t hint_n = 0;
  float* d_absmax = nullptr;    // n_max
  int64_t fallbacks = 0;        // exact-scale recomputations (+ TF32X3 last resorts)
  int* h_ovf = nullptr;         // pinned
  // host-buffer entry (fs_chol_solve_host): device copies of S, v, x, an upload stream and
  // one event per uploaded row chunk (all lazy)
  void* d_Sin = nullptr;
  size_t Sin_bytes = 0;
  double* d_vin = nullptr;      // m_max doubles (holds v in its own dtype)
  double* d_xin = nullptr;      // m_max doubles
  int* d_flag = nullptr;        // non-finite input flag
  int* h_flag = nullptr;        // pinned
  cudaStream_t up_st = nullptr;
  static constexpr int kMaxChunks = 64;
  cudaEvent_t ev_chunk[kMaxChunks] = {};
  cudaEvent_t ev_free = nullptr;
  // host entry: x is copied to the caller's buffer on up_st as soon as the first x pass ends,
  // overlapping the residual pass (state 1 = the copy holds the final x, 2 = x changed since)
  double* early_x_host = nullptr;
  int early_x_state = 0;
  cudaEvent_t ev_xready = nullptr, ev_xcopy = nullptr;
  // z-space refinement: |d|, |z| of a correction fetched on a side stream, so the host decides on
  // the next step while the current x + y pass still runs (no idle gap between the steps)
  cudaStream_t dz_st = nullptr;
  cudaEvent_t ev_dz = nullptr, ev_dz_done = nullptr;
  double* h_dz = nullptr;       // pinned, 2 doubles
  // stage timing (fs_profile_enable): events recorded on the solve stream after each stage,
  // in chronological order; stage time = gap to the previous mark
  static constexpr int kMaxMarks = 24;
  bool prof_on = false;
  cudaEvent_t ev[kMaxMarks] = {};
  int ev_stage[kMaxMarks] = {};
  int n_marks = 0;
  double prof_ms[FS_PROF_STAGES] = {};
};

namespace {
// NVTX ranges per solve stage (header-only NVTX v3: free unless a profiler attaches)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

inline void prof_mark(fs_ctx* ctx, int stage, cudaStream_t st) {
  if (ctx->prof_on && ctx->n_marks < fs_ctx::kMaxMarks && ctx->ev[ctx->n_marks]) {
    cudaEventRecord(ctx->ev[ctx->n_marks], st);
    ctx->ev_stage[ctx->n_marks++] = stage;
  }
}
}  // namespace

namespace {

const double kEps = 2.220446049250313e-16;  // core.py:16

size_t packed_len(int64_t n) { return (size_t)(n * (n + 1) / 2 + n); }

struct Sizes {
  size_t packed, W, vec, partials, block_sums, r, syrk, potrf;
};

Sizes sizes_for(int64_t n, int64_t m, int num_sms) {
  Sizes s;
  s.packed = packed_len(n) * sizeof(double);
  s.W = (size_t)n * n * sizeof(double);
  s.vec = (size_t)n * sizeof(double);
  // row-GEMV chunk partials; also the F16X2 direct SYRK's per-split u partials (its split count
  // P <= KB / 8 = ceil(m / 64) / 8 <= ceil(m / 512) = the fp64 chunk count)
  s.partials = (size_t)fs::gemv_rows_chunks(m, true) * n * sizeof(double);
  s.block_sums = (size_t)fs::residual_cols_blocks(m, true) * 2 * sizeof(double);
  s.r = (size_t)m * sizeof(double);
  s.syrk = std::max(fs::syrk_dmma_workspace_bytes(n, m, num_sms), fs::syrk_tc_workspace_bytes(n, m, num_sms));
  s.potrf = (size_t)fs::potrf_scratch_doubles(n) * sizeof(double);
  return s;
}

int fail(fs_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_fail(fs_ctx* ctx, cudaError_t e, const char* where) {
  return fail(ctx, FS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define FS_CK(expr, where)                          \
  do {                                              \
    cudaError_t _e = (expr);                        \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, where); \
  } while (0)

int check_shape(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS) {
  if (!ctx) return FS_EINVAL;
  if (dtype != FS_F32 && dtype != FS_F64) return fail(ctx, FS_EINVAL, "dtype must be FS_F32 or FS_F64");
  if (!S) return fail(ctx, FS_EINVAL, "S is NULL");
  if (n < 1 || m < 1) return fail(ctx, FS_EINVAL, "score matrix needs at least one row and column");
  if (ldS < m) return fail(ctx, FS_EINVAL, "ldS must be >= m");
  if (n > ctx->n_max || m > ctx->m_max) return fail(ctx, FS_ENOMEM, "problem exceeds the context's n_max/m_max");
  return FS_OK;
}

int check_lam(fs_ctx* ctx, double lam) {
  if (!(lam > 0.0) || !isfinite(lam)) return fail(ctx, FS_EINVAL, "damping must be finite and > 0");
  return FS_OK;
}

// use_tc: 0 = fp64 SIMT, 1 = TF32X3, 2 = F16X2
int resolve_precision(fs_ctx* ctx, int dtype, int precision, const void* S, int64_t ldS, int* use_tc) {
  *use_tc = 0;
  if (precision == FS_PREC_FP64) return FS_OK;
  if (precision == FS_PREC_TF32X3 || precision == FS_PREC_F16X2 || precision == FS_PREC_AUTO) {
    if (dtype != FS_F32) {
      if (precision == FS_PREC_AUTO) return FS_OK;
      return fail(ctx, FS_EUNSUPPORTED, "TF32X3 / F16X2 precision needs fp32 scores");
    }
    *use_tc = precision == FS_PREC_TF32X3 ? 1 : 2;
    return FS_OK;
  }
  return fail(ctx, FS_EINVAL, "unknown precision mode");
}

// The tiled copy S_t is sized for the context's (n_max, m_max) in the layout the mode needs
// (F16X2: two fp16 planes, 4 bytes per score; TF32X3: two tf32 planes, 8 bytes) and allocated on
// first use — fp64-only users never pay for it, and an F16X2 user at the per-rank shard of
// n = 16384, m = 1e7 / 8 (82 GB of scores) is not charged the 164 GB TF32X3 layout.
// The tiled copy is capped at tile_cap_bytes() (16 GB): a larger (n, m) is split into K-chunks that each
// fit (retile a column range, SYRK its K-blocks, accumulate), so an F16X2 solve needs S plus at
// most 16 GB (n = 16384, m = 2e6: 131 GB of scores, one B200).
size_t tile_cap_bytes() {   // FS_TILE_CAP_MB overrides (tests force the K-chunked path with it)
  static const size_t cap = getenv("FS_TILE_CAP_MB") ? (size_t)atoll(getenv("FS_TILE_CAP_MB")) << 20
                                                     : (size_t)16 << 30;
  return cap;
}
int ensure_tiles(fs_ctx* ctx, bool f16) {
  const size_t need = std::min(tile_cap_bytes(), f16 ? fs::tiles16_bytes(ctx->n_max, ctx->m_max)
                                                  : fs::tiles_bytes(ctx->n_max, ctx->m_max));
  if (ctx->St_bytes >= need) return FS_OK;
  if (ctx->d_St) cudaFree(ctx->d_St);
  ctx->d_St = nullptr;
  ctx->St_bytes = 0;
  if (cudaMalloc((void**)&ctx->d_St, need) != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, FS_ENOMEM, f16 ? "cannot allocate the fp16 planes of S (F16X2)"
                                    : "cannot allocate the tf32 planes of S (TF32X3)");
  }
  ctx->St_bytes = need;
  return FS_OK;
}

int ensure_ring(fs_ctx* ctx) {
  if (ctx->d_ring) return FS_OK;
  bool ok = cudaMalloc((void**)&ctx->d_ring, fs::syrk_ring_bytes()) == cudaSuccess &&
            cudaMalloc((void**)&ctx->d_ring_cnt, 2 * 74 * 16 * sizeof(int)) == cudaSuccess &&
            cudaMalloc((void**)&ctx->d_ring_upart, fs::syrk_ring_upart_doubles(ctx->n_max) * sizeof(double)) ==
                cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    cudaFree(ctx->d_ring); cudaFree(ctx->d_ring_cnt); cudaFree(ctx->d_ring_upart);
    ctx->d_ring = nullptr; ctx->d_ring_cnt = nullptr; ctx->d_ring_upart = nullptr;
    return fail(ctx, FS_ENOMEM, "cannot allocate the F16X2 tile ring");
  }
  return FS_OK;
}

// F16X2 ring SYRK for this shape (FS_F16_RING=0 turns it off; FS_F16_DIRECT wins when set)
bool use_ring(fs_ctx* ctx, const void* S, int64_t n, int64_t m, int64_t ldS) {
  return fs::syrk_tc_supported(S, ldS) && fs::syrk_ring_ok(n, m, ctx->num_sms);
}

int ensure_eig(fs_ctx* ctx) {
  if (ctx->d_eig) return FS_OK;
  if (ctx->n_max > fs::syevj_max_n()) return fail(ctx, FS_EUNSUPPORTED, "eigh route supports n <= 16384");
  const int64_t n = ctx->n_max;
  bool ok = cudaMalloc(&ctx->d_eig, fs::syevj_workspace_bytes(n, ctx->num_sms)) == cudaSuccess &&
            cudaMalloc((void**)&ctx->d_U, (size_t)n * n * sizeof(double)) == cudaSuccess &&
            cudaMalloc((void**)&ctx->d_w, (size_t)n * sizeof(double)) == cudaSuccess &&
            (ctx->d_t || cudaMalloc((void**)&ctx->d_t, (size_t)n * sizeof(double)) == cudaSuccess) &&
            (ctx->d_info || cudaMalloc((void**)&ctx->d_info, 2 * sizeof(int)) == cudaSuccess) &&
            (ctx->h_info || cudaMallocHost((void**)&ctx->h_info, 2 * sizeof(int)) == cudaSuccess) &&
            cudaMallocHost((void**)&ctx->h_w, (size_t)n * sizeof(double)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return fail(ctx, FS_ENOMEM, "cannot allocate the eigensolver workspace");
  }
  return FS_OK;
}

int ensure_svd(fs_ctx* ctx, int64_t n) {
  const size_t need = std::max(fs::jacobi_svd_workspace_bytes(n), (size_t)n * n * sizeof(double));
  if (ctx->svd_bytes >= need) return FS_OK;
  if (ctx->d_svd) cudaFree(ctx->d_svd);
  ctx->d_svd = nullptr;
  ctx->svd_bytes = 0;
  bool ok = cudaMalloc(&ctx->d_svd, need) == cudaSuccess;
  if (ok && !ctx->d_info) ok = cudaMalloc((void**)&ctx->d_info, 2 * sizeof(int)) == cudaSuccess;
  if (ok && !ctx->h_info) ok = cudaMallocHost((void**)&ctx->h_info, 2 * sizeof(int)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return fail(ctx, FS_ENOMEM, "cannot allocate the SVD workspace");
  }
  ctx->svd_bytes = need;
  return FS_OK;
}

// Eigenpairs of the packed Gram (no shift) into ctx->d_w (descending) / ctx->d_U; synchronises
// to read the convergence word and w (ctx->h_w).
int eig_impl(fs_ctx* ctx, const double* Gp, int64_t n, cudaStream_t st, double tol = 1e-14) {
  int rc = ensure_eig(ctx);
  if (rc) return rc;
  int l = 0;
  // tolerance: off(A) <= tol ||A||_F (1e-14 unless the caller's Gram is itself less accurate),
  // at most 40 sweeps (quadratic convergence: ~6-11)
  cudaError_t e = fs::syevj(Gp, n, ctx->d_w, ctx->d_U, n, 40, tol, ctx->d_eig, ctx->num_sms, ctx->d_info, st, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "syevj");
  FS_CK(cudaMemcpyAsync(ctx->h_info, ctx->d_info, 2 * sizeof(int), cudaMemcpyDeviceToHost, st), "info d2h");
  FS_CK(cudaMemcpyAsync(ctx->h_w, ctx->d_w, n * sizeof(double), cudaMemcpyDeviceToHost, st), "w d2h");
  FS_CK(cudaStreamSynchronize(st), "sync");
  if (ctx->h_info[1]) return fail(ctx, FS_ENOCONV, "eigendecomposition did not converge");
  return FS_OK;
}

// F16X2 direct (the SYRK splits fp32 S itself, no S_t16 copy), FS_F16_DIRECT=1.  Off by default:
// the in-kernel split moves 288 KB of shared memory per K-block and CTA (TMA write + converter
// read/write + MMA operand reads) against 160 KB for the pre-tiled planes, and the 128 B/clk
// crossbar makes it slower than retile16 + the pre-tiled SYRK (4.3 vs 2.8 + 1.3 ms).
bool f16_direct() {
  static const int env = getenv("FS_F16_DIRECT") ? atoi(getenv("FS_F16_DIRECT")) : 0;
  return env != 0;
}

// F16X2 row scales: exact from a row-max hint (the caller's fs_set_row_absmax, or this context's
// own pass after an overflow), else from the sampled head of each row (overflow -> exact retry).
cudaError_t f16_scales(fs_ctx* ctx, const float* S, int64_t n, int64_t m, int64_t ldS, cudaStream_t st, int* l) {
  if (ctx->hint_absmax && ctx->hint_n == n) return fs::scales_from_max(ctx->hint_absmax, n, ctx->d_scale, ctx->d_inv_scale, st, l);
  return fs::row_scales(S, n, m, ldS, ctx->d_scale, ctx->d_inv_scale, st, l);
}

// after an fp16 overflow of the sampled scales: the exact row maxima of S (one streaming pass),
// used as the hint of the recomputation
cudaError_t exact_row_max(fs_ctx* ctx, const float* S, int64_t n, int64_t m, int64_t ldS, cudaStream_t st) {
  int l = 0;
  cudaError_t e = cudaMemsetAsync(ctx->d_absmax, 0, n * sizeof(float), st);
  if (e == cudaSuccess)
    e = fs::check_finite(S, false, n, m, ldS, ctx->d_ovf, ctx->num_sms, st, &l, (unsigned*)ctx->d_absmax);
  ctx->launches += l;
  ctx->hint_absmax = ctx->d_absmax;
  ctx->hint_n = n;
  ctx->fallbacks += 1;
  return e;
}

// Gram stage.  TF32X3: retile S into S_t (optionally fused with u = S w), then the CTA-pair
// tcgen05 SYRK on S_t.  FP64: exact-product SIMT SYRK on S.
int gram_impl(fs_ctx* ctx, int dtype, int precision, const void* S, int64_t n, int64_t m,
              int64_t ldS, double lam, double* Gp, cudaStream_t st, const float* w32 = nullptr,
              double* u = nullptr) {
  int use_tc = 0;
  int rc = resolve_precision(ctx, dtype, precision, S, ldS, &use_tc);
  if (rc) return rc;
  int l = 0;
  cudaError_t e;
  if (use_tc == 2 && f16_direct() && fs::syrk_tc_supported(S, ldS)) {
    // F16X2 direct: row scales from a sample, then the SYRK splits fp32 S itself (no S_t16 copy)
    // and forms u = S w in the same pass.  The overflow flag is checked by the caller at its next
    // host synchronisation.
    e = cudaMemsetAsync(ctx->d_ovf, 0, sizeof(int), st);
    if (e == cudaSuccess) e = f16_scales(ctx, (const float*)S, n, m, ldS, st, &l);
    if (e == cudaSuccess && w32) prof_mark(ctx, FS_PROF_GEMV_SV, st);
    if (e == cudaSuccess)
      e = fs::syrk_f16_direct((const float*)S, ldS, n, m, ctx->d_scale, ctx->d_inv_scale, w32, ctx->d_ovf,
                              ctx->d_partials, u, lam, Gp, ctx->d_syrk_ws, ctx->num_sms, st, &l);
  } else if (use_tc == 2 && use_ring(ctx, S, n, m, ldS) && (rc = ensure_ring(ctx)) == FS_OK) {
    // F16X2 ring: row scales, then ONE kernel splits S into the L2-resident tile ring, forms
    // u = S w and the Gram from it (no S_t16 round trip through HBM)
    e = cudaMemsetAsync(ctx->d_ovf, 0, sizeof(int), st);
    if (e == cudaSuccess) e = f16_scales(ctx, (const float*)S, n, m, ldS, st, &l);
    if (e == cudaSuccess && w32) prof_mark(ctx, FS_PROF_GEMV_SV, st);
    if (e == cudaSuccess)
      e = fs::syrk_f16_ring((const float*)S, ldS, n, m, ctx->d_scale, ctx->d_inv_scale, w32, ctx->d_ovf,
                            ctx->d_ring_upart, u, lam, Gp, ctx->d_syrk_ws, ctx->d_ring, ctx->d_ring_cnt,
                            ctx->num_sms, st, &l);
  } else if (use_tc == 2 && ((rc = FS_OK), true) && (rc = ensure_tiles(ctx, true)) == FS_OK &&
             fs::tiles16_bytes(n, m) <= ctx->St_bytes) {
    // F16X2: row scales, split planes (+ u = S w), kind::f16 SYRK.  The overflow flag is checked
    // by the caller at its next host synchronisation.  (A failed ring allocation falls back here.)
    e = cudaMemsetAsync(ctx->d_ovf, 0, sizeof(int), st);
    if (e == cudaSuccess) e = f16_scales(ctx, (const float*)S, n, m, ldS, st, &l);
    if (e == cudaSuccess)
      e = fs::retile16_cols((const float*)S, n, m, ldS, w32, ctx->d_partials, ctx->d_St, ctx->d_scale, 0, m,
                            ctx->d_ovf, st, &l);
    if (e == cudaSuccess && w32) e = fs::reduce_row_partials(ctx->d_partials, n, m, u, st, &l);
    if (e == cudaSuccess && w32) prof_mark(ctx, FS_PROF_GEMV_SV, st);
    if (e == cudaSuccess)
      e = fs::syrk_f16(ctx->d_St, n, m, ctx->d_inv_scale, lam, Gp, ctx->d_syrk_ws, ctx->num_sms, st, &l);
  } else if (use_tc && !rc && (rc = ensure_tiles(ctx, use_tc == 2)) == FS_OK) {
    // K-chunked: the tiled copy of all of S would exceed the cap.  Each chunk of K-blocks is
    // retiled into the same buffer (addressed through a base shifted by the chunk's first
    // K-block, so the kernels' absolute tile offsets land in it), its SYRK share accumulated
    // into Gp (lam added once); stream order keeps a chunk's SYRK ahead of the next retile.
    const bool f16 = use_tc == 2;
    const int64_t nb = fs::tiles_nb(n), tile_cols = f16 ? fs::kTile16Cols : fs::kTileCols;
    const size_t kb_bytes = (size_t)nb * (f16 ? 2 : 1) * fs::kTileBytes;
    const int64_t KB = (m + tile_cols - 1) / tile_cols;
    const int64_t align = fs::gemv_rows_chunk_cols() / tile_cols;   // column chunks of the u partials
    const int64_t fit = (int64_t)(ctx->St_bytes / kb_bytes);
    const int64_t kbc = fit >= KB ? KB : fit / align * align;   // one chunk when everything fits
    if (kbc < 1) return fail(ctx, FS_ENOMEM, "tiled copy too small for one K-chunk");
    e = cudaMemsetAsync(ctx->d_ovf, 0, sizeof(int), st);
    if (e == cudaSuccess && f16) e = f16_scales(ctx, (const float*)S, n, m, ldS, st, &l);
    for (int64_t kb0 = 0; kb0 < KB && e == cudaSuccess; kb0 += kbc) {
      const int64_t kb1 = std::min(KB, kb0 + kbc), c0 = kb0 * tile_cols, c1 = std::min(m, kb1 * tile_cols);
      uint8_t* base = ctx->d_St - (ptrdiff_t)(kb0 * (int64_t)kb_bytes);
      const double lam_c = kb0 == 0 ? lam : 0.0;
      if (f16) {
        e = fs::retile16_cols((const float*)S, n, m, ldS, w32, ctx->d_partials, base, ctx->d_scale, c0, c1,
                              ctx->d_ovf, st, &l);
        if (e == cudaSuccess)
          e = fs::syrk_f16(base, n, m, ctx->d_inv_scale, lam_c, Gp, ctx->d_syrk_ws, ctx->num_sms, st, &l, (int)kb0,
                           (int)kb1, kb0 > 0);
      } else {
        e = fs::retile_cols((const float*)S, n, m, ldS, w32, ctx->d_partials, base, c0, c1, ctx->d_ovf, st, &l);
        if (e == cudaSuccess)
          e = fs::syrk_tc(base, n, m, lam_c, Gp, ctx->d_syrk_ws, ctx->num_sms, st, &l, 0, -1, (int)kb0, (int)kb1,
                          kb0 > 0);
      }
    }
    if (e == cudaSuccess && w32) e = fs::reduce_row_partials(ctx->d_partials, n, m, u, st, &l);
    if (e == cudaSuccess && w32) prof_mark(ctx, FS_PROF_GEMV_SV, st);
  } else if (use_tc) {
    return rc;
  } else {
    e = fs::syrk_dmma(dtype == FS_F64, S, n, m, ldS, lam, Gp, ctx->d_syrk_ws, ctx->syrk_bytes, ctx->num_sms, st, &l);
  }
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gram");
  prof_mark(ctx, FS_PROF_GRAM, st);
  return FS_OK;
}

}  // namespace

// Everything after the Gram/u stage of _solve_chol_impl: all-reduce, potrf, _chol_apply,
// residual, optional refinement, status + norms read-back (one host synchronisation per pass).
// internal: the F16X2 Gram overflowed on some rank -> recompute with TF32X3
constexpr int kRetryTf32 = 100;

// ---- multi-rank failure protocol ----
// With an all-reduce callback every rank must issue the same collectives in the same order, so
// no rank may return between two of them.  A rank whose local step fails (a CUDA error, a lazy
// allocation that does not fit, an empty shard's missing data) becomes "idle": it records the
// first failure, skips its remaining kernels, contributes zeros to every collective and keeps
// joining them.  The norms all-reduce carries a status slot (sums[3] = idle + 1024 * non-finite
// input), so every rank learns at the same host synchronisation that the solve failed and all
// return an error together (the failing rank its own status, the others FS_ECUDA / FS_EINVAL
// naming a peer).  Host-side control flow between collectives depends only on all-reduced values
// (the norms, the overflow flag) or on arguments every rank shares, so ranks cannot diverge.
// One rank (no callback) keeps the direct early returns.
constexpr double kStatusIdle = 1.0, kStatusNonFinite = 1024.0;

namespace {
void poison(fs_ctx* ctx, int rc) {
  if (!ctx->poison_rc) {
    ctx->poison_rc = rc;
    ctx->poison_msg = ctx->err;
  }
}

__global__ void status_slot_kernel(const int* nonfinite, int idle, int host_nonfinite, double* out) {
  double s = idle ? kStatusIdle : 0.0;
  if (host_nonfinite || (nonfinite && (*nonfinite & 1))) s += kStatusNonFinite;
  *out = s;
}

// z-space refinement (see finish_x): t = lam (y - z_acc) into dz
__global__ void zres_kernel(const double* __restrict__ y, const double* __restrict__ zacc, double lam, int64_t n,
                            double* __restrict__ dz) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dz[i] = lam * (y[i] - zacc[i]);
}
// z_acc += dz; sums[0] = |dz|^2, sums[1] = |z_acc|^2 (one CTA, fixed order: deterministic)
__global__ void zadd_kernel(double* __restrict__ zacc, const double* __restrict__ dz, int64_t n,
                            double* __restrict__ sums) {
  __shared__ double red[2][32];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = dz[i], z = zacc[i] + d;
    zacc[i] = z;
    a = fma(d, d, a);
    b = fma(z, z, b);
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = a; red[1][threadIdx.x >> 5] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { sa += red[0][w]; sb += red[1][w]; }
    sums[0] = sa;
    sums[1] = sb;
  }
}

// after the norms all-reduce: the collective decision when the status slot is set
int collective_failure(fs_ctx* ctx, double status) {
  const long long nf = (long long)(status / kStatusNonFinite);
  if (ctx->poison_rc) {
    ctx->err = ctx->poison_msg;
    return ctx->poison_rc;
  }
  if (ctx->local_nonfinite) return fail(ctx, FS_EINVAL, "score matrix and right-hand side must contain only finite entries");
  if (nf > 0) return fail(ctx, FS_EINVAL, "a peer rank's score shard or right-hand side has non-finite entries");
  return fail(ctx, FS_ECUDA, "a peer rank failed during the collective solve");
}
}  // namespace

// a local step inside a collective solve: single rank -> return the failure; multi-rank -> idle
#define FS_STEP(expr)                          \
  do {                                         \
    int _r = (expr);                           \
    if (_r) {                                  \
      if (!multi) return _r;                   \
      poison(ctx, _r);                         \
    }                                          \
  } while (0)
#define FS_CKS(expr, where) FS_STEP(([&]() -> int { cudaError_t _e = (expr); \
                                      return _e == cudaSuccess ? FS_OK : cuda_fail(ctx, _e, where); })())

static int finish_x(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS, const void* v, int vdt,
                    double lam, double* x, fs_allreduce_fn allreduce, void* allreduce_user, int flags,
                    double refine_above, int64_t* pivot, double* out_res, cudaStream_t st, const int* ovf,
                    const int* nonfinite = nullptr);

// ovf: F16X2 retile flag word (bit 2 = fp16 overflow) or NULL.  The bit joins the norms
// all-reduce, so every rank takes the same retry decision.
static int solve_tail(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS, const void* v, int vdt,
               double lam, double* x, fs_allreduce_fn allreduce, void* allreduce_user, int flags,
               double refine_above, int64_t* pivot, double* out_res, cudaStream_t st, const int* ovf = nullptr,
               const int* nonfinite = nullptr) {
  const bool multi = allreduce != nullptr;
  void* stream = (void*)st;
  double* u = ctx->d_packed + n * (n + 1) / 2;
  NvtxRange range("fs: allreduce + potrf + trsv");
  if (multi) {
    if (ctx->poison_rc || ctx->empty_shard) cudaMemsetAsync(ctx->d_packed, 0, packed_len(n) * sizeof(double), st);
    if (allreduce(ctx->d_packed, (int64_t)packed_len(n), allreduce_user, stream) != 0)
      return fail(ctx, FS_ECUDA, "allreduce of [W | u] failed");
  }
  prof_mark(ctx, FS_PROF_ALLREDUCE, st);
  // 2. W = G + lam I, L = chol(W) (redundant on every rank, deterministic: identical L)
  bool solved = false;
  if (!ctx->poison_rc) FS_STEP(fs_unpack_lower(ctx, ctx->d_packed, n, lam, ctx->d_W, n, stream));
  if (!ctx->poison_rc) {
    // L = chol(W) with the TRSV pair z = L^-T L^-1 u fused into the same persistent kernel
    FS_CKS(cudaMemsetAsync(ctx->d_status, 0, sizeof(int64_t), st), "potrf status reset");
    int l = 0;
    // the TRSV pair rides along inside the factorisation kernel up to FS_POTRF_FUSE_MAXN; above
    // it the flag-chained TRSV kernel is faster than the fused grid-barrier steps
    static const int64_t fuse_maxn = getenv("FS_POTRF_FUSE_MAXN") ? atoll(getenv("FS_POTRF_FUSE_MAXN")) : 4096;
    const double* u_fused = n <= fuse_maxn ? u : nullptr;
    if (!ctx->poison_rc) FS_CKS(fs::potrf_lower(ctx->d_W, n, n, ctx->d_status, ctx->d_potrf, st, &l, u_fused, ctx->d_z, &solved),
                                "potrf");
    ctx->launches += l;
  }
  prof_mark(ctx, FS_PROF_POTRF, st);
  if (!solved && !ctx->poison_rc) {
    FS_CKS(cudaMemcpyAsync(ctx->d_z, u, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy u");
    int l = 0;
    if (!ctx->poison_rc) FS_CKS(fs::trsv_pair(ctx->d_W, n, n, ctx->d_potrf, ctx->d_z, ctx->d_status, st, &l), "trsv_pair");
    ctx->launches += l;
  }
  prof_mark(ctx, FS_PROF_TRSV, st);
  return finish_x(ctx, dtype, S, n, m, ldS, v, vdt, lam, x, allreduce, allreduce_user, flags, refine_above, pivot,
                  out_res, st, ovf, nonfinite);
}

// From z (in ctx->d_z) to x = (v - S^T z)/lam, the residual diagnostics and the optional
// refinement with the Cholesky factor in ctx->d_W (solvers.py:122-126, :160-194).
static int finish_x(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS, const void* v, int vdt,
                    double lam, double* x, fs_allreduce_fn allreduce, void* allreduce_user, int flags,
                    double refine_above, int64_t* pivot, double* out_res, cudaStream_t st, const int* ovf,
                    const int* nonfinite) {
  const bool multi = allreduce != nullptr;
  void* stream = (void*)st;
  const int nsums = multi ? 4 : (ovf ? 3 : 2);
  const bool want_res = (flags & FS_FLAG_RESIDUAL) != 0;
  const bool want_refine = (flags & FS_FLAG_REFINE) != 0;
  auto idle = [&]() { return ctx->poison_rc != 0 || ctx->empty_shard; };
  // 3. x = (v - S^T z) / lam on the local shard; with diagnostics fused with y = S x (one
  //    HBM pass; falls back to two passes when n is too large for the fused kernel)
  bool y_ready = false;
  auto solve_cols = [&](const void* rhs, int rhs_f64, double l, bool accumulate) -> int {
    int lc = 0;
    cudaError_t e = cudaErrorNotSupported;
    if (want_res)
      e = fs::gemv_cols_solve_y(dtype == FS_F64, S, n, m, ldS, ctx->d_z, rhs, rhs_f64, l, accumulate, x,
                                ctx->d_partials, fs::gemv_rows_chunks(ctx->m_max, true) * ctx->n_max / n, ctx->d_y,
                                ctx->num_sms,
                                st, &lc);
    if (e == cudaErrorNotSupported) {
      cudaGetLastError();
      y_ready = false;
      e = fs::gemv_cols_solve(dtype == FS_F64, S, n, m, ldS, ctx->d_z, rhs, rhs_f64, l, accumulate, x, st, &lc);
    } else {
      y_ready = true;
    }
    ctx->launches += lc;
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gemv_cols_solve");
    return FS_OK;
  };
  {
    NvtxRange r("fs: x = (v - S^T z)/lam, y = S x");
    if (!idle()) FS_STEP(solve_cols(v, vdt == FS_F64, lam, false));
  }
  prof_mark(ctx, FS_PROF_GEMV_STZ, st);
  if (ctx->early_x_host && !idle()) {   // host entry: x -> host on up_st while the residual pass runs
    FS_CK(cudaEventRecord(ctx->ev_xready, st), "event");
    FS_CK(cudaStreamWaitEvent(ctx->up_st, ctx->ev_xready, 0), "event wait");
    FS_CK(cudaMemcpyAsync(ctx->early_x_host, x, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->up_st),
          "x d2h (early)");
    FS_CK(cudaEventRecord(ctx->ev_xcopy, ctx->up_st), "event");
    ctx->early_x_state = 1;
  }
  // the status slot and the overflow flag of one norms all-reduce (multi-rank: always 4 doubles)
  auto fill_flags = [&]() -> int {
    if (ovf && !idle()) {
      int lf = 0;
      FS_CKS(fs::flag_bit_to_double(ovf, 2, ctx->d_sums + 2, st, &lf), "overflow flag");
      ctx->launches += lf;
    } else if (multi) {
      cudaMemsetAsync(ctx->d_sums + 2, 0, sizeof(double), st);
    }
    if (multi) {
      status_slot_kernel<<<1, 1, 0, st>>>(nonfinite, ctx->poison_rc != 0 ? 1 : 0, ctx->local_nonfinite ? 1 : 0,
                                          ctx->d_sums + 3);
      ctx->launches += 1;
    }
    return FS_OK;
  };
  // ---- z-space refinement (FS_FLAG_REFINE_Z, the fp32-split modes) ----
  // x = (v - S^T z)/lam depends on S only through the n-vector z = W^-1 S v, W = S S^T + lam I.
  // The split Gram's factor solves W~ = W + E instead; refining z on the n x n system W z = u
  // contracts by ||W~^-1 E|| ~ 2^-21 kappa(W) per step, whereas refining x on the m x m system
  // (the reference's scheme) contracts by ~2^-21 sigma_max^2 / lam — no contraction at all at
  // the headline (sigma^2/lam ~ 1e6).  The z residual needs no extra pass: with y = S x (already
  // formed by the fused x + y pass, exact fp64 products), lam (y - z) = S v - S S^T z - lam z =
  // u - W z exactly.  A step is: d = W~^-1 lam (y - z) (the TRSV pair), z += d, and one fused pass
  // x += (0 - S^T d)/lam, y = S x.  Single rank: stop once |d| <= 1e-12 |z|; multi-rank: the
  // fixed step count (control flow may not depend on rank-local data).  Profiled as
  // FS_PROF_REFINE.
  const bool want_z = (flags & FS_FLAG_REFINE_Z) != 0 && want_res;
  const int zsteps = want_z ? std::max(1, (flags >> 8) & 0xFF) : 0;
  int zdone = 0;
  // single rank: fetch (|d|^2, |z|^2) of the step on the side stream (created on first use;
  // false -> the caller synchronises the stream instead)
  auto fetch_dz = [&]() -> bool {
    if (!ctx->dz_st) {
      if (cudaStreamCreateWithFlags(&ctx->dz_st, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx->ev_dz, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx->ev_dz_done, cudaEventDisableTiming) != cudaSuccess ||
          cudaMallocHost((void**)&ctx->h_dz, 2 * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
    }
    return cudaEventRecord(ctx->ev_dz, st) == cudaSuccess && cudaStreamWaitEvent(ctx->dz_st, ctx->ev_dz, 0) == cudaSuccess &&
           cudaMemcpyAsync(ctx->h_dz, ctx->d_sums, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->dz_st) == cudaSuccess &&
           cudaEventRecord(ctx->ev_dz_done, ctx->dz_st) == cudaSuccess;
  };
  bool dz_async = false;
  // one z-space step: d = W~^-1 lam (y - z_acc), z_acc += d, x += -S^T d / lam, y = S x
  auto z_step = [&](bool fetch) -> int {
    NvtxRange r("fs: z-space refinement step");
    if (!y_ready && !idle()) FS_STEP(fs_gemv_rows(ctx, dtype, S, n, m, ldS, x, FS_F64, ctx->d_y, stream));
    if (multi) {
      if (idle()) cudaMemsetAsync(ctx->d_y, 0, n * sizeof(double), st);
      if (allreduce(ctx->d_y, n, allreduce_user, stream) != 0) return fail(ctx, FS_ECUDA, "allreduce of y failed");
    }
    if (!ctx->poison_rc) {
      const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 64);
      zres_kernel<<<g, 256, 0, st>>>(ctx->d_y, ctx->d_zacc, lam, n, ctx->d_z);
      int l = 0;
      if (ctx->z_solver == 1)   // eigh route: d = U_r diag(1 / (w_r + lam)) U_r^T e (in place)
        FS_CKS(fs::eig_apply(ctx->d_U, n, n, ctx->eig_rank, ctx->d_z, ctx->d_w, lam, ctx->d_t, ctx->d_z, st, &l),
               "eig_apply (z refine)");
      else
        FS_CKS(fs::trsv_pair(ctx->d_W, n, n, ctx->d_potrf, ctx->d_z, ctx->d_status, st, &l), "trsv_pair (z refine)");
      zadd_kernel<<<1, 1024, 0, st>>>(ctx->d_zacc, ctx->d_z, n, ctx->d_sums);
      ctx->launches += l + 2;
    }
    static const bool dz_env = getenv("FS_DZ_ASYNC") ? atoi(getenv("FS_DZ_ASYNC")) != 0 : true;
    dz_async = fetch && !multi && dz_env && fetch_dz();
    if (ctx->early_x_state == 1) {   // x changes: the early copy must finish reading it first
      FS_CK(cudaStreamWaitEvent(st, ctx->ev_xcopy, 0), "event wait");
      ctx->early_x_state = 2;
    }
    if (!idle()) FS_STEP(solve_cols(ctx->d_r, 1, lam, true));
    prof_mark(ctx, FS_PROF_REFINE, st);
    ++zdone;
    return FS_OK;
  };
  if (want_z) {
    if (!idle()) FS_CKS(cudaMemcpyAsync(ctx->d_zacc, ctx->d_z, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "z copy");
    if (!idle()) FS_CKS(cudaMemsetAsync(ctx->d_r, 0, m * sizeof(double), st), "zero rhs");
    for (int step = 0; step < zsteps; ++step) {
      const bool check = !multi && step + 1 < zsteps;
      if (int rc = z_step(check)) return rc;
      if (check) {
        const double* hs = ctx->h_sums;
        if (dz_async) {
          FS_CK(cudaEventSynchronize(ctx->ev_dz_done), "dz wait");
          hs = ctx->h_dz;
        } else {
          FS_CK(cudaMemcpyAsync(ctx->h_sums, ctx->d_sums, 2 * sizeof(double), cudaMemcpyDeviceToHost, st), "dz d2h");
          FS_CK(cudaStreamSynchronize(st), "sync");
        }
        // the last correction moved z by <= 1e-12 of its size: x is at (or next to) the fp64
        // residual floor; the residual below decides whether one more step is needed
        if (!(hs[0] > 1e-24 * hs[1])) break;
      }
    }
  }
  double abs_res = NAN, rel_res = NAN;
  // refinement steps: FS_FLAG_REFINE alone = the reference's single step; bits 8-15 raise it
  const int max_steps = want_refine && !want_z ? std::max(1, (flags >> 8) & 0xFF) : 0;
  double prev_rel = INFINITY;
  // z-space mode, one rank: the reference's rule on the measured residual — if it is above
  // refine_above and steps remain, one more step and a fresh residual (the |d| test above stops
  // at the fp64 floor of z, which at large m can leave x's residual slightly above 1e-10)
  for (int zround = 0;; ++zround) {
    if (zround > 0) {
      if (int rc = z_step(false)) return rc;
    }
    for (int pass = 0; want_res && pass <= max_steps; ++pass) {
      NvtxRange r("fs: residual (+ x-space refinement)");
      // residual: y = S x (all-reduced), r = S^T y + lam x - v, norms all-reduced
      if (!y_ready && !idle()) FS_STEP(fs_gemv_rows(ctx, dtype, S, n, m, ldS, x, FS_F64, ctx->d_y, stream));
      if (multi) {
        if (idle()) cudaMemsetAsync(ctx->d_y, 0, n * sizeof(double), st);
        if (allreduce(ctx->d_y, n, allreduce_user, stream) != 0) return fail(ctx, FS_ECUDA, "allreduce of y failed");
      }
      if (!idle()) {
        int l = 0;
        FS_CKS(fs::residual_cols(dtype == FS_F64, S, n, m, ldS, ctx->d_y, x, v, vdt == FS_F64, lam,
                                 pass < max_steps ? ctx->d_r : nullptr, ctx->d_block_sums, ctx->d_sums, st, &l),
               "residual_cols");
        ctx->launches += l;
      }
      if (idle()) cudaMemsetAsync(ctx->d_sums, 0, 2 * sizeof(double), st);
      if (int r = fill_flags()) return r;
      if (multi && allreduce(ctx->d_sums, nsums, allreduce_user, stream) != 0)
        return fail(ctx, FS_ECUDA, "allreduce of residual norms failed");
      prof_mark(ctx, FS_PROF_RESIDUAL, st);
      FS_CK(cudaMemcpyAsync(ctx->h_sums, ctx->d_sums, nsums * sizeof(double), cudaMemcpyDeviceToHost, st), "norms d2h");
      FS_CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "status d2h");
      FS_CK(cudaStreamSynchronize(st), "sync");
      if (multi && ctx->h_sums[3] > 0.0) return collective_failure(ctx, ctx->h_sums[3]);
      if (ovf && ctx->h_sums[2] > 0.0) return kRetryTf32;
      if (*ctx->h_status != 0) break;
      abs_res = sqrt(ctx->h_sums[0]);
      rel_res = abs_res / std::max(sqrt(ctx->h_sums[1]), kEps);
      if (pass == max_steps || !(rel_res > refine_above)) break;
      // iterative mode: stop once a step no longer halves the residual (no contraction left)
      if (pass > 0 && !(rel_res < 0.5 * prev_rel)) break;
      prev_rel = rel_res;
      // one correction pass with the same factor (solvers.py:183-194): d = chol_apply(-r)
      // residual_cols stored r = (S^T y + lam x) - v; refinement right-hand side is -r
      if (!idle()) FS_STEP(fs_gemv_rows(ctx, dtype, S, n, m, ldS, ctx->d_r, FS_F64, ctx->d_z, stream));
      if (multi) {
        if (idle()) cudaMemsetAsync(ctx->d_z, 0, n * sizeof(double), st);
        if (allreduce(ctx->d_z, n, allreduce_user, stream) != 0)
          return fail(ctx, FS_ECUDA, "allreduce of refinement u failed");
      }
      if (!ctx->poison_rc) {
        int l = 0;
        FS_CKS(fs::trsv_pair(ctx->d_W, n, n, ctx->d_potrf, ctx->d_z, ctx->d_status, st, &l), "trsv_pair (refine)");
        ctx->launches += l;
      }
      // x += (-r - S^T z') / lam  ==  x - (r + S^T z') / lam ; z' = W^-1 S r  (linearity)
      if (ctx->early_x_state == 1) {   // x changes: the early copy must finish reading it first
        FS_CK(cudaStreamWaitEvent(st, ctx->ev_xcopy, 0), "event wait");
        ctx->early_x_state = 2;
      }
      if (!idle()) FS_STEP(solve_cols(ctx->d_r, 1, -lam, true));
    }
    // (at most one such step, like the reference's single correction pass, solvers.py:183-194)
    if (!(want_z && !multi && zround == 0 && rel_res > refine_above && zdone < zsteps && *ctx->h_status == 0 &&
          !ctx->poison_rc))
      break;
  }
  if (!want_res) {
    const int off = 2, cnt = multi ? 2 : 1;
    if (ovf || multi) {
      if (int r = fill_flags()) return r;
      if (multi && allreduce(ctx->d_sums + off, cnt, allreduce_user, stream) != 0)
        return fail(ctx, FS_ECUDA, "allreduce of the overflow / status flags failed");
      FS_CK(cudaMemcpyAsync(ctx->h_sums + off, ctx->d_sums + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, st),
            "flag d2h");
    }
    FS_CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "status d2h");
    FS_CK(cudaStreamSynchronize(st), "sync");
    if (multi && ctx->h_sums[3] > 0.0) return collective_failure(ctx, ctx->h_sums[3]);
    if (ovf && ctx->h_sums[2] > 0.0) return kRetryTf32;
  }
  if (ctx->poison_rc) {   // single rank never gets here idle; multi-rank: the status slot said so
    ctx->err = ctx->poison_msg;
    return ctx->poison_rc;
  }
  if (ctx->prof_on) {
    // each mark closes the stage it names (refinement passes fold into their stages)
    for (int k = 0; k < FS_PROF_STAGES; ++k) ctx->prof_ms[k] = 0.0;
    for (int i = 1; i < ctx->n_marks; ++i) {
      float ms = 0.f;
      const int sidx = ctx->ev_stage[i];
      if (sidx >= 0 && sidx < FS_PROF_STAGES && cudaEventElapsedTime(&ms, ctx->ev[i - 1], ctx->ev[i]) == cudaSuccess)
        ctx->prof_ms[sidx] += ms;
    }
  }
  if (*ctx->h_status != 0) {
    if (pivot) *pivot = *ctx->h_status - 1;
    return fail(ctx, FS_NOT_PD, "Gram matrix is not positive definite at pivot " + std::to_string(*ctx->h_status - 1));
  }
  if (out_res) { out_res[0] = abs_res; out_res[1] = rel_res; }
  return FS_OK;
}


extern "C" {

const char* fs_version(void) { return "fisher-b200 0.1.0 sm_100a"; }

size_t fs_workspace_bytes(int64_t n, int64_t m, int dtype, int precision) {
  // device bytes one solve of (n, m) touches besides S, v and x (feeds WorkspaceMeter)
  Sizes s = sizes_for(n, m, 148);
  const bool tc = dtype == FS_F32 && precision != FS_PREC_FP64;
  const size_t gram = tc ? fs::syrk_tc_plan_bytes(n, m, 148) : fs::syrk_dmma_plan_bytes(n, m, 148);
  return s.packed + s.W + 2 * s.vec + s.partials + s.block_sums + 4 * sizeof(double) + 2 * s.r + gram + s.potrf +
         sizeof(int64_t);
}

int fs_ctx_create(fs_ctx** out, int device, int64_t n_max, int64_t m_max) {
  if (!out || n_max < 1 || m_max < 1) return FS_EINVAL;
  *out = nullptr;
  fs_ctx* ctx = new fs_ctx();
  ctx->device = device;
  ctx->n_max = n_max;
  ctx->m_max = m_max;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete ctx; return FS_ECUDA; }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (sms > 0) ctx->num_sms = sms;
  Sizes s = sizes_for(n_max, m_max, ctx->num_sms);
  bool ok = true;
  auto A = [&](void** p, size_t b) { if (ok && cudaMalloc(p, std::max<size_t>(b, 16)) != cudaSuccess) ok = false; };
  A((void**)&ctx->d_packed, s.packed);
  A((void**)&ctx->d_W, s.W);
  A((void**)&ctx->d_z, s.vec);
  A((void**)&ctx->d_y, s.vec);
  A((void**)&ctx->d_zacc, s.vec);
  A((void**)&ctx->d_partials, s.partials);
  A((void**)&ctx->d_block_sums, s.block_sums);
  A((void**)&ctx->d_sums, 4 * sizeof(double));
  A((void**)&ctx->d_r, s.r);
  A((void**)&ctx->d_v64, s.r);
  A((void**)&ctx->d_syrk_ws, s.syrk);
  ctx->syrk_bytes = s.syrk;
  A((void**)&ctx->d_potrf, s.potrf);
  A((void**)&ctx->d_status, sizeof(int64_t));
  A((void**)&ctx->d_scale, n_max * sizeof(float));
  A((void**)&ctx->d_inv_scale, n_max * sizeof(double));
  A((void**)&ctx->d_ovf, sizeof(int));
  A((void**)&ctx->d_absmax, n_max * sizeof(float));
  if (ok && cudaMallocHost((void**)&ctx->h_ovf, sizeof(int)) != cudaSuccess) ok = false;
  if (ok && cudaMallocHost((void**)&ctx->h_status, sizeof(int64_t)) != cudaSuccess) ok = false;
  if (ok && cudaMallocHost((void**)&ctx->h_sums, 4 * sizeof(double)) != cudaSuccess) ok = false;
  if (!ok) {
    cudaGetLastError();
    fs_ctx_destroy(ctx);
    return FS_ENOMEM;
  }
  for (int i = 0; i < fs_ctx::kMaxMarks; ++i) cudaEventCreate(&ctx->ev[i]);
  ctx->ws_bytes = s.packed + s.W + 2 * s.vec + s.partials + s.block_sums + s.r + s.syrk;
  cudaMemset(ctx->d_status, 0, sizeof(int64_t));
  cudaMemset(ctx->d_ovf, 0, sizeof(int));
  *out = ctx;
  return FS_OK;
}

void fs_ctx_destroy(fs_ctx* ctx) {
  if (!ctx) return;
  cudaFree(ctx->d_packed); cudaFree(ctx->d_W); cudaFree(ctx->d_z); cudaFree(ctx->d_y); cudaFree(ctx->d_zacc);
  cudaFree(ctx->d_partials); cudaFree(ctx->d_block_sums); cudaFree(ctx->d_sums);
  cudaFree(ctx->d_r); cudaFree(ctx->d_v64); cudaFree(ctx->d_syrk_ws); cudaFree(ctx->d_status);
  cudaFree(ctx->d_potrf);
  cudaFree(ctx->d_scale); cudaFree(ctx->d_inv_scale); cudaFree(ctx->d_ovf); cudaFree(ctx->d_absmax);
  if (ctx->d_eig) cudaFree(ctx->d_eig);
  if (ctx->d_svd) cudaFree(ctx->d_svd);
  if (ctx->d_U) cudaFree(ctx->d_U);
  if (ctx->d_w) cudaFree(ctx->d_w);
  if (ctx->d_t) cudaFree(ctx->d_t);
  if (ctx->d_info) cudaFree(ctx->d_info);
  if (ctx->h_info) cudaFreeHost(ctx->h_info);
  if (ctx->h_w) cudaFreeHost(ctx->h_w);
  if (ctx->h_ovf) cudaFreeHost(ctx->h_ovf);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->h_sums) cudaFreeHost(ctx->h_sums);
  for (int i = 0; i < fs_ctx::kMaxMarks; ++i)
    if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
  if (ctx->d_St) cudaFree(ctx->d_St);
  cudaFree(ctx->d_ring); cudaFree(ctx->d_ring_cnt); cudaFree(ctx->d_ring_upart);
  if (ctx->d_Sin) cudaFree(ctx->d_Sin);
  if (ctx->d_vin) cudaFree(ctx->d_vin);
  if (ctx->d_xin) cudaFree(ctx->d_xin);
  if (ctx->d_flag) cudaFree(ctx->d_flag);
  if (ctx->h_flag) cudaFreeHost(ctx->h_flag);
  for (int i = 0; i < fs_ctx::kMaxChunks; ++i)
    if (ctx->ev_chunk[i]) cudaEventDestroy(ctx->ev_chunk[i]);
  if (ctx->ev_free) cudaEventDestroy(ctx->ev_free);
  if (ctx->dz_st) cudaStreamDestroy(ctx->dz_st);
  if (ctx->ev_dz) cudaEventDestroy(ctx->ev_dz);
  if (ctx->ev_dz_done) cudaEventDestroy(ctx->ev_dz_done);
  if (ctx->h_dz) cudaFreeHost(ctx->h_dz);
  if (ctx->ev_xready) cudaEventDestroy(ctx->ev_xready);
  if (ctx->ev_xcopy) cudaEventDestroy(ctx->ev_xcopy);
  if (ctx->up_st) cudaStreamDestroy(ctx->up_st);
  delete ctx;
}

const char* fs_last_error(const fs_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t fs_launch_count(const fs_ctx* ctx) { return ctx ? ctx->launches : 0; }

int fs_profile_enable(fs_ctx* ctx, int on) {
  if (!ctx) return FS_EINVAL;
  ctx->prof_on = on != 0;
  return FS_OK;
}

int fs_profile_read(fs_ctx* ctx, double* ms, int count) {
  if (!ctx || !ms || count < 1) return FS_EINVAL;
  for (int i = 0; i < count && i < FS_PROF_STAGES; ++i) ms[i] = ctx->prof_ms[i];
  return FS_OK;
}

int fs_gram_packed(fs_ctx* ctx, int dtype, int precision, const void* S, int64_t n, int64_t m,
                   int64_t ldS, double lam, double* G_packed, void* stream) {
  int rc = check_shape(ctx, dtype, S, n, m, ldS);
  if (rc) return rc;
  if (!(lam >= 0.0) || !isfinite(lam)) return fail(ctx, FS_EINVAL, "diagonal shift must be finite and >= 0");
  if (!G_packed) return fail(ctx, FS_EINVAL, "G_packed is NULL");
  int use_tc = 0;
  if ((rc = resolve_precision(ctx, dtype, precision, S, ldS, &use_tc))) return rc;
  if ((rc = gram_impl(ctx, dtype, precision, S, n, m, ldS, lam, G_packed, (cudaStream_t)stream))) return rc;
  if (use_tc == 2) {   // F16X2 overflow -> TF32X3 (one host synchronisation)
    cudaStream_t st = (cudaStream_t)stream;
    FS_CK(cudaMemcpyAsync(ctx->h_ovf, ctx->d_ovf, sizeof(int), cudaMemcpyDeviceToHost, st), "flag d2h");
    FS_CK(cudaStreamSynchronize(st), "sync");
    if (*ctx->h_ovf & 2) {   // the sampled scales overflowed: exact row scales, F16X2 again
      FS_CK(exact_row_max(ctx, (const float*)S, n, m, ldS, st), "row max");
      rc = gram_impl(ctx, dtype, FS_PREC_F16X2, S, n, m, ldS, lam, G_packed, st);
      ctx->hint_absmax = nullptr;
      return rc;
    }
  }
  ctx->hint_absmax = nullptr;
  return FS_OK;
}

int fs_gemv_rows(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS,
                 const void* w, int wdtype, double* u, void* stream) {
  int rc = check_shape(ctx, dtype, S, n, m, ldS);
  if (rc) return rc;
  if (!w || !u) return fail(ctx, FS_EINVAL, "NULL vector");
  int l = 0;
  cudaError_t e = cudaErrorNotSupported;
  if (wdtype == FS_F64)   // exact fp64 products: the panel pass (same order as the fused solve's y)
    e = fs::gemv_rows_panel(dtype == FS_F64, S, n, m, ldS, (const double*)w, ctx->d_partials,
                            fs::gemv_rows_chunks(ctx->m_max, true) * ctx->n_max / n, u, ctx->num_sms,
                            (cudaStream_t)stream, &l);
  if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    e = fs::gemv_rows(dtype == FS_F64, S, n, m, ldS, w, wdtype == FS_F64, ctx->d_partials, u, (cudaStream_t)stream,
                      &l);
  }
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gemv_rows");
  return FS_OK;
}

int fs_unpack_lower(fs_ctx* ctx, const double* G_packed, int64_t n, double add_diag, double* W,
                    int64_t ldW, void* stream) {
  if (!ctx || !G_packed || !W || n < 1 || ldW < n) return fail(ctx, FS_EINVAL, "bad unpack arguments");
  int l = 0;
  cudaError_t e = fs::unpack_lower(G_packed, n, add_diag, W, ldW, (cudaStream_t)stream, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "unpack_lower");
  return FS_OK;
}

int fs_potrf_async(fs_ctx* ctx, double* W, int64_t n, int64_t ldW, void* stream) {
  if (!ctx || !W || n < 1 || ldW < n) return fail(ctx, FS_EINVAL, "bad potrf arguments");
  if (n > ctx->n_max) return fail(ctx, FS_ENOMEM, "n exceeds n_max");
  cudaStream_t st = (cudaStream_t)stream;
  FS_CK(cudaMemsetAsync(ctx->d_status, 0, sizeof(int64_t), st), "potrf status reset");
  int l = 0;
  cudaError_t e = fs::potrf_lower(W, n, ldW, ctx->d_status, ctx->d_potrf, st, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "potrf");
  return FS_OK;
}

int64_t fs_status_read(fs_ctx* ctx, void* stream) {
  if (!ctx) return -1;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess) return -1;
  if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
  return *ctx->h_status;
}

int fs_potrf(fs_ctx* ctx, double* W, int64_t n, int64_t ldW, int64_t* pivot, void* stream) {
  int rc = fs_potrf_async(ctx, W, n, ldW, stream);
  if (rc) return rc;
  const int64_t s = fs_status_read(ctx, stream);
  if (s < 0) return fail(ctx, FS_ECUDA, "potrf status read failed");
  if (pivot) *pivot = s > 0 ? s - 1 : -1;
  if (s > 0) return fail(ctx, FS_NOT_PD, "Gram matrix is not positive definite");
  return FS_OK;
}

int fs_trsv_pair(fs_ctx* ctx, const double* L, int64_t n, int64_t ldL, double* z, void* stream) {
  if (!ctx || !L || !z || n < 1 || ldL < n) return fail(ctx, FS_EINVAL, "bad trsv arguments");
  if (n > ctx->n_max) return fail(ctx, FS_ENOMEM, "n exceeds n_max");
  int l = 0;
  cudaError_t e = fs::invert_diag_blocks(L, n, ldL, ctx->d_potrf, (cudaStream_t)stream, &l);
  if (e == cudaSuccess) e = fs::trsv_pair(L, n, ldL, ctx->d_potrf, z, nullptr, (cudaStream_t)stream, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "trsv_pair");
  return FS_OK;
}

int fs_gemv_cols_solve(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS,
                       const double* z, const void* v, int vdtype, double lam, int accumulate,
                       double* x, void* stream) {
  int rc = check_shape(ctx, dtype, S, n, m, ldS);
  if (rc) return rc;
  if ((rc = check_lam(ctx, lam))) return rc;
  if (!z || !v || !x) return fail(ctx, FS_EINVAL, "NULL vector");
  int l = 0;
  cudaError_t e = fs::gemv_cols_solve(dtype == FS_F64, S, n, m, ldS, z, v, vdtype == FS_F64, lam,
                                      accumulate != 0, x, (cudaStream_t)stream, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gemv_cols_solve");
  return FS_OK;
}

int fs_residual_cols(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS,
                     const double* y, const double* x, const void* v, int vdtype, double lam,
                     double* r, double* sums, void* stream) {
  int rc = check_shape(ctx, dtype, S, n, m, ldS);
  if (rc) return rc;
  if (!y || !x || !v || !sums) return fail(ctx, FS_EINVAL, "NULL vector");
  int l = 0;
  cudaError_t e = fs::residual_cols(dtype == FS_F64, S, n, m, ldS, y, x, v, vdtype == FS_F64, lam, r,
                                    ctx->d_block_sums, sums, (cudaStream_t)stream, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "residual_cols");
  return FS_OK;
}

// one solve's local state of the multi-rank protocol starts clean
static void begin_solve(fs_ctx* ctx, bool empty) {
  ctx->poison_rc = 0;
  ctx->poison_msg.clear();
  ctx->empty_shard = empty;
  ctx->local_nonfinite = false;
}

static int chol_solve_impl(fs_ctx* ctx, int dtype, int precision, const void* S, int64_t n, int64_t m, int64_t ldS,
                           const void* v, double lam, double* x, fs_allreduce_fn allreduce, void* allreduce_user,
                           int flags, double refine_above, int64_t* pivot, double* out_res, void* stream,
                           const int* nonfinite = nullptr) {
  const bool multi = allreduce != nullptr;
  // an empty column shard (m < world) still joins every collective with zero contributions
  const bool empty = multi && m == 0;
  int rc = empty ? (ctx && n >= 1 && n <= ctx->n_max ? FS_OK : check_shape(ctx, dtype, S, n, 1, 1))
                 : check_shape(ctx, dtype, S, n, m, ldS);
  if (rc) return rc;
  if ((rc = check_lam(ctx, lam))) return rc;
  if (!empty && (!v || !x)) return fail(ctx, FS_EINVAL, "NULL vector");
  int use_tc = 0;
  if ((rc = resolve_precision(ctx, dtype, precision, S, ldS, &use_tc))) return rc;
  if (pivot) *pivot = -1;
  begin_solve(ctx, empty);
  if (flags & FS_FLAG_INVALID_SHARD) {
    // the caller found non-finite entries in this rank's shard: fail, on every rank together
    fail(ctx, FS_EINVAL, "score matrix and right-hand side must contain only finite entries");
    if (!multi) return FS_EINVAL;
    poison(ctx, FS_EINVAL);
    ctx->local_nonfinite = true;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int vdt = dtype;  // v has the dtype of S
  if (dtype == FS_F32 && !use_tc && !empty && !ctx->poison_rc) {
    // fp64 precision mode on fp32 scores: widen v once so every GEMV product is exact fp64
    int l = 0;
    FS_CKS(fs::widen_f32((const float*)v, m, ctx->d_v64, st, &l), "widen v");
    ctx->launches += l;
    v = ctx->d_v64;
    vdt = FS_F64;
  }
  double* u = ctx->d_packed + n * (n + 1) / 2;
  ctx->n_marks = 0;
  prof_mark(ctx, -1, st);
  // 1. partial Gram (no shift) and u = S v, packed for one all-reduce (tensor-core modes: one
  //    fused streaming pass computes u and writes the tiled copy the SYRK reads)
  if (!empty && !ctx->poison_rc) {
    NvtxRange r("fs: gram + u = S v");
    if (use_tc && vdt == FS_F32) {
      FS_STEP(gram_impl(ctx, dtype, precision, S, n, m, ldS, 0.0, ctx->d_packed, st, (const float*)v, u));
    } else {
      FS_STEP(gram_impl(ctx, dtype, precision, S, n, m, ldS, 0.0, ctx->d_packed, st));
      if (!ctx->poison_rc) FS_STEP(fs_gemv_rows(ctx, dtype, S, n, m, ldS, v, vdt, u, stream));
      prof_mark(ctx, FS_PROF_GEMV_SV, st);
    }
  }
  if ((flags & FS_FLAG_REFINE_Z) && vdt == FS_F32 && !empty && !ctx->poison_rc) {
    // z-space refinement: every x pass in exact fp64 products (the first one's fp32 rounding
    // would otherwise stay in x's component outside the row space of S, ~1e-9 of the residual)
    int l = 0;
    FS_CKS(fs::widen_f32((const float*)v, m, ctx->d_v64, st, &l), "widen v");
    ctx->launches += l;
    v = ctx->d_v64;
    vdt = FS_F64;
  }
  rc = solve_tail(ctx, dtype, S, n, m, ldS, v, vdt, lam, x, allreduce, allreduce_user, flags, refine_above, pivot,
                  out_res, st, use_tc == 2 ? ctx->d_ovf : nullptr, nonfinite);
  const bool had_hint = ctx->hint_absmax != nullptr;
  ctx->hint_absmax = nullptr;
  if (rc == kRetryTf32) {
    // some rank's sampled fp16 scales overflowed (the decision is collective): every rank
    // recomputes in F16X2 with exact row scales (no second copy of S); exact scales cannot
    // overflow, so the TF32X3 recomputation is only a last resort
    if (!had_hint) {
      if (!ctx->poison_rc && !ctx->empty_shard) FS_CKS(exact_row_max(ctx, (const float*)S, n, m, ldS, st), "row max");
      return chol_solve_impl(ctx, dtype, FS_PREC_F16X2, S, n, m, ldS, v, lam, x, allreduce, allreduce_user, flags,
                             refine_above, pivot, out_res, stream, nonfinite);
    }
    ctx->fallbacks += 1;
    return chol_solve_impl(ctx, dtype, FS_PREC_TF32X3, S, n, m, ldS, v, lam, x, allreduce, allreduce_user, flags,
                           refine_above, pivot, out_res, stream, nonfinite);
  }
  return rc;
}

int fs_chol_solve(fs_ctx* ctx, int dtype, int precision, const void* S, int64_t n, int64_t m,
                  int64_t ldS, const void* v, double lam, double* x, fs_allreduce_fn allreduce,
                  void* allreduce_user, int flags, double refine_above, int64_t* pivot,
                  double* out_res, void* stream) {
  NvtxRange range("fs_chol_solve");
  return chol_solve_impl(ctx, dtype, precision, S, n, m, ldS, v, lam, x, allreduce, allreduce_user, flags,
                         refine_above, pivot, out_res, stream);
}

int fs_chol_solve_host(fs_ctx* ctx, int dtype, int precision, const void* S_host, int64_t n, int64_t m,
                       int64_t ldS, const void* v_host, double lam, double* x_host, fs_allreduce_fn allreduce,
                       void* allreduce_user, int flags, double refine_above, int64_t* pivot,
                       double* out_res, void* stream) {
  int rc = check_shape(ctx, dtype, S_host, n, m, ldS);
  if (rc) return rc;
  if ((rc = check_lam(ctx, lam))) return rc;
  if (!v_host || !x_host) return fail(ctx, FS_EINVAL, "NULL vector");
  if (pivot) *pivot = -1;
  int use_tc = 0;
  if ((rc = resolve_precision(ctx, dtype, precision, S_host, ldS, &use_tc))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const bool multi = allreduce != nullptr;   // see solve_tail: no rank returns between collectives
  begin_solve(ctx, false);
  const size_t elem = dtype == FS_F64 ? 8 : 4;
  const int64_t per16 = 16 / (int64_t)elem;
  const int64_t ldd = (m + per16 - 1) / per16 * per16;   // device rows start on 16-byte boundaries
  const size_t need = (size_t)n * ldd * elem;
  // ---- lazy resources ----
  if (ctx->Sin_bytes < need) {
    if (ctx->d_Sin) { cudaStreamSynchronize(st); cudaFree(ctx->d_Sin); }
    ctx->d_Sin = nullptr;
    ctx->Sin_bytes = 0;
    if (cudaMalloc(&ctx->d_Sin, need) != cudaSuccess) {
      cudaGetLastError();
      ctx->d_Sin = nullptr;
      FS_STEP(fail(ctx, FS_ENOMEM, "cannot allocate the device copy of S"));
    } else {
      ctx->Sin_bytes = need;
    }
  }
  if (!ctx->d_vin && !ctx->poison_rc) {
    bool ok = cudaMalloc((void**)&ctx->d_vin, ctx->m_max * sizeof(double)) == cudaSuccess &&
              cudaMalloc((void**)&ctx->d_xin, ctx->m_max * sizeof(double)) == cudaSuccess &&
              cudaMalloc((void**)&ctx->d_flag, sizeof(int)) == cudaSuccess &&
              cudaMallocHost((void**)&ctx->h_flag, sizeof(int)) == cudaSuccess &&
              cudaStreamCreateWithFlags(&ctx->up_st, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->ev_free, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->ev_xready, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&ctx->ev_xcopy, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < fs_ctx::kMaxChunks; ++i)
      ok = cudaEventCreateWithFlags(&ctx->ev_chunk[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      FS_STEP(fail(ctx, FS_ENOMEM, "cannot allocate the host-entry buffers"));
    }
  }
  const bool direct = use_tc == 2 && f16_direct() && fs::syrk_tc_supported(ctx->d_Sin, ldd);
  if (use_tc && !direct && !ctx->poison_rc) FS_STEP(ensure_tiles(ctx, use_tc == 2));
  ctx->n_marks = 0;
  prof_mark(ctx, -1, st);
  int l = 0;
  if (!ctx->poison_rc) {
    FS_CKS(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), st), "flag reset");
    FS_CKS(cudaMemcpyAsync(ctx->d_vin, v_host, m * elem, cudaMemcpyHostToDevice, st), "v h2d");
    FS_CKS(fs::check_finite(ctx->d_vin, dtype == FS_F64, 1, m, m, ctx->d_flag, ctx->num_sms, st, &l), "check v");
    // the upload stream must not overwrite d_Sin while earlier work on `st` still reads it
    FS_CKS(cudaEventRecord(ctx->ev_free, st), "event");
    FS_CKS(cudaStreamWaitEvent(ctx->up_st, ctx->ev_free, 0), "event wait");
  }
  const int64_t hpitch = ldS * (int64_t)elem, dpitch = ldd * (int64_t)elem;
  // upload columns [c0, c1) of every row (2-D copy: n segments of (c1-c0) elements)
  auto upload = [&](int64_t c0, int64_t c1, int ev) -> cudaError_t {
    const char* src = (const char*)S_host + c0 * (int64_t)elem;
    char* dst = (char*)ctx->d_Sin + c0 * (int64_t)elem;
    cudaError_t e = (c0 == 0 && c1 == m && hpitch == dpitch)
                        ? cudaMemcpyAsync(dst, src, (size_t)n * hpitch, cudaMemcpyHostToDevice, ctx->up_st)
                        : cudaMemcpy2DAsync(dst, dpitch, src, hpitch, (c1 - c0) * elem, n, cudaMemcpyHostToDevice,
                                            ctx->up_st);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_chunk[ev], ctx->up_st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ctx->ev_chunk[ev], 0);
    return e;
  };
  const void* S = ctx->d_Sin;
  const void* v = ctx->d_vin;
  double* x = ctx->d_xin;
  ctx->early_x_host = x_host;   // finish_x starts the x download as soon as x exists
  struct EarlyReset {          // every exit path leaves the context without a pending host target
    fs_ctx* c;
    ~EarlyReset() { c->early_x_host = nullptr; c->early_x_state = 0; }
  } early_reset{ctx};
  const int* nonfinite = ctx->d_flag;
  if (ctx->poison_rc) {
    // this rank failed before the first collective: join them idle (multi-rank only)
    rc = solve_tail(ctx, dtype, S, n, m, ldd, v, dtype, lam, x, allreduce, allreduce_user, flags, refine_above,
                    pivot, out_res, st, nullptr, nullptr);
  } else if (use_tc) {
    // K-chunks of >= 32 MB (about 16, then tapering): upload columns [c0, c1) of all rows -> retile them (+ u
    // partials + finiteness) -> SYRK over their K-blocks, accumulated into the packed Gram.  The
    // transfer of chunk c+1 overlaps the kernels of chunk c; only the last chunk's share is exposed.
    double* u = ctx->d_packed + n * (n + 1) / 2;
    const int64_t CW = fs::gemv_rows_chunk_cols();
    const int64_t by_bytes = ((int64_t)(32 << 20) / (n * (int64_t)elem) + CW - 1) / CW * CW;
    const int64_t by_count = (m + 16 * CW - 1) / (16 * CW) * CW;
    const int64_t W = std::max<int64_t>(CW, std::max(by_bytes, by_count));
    // tapered schedule: full chunks while more than two remain, then halving ones, so the Gram
    // share left exposed after the last transfer is a few K-blocks instead of a full chunk
    auto next_width = [&](int64_t rest) -> int64_t {
      if (rest > 2 * W) return W;
      const int64_t w = std::max<int64_t>(CW, (rest / 2 + CW - 1) / CW * CW);
      return rest - w < CW ? rest : w;
    };
    int c = 0;
    for (int64_t c0 = 0, c1 = 0; c0 < m && !ctx->poison_rc; c0 = c1, ++c) {
      c1 = std::min(m, c0 + (c + 1 < fs_ctx::kMaxChunks ? next_width(m - c0) : m - c0));
      FS_CKS(upload(c0, c1, c % fs_ctx::kMaxChunks), "S h2d");
      // the chunk's tiles at the start of the (capped) tiled copy: a base shifted by its first
      // K-block keeps the kernels' absolute offsets; stream order keeps chunk c's SYRK ahead of
      // chunk c+1's retile
      const int64_t tcols = use_tc == 2 ? fs::kTile16Cols : fs::kTileCols;
      const size_t kbb = (size_t)fs::tiles_nb(n) * (use_tc == 2 ? 2 : 1) * fs::kTileBytes;
      uint8_t* St_c = ctx->d_St ? ctx->d_St - (ptrdiff_t)((c0 / tcols) * (int64_t)kbb) : nullptr;
      if (!direct && (size_t)((c1 - c0 + tcols - 1) / tcols) * kbb > ctx->St_bytes)   // (c0 % tcols == 0)
        FS_STEP(fail(ctx, FS_ENOMEM, "a host-entry K-chunk exceeds the tiled copy"));
      if (ctx->poison_rc) break;
      if (use_tc == 2 && direct) {
        // F16X2 direct: row scales from the first chunk's columns, then the K-range SYRK splits the
        // chunk in-kernel and accumulates u = S v
        if (c == 0)
          FS_CKS(fs::row_scales((const float*)S, n, m, ldd, ctx->d_scale, ctx->d_inv_scale, st, &l, c1), "scales");
        FS_CKS(fs::syrk_f16_direct((const float*)S, ldd, n, m, ctx->d_scale, ctx->d_inv_scale, (const float*)v,
                                  ctx->d_flag, ctx->d_partials, u, 0.0, ctx->d_packed, ctx->d_syrk_ws, ctx->num_sms,
                                  st, &l, (int)(c0 / fs::kTile16Cols),
                                  (int)((c1 + fs::kTile16Cols - 1) / fs::kTile16Cols), c > 0),
              "syrk_f16_direct");
      } else if (use_tc == 2) {
        // F16X2: row scales from the first chunk's columns, then split planes + K-range SYRK
        if (c == 0)
          FS_CKS(fs::row_scales((const float*)S, n, m, ldd, ctx->d_scale, ctx->d_inv_scale, st, &l, c1), "scales");
        FS_CKS(fs::retile16_cols((const float*)S, n, m, ldd, (const float*)v, ctx->d_partials, St_c,
                                ctx->d_scale, c0, c1, ctx->d_flag, st, &l),
              "retile16");
        FS_CKS(fs::syrk_f16(St_c, n, m, ctx->d_inv_scale, 0.0, ctx->d_packed, ctx->d_syrk_ws, ctx->num_sms, st,
                           &l, (int)(c0 / fs::kTile16Cols), (int)((c1 + fs::kTile16Cols - 1) / fs::kTile16Cols),
                           c > 0),
              "syrk_f16");
      } else {
        FS_CKS(fs::retile_cols((const float*)S, n, m, ldd, (const float*)v, ctx->d_partials, St_c, c0, c1,
                              ctx->d_flag, st, &l),
              "retile");
        FS_CKS(fs::syrk_tc(St_c, n, m, 0.0, ctx->d_packed, ctx->d_syrk_ws, ctx->num_sms, st, &l, 0, -1,
                          (int)(c0 / fs::kTileCols), (int)((c1 + fs::kTileCols - 1) / fs::kTileCols), c > 0),
              "syrk_tc");
      }
    }
    if (!(use_tc == 2 && direct) && !ctx->poison_rc) FS_CKS(fs::reduce_row_partials(ctx->d_partials, n, m, u, st, &l), "u reduce");
    ctx->launches += l;
    prof_mark(ctx, FS_PROF_GRAM, st);
    int vdt = dtype;
    if ((flags & FS_FLAG_REFINE_Z) && dtype == FS_F32 && !ctx->poison_rc) {   // exact x passes (chol_solve_impl)
      FS_CKS(fs::widen_f32((const float*)v, m, ctx->d_v64, st, &l), "widen v");
      v = ctx->d_v64;
      vdt = FS_F64;
    }
    rc = solve_tail(ctx, dtype, S, n, m, ldd, v, vdt, lam, x, allreduce, allreduce_user, flags, refine_above,
                    pivot, out_res, st, use_tc == 2 ? ctx->d_flag : nullptr, nonfinite);
    v = ctx->d_vin;
    if (rc == kRetryTf32) {   // fp16 overflow of the sampled scales: S is on the device already
      if (!ctx->poison_rc) FS_CKS(exact_row_max(ctx, (const float*)S, n, m, ldd, st), "row max");
      rc = chol_solve_impl(ctx, dtype, FS_PREC_F16X2, S, n, m, ldd, v, lam, x, allreduce, allreduce_user, flags,
                           refine_above, pivot, out_res, stream, nonfinite);
    }
  } else {
    FS_CKS(upload(0, m, 0), "S h2d");
    if (!ctx->poison_rc)
      FS_CKS(fs::check_finite(S, dtype == FS_F64, n, m, ldd, ctx->d_flag, ctx->num_sms, st, &l), "check S");
    ctx->launches += l;
    if (ctx->poison_rc)
      rc = solve_tail(ctx, dtype, S, n, m, ldd, v, dtype, lam, x, allreduce, allreduce_user, flags, refine_above,
                      pivot, out_res, st, nullptr, nullptr);
    else
      rc = chol_solve_impl(ctx, dtype, precision, S, n, m, ldd, v, lam, x, allreduce, allreduce_user, flags,
                           refine_above, pivot, out_res, stream, nonfinite);
  }
  const int early = ctx->early_x_state;
  ctx->early_x_host = nullptr;
  ctx->early_x_state = 0;
  if (early) FS_CK(cudaStreamWaitEvent(st, ctx->ev_xcopy, 0), "event wait");   // the early copy is done
  if ((rc != FS_OK && rc != FS_NOT_PD && rc != FS_EINVAL) || !ctx->d_flag || !ctx->h_flag) {
    cudaStreamSynchronize(st);
    return rc;
  }
  FS_CK(cudaMemcpyAsync(ctx->h_flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st), "flag d2h");
  if (rc == FS_OK && early != 1)
    FS_CK(cudaMemcpyAsync(x_host, x, m * sizeof(double), cudaMemcpyDeviceToHost, st), "x d2h");
  FS_CK(cudaStreamSynchronize(st), "sync");
  if (*ctx->h_flag & 1) {
    if (pivot) *pivot = -1;
    return fail(ctx, FS_EINVAL, "score matrix and right-hand side must contain only finite entries");
  }
  return rc;
}

int fs_syevj_packed(fs_ctx* ctx, const double* G_packed, int64_t n, double* w, double* U, int64_t ldU, int* sweeps,
                    void* stream) {
  if (!ctx || !G_packed || !w || !U || n < 1 || ldU < n) return fail(ctx, FS_EINVAL, "bad syevj arguments");
  if (n > ctx->n_max) return fail(ctx, FS_ENOMEM, "n exceeds n_max");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = eig_impl(ctx, G_packed, n, st);
  if (sweeps && ctx->h_info) *sweeps = ctx->h_info[0];
  if (rc) return rc;
  FS_CK(cudaMemcpyAsync(w, ctx->d_w, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "w copy");
  FS_CK(cudaMemcpy2DAsync(U, ldU * sizeof(double), ctx->d_U, n * sizeof(double), n * sizeof(double), n,
                          cudaMemcpyDeviceToDevice, st),
        "U copy");
  return FS_OK;
}

int fs_eigh_solve(fs_ctx* ctx, int dtype, int precision, const void* S, int64_t n, int64_t m, int64_t ldS,
                  const void* v, double lam, double sigma_floor, double* x, fs_allreduce_fn allreduce,
                  void* allreduce_user, int flags, int64_t* rank, double* out_res, void* stream) {
  int rc = check_shape(ctx, dtype, S, n, m, ldS);
  if (rc) return rc;
  if ((rc = check_lam(ctx, lam))) return rc;
  if (!(sigma_floor >= 0.0) || !isfinite(sigma_floor)) return fail(ctx, FS_EINVAL, "sigma_floor must be finite and >= 0");
  if (n > m) return fail(ctx, FS_EINVAL, "the eigh route requires n <= m (solvers.py:254-255)");
  if (!v || !x) return fail(ctx, FS_EINVAL, "NULL vector");
  cudaStream_t st = (cudaStream_t)stream;
  int use_tc = 0;
  if ((rc = resolve_precision(ctx, dtype, precision, S, ldS, &use_tc))) return rc;
  begin_solve(ctx, false);
  int vdt = dtype;
  const bool refine_z = (flags & FS_FLAG_REFINE_Z) != 0 && (flags & FS_FLAG_RESIDUAL) != 0 && use_tc;
  if (dtype == FS_F32 && !use_tc) {
    int l = 0;
    cudaError_t e = fs::widen_f32((const float*)v, m, ctx->d_v64, st, &l);
    ctx->launches += l;
    if (e != cudaSuccess) return cuda_fail(ctx, e, "widen v");
    v = ctx->d_v64;
    vdt = FS_F64;
  }
  double* u = ctx->d_packed + n * (n + 1) / 2;
  ctx->n_marks = 0;
  prof_mark(ctx, -1, st);
  // 1. Gram (no shift) and u = S v, packed for one all-reduce (solvers.py:257-259)
  if (use_tc && vdt == FS_F32) {
    if ((rc = gram_impl(ctx, dtype, precision, S, n, m, ldS, 0.0, ctx->d_packed, st, (const float*)v, u))) return rc;
  } else {
    if ((rc = gram_impl(ctx, dtype, precision, S, n, m, ldS, 0.0, ctx->d_packed, st))) return rc;
    if ((rc = fs_gemv_rows(ctx, dtype, S, n, m, ldS, v, vdt, u, stream))) return rc;
    prof_mark(ctx, FS_PROF_GEMV_SV, st);
  }
  if (allreduce && allreduce(ctx->d_packed, (int64_t)packed_len(n), allreduce_user, stream) != 0)
    return fail(ctx, FS_ECUDA, "allreduce of [G | u] failed");
  prof_mark(ctx, FS_PROF_ALLREDUCE, st);
  // 2. G = U diag(w) U^T, w descending (solvers.py:261-266); sigma floor (solvers.py:267-271)
  const bool had_hint = ctx->hint_absmax != nullptr;
  ctx->hint_absmax = nullptr;
  // the split Grams carry ~2^-22 ||G|| of error: a Jacobi backward error of 1e-8 ||G|| is below
  // it (one sweep fewer at the headline, 16.0 -> 14.6 ms); z-space refinement takes x the rest
  // of the way.  Exact-product (fp64) Grams keep 1e-14.
  if ((rc = eig_impl(ctx, ctx->d_packed, n, st, use_tc ? 1e-8 : 1e-14))) return rc;
  if (use_tc == 2) {   // an F16X2 overflow shows up here already (the eigh path synchronises)
    FS_CK(cudaMemcpyAsync(ctx->h_ovf, ctx->d_ovf, sizeof(int), cudaMemcpyDeviceToHost, st), "flag d2h");
    FS_CK(cudaStreamSynchronize(st), "sync");
    if (*ctx->h_ovf & 2) {   // sampled scales overflowed: exact row scales (TF32X3 only as a last resort)
      if (!had_hint) FS_CK(exact_row_max(ctx, (const float*)S, n, m, ldS, st), "row max");
      else ctx->fallbacks += 1;
      return fs_eigh_solve(ctx, dtype, had_hint ? FS_PREC_TF32X3 : FS_PREC_F16X2, S, n, m, ldS, v, lam, sigma_floor, x,
                           allreduce, allreduce_user, flags, rank, out_res, stream);
    }
  }
  prof_mark(ctx, FS_PROF_POTRF, st);
  const double s0 = sqrt(std::max(ctx->h_w[0], 0.0));
  int64_t r = 0;
  while (r < n && sqrt(std::max(ctx->h_w[r], 0.0)) > sigma_floor * s0) ++r;
  if (rank) *rank = r;
  // 3. z = U_r (w_r + lam)^-1 U_r^T u  ==  the V (s^2+lam)^-1 V^T v part of solvers.py:315-317
  //    rewritten through S^T: x = (v - S^T z') / lam with z' = -(...); here z = U_r diag(...) U_r^T u
  //    and x = (v - S^T z)/lam follows from (v - V V^T v)/lam + V (s^2+lam)^-1 V^T v.
  {
    int l = 0;
    cudaError_t e = fs::eig_apply(ctx->d_U, n, n, r, u, ctx->d_w, lam, ctx->d_t, ctx->d_z, st, &l);
    ctx->launches += l;
    if (e != cudaSuccess) return cuda_fail(ctx, e, "eig_apply");
  }
  prof_mark(ctx, FS_PROF_TRSV, st);
  FS_CK(cudaMemsetAsync(ctx->d_status, 0, sizeof(int64_t), st), "status reset");
  // 4. x and the residual against S (solvers.py:318-322 -> _finish).  The fp32-split modes may
  //    refine z on the kept eigen-subspace like the chol route (the reference's eigh route has
  //    no refinement; its fp64 result is what the refined one converges to): exact fp64 x passes
  int fl = flags & FS_FLAG_RESIDUAL;
  if (refine_z) {
    fl |= flags & (FS_FLAG_REFINE_Z | (0xFF << 8));
    if (vdt == FS_F32) {
      int l = 0;
      cudaError_t e = fs::widen_f32((const float*)v, m, ctx->d_v64, st, &l);
      ctx->launches += l;
      if (e != cudaSuccess) return cuda_fail(ctx, e, "widen v");
      v = ctx->d_v64;
      vdt = FS_F64;
    }
  }
  int64_t piv = -1;
  ctx->z_solver = 1;
  ctx->eig_rank = r;
  rc = finish_x(ctx, dtype, S, n, m, ldS, v, vdt, lam, x, allreduce, allreduce_user, fl, 1e-10 /* solvers.py:43 */, &piv,
                out_res, st, nullptr);
  ctx->z_solver = 0;
  return rc;
}

int fs_embed_complex(fs_ctx* ctx, int kind, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS, void* out,
                     int64_t ldo, void* stream) {
  if (!ctx || !S || !out || n < 1 || m < 1 || ldS < m || (kind != 0 && kind != 1))
    return fail(ctx, FS_EINVAL, "bad embed arguments");
  if (dtype != FS_F32 && dtype != FS_F64) return fail(ctx, FS_EINVAL, "dtype must be FS_F32 or FS_F64");
  if (ldo < (kind == 0 ? m : 2 * m)) return fail(ctx, FS_EINVAL, "ldo too small");
  int l = 0;
  cudaError_t e = fs::embed_complex(dtype == FS_F64, S, n, m, ldS, kind, out, ldo, ctx->num_sms, (cudaStream_t)stream, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "embed_complex");
  return FS_OK;
}

int fs_hermitian_gram(fs_ctx* ctx, const double* G2_packed, int64_t n, double lam, double* W, int64_t ldW,
                      void* stream) {
  if (!ctx || !G2_packed || !W || n < 1 || ldW < n) return fail(ctx, FS_EINVAL, "bad hermitian_gram arguments");
  if (!(lam >= 0.0) || !isfinite(lam)) return fail(ctx, FS_EINVAL, "diagonal shift must be finite and >= 0");
  int l = 0;
  cudaError_t e = fs::hermitian_gram(G2_packed, n, lam, W, ldW, ctx->num_sms, (cudaStream_t)stream, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "hermitian_gram");
  return FS_OK;
}

static int apply_rows_impl(fs_ctx* ctx, int dtype, const double* T, int64_t r, int64_t n, int64_t ldT, const void* X,
                           int64_t m, int64_t ldX, double* Y, int64_t ldY, void* stream, bool lower) {
  if (!ctx) return FS_EINVAL;
  if (dtype != FS_F32 && dtype != FS_F64) return fail(ctx, FS_EINVAL, "dtype must be FS_F32 or FS_F64");
  if (!T || !X || !Y || r < 1 || n < 1 || m < 1 || ldT < n || ldX < m || ldY < m)
    return fail(ctx, FS_EINVAL, "bad apply_rows arguments");
  int l = 0;
  cudaError_t e = fs::apply_rows(dtype == FS_F64, T, r, n, ldT, X, m, ldX, Y, ldY, (cudaStream_t)stream, &l, lower);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "apply_rows");
  return FS_OK;
}

int fs_apply_rows(fs_ctx* ctx, int dtype, const double* T, int64_t r, int64_t n, int64_t ldT, const void* X,
                  int64_t m, int64_t ldX, double* Y, int64_t ldY, void* stream) {
  return apply_rows_impl(ctx, dtype, T, r, n, ldT, X, m, ldX, Y, ldY, stream, false);
}

int fs_apply_rows_lower(fs_ctx* ctx, int dtype, const double* T, int64_t r, int64_t n, int64_t ldT, const void* X,
                        int64_t m, int64_t ldX, double* Y, int64_t ldY, void* stream) {
  return apply_rows_impl(ctx, dtype, T, r, n, ldT, X, m, ldX, Y, ldY, stream, true);
}

int fs_heevj_packed(fs_ctx* ctx, const double* G2_packed, int64_t n, double* w, double* U, int64_t ldU, int* sweeps,
                    void* stream) {
  if (!ctx || !G2_packed || !w || !U || n < 1 || ldU != n) return fail(ctx, FS_EINVAL, "bad heevj arguments");
  if (2 * n > ctx->n_max) return fail(ctx, FS_ENOMEM, "2n exceeds n_max");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_svd(ctx, 2 * n);
  if (rc) return rc;
  double* R = (double*)ctx->d_svd;                       // packed rho(G): n (2n + 1) doubles
  double* scratch = R + n * (2 * n + 1);                 // 2n doubles (extraction candidate)
  int* kept = (int*)(scratch + 2 * n);
  int l = 0;
  cudaError_t e = fs::rho_gram(G2_packed, n, R, ctx->num_sms, st, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "rho_gram");
  if ((rc = eig_impl(ctx, R, 2 * n, st))) {
    if (sweeps && ctx->h_info) *sweeps = ctx->h_info[0];
    return rc;
  }
  if (sweeps) *sweeps = ctx->h_info[0];
  // clusters: eigenvalues of rho(G) within 1e-9 |w|_max of their neighbour
  const double wmax = std::max(fabs(ctx->h_w[0]), fabs(ctx->h_w[2 * n - 1]));
  l = 0;
  e = fs::herm_extract(ctx->d_U, ctx->d_w, n, 1e-9 * std::max(wmax, 1e-300), U, w, kept, scratch, st, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "herm_extract");
  FS_CK(cudaMemcpyAsync(ctx->h_info, kept, sizeof(int), cudaMemcpyDeviceToHost, st), "kept d2h");
  FS_CK(cudaStreamSynchronize(st), "sync");
  if (ctx->h_info[0] != n) return fail(ctx, FS_ENOCONV, "Hermitian eigenvector extraction incomplete");
  return FS_OK;
}

int fs_tri_inverse(fs_ctx* ctx, const double* L, int64_t n, int64_t ldL, double* Linv, int64_t ldo, void* stream) {
  if (!ctx || !L || !Linv || n < 1 || ldL < n || ldo < n) return fail(ctx, FS_EINVAL, "bad tri_inverse arguments");
  int rc = ensure_svd(ctx, n);
  if (rc) return rc;
  int l = 0;
  cudaError_t e = fs::tri_inverse(L, n, ldL, Linv, ldo, (double*)ctx->d_svd, ctx->num_sms, (cudaStream_t)stream, &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "tri_inverse");
  return FS_OK;
}

int fs_jacobi_svd(fs_ctx* ctx, const double* A, int64_t n, int64_t lda, double* sigma, double* U, int64_t ldu,
                  double* Zt, int64_t ldz, int* sweeps, void* stream) {
  if (!ctx || !A || !sigma || !U || !Zt || n < 1 || lda < n || ldu < n || ldz < n)
    return fail(ctx, FS_EINVAL, "bad jacobi_svd arguments");
  if (n > 16384) return fail(ctx, FS_EUNSUPPORTED, "the Jacobi SVD supports n <= 16384");
  int rc = ensure_svd(ctx, n);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  // rows orthogonal to sqrt(n) u (LAPACK dgesvj's default): the factor solve amplifies the
  // singular vectors' error by sigma^2/lam (n u left the headline's full route at rel_residual
  // 4.5e-8; sqrt(n) u: 8.6e-9, +7 ms of 570)
  const double tol = std::max(1e-15, std::sqrt((double)n) * 1.1102230246251565e-16);
  int l = 0;
  cudaError_t e = fs::jacobi_svd(A, n, lda, sigma, U, ldu, Zt, ldz, 60, tol, ctx->d_svd, ctx->num_sms, ctx->d_info, st,
                                 &l);
  ctx->launches += l;
  if (e != cudaSuccess) return cuda_fail(ctx, e, "jacobi_svd");
  FS_CK(cudaMemcpyAsync(ctx->h_info, ctx->d_info, 2 * sizeof(int), cudaMemcpyDeviceToHost, st), "info d2h");
  FS_CK(cudaStreamSynchronize(st), "sync");
  if (sweeps) *sweeps = ctx->h_info[0];
  if (ctx->h_info[1]) return fail(ctx, FS_ENOCONV, "SVD did not converge");
  return FS_OK;
}

int fs_factor_solve(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS, const void* v,
                    double lam, const double* U, int64_t ldU, const double* w, int64_t r, double* x, int flags,
                    double* out_res, void* stream) {
  int rc = check_shape(ctx, dtype, S, n, m, ldS);
  if (rc) return rc;
  if ((rc = check_lam(ctx, lam))) return rc;
  if (!v || !x || (r > 0 && (!U || !w)) || r < 0 || r > n || ldU < r) return fail(ctx, FS_EINVAL, "bad factor_solve arguments");
  cudaStream_t st = (cudaStream_t)stream;
  begin_solve(ctx, false);
  int vdt = dtype;
  if (dtype == FS_F32) {   // exact fp64 GEMV products on this route
    int l = 0;
    cudaError_t e = fs::widen_f32((const float*)v, m, ctx->d_v64, st, &l);
    ctx->launches += l;
    if (e != cudaSuccess) return cuda_fail(ctx, e, "widen v");
    v = ctx->d_v64;
    vdt = FS_F64;
  }
  ctx->n_marks = 0;
  double* u = ctx->d_packed + n * (n + 1) / 2;
  if ((rc = fs_gemv_rows(ctx, dtype, S, n, m, ldS, v, vdt, u, stream))) return rc;
  if (!ctx->d_t && cudaMalloc((void**)&ctx->d_t, (size_t)ctx->n_max * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, FS_ENOMEM, "cannot allocate the factor-solve scratch");
  }
  {
    int l = 0;
    cudaError_t e = fs::eig_apply(U, ldU, n, r, u, w, lam, ctx->d_t, ctx->d_z, st, &l);
    ctx->launches += l;
    if (e != cudaSuccess) return cuda_fail(ctx, e, "factor apply");
  }
  FS_CK(cudaMemsetAsync(ctx->d_status, 0, sizeof(int64_t), st), "status reset");
  int64_t piv = -1;
  return finish_x(ctx, dtype, S, n, m, ldS, v, vdt, lam, x, nullptr, nullptr, flags & FS_FLAG_RESIDUAL, 0.0, &piv,
                  out_res, st, nullptr);
}

int fs_row_absmax(int dtype, const void* a, int64_t rows, int64_t cols, int64_t ld, float* out, void* stream) {
  if (!a || !out || rows < 1 || cols < 0 || ld < cols || (dtype != FS_F32 && dtype != FS_F64)) return FS_EINVAL;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return FS_ECUDA;
  struct Flag { int* d = nullptr; int* h = nullptr; };
  static Flag flags[64];
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) return FS_EINVAL;
  Flag& f = flags[dev];
  if (!f.d && (cudaMalloc((void**)&f.d, sizeof(int)) != cudaSuccess ||
               cudaMallocHost((void**)&f.h, sizeof(int)) != cudaSuccess))
    return FS_ENOMEM;
  cudaStream_t st = (cudaStream_t)stream;
  int l = 0;
  if (cudaMemsetAsync(f.d, 0, sizeof(int), st) != cudaSuccess ||
      cudaMemsetAsync(out, 0, rows * sizeof(float), st) != cudaSuccess ||
      (cols > 0 && fs::check_finite(a, dtype == FS_F64, rows, cols, ld, f.d, sms, st, &l, (unsigned*)out) != cudaSuccess) ||
      cudaMemcpyAsync(f.h, f.d, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return FS_ECUDA;
  return (*f.h & 1) ? FS_EINVAL : FS_OK;
}

int fs_set_row_absmax(fs_ctx* ctx, const float* row_absmax, int64_t n) {
  if (!ctx || n < 0) return FS_EINVAL;
  ctx->hint_absmax = row_absmax;
  ctx->hint_n = row_absmax ? n : 0;
  return FS_OK;
}

int64_t fs_fallback_count(const fs_ctx* ctx) { return ctx ? ctx->fallbacks : 0; }

int fs_gram_splits(const fs_ctx* ctx, int64_t n, int64_t m, int precision) {
  if (!ctx || n < 1 || m < 1) return -1;
  if (precision != FS_PREC_FP64) return -1;
  return fs::syrk_dmma_splits(n, m, ctx->num_sms, ctx->syrk_bytes);
}

int fs_all_finite(int dtype, const void* a, int64_t rows, int64_t cols, int64_t ld, void* stream) {
  if (!a || rows < 0 || cols < 0 || ld < cols || (dtype != FS_F32 && dtype != FS_F64)) return FS_EINVAL;
  if (rows == 0 || cols == 0) return FS_OK;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return FS_ECUDA;
  // one flag word per device (device int + page-locked host copy), created on first use
  struct Flag { int* d = nullptr; int* h = nullptr; };
  static Flag flags[64];
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) return FS_EINVAL;
  Flag& f = flags[dev];
  if (!f.d && (cudaMalloc((void**)&f.d, sizeof(int)) != cudaSuccess ||
               cudaMallocHost((void**)&f.h, sizeof(int)) != cudaSuccess))
    return FS_ENOMEM;
  cudaStream_t st = (cudaStream_t)stream;
  int l = 0;
  if (cudaMemsetAsync(f.d, 0, sizeof(int), st) != cudaSuccess ||
      fs::check_finite(a, dtype == FS_F64, rows, cols, ld, f.d, sms, st, &l) != cudaSuccess ||
      cudaMemcpyAsync(f.h, f.d, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return FS_ECUDA;
  return (*f.h & 1) ? FS_EINVAL : FS_OK;
}

}  // extern "C"
