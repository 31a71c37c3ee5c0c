/*
 * fs.h — C ABI of the B200-native damped-Fisher Cholesky solve.
 *
 * Solves (S^T S + lam I) x = v for a wide score matrix S (n x m, one sample per
 * row, row-major, leading dimension ldS >= m) by the paper's Algorithm 1:
 *   W = S S^T + lam I  ->  L = chol(W)  ->  z = L^-T L^-1 (S v)  ->  x = (v - S^T z) / lam
 *
 * Every pointer argument named S, v, x, W, L, u, z, y, r is a DEVICE pointer;
 * every call is ordered on the given CUDA stream (cudaStream_t passed as void*,
 * NULL = legacy default stream).  Device memory: fs_ctx_create allocates every
 * workspace of the fp64 chol path; a mode's larger workspaces are allocated by the
 * context on the FIRST call that needs them and kept for later calls (the tensor-core
 * modes' tiled copy of S, capped at 16 GB; the eigh route's Jacobi buffers; the svd
 * route's scratch; the host entry's device copy of S) — a caller that must not
 * allocate inside a timed or captured region warms the context up with one call
 * first.  Plain C types only: no torch, no C++ in the signatures.
 *
 * This ABI replaces the numpy/scipy calls of the reference package
 * (/root/reference/pkg/src/fisher_solve/, cited per entry point below).  The
 * Python mirror of the reference's public API (solve_chol, solve_svd_eigh,
 * solve_svd_direct, gram, residual, ...) lives in paper_2310_17556_b200/ and
 * binds these symbols with ctypes; see INTEGRATION.md.
 */
#ifndef FS_H_
#define FS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FS_OK = 0,
  FS_EINVAL = 1,      /* bad argument -> Python ValueError (core.py:99-119)            */
  FS_NOT_PD = 2,      /* Cholesky breakdown -> FactorizationError(pivot) (solvers.py:82-87) */
  FS_ECUDA = 3,       /* CUDA runtime/driver error                                      */
  FS_ENOMEM = 4,      /* problem larger than the context was created for               */
  FS_EUNSUPPORTED = 5, /* e.g. precision mode not available for this dtype             */
  FS_ENOCONV = 6       /* eigendecomposition did not converge (solvers.py:262-263)       */
} fs_status;

typedef enum { FS_F32 = 0, FS_F64 = 1 } fs_dtype;

/* How the Gram product S S^T is computed (the only dense contraction). */
typedef enum {
  FS_PREC_FP64 = 0,   /* exact-product fp64 FMA (the reference's arithmetic)            */
  FS_PREC_TF32X3 = 1, /* fp32 input, tcgen05 kind::tf32, hi*hi + hi*lo + lo*hi, fp64 drain */
  FS_PREC_AUTO = 2,   /* FP64 for fp64 input, F16X2 for fp32 input                      */
  FS_PREC_F16X2 = 3   /* fp32 input split per row-scaled element into two fp16 planes
                         (22 significant bits), tcgen05 kind::f16 hi*hi + hi*lo + lo*hi,
                         fp64 drain; row scales exact (fs_set_row_absmax) or sampled, an
                         overflow of sampled scales recomputes with exact ones (below)     */
} fs_precision;

/* Host-supplied sum-all-reduce over ranks of `count` doubles in device memory,
 * in place, ordered on `stream`.  NULL = single rank.  Returns 0 on success. */
typedef int (*fs_allreduce_fn)(double* buf, int64_t count, void* user, void* stream);

typedef struct fs_ctx fs_ctx;

/* Version string "fisher-b200 <semver> sm_100a". */
const char* fs_version(void);

/* Create a context on `device` able to solve problems with n <= n_max and
 * local column count m <= m_max.  Owns every device workspace (Gram partials,
 * W/L, GEMV partials, status word).  Replaces nothing in the reference (numpy
 * allocates per call); it is the B200 analogue of CholWorkspace (solvers.py:57-71). */
int fs_ctx_create(fs_ctx** out, int device, int64_t n_max, int64_t m_max);
void fs_ctx_destroy(fs_ctx* ctx);
const char* fs_last_error(const fs_ctx* ctx);
/* Device bytes one solve of (n, m) in (dtype, precision) touches besides S, v, x
 * (feeds WorkspaceMeter, core.py:63-96; a context may own more to serve any smaller problem).
 * Not counted: the tensor-core modes' re-laid-out copy of S itself (F16X2 and TF32X3: 4 n m
 * bytes, capped at 16 GB with a K-chunked Gram beyond; allocated on first use of that mode,
 * sized for the context's n_max x m_max). */
size_t fs_workspace_bytes(int64_t n, int64_t m, int dtype, int precision);
/* Number of kernels this context launched since creation (bench evidence). */
int64_t fs_launch_count(const fs_ctx* ctx);

/* Stage timing of fs_chol_solve with CUDA events on the solve stream (no extra syncs).
 * fs_profile_read fills ms[stage] for the most recent solve, stages in this order: */
#define FS_PROF_GRAM 0       /* S S^T (tcgen05 / fp64 SYRK + split-K reduce)   */
#define FS_PROF_GEMV_SV 1    /* u = S v                                         */
#define FS_PROF_ALLREDUCE 2  /* caller's all-reduce of [W | u] (0 for one rank) */
#define FS_PROF_POTRF 3      /* unpack + lam + Cholesky                         */
#define FS_PROF_TRSV 4       /* z = L^-T L^-1 u                                 */
#define FS_PROF_GEMV_STZ 5   /* x = (v - S^T z) / lam                           */
#define FS_PROF_RESIDUAL 6   /* y = S x, r = S^T y + lam x - v, norms (+ x-space refinement) */
#define FS_PROF_REFINE 7     /* z-space refinement steps (FS_FLAG_REFINE_Z)      */
#define FS_PROF_STAGES 8
int fs_profile_enable(fs_ctx* ctx, int on);
int fs_profile_read(fs_ctx* ctx, double* ms, int count);

/* ---- stage entry points (parity tests, ncu isolation, multi-rank drivers) ---- */

/* Gram: packed-lower G[i(i+1)/2 + j] = sum_k S[i,k] S[j,k] (+ lam on i == j), fp64.
 * Replaces core.py:284-289 (numpy A @ A.T -> dsyrk, symmetrize, diagonal shift). */
int fs_gram_packed(fs_ctx* ctx, int dtype, int precision, const void* S, int64_t n, int64_t m,
                   int64_t ldS, double lam, double* G_packed, void* stream);

/* Row GEMV: u[i] = sum_k S[i,k] w[k], fp64 accumulation, w of type `wdtype`.
 * Replaces solvers.py:110 (t1 = A @ b) and core.py:297 (A @ x). */
int fs_gemv_rows(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS,
                 const void* w, int wdtype, double* u, void* stream);

/* Unpack a packed lower Gram into a full row-major n x n matrix (upper zeroed). */
int fs_unpack_lower(fs_ctx* ctx, const double* G_packed, int64_t n, double add_diag, double* W,
                    int64_t ldW, void* stream);

/* In-place lower Cholesky of W (row-major, lower triangle read, upper left zero).
 * Synchronizes `stream`.  On breakdown returns FS_NOT_PD and *pivot = 0-based index
 * of the first non-positive/NaN pivot (LAPACK info-1).  Replaces solvers.py:74-90 (dpotrf). */
int fs_potrf(fs_ctx* ctx, double* W, int64_t n, int64_t ldW, int64_t* pivot, void* stream);
/* Asynchronous variant: leaves the status word on the device (read via fs_status_read). */
int fs_potrf_async(fs_ctx* ctx, double* W, int64_t n, int64_t ldW, void* stream);
/* Synchronizes `stream` and returns the device status: 0 ok, else pivot+1. */
int64_t fs_status_read(fs_ctx* ctx, void* stream);

/* In place: z <- L^-T L^-1 z.  Replaces solvers.py:111 and :114 (two dtrtrs). */
int fs_trsv_pair(fs_ctx* ctx, const double* L, int64_t n, int64_t ldL, double* z, void* stream);

/* Column GEMV + epilogue: x[k] = (x_prev[k] if accumulate) + (v[k] - sum_i z[i] S[i,k]) / lam.
 * Replaces solvers.py:122-126 (w = t3 @ A; x = (b - w)/lam) and the refinement x += d (:188). */
int fs_gemv_cols_solve(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS,
                       const double* z, const void* v, int vdtype, double lam, int accumulate,
                       double* x, void* stream);

/* Residual tail: r[k] = sum_i y[i] S[i,k] + lam x[k] - v[k] (y = S x), and
 * sums[0] += ||r||^2, sums[1] += ||v||^2 (deterministic, fp64).  r may be NULL.
 * Replaces core.py:297 ((A@x)@A + lam*x) and core.py:319-321 (norms). */
int fs_residual_cols(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS,
                     const double* y, const double* x, const void* v, int vdtype, double lam,
                     double* r, double* sums, void* stream);

/* ---- one-shot solve (the drop-in for solvers.py:151-206) ----
 * S, v: device, this rank's column shard.  x: device fp64 out (length m).
 * allreduce: NULL for one rank, else called on [G_packed | u], y and the norm pair.
 * flags: bit0 = compute residual diagnostics, bit1 = allow the reference's one-step
 * refinement (solvers.py:183-194) when rel_residual > refine_above.
 * out_res: host double[2] = {abs_residual, rel_residual} (if bit0).  Synchronizes. */
#define FS_FLAG_RESIDUAL 1
#define FS_FLAG_REFINE 2
/* iterative refinement: up to k correction steps with the same factor while
 * rel_residual > refine_above and each step at least halves it; k = 1 is the reference rule */
#define FS_FLAG_REFINE_STEPS(k) (FS_FLAG_REFINE | (((k) & 0xFF) << 8))
/* z-space refinement (the fp32-split modes; needs FS_FLAG_RESIDUAL): up to k steps of
 * z += W~^-1 (S v - W z) on the n x n system, the residual read off the fused x + y pass
 * (lam (y - z) = S v - W z), each step one TRSV pair and one fused pass over S.  Contracts by
 * ~2^-21 kappa(W) per step whatever sigma_max^2/lam is (the x-space scheme contracts by
 * ~2^-21 sigma_max^2/lam and stalls once that nears 1).  Takes precedence over FS_FLAG_REFINE. */
#define FS_FLAG_REFINE_Z 4
#define FS_FLAG_REFINE_Z_STEPS(k) (FS_FLAG_REFINE_Z | (((k) & 0xFF) << 8))
/* multi-rank: the caller's validation found non-finite entries in this rank's shard.  The rank
 * still joins every collective (contributing zeros) and every rank returns FS_EINVAL together;
 * with no all-reduce callback the call just returns FS_EINVAL.  More generally, with a callback
 * no rank returns between two all-reduces: a rank whose local step fails joins the remaining
 * collectives idle and the failure reaches every rank through a status slot of the norms
 * all-reduce (all return an error together: the failing rank its own status, the others
 * FS_ECUDA, or FS_EINVAL for a peer's non-finite input).  A zero-column shard (m = 0, S / v / x
 * may be NULL) is valid with a callback: it contributes nothing. */
#define FS_FLAG_INVALID_SHARD 0x10000
int fs_chol_solve(fs_ctx* ctx, int dtype, int precision, const void* S, int64_t n, int64_t m,
                  int64_t ldS, const void* v, double lam, double* x, fs_allreduce_fn allreduce,
                  void* allreduce_user, int flags, double refine_above, int64_t* pivot,
                  double* out_res, void* stream);

/* ---- one-shot solve from HOST buffers (the same call with S, v, x in host memory) ----
 * What a numpy caller of solvers.py:197 solve_chol(system) hands over: S (n x m, leading
 * dimension ldS, row-major), v (length m, S's dtype) and x (fp64 out) in host memory —
 * page-locked for full overlap.  S is uploaded in column chunks (>= 32 MB, about 16; 2-D
 * copies of all rows) on a second stream; the Gram and u = S v of each chunk's K range run
 * while the next chunk is in flight, so the transfer hides all but the last chunk's share.  Non-finite entries in S or v are detected on the device
 * and return FS_EINVAL (core.py:108-119 rejects them).  The last chunks taper (halving widths)
 * so little Gram work is left after the final transfer, and x is downloaded while the residual
 * pass runs; unless FS_OK is returned the contents of x are unspecified.  Synchronizes. */
int fs_chol_solve_host(fs_ctx* ctx, int dtype, int precision, const void* S_host, int64_t n, int64_t m,
                       int64_t ldS, const void* v_host, double lam, double* x_host, fs_allreduce_fn allreduce,
                       void* allreduce_user, int flags, double refine_above, int64_t* pivot,
                       double* out_res, void* stream);

/* ---- eigh comparison route (solvers.py:243-277, :294-354) ----
 * fs_syevj_packed: eigenpairs of a packed lower symmetric fp64 matrix (device): w (n) descending,
 * U (n x n, leading dimension ldU, column j <-> w[j]); parallel Jacobi on the GPU (replaces
 * np.linalg.eigh -> dsyevd).  n <= 16384.  *sweeps = Jacobi sweeps run.  Synchronizes.
 * fs_eigh_solve: solve_svd_eigh — Gram (precision as fs_chol_solve), eigh, singular values
 * floored at sigma_floor * sigma_max (*rank = kept count), x from the kept eigenpairs, residual
 * against S (flags: FS_FLAG_RESIDUAL; with it, FS_FLAG_REFINE_Z_STEPS(k) in the fp32-split
 * precisions refines z with the kept-eigenpair apply as the correction solve — the reference's
 * route has no refinement, the refined x converges to its fp64 result; FS_FLAG_REFINE is
 * ignored).  Synchronizes. */
int fs_syevj_packed(fs_ctx* ctx, const double* G_packed, int64_t n, double* w, double* U, int64_t ldU, int* sweeps,
                    void* stream);
/* fs_heevj_packed: eigenpairs of G = S S^H (complex scores; solvers.py:258-266 with A.conj().T)
 * from G2_packed, the packed Gram of [Re S; Im S] (2n rows): the Jacobi eigensolver runs on the
 * real 2n x 2n representation [[Re G, -Im G], [Im G, Re G]] (each eigenvalue twice) and one
 * eigenvector per complex direction is extracted; w (n) descending, U (n x n, interleaved
 * complex, ldU = n, column j <-> w[j]).  The context needs n_max >= 2n.  Synchronizes. */
int fs_heevj_packed(fs_ctx* ctx, const double* G2_packed, int64_t n, double* w, double* U, int64_t ldU, int* sweeps,
                    void* stream);
int fs_eigh_solve(fs_ctx* ctx, int dtype, int precision, const void* S, int64_t n, int64_t m, int64_t ldS,
                  const void* v, double lam, double sigma_floor, double* x, fs_allreduce_fn allreduce,
                  void* allreduce_user, int flags, int64_t* rank, double* out_res, void* stream);

/* ---- complex scores (solvers.py:209-240) ----
 * S: device, n x m complex (interleaved re, im of `dtype`; ldS in complex elements).
 * kind 0: out = [Re S; Im S] (2n x m) — solve_realpart's C (sr.py:61-70), C^T C = Re[S^H S].
 * kind 1: out = [[Re S, -Im S], [Im S, Re S]] (2n x 2m) — the real representation under which
 *         solve_chol_hermitian's (S^H S + lam I) x = v is the plain system on [Re x; Im x].
 * out: device, real `dtype`, leading dimension ldo.  The caller then runs fs_chol_solve. */
int fs_embed_complex(fs_ctx* ctx, int kind, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS, void* out,
                     int64_t ldo, void* stream);

/* W = S S^H + lam I for complex S (core.py:279-290): G2_packed is the packed lower Gram of the
 * kind-0 embedding [Re S; Im S] (2n rows, from fs_embed_complex + fs_gram_packed with shift 0);
 * W is n x n complex (interleaved re, im doubles, leading dimension ldW in complex elements),
 * exactly Hermitian, lam added on the diagonal. */
int fs_hermitian_gram(fs_ctx* ctx, const double* G2_packed, int64_t n, double lam, double* W, int64_t ldW,
                      void* stream);

/* Y = T X (fp64 tensor cores, exact fp64 products): T r x n fp64 (row-major, ldT), X n x m in the
 * score layout (row-major, ldX, dtype fp32/fp64), Y r x m fp64 (row-major, ldY).  The factor
 * products of the comparison routes: thin_svd_eigh's V^T = (U / sigma)^T S (replaces
 * solvers.py:272-276, A.T @ B -> dgemm) and the svd route's Q^T = L^-1 S, V^T = W^T Q^T. */
int fs_apply_rows(fs_ctx* ctx, int dtype, const double* T, int64_t r, int64_t n, int64_t ldT, const void* X,
                  int64_t m, int64_t ldX, double* Y, int64_t ldY, void* stream);
/* The same with T lower triangular (its strictly upper part is never read: every row tile stops
 * its contraction at its last row, ~half the products): the CholeskyQR steps' Q^T = L^-1 X and
 * the triangular factor products. */
int fs_apply_rows_lower(fs_ctx* ctx, int dtype, const double* T, int64_t r, int64_t n, int64_t ldT, const void* X,
                        int64_t m, int64_t ldX, double* Y, int64_t ldY, void* stream);

/* ---- direct-SVD comparison route ("svda", solvers.py:280-291, :357-364) ----
 * The reference calls dgesdd on S.  The GPU route: shifted CholeskyQR3 of S^T (fs_gram_packed in
 * FP64 on S and on Q^T, fs_potrf, fs_tri_inverse, fs_apply_rows) gives S = L Q^T; the one-sided
 * Jacobi SVD of the n x n factor L = W diag(sigma) Z^T gives S = W diag(sigma) (Q Z)^T.
 * fs_tri_inverse: Linv = L^-1 for a lower-triangular L (row-major; Linv's upper triangle zero).
 * fs_jacobi_svd: A (n x n, row-major) = U diag(sigma) Zt with sigma descending (>= 0), U and Zt
 *   n x n row-major (U's column j and Zt's row j belong to sigma[j]); works on A's columns, so
 *   the condition number is not squared.  Synchronizes; FS_ENOCONV if not converged.
 * fs_factor_solve: the solve from left factors, x = (v - S^T z)/lam with z = U_r diag(1/(w + lam))
 *   U_r^T (S v) (U n x r, ldU; w length r, e.g. sigma^2) — equal to solvers.py:315-317's
 *   V (sigma^2+lam)^-1 V^T v + (v - V V^T v)/lam for V = S^T U diag(1/sigma), without forming V
 *   or dividing by sigma; flags: FS_FLAG_RESIDUAL (residual against S).  Synchronizes. */
int fs_tri_inverse(fs_ctx* ctx, const double* L, int64_t n, int64_t ldL, double* Linv, int64_t ldo, void* stream);
int fs_jacobi_svd(fs_ctx* ctx, const double* A, int64_t n, int64_t lda, double* sigma, double* U, int64_t ldu,
                  double* Zt, int64_t ldz, int* sweeps, void* stream);
int fs_factor_solve(fs_ctx* ctx, int dtype, const void* S, int64_t n, int64_t m, int64_t ldS, const void* v,
                    double lam, const double* U, int64_t ldU, const double* w, int64_t r, double* x, int flags,
                    double* out_res, void* stream);

/* ---- F16X2 row scales ----
 * fs_row_absmax: out[i] = max_j |a[i, j]| (float, device, `rows` entries) in one streaming pass,
 *   FS_EINVAL when an entry is not finite (so it doubles as the construction-time validation of
 *   core.py:108-119).  Context-free; synchronizes.
 * fs_set_row_absmax: hand those maxima to the next F16X2 Gram / solve on this context (device
 *   pointer, valid until that call returns; consumed by it).  With exact maxima every row is
 *   scaled to max |S_i| 2^k in [2^14, 2^15): no fp16 overflow is possible.  Without them the
 *   scale comes from each row's first 4096 columns; an overflow is detected and that solve (on
 *   every rank together) recomputes once in F16X2 with exact row scales from its own pass over S
 *   — no second copy of S, unlike a TF32X3 recomputation (kept only as a last resort).
 * fs_fallback_count: how many such recomputations this context has made. */
int fs_row_absmax(int dtype, const void* a, int64_t rows, int64_t cols, int64_t ld, float* out, void* stream);
int fs_set_row_absmax(fs_ctx* ctx, const float* row_absmax, int64_t n);
int64_t fs_fallback_count(const fs_ctx* ctx);
/* Split-K count the FP64 Gram takes for (n, m) on this context (plan query for tests; -1 for the
 * other precision modes). */
int fs_gram_splits(const fs_ctx* ctx, int64_t n, int64_t m, int precision);

/* ---- input validation (core.py:108-119: np.isfinite(S).all() on construction) ----
 * FS_OK when all rows x cols entries (row-major, leading dimension ld) of the device array a are
 * finite, FS_EINVAL when one is not (or on bad arguments).  One streaming pass on the device of
 * the current CUDA context, no temporaries; complex data is passed as its real view (2 cols per
 * element).  No context needed.  Synchronizes `stream`. */
int fs_all_finite(int dtype, const void* a, int64_t rows, int64_t cols, int64_t ld, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FS_H_ */
