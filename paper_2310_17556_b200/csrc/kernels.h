// kernels.h — host-side launchers of the fisher-b200 CUDA kernels (internal, C++).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fs {

// ---- gemv.cu (HBM-bound streaming passes over S) ----
// flag |= 1 if any entry is non-finite; rowmax (optional, zero-initialised): per-row max |a| as float bits
cudaError_t check_finite(const void* a, bool is64, int64_t rows, int64_t cols, int64_t ld, int* flag, int num_sms,
                         cudaStream_t st, int* launches, unsigned* rowmax = nullptr);
// F16X2 row scales 2^k from exact row maxima (max |S_i| 2^k in [2^14, 2^15): no fp16 overflow)
cudaError_t scales_from_max(const float* absmax, int64_t n, float* scale, double* inv_scale, cudaStream_t st,
                            int* launches);
cudaError_t widen_f32(const float* in, int64_t m, double* out, cudaStream_t st, int* launches);
// fp32 u = S w (w may be NULL: retile only) that also writes the tiled copy S_t (tiles.cuh)
// rows [r0, r1) only (r1 < 0: all; when r1 == n the tiled copy's zero padding rows are written
// too); nonfinite (may be NULL) is OR-ed with 1 if any element read is not finite
cudaError_t gemv_rows_retile(const float* S, int64_t n, int64_t m, int64_t ldS, const float* w, double* partials,
                             double* u, uint8_t* St, cudaStream_t st, int* launches, int64_t r0 = 0, int64_t r1 = -1,
                             int* nonfinite = nullptr);
// column range [c0, c1) of all rows (c0 a multiple of gemv_rows_chunk_cols()): tiled copy + the
// u-partials of its column chunks; no reduction (reduce_row_partials finishes u)
cudaError_t retile_cols(const float* S, int64_t n, int64_t m, int64_t ldS, const float* w, double* partials,
                        uint8_t* St, int64_t c0, int64_t c1, int* nonfinite, cudaStream_t st, int* launches);
// F16X2 (tiles.cuh): per-row power-of-two scales from a column sample, then the split planes
// of columns [c0, c1) of all rows (+ u partials of w, flags |= 1 non-finite, |= 2 fp16 overflow)
cudaError_t row_scales(const float* S, int64_t n, int64_t m, int64_t ldS, float* scale, double* inv_scale,
                       cudaStream_t st, int* launches, int64_t sample_cols = 0);
// *out = (*flags & bit) ? 1 : 0 (an overflow flag joins a norms all-reduce)
cudaError_t flag_bit_to_double(const int* flags, int bit, double* out, cudaStream_t st, int* launches);
cudaError_t retile16_cols(const float* S, int64_t n, int64_t m, int64_t ldS, const float* w, double* partials,
                          uint8_t* St, const float* scale, int64_t c0, int64_t c1, int* flags, cudaStream_t st,
                          int* launches);
cudaError_t reduce_row_partials(const double* partials, int64_t n, int64_t m, double* u, cudaStream_t st,
                                int* launches);
int64_t gemv_rows_chunk_cols();
// Number of column chunks the row-GEMV splits m into (partials buffer = chunks * n doubles).
int64_t gemv_rows_chunks(int64_t m, bool s_is_f64);
cudaError_t gemv_rows(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS, const void* w,
                      bool w_f64, double* partials, double* u, cudaStream_t st, int* launches);
cudaError_t gemv_cols_solve(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS,
                            const double* z, const void* v, bool v_f64, double lam, bool accumulate,
                            double* x, cudaStream_t st, int* launches);
int64_t residual_cols_blocks(int64_t m, bool s_is_f64);
// x = (v - S^T z)/lam (x += ... if accumulate) fused with y = S x (exact fp64 products):
// one HBM pass, the second read of each column panel hits L2.  ypart: >= ypart_rows x n
// doubles of scratch.  Returns cudaErrorNotSupported when n is too large for the per-CTA
// accumulators (callers then run gemv_cols_solve + gemv_rows).
cudaError_t gemv_cols_solve_y(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS, const double* z,
                              const void* v, bool v_f64, double lam, bool accumulate, double* x, double* ypart,
                              int64_t ypart_rows, double* y, int num_sms, cudaStream_t st, int* launches);
// y = S x (fp64 x, exact fp64 products) with the panel order of gemv_cols_solve_y (same
// support rule: cudaErrorNotSupported -> use gemv_rows)
cudaError_t gemv_rows_panel(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS, const double* x,
                            double* ypart, int64_t ypart_rows, double* y, int num_sms, cudaStream_t st,
                            int* launches);
cudaError_t residual_cols(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS,
                          const double* y, const double* x, const void* v, bool v_f64, double lam,
                          double* r, double* block_sums, double* sums, cudaStream_t st,
                          int* launches);

// ---- syrk_dmma.cu (exact-product fp64 Gram on the fp64 tensor cores, any dtype) ----
size_t syrk_dmma_workspace_bytes(int64_t n, int64_t m, int num_sms);   // a context for (n, m): every smaller plan fits
size_t syrk_dmma_plan_bytes(int64_t n, int64_t m, int num_sms);        // tiles x splits (partials + flush slots)
int syrk_dmma_splits(int64_t n, int64_t m, int num_sms, size_t ws_bytes);   // split count the plan takes
// cols > 0: update only C's first `cols` columns (all nt rows; a whole number of 128-col tiles)
cudaError_t syrk_dmma_trail(const double* P, int64_t nt, int64_t K, int64_t ldP, double* C, int64_t ldc,
                            const int64_t* status, cudaStream_t st, int* launches, int64_t cols = 0);
cudaError_t syrk_dmma(bool s_f64, const void* S, int64_t n, int64_t m, int64_t ldS, double lam, double* Gp,
                      double* ws, size_t ws_bytes, int num_sms, cudaStream_t st, int* launches);

// ---- syrk_tc.cu (tcgen05 3xTF32 Gram, fp32 input) ----
size_t syrk_tc_workspace_bytes(int64_t n, int64_t m, int num_sms);
size_t syrk_tc_plan_bytes(int64_t n, int64_t m, int num_sms);
// St: the tiled copy written by gemv_rows_retile
// pair rows [prow0, prow1) of the lower Gram (pair row p = 128-row blocks 2p, 2p+1) over the
// K-blocks [kb_begin, kb_end) of S_t (-1 = all); accum != 0 adds into G_packed instead of storing
cudaError_t syrk_tc(const uint8_t* St, int64_t n, int64_t m, double lam, double* G_packed, double* ws, int num_sms,
                    cudaStream_t st, int* launches, int prow0 = 0, int prow1 = -1, int kb_begin = 0, int kb_end = -1,
                    int accum = 0);
// F16X2 Gram on the split planes (tiles.cuh): kind::f16 MMAs hi*hi + hi*lo + lo*hi per
// 64-column K-block; inv_scale[i] = 2^-k_i undoes the row scales in the fp64 result
cudaError_t syrk_f16(const uint8_t* St16, int64_t n, int64_t m, const double* inv_scale, double lam, double* G_packed,
                     double* ws, int num_sms, cudaStream_t st, int* launches, int kb_begin = 0, int kb_end = -1,
                     int accum = 0);
// true when S (fp32, pitch ldS) meets the TMA alignment rules (16-byte base and pitch)
bool syrk_tc_supported(const void* S, int64_t ldS);
// F16X2 without the S_t16 copy: the SYRK reads fp32 S (row-major, pitch ldS) with 2-D TMA and
// splits it in-kernel (identical hi/lo to retile16); u (+)= S v (v fp32, may be null) from the
// diagonal tiles' converter pass via upart ([splits][n] doubles, splits <= num_sms / 2).
cudaError_t syrk_f16_direct(const float* S, int64_t ldS, int64_t n, int64_t m, const float* scale,
                            const double* inv_scale, const float* v, int* flags, double* upart, double* u, double lam,
                            double* G_packed, double* ws, int num_sms, cudaStream_t st, int* launches,
                            int kb_begin = 0, int kb_end = -1, int accum = 0);
// F16X2 "ring": fp32 S is split ONCE per element by the SYRK's own converter warps (each
// (K-block, row block) tile by one CTA of its split group) into an L2-resident ring of
// pre-swizzled hi/lo tiles (ring: syrk_ring_bytes(); counters: 2 * 74 * 16 ints), from which every
// consumer bulk-copies as in the pre-tiled mode — no S_t16 copy in HBM and no separate retile
// pass.  u (+)= S v (v may be null) through upart (syrk_ring_upart_doubles(n)).
// cudaErrorNotSupported when the shape does not qualify (syrk_ring_ok).
size_t syrk_ring_bytes();
size_t syrk_ring_upart_doubles(int64_t n);
bool syrk_ring_ok(int64_t n, int64_t m, int num_sms);
cudaError_t syrk_f16_ring(const float* S, int64_t ldS, int64_t n, int64_t m, const float* scale,
                          const double* inv_scale, const float* v, int* flags, double* upart, double* u, double lam,
                          double* G_packed, double* ws, uint8_t* ring, int* counters, int num_sms, cudaStream_t st,
                          int* launches, int kb_begin = 0, int kb_end = -1, int accum = 0);

// ---- potrf.cu / trsv.cu (fp64 small dense factor + solves) ----
cudaError_t unpack_lower(const double* Gp, int64_t n, double add_diag, double* W, int64_t ldW,
                         cudaStream_t st, int* launches);
// scratch = potrf_scratch_doubles(n) doubles; on return it starts with the inverted 64x64
// diagonal blocks of L (Linv), which trsv_pair consumes
int64_t potrf_scratch_doubles(int64_t n);
int64_t potrf_trsv_flags_offset(int64_t n);   // doubles before trsv_pair's block flags in that scratch
// u / z (optional): the TRSV pair z = L^-T L^-1 u fused into the factorisation's persistent
// kernel (*solved = true when it ran; otherwise call trsv_pair)
cudaError_t potrf_lower(double* W, int64_t n, int64_t ldW, int64_t* d_status, double* scratch,
                        cudaStream_t st, int* launches, const double* u = nullptr, double* z = nullptr,
                        bool* solved = nullptr);
cudaError_t invert_diag_blocks(const double* L, int64_t n, int64_t ldL, double* scratch, cudaStream_t st,
                               int* launches);
// potrf's fused TRSVs: the backward half on the TRSV cluster (from potrf's forward result t)
bool trsv_cluster_ok(int64_t n);
cudaError_t trsv_backward_cluster(const double* L, int64_t n, int64_t ldL, const double* Linv, const double* t,
                                  double* z, const int64_t* d_status, cudaStream_t st, int* launches);
cudaError_t trsv_pair(const double* L, int64_t n, int64_t ldL, const double* Linv, double* z,
                      const int64_t* d_status, cudaStream_t st, int* launches);

// ---- syevj.cu (eigh comparison route) ----
size_t syevj_workspace_bytes(int64_t n, int num_sms);
int64_t syevj_max_n();
// eigenpairs of the packed lower symmetric Gp: w descending, U (n x n, ldu) column j <-> w[j];
// d_info[0] = sweeps run, d_info[1] = 1 if not converged within max_sweeps
cudaError_t syevj(const double* Gp, int64_t n, double* w, double* U, int64_t ldu, int max_sweeps, double tol,
                  void* ws, int num_sms, int* d_info, cudaStream_t st, int* launches);
// z = U_r diag(1/(max(w,0)+lam)) U_r^T u (t: r doubles of scratch)
cudaError_t eig_apply(const double* U, int64_t ldu, int64_t n, int64_t r, const double* u, const double* w, double lam,
                      double* t, double* z, cudaStream_t st, int* launches);

// ---- complex.cu: kind 0 -> [Re S; Im S] (2n x m), kind 1 -> [[Re, -Im], [Im, Re]] (2n x 2m) ----
cudaError_t embed_complex(bool f64, const void* S, int64_t n, int64_t m, int64_t ldS, int kind, void* out, int64_t ldo,
                          int num_sms, cudaStream_t st, int* launches);
// W (n x n interleaved complex) = S S^H + lam I from the packed Gram of [Re S; Im S] (2n rows)
cudaError_t hermitian_gram(const double* G2, int64_t n, double lam, double* W, int64_t ldW, int num_sms,
                           cudaStream_t st, int* launches);

// packed lower rho(G) (2n x 2n) of G = S S^H from the packed Gram of [Re S; Im S]
cudaError_t rho_gram(const double* G2, int64_t n, double* R, int num_sms, cudaStream_t st, int* launches);
// complex eigenvectors of G (n x n interleaved, column j <-> w[j]) from rho(G)'s eigenpairs (Y, w2)
cudaError_t herm_extract(const double* Y, const double* w2, int64_t n, double tol, double* U, double* w, int* kept,
                         double* scratch, cudaStream_t st, int* launches);

// ---- apply.cu: Y (r x m, fp64) = T (r x n, fp64) X (n x m, fp32/fp64 row-major), fp64 tensor cores ----
cudaError_t apply_rows(bool x_f64, const double* T, int64_t r, int64_t n, int64_t ldT, const void* X, int64_t m,
                       int64_t ldX, double* Y, int64_t ldY, cudaStream_t st, int* launches, bool lower = false);

// ---- svd.cu: the direct-SVD route's n x n pieces ----
// Linv = L^-1 (lower, row-major ldo; upper zeroed); scratch: n*n doubles
cudaError_t tri_inverse(const double* L, int64_t n, int64_t ldL, double* Linv, int64_t ldo, double* scratch,
                        int num_sms, cudaStream_t st, int* launches);
size_t jacobi_svd_workspace_bytes(int64_t n);
// one-sided Jacobi SVD of A (n x n): A = U diag(sigma) Zt, sigma descending (>= 0);
// d_info[0] = sweeps, d_info[1] = 1 if not converged within max_sweeps
cudaError_t jacobi_svd(const double* A, int64_t n, int64_t lda, double* sigma, double* U, int64_t ldu, double* Zt,
                       int64_t ldz, int max_sweeps, double tol, void* ws, int num_sms, int* d_info, cudaStream_t st,
                       int* launches);

// ---- tmap.cu: 2-D tensor map (no swizzle) over a row-major array of `outer` rows ----
cudaError_t make_tensor_map_2d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, uint64_t inner,
                               uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                               CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_NONE);

}  // namespace fs
