/*
 * cnmf_b200.h — C ABI of the B200-native compressed-NMF hot path.
 *
 * The reference (arxiv/paper_1505_04650, package `cnmf`) is pure Python/numpy;
 * its FFI for this path would be a ctypes binding of exactly these entry
 * points (see INTEGRATION.md for the stub). Every pointer argument marked
 * "device" is CUDA device memory on the current device; `stream` is a
 * cudaStream_t (NULL = legacy default stream). Calls are stream-ordered unless
 * they return host-visible results, in which case they synchronise `stream`.
 *
 * Layouts
 *   A        : fp32 row-major m x n, leading dimension lda (elements),
 *              lda % 4 == 0 and 16-byte aligned base (TMA requirement).
 *   panel    : a tall-skinny matrix with s logical columns stored row-major
 *              with leading dimension ldp = cnmf_panel_ld(s) >= s; the
 *              padding columns are kept zero. Q (m x s), the row-space basis
 *              R^T (n x s) and the reduced matrix (Q^T A)^T (n x s) are panels.
 *
 * Every function returns a cnmf_status; cnmf_last_error() describes the most
 * recent failure on the calling thread. Error codes map one-to-one onto the
 * reference's exception classes (errors.py).
 */
#ifndef CNMF_B200_H
#define CNMF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CNMF_OK = 0,
  CNMF_ERR_ARGUMENT = 1,          /* errors.py:13  ArgumentError */
  CNMF_ERR_INFEASIBLE_RANK = 2,   /* errors.py:17  InfeasibleRankError */
  CNMF_ERR_NUMERIC = 3,           /* errors.py:21  NumericError */
  CNMF_ERR_RANK_DEFICIENCY = 4,   /* errors.py:48  RankDeficiencyError */
  CNMF_ERR_CONVERGENCE = 5,       /* errors.py:30  ConvergenceError */
  CNMF_ERR_DIVERGENCE = 6,        /* errors.py:39  DivergenceError */
  CNMF_ERR_UNDEFINED_METRIC = 7,  /* errors.py:57  UndefinedMetricError */
  CNMF_ERR_CUDA = 8,              /* device / launch failure (no reference analogue) */
} cnmf_status;

typedef enum { CNMF_F32 = 0, CNMF_F64 = 1 } cnmf_dtype;

/* ---- library ------------------------------------------------------------ */
int cnmf_abi_version(void);
const char* cnmf_last_error(void);
/* padded leading dimension used for s-column panels (multiple of 32) */
int cnmf_panel_ld(int s);
/* instrumentation: kernels launched by this library so far (process-wide),
 * and optional CUDA-event timing of the streaming passes over A: total
 * device milliseconds, launch count and algorithmic bytes since enabled. */
int64_t cnmf_launch_count(void);
void cnmf_set_pass_profiling(int on);
/* streaming-pass implementation: 1 = tcgen05 3xTF32 (default; panel widths
 * 32 and 64), 0 = FFMA (all widths; also selected by env CNMF_PASS=ffma) */
void cnmf_set_pass_impl(int impl);
int cnmf_pass_stats(double* total_ms, int64_t* launches, double* bytes);

/* ---- RNG (rng.py) --------------------------------------------------------
 * cnmf_child_seed             replaces rng.py:73 child_seed / rng.py:56 Rng.child
 * cnmf_gaussian_fill          replaces compress.py:115 _drawn_in_chunks /
 *                             compress.py:125 draw_test_matrix (chunk_rows=4096)
 *                             and rng.py:78 gaussian_matrix (chunk_rows=0).
 *                             Bit-identical to numpy Generator(Philox(key))
 *                             .standard_normal. out: device, rows x cols, ld.
 * cnmf_uniform_fill           replaces rng.py:63 Rng.uniform (row-major
 *                             rows x cols stream); transpose=1 stores the
 *                             stream transposed (cols x rows, ld=rows).
 */
uint64_t cnmf_child_seed(uint64_t seed, const char* tag);
int cnmf_gaussian_fill(uint64_t seed, int64_t rows, int64_t cols, int64_t chunk_rows, int dtype, void* out,
                       int64_t ld, void* stream);
int cnmf_uniform_fill(uint64_t seed, int64_t rows, int64_t cols, double low, double high, int dtype,
                      int transpose, void* out, void* stream);
/* Stream continuation (rng.py:38-70: successive draws on one Rng continue
 * numpy's Philox stream). Raw 64-bit draw `start` is the first one used.
 * cnmf_uniform_fill_at   Rng.uniform from raw position `start` (one raw draw
 *                        per variate: the next position is start + rows*cols).
 * cnmf_normal_fill_at    Rng.standard_normal: `count` variates from raw
 *                        position `start` into out (device, contiguous);
 *                        *d_end (device int64) receives the raw position after
 *                        the last variate (the ziggurat consumes a variable
 *                        number of draws). */
int cnmf_uniform_fill_at(uint64_t seed, int64_t start, int64_t rows, int64_t cols, double low, double high, int dtype,
                         int transpose, void* out, void* stream);
int cnmf_normal_fill_at(uint64_t seed, int64_t start, int64_t count, int dtype, void* out, int64_t* d_end,
                        void* stream);

/* ---- streaming passes over A (store.py:578 matmul_blocked,
 *      store.py:600 matmul_transposed_blocked) --------------------------------
 * forward  : Y (m x s panel)  = A X,    X (n x s panel)
 * transpose: Z (n x s panel)  = A^T W,  W (m x s panel)
 * Outputs are overwritten (the kernels zero them first).
 */
int cnmf_pass_forward(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int s, float* Y,
                      void* stream);
int cnmf_pass_transpose(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, int s, float* Z,
                        void* stream);
/* Both at once: Y = A X and Z = A^T W in one launch (the two range finders'
 * passes of a power step; one pipeline ramp-up and tail instead of two). */
int cnmf_pass_pair(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, const float* W,
                   float* Z, int s, void* stream);

/* ---- structured compression (compress.py:156 structured_compress,
 *      compress.py:202 structured_compress_rows, nmf.py:120 _compression_pair)
 * side = 0: Q (m x s panel) spans the dominant column space of A.
 * side = 1: Q (n x s panel) spans the dominant row space (= basis of A^T).
 * Power passes are re-orthonormalised implicitly (CholeskyQR2 with fp64
 * Gram matrices); the final basis is sign-canonical (diag(R) > 0).
 * The Gaussian test matrix is the reference's, drawn from `seed`.
 * ws: device workspace of cnmf_compress_workspace(m, n, s) bytes.
 */
size_t cnmf_compress_workspace(int64_t m, int64_t n, int s);
int cnmf_structured_compress(const float* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed,
                             int side, float* Q, void* ws, size_t ws_bytes, void* stream);
/* Same as cnmf_structured_compress without the final host synchronisation:
 * the numeric status stays in `ws` until cnmf_compress_check(ws, m, n, s)
 * reads it (synchronising `stream`). Lets a caller enqueue several range
 * finders and projections back to back. */
int cnmf_structured_compress_async(const float* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed,
                                   int side, float* Q, void* ws, size_t ws_bytes, void* stream);
int cnmf_compress_check(const void* ws, int64_t m, int64_t n, int s, void* stream);
/* Both bases of the compressed NMF at once (nmf.py:120 _compression_pair):
 * QL (m x s panel) = cnmf_structured_compress(side 0, seed_left) and
 * QR (n x s panel) = cnmf_structured_compress(side 1, seed_right), the same
 * kernels and arithmetic; the two range finders are interleaved on `stream`
 * (column-chain pass, row-chain pass, one CholeskyQR sweep launch for both).
 * ws_left / ws_right: cnmf_compress_workspace bytes each; status via
 * cnmf_compress_check on each workspace. Asynchronous. */
int cnmf_compress_pair_async(const float* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed_left,
                             uint64_t seed_right, float* QL, float* QR, void* ws_left, void* ws_right,
                             size_t ws_bytes, void* stream);
/* orthonormalise a panel in place (compress.py:136 canonical_qr, Q factor);
 * R (s x s, fp64, device, may be NULL) receives the triangular factor. */
int cnmf_orthonormalize(float* P, int64_t rows, int s, double* R, void* ws, size_t ws_bytes, void* stream);
/* CholeskyQR pieces for panels whose rows are spread over several GPUs
 * (the Gram matrix is all-reduced between them):
 * cnmf_cholesky_inverse  G (S x S fp64, device, upper triangle used) = R^T R;
 *                        Rinv = R^{-1} and R (S x S, device; R may be NULL),
 *                        zero outside the leading s x s block. G is consumed
 *                        (returned zeroed). Synchronises `stream`; a Gram
 *                        matrix that is not finite or not factorable after a
 *                        1e-12 diagonal shift returns CNMF_ERR_NUMERIC.
 * cnmf_panel_apply       P <- P T in place (T upper triangular S x S fp64). */
int cnmf_cholesky_inverse(double* G, int s, int S, double* Rinv, double* R, void* stream);
/* Asynchronous variants for a whole sharded range finder with one status
 * check: `ws` is a small workspace of cnmf_small_workspace(s) bytes (Gram
 * scratch, counters, failure word). cnmf_status_reset clears it, the async
 * calls record failures in it, cnmf_status_check synchronises and reports
 * CNMF_ERR_NUMERIC if any recorded failure. */
size_t cnmf_small_workspace(int s);
int cnmf_status_reset(void* ws, int s, void* stream);
int cnmf_status_check(const void* ws, int s, void* stream);
int cnmf_orthonormalize_async(float* P, int64_t rows, int s, double* R, void* ws, size_t ws_bytes, void* stream);
int cnmf_cholesky_inverse_async(double* G, int s, int S, double* Rinv, double* R, void* ws, void* stream);
int cnmf_panel_apply(float* P, int64_t rows, int S, const double* T, void* stream);

/* ---- separable NMF (snmf.py) ---------------------------------------------
 * The reduced matrix (Q^T A, s x n) is kept transposed: W (n x ld, fp64,
 * device) holds column j of the reduced matrix in row j.
 * cnmf_panel_to_f64     converts an fp32 panel (rows x S) into such a W.
 * cnmf_select_spa       replaces snmf.py:39 select_columns_spa. W is
 *                       overwritten by the projected residual. picks: host
 *                       int64[r]; *n_picks = picks found (also on
 *                       CNMF_ERR_RANK_DEFICIENCY, errors.py:48 .picks).
 * cnmf_select_xray      replaces snmf.py:74 select_columns_xray (mass: device
 *                       s-vector, the column-mass functional).
 * cnmf_right_factor     replaces snmf.py:129 snmf_right_factor: Ht (n x k) =
 *                       NNLS coefficients (transposed) of every column over
 *                       the k picked ones; d_picks: device int64[k].
 *                       *n_capped = columns that hit the exchange cap.
 *                       When the call follows cnmf_select_xray on the same W
 *                       with the same picks and tolerance, the active-set
 *                       iteration starts from that selection's last refit
 *                       (the same NNLS problem) instead of h = 0: the same
 *                       KKT tolerance is met, in a fraction of the exchanges.
 * cnmf_refit_norms      out[0] = ||W - W[:,K] H||^2, out[1] = ||W||^2 (device)
 *                       (snmf.py:218-221 rel_error_reduced).
 */
size_t cnmf_spa_workspace(int64_t n, int s);
int cnmf_panel_to_f64(const float* src, int64_t rows, int S, double* dst, int64_t ld, void* stream);
int cnmf_select_spa(double* W, int64_t n, int s, int64_t ld, int r, int64_t* picks, int* n_picks, void* ws,
                    size_t ws_bytes, void* stream);
int cnmf_select_xray(const double* W, int64_t n, int s, int64_t ld, int r, const double* mass, double nnls_tol,
                     int64_t* picks, int* n_picks, void* stream);
int cnmf_right_factor(const double* W, int64_t n, int s, int64_t ld, const int64_t* d_picks, int k, double tol,
                      double* Ht, int64_t* n_capped, void* stream);
int cnmf_refit_norms(const double* W, int64_t n, int s, int64_t ld, const int64_t* d_picks, int k,
                     const double* Ht, double* out, void* stream);
/* batched active-set NNLS (nnls.py:21 nnls_solve) on precomputed Gram
 * products: gram (q x q) = C^T C, target (k x q) = (C^T D)^T, H (k x q) out;
 * fp64, device. tol / max_exchanges (0 = 3q) as in the reference. */
int cnmf_nnls_gram(const double* gram, const double* target, int64_t k, int q, double tol, int max_exchanges,
                   double* H, int64_t* n_capped, void* stream);
/* out (a x b, fp64, device) = X^T Y for row-aligned fp64 X (p x a), Y (p x b):
 * the shared Gram products of nnls.py:64-65. */
int cnmf_gram_f64(const double* X, int64_t p, int a, const double* Y, int b, double* out, void* stream);

/* ---- projections (nmf.py:138 _projected_data, nmf.py:329-332) ------------
 * out (S x S, fp64, device) = P1^T P2 for row-aligned panels (S = 32, 64, 128). */
int cnmf_panel_cross(const float* P1, const float* P2, int64_t rows, int S, double* out, void* stream);

/* ---- relative error (nmf.py:53 relative_error) ---------------------------
 * out[0] = ||A - X Y||_F^2, out[1] = ||A||_F^2 (device, fp64).
 * X: m x r fp64 row-major, Yt: n x r fp64 row-major (Y transposed).
 * cols (optional, may be NULL): when given, X is gathered as A[:, cols]
 * (snmf.py:223-230 full-space error; X must then be NULL). */
int cnmf_residual_norms(const float* A, int64_t m, int64_t n, int64_t lda, const double* X, const int64_t* cols,
                        const double* Yt, int r, double* out, void* stream);

/* ---- compressed ADMM NMF (nmf.py:306 nmf_admm) --------------------------
 * core : s x s fp64 (L^T A R^T), L : m x s panel, Rt : n x s panel (fp32).
 * u, du: m x r fp64; vt, dvt: n x r fp64 (V and its dual, transposed).
 * u / vt hold the initial splits on entry; du / dvt are zeroed here.
 * xc (s x r), yc (r x s) fp64 device. trace / scores: device fp64[max_iter].
 * Runs up to max_iter iterations with the reference's stopping rule (max KKT
 * residual < tol) and divergence rule (10x over 50 iterations), checked on
 * the device; *iterations (host) receives the iteration count.
 * Returns CNMF_ERR_DIVERGENCE with *iterations = detection iteration + 1.
 */
size_t cnmf_admm_workspace(int64_t m, int64_t n, int s, int r);
/* resume = 0 starts from the initial splits; resume = 1 continues a run
 * (same workspace). step_limit > 0 runs at most that many iterations in this
 * call (used to drive the reference's on_iteration callback); 0 = run to
 * completion. *done (host) = 1 once the run has stopped. */
int cnmf_admm_run(const double* core, const float* L, int64_t m, const float* Rt, int64_t n, int s, int r,
                  double* u, double* du, double* vt, double* dvt, double* xc, double* yc, double pu, double pv,
                  double step, int max_iter, double tol, double* trace, double* scores, int* iterations, int* done,
                  int resume, int step_limit, void* ws, size_t ws_bytes, void* stream);

/* ---- uncompressed ADMM (nmf_admm(compressed=False), nmf.py:306-377 with
 * identity bases: a_comp = A) ------------------------------------------------
 * A (m x n fp32, device); u (m x r), vt (n x r) hold the seeded starts on
 * entry (resume = 0) and U, V^T on return; du, dvt, xc (m x r) and yct
 * (n x r, yc^T) are fp64 device buffers the call owns. trace / scores get one
 * entry per iteration (nmf.py:362, 366). Protocol of cnmf_admm_run
 * (resume, step_limit, *done). r <= 32. DivergenceError ->
 * CNMF_ERR_DIVERGENCE with *iterations = the diverging iteration + 1. */
size_t cnmf_admm_full_workspace(int64_t m, int64_t n, int r);
int cnmf_admm_full_run(const float* A, int64_t m, int64_t n, int64_t lda, int r, double* u, double* du, double* vt,
                       double* dvt, double* xc, double* yct, double pu, double pv, double step, int max_iter,
                       double tol, double* trace, double* scores, int* iterations, int* done, int resume,
                       int step_limit, void* ws, size_t ws_bytes, void* stream);


/* ---- column-sharded multi-GPU pieces (paper_1505_04650_b200/distributed.py)
 * The host drives these one phase at a time and all-reduces between them
 * (NCCL through torch.distributed); every buffer is device memory.
 *
 * Compressed ADMM with U / dU row-sharded (the rows of L this rank owns) and
 * V^T / dV^T column-sharded (the rows of R^T of this rank's columns),
 * nmf.py:334-377: per iteration
 *   cnmf_admm_shard_core   the replicated core step (KKT score of the previous
 *                          iteration from the all-reduced sums, the stop and
 *                          divergence rules, the two ridge solves);
 *   cnmf_admm_shard_sweep  this rank's rows: x = max(P z + dx / p, 0), the dual
 *                          update, and the partial sums L_i^T U_i, L_i^T dU_i,
 *                          R_i V_i^T and the four KKT sums per side, written at
 *                          byte offset cnmf_admm_shard_sums_offset() of ws
 *                          (2 x (2 s r + 4) doubles; the dual projections are
 *                          not reduced -- the core step carries L^T dU and
 *                          R dV^T by the recurrence L^T dU += step pu (G_L xc -
 *                          L^T U), G_L = L^T L, likewise G_R = R R^T) -- the
 *                          block the host all-reduces (SUM) before the next
 *                          core step.
 * ws: cnmf_admm_shard_workspace(s, r) bytes; cnmf_admm_shard_begin resets it
 * and takes G_L, G_R (ld x ld fp64, ld = the panel width, summed over all
 * ranks' rows);
 * cnmf_admm_shard_status copies (next iteration, done, iterations, diverged
 * iteration or -1) to the host int[4] (synchronises).
 *
 * Column selection on a column shard W_i (n_i x ld, fp64, the local rows of
 * (Q^T A)^T), snmf.py:39-126:
 *   cnmf_shard_argmax      (value, index) of the best unpicked entry of v
 *                          (ties -> lowest index), into device scalars; the
 *                          host all-gathers the pairs of all ranks;
 *   cnmf_spa_shard_step    project every local column off v (NULL: none) and
 *                          store the residual squared norms (picked -> 0);
 *   cnmf_xray_shard_scores score_c = (r_j . W_c) / denom_c for the broadcast
 *                          residual column r_j;
 *   cnmf_col_mass          denom_c = mass . W_c;
 *   cnmf_right_factor_given / cnmf_refit_given  NNLS coefficients of every
 *                          local column over k picked columns given
 *                          explicitly (P: k x ld fp64, replicated), and the
 *                          residual R / squared norms sq / (res, ref) totals.
 */
size_t cnmf_admm_shard_workspace(int s, int r);
size_t cnmf_admm_shard_sums_offset(void);
int cnmf_admm_shard_begin(void* ws, int s, int r, const double* GL, const double* GR, int ld, void* stream);
int cnmf_admm_shard_sweep(void* ws, const float* L, int64_t m, const float* Rt, int64_t n, int s, int r, double* u,
                          double* du, double* vt, double* dvt, double pu, double pv, double step, int update,
                          void* stream);
int cnmf_admm_shard_core(void* ws, const double* core, double* xc, double* yc, int s, int r, double pu, double pv,
                         double step, double tol, double* trace, double* scores, int k, int max_iter, int first,
                         int solve, void* stream);
int cnmf_admm_shard_status(const void* ws, int* state, void* stream);
int cnmf_shard_argmax(const double* v, int64_t n, const uint8_t* picked, const uint8_t* valid, double* out_v,
                      int64_t* out_i, void* stream);
int cnmf_spa_shard_step(double* W, int64_t n, int s, int64_t ld, const double* v, const uint8_t* picked, double* sq,
                        void* stream);
int cnmf_xray_shard_scores(const double* W, int64_t n, int s, int64_t ld, const double* rj, const double* denom,
                           double* score, void* stream);
int cnmf_col_mass(const double* W, int64_t n, int s, int64_t ld, const double* mass, double* denom, void* stream);
int cnmf_right_factor_given(const double* W, int64_t n, int s, int64_t ld, const double* P, int k, double tol,
                            double* Ht, int64_t* n_capped, void* stream);
int cnmf_refit_given(const double* W, int64_t n, int s, int64_t ld, const double* P, int k, const double* Ht,
                     double* R, double* sq, double* tot, void* stream);


/* ---- fp64 path for float64 inputs (BASELINE.json configs[0] is an fp64
 * workload; compress.py:156-227, snmf.py:154-232 with precision="fp64") ----
 * A: fp64 row-major m x n (lda >= n); panels fp64 with ld = cnmf_panel_ld(s)
 * (s <= 64). The same algorithm as the fp32 path -- seeded test matrix,
 * 2w + 1 passes, every pass output re-orthonormalised (CholeskyQR2 in fp64)
 * -- with DFMA passes (plain tiled kernels, meant for CPU-sized inputs).
 * cnmf_structured_compress_f64  Q (m x S or n x S for side 1), synchronises
 *                               (NumericError if a Gram matrix fails).
 * cnmf_pass_transpose_f64       Z (n x S) = A^T W.
 * cnmf_residual_norms_f64       out[0] = ||A - X Y||^2, out[1] = ||A||^2
 *                               (X: m x r fp64, or A[:, cols]; Yt: n x r). */
size_t cnmf_compress_f64_workspace(int64_t m, int64_t n, int s);
int cnmf_structured_compress_f64(const double* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed,
                                 int side, double* Q, void* ws, size_t ws_bytes, void* stream);
int cnmf_pass_transpose_f64(const double* A, int64_t m, int64_t n, int64_t lda, const double* W, int s, double* Z,
                            void* stream);
int cnmf_residual_norms_f64(const double* A, int64_t m, int64_t n, int64_t lda, const double* X, const int64_t* cols,
                            const double* Yt, int r, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CNMF_B200_H */
