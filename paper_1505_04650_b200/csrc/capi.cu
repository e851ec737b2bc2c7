// extern "C" entry points (include/cnmf_b200.h). Thin: argument checks and
// dispatch into the cnmf:: implementations; no torch types cross this line.
#include "common.cuh"
#include "pass.cuh"

namespace cnmf {
const char* last_error();
int panel_ld(int s);
int gaussian_fill(uint64_t, int64_t, int64_t, int64_t, int, void*, int64_t, cudaStream_t);
int uniform_fill(uint64_t, int64_t, int64_t, double, double, int, int, void*, cudaStream_t);
int uniform_fill_at(uint64_t, int64_t, int64_t, int64_t, double, double, int, int, void*, cudaStream_t);
int normal_fill_at(uint64_t, int64_t, int64_t, int, void*, int64_t*, cudaStream_t);

int panel_cross(const float*, const float*, int64_t, int, double*, cudaStream_t);
size_t admm_full_workspace(int64_t m, int64_t n, int r);
int admm_full_run(const float* A, int64_t m, int64_t n, int64_t lda, int r, double* u, double* du, double* vt,
                  double* dvt, double* xc, double* yct, double pu, double pv, double step, int max_iter, double tol,
                  double* trace, double* scores, int* iterations, int* done, int resume, int step_limit, void* ws,
                  size_t ws_bytes, cudaStream_t st);
int cholesky_inverse(double*, int, int, double*, double*, cudaStream_t);
int status_reset(void*, int, cudaStream_t);
size_t small_workspace(int);
int status_check(const void*, int, const char*, cudaStream_t);
int orthonormalize_async(float*, int64_t, int, double*, void*, size_t, cudaStream_t);
int cholesky_inverse_async(double*, int, int, double*, double*, void*, cudaStream_t);
int panel_finalize(float*, int64_t, int, const double*, double*, cudaStream_t);
size_t compress_workspace(int64_t, int64_t, int);
int structured_compress(const float*, int64_t, int64_t, int64_t, int, int, uint64_t, int, float*, void*, size_t,
                        cudaStream_t, bool);
int compress_check(const void*, int64_t, int64_t, int, cudaStream_t);
int structured_compress_pair(const float*, int64_t, int64_t, int64_t, int, int, uint64_t, uint64_t, float*, float*,
                             void*, void*, size_t, cudaStream_t);
int orthonormalize(float*, int64_t, int, double*, void*, size_t, cudaStream_t);
size_t spa_workspace(int64_t, int);
int panel_to_f64(const float*, int64_t, int, double*, int64_t, cudaStream_t);
int select_spa(double*, int64_t, int, int64_t, int, int64_t*, int*, void*, size_t, cudaStream_t);
int select_xray(const double*, int64_t, int, int64_t, int, const double*, double, int64_t*, int*, cudaStream_t);
int right_factor(const double*, int64_t, int, int64_t, const int64_t*, int, double, double*, double*, int64_t*,
                 cudaStream_t, const double* H0 = nullptr, int q0 = 0, double* fstate = nullptr, size_t fstride = 0,
                 int tld = 0);
int right_factor_after_selection(const double*, int64_t, int, int64_t, const int64_t*, int, double, double*, double*,
                                 int64_t*, cudaStream_t);
int refit_norms(const double*, int64_t, int, int64_t, const int64_t*, int, const double*, double*, double*, double*,
                cudaStream_t);
int nnls_gram(const double*, const double*, int64_t, int, double, int, double*, int64_t*, cudaStream_t,
              const double* H0 = nullptr, int q0 = 0, double* fstate = nullptr, size_t fstride = 0, int tld = 0);
size_t nnls_state_stride(int qmax);
int residual_norms(const float*, int64_t, int64_t, int64_t, const double*, const int64_t*, const double*, int,
                   double*, cudaStream_t);
size_t admm_workspace(int64_t, int64_t, int, int);
int admm_run(const double*, const float*, int64_t, const float*, int64_t, int, int, double*, double*, double*,
             double*, double*, double*, double, double, double, int, double, double*, double*, int*, void*, size_t,
             int, int, cudaStream_t);
int64_t launch_count();
size_t compress_f64_workspace(int64_t, int64_t, int);
int structured_compress_f64(const double*, int64_t, int64_t, int64_t, int, int, uint64_t, int, double*, void*, size_t,
                            cudaStream_t);
int pass_transpose_f64(const double*, int64_t, int64_t, int64_t, const double*, int, double*, cudaStream_t);
int residual_norms_f64(const double*, int64_t, int64_t, int64_t, const double*, const int64_t*, const double*, int,
                       double*, cudaStream_t);
size_t admm_shard_workspace(int, int);
size_t admm_shard_sums_offset();
int admm_shard_begin(void*, int, int, const double*, const double*, int, cudaStream_t);
int admm_shard_sweep(void*, const float*, int64_t, const float*, int64_t, int, int, double*, double*, double*,
                     double*, double, double, double, int, cudaStream_t);
int admm_shard_core(void*, const double*, double*, double*, int, int, double, double, double, double, double*,
                    double*, int, int, int, int, cudaStream_t);
int admm_shard_status(const void*, int*, cudaStream_t);
int shard_argmax(const double*, int64_t, const uint8_t*, const uint8_t*, double*, int64_t*, cudaStream_t);
int spa_shard_step(double*, int64_t, int, int64_t, const double*, const uint8_t*, double*, cudaStream_t);
int xray_shard_scores(const double*, int64_t, int, int64_t, const double*, const double*, double*, cudaStream_t);
int col_mass_denoms(const double*, int64_t, int, int64_t, const double*, double*, cudaStream_t);
int right_factor_given(const double*, int64_t, int, int64_t, const double*, int, double, double*, int64_t*,
                       cudaStream_t);
int refit_given(const double*, int64_t, int, int64_t, const double*, int, const double*, double*, double*, double*,
                cudaStream_t);
void set_pass_impl(int);
void set_pass_profiling(int);
int pass_stats(double*, int64_t*, double*);
}  // namespace cnmf

using namespace cnmf;

#define STREAM(s) reinterpret_cast<cudaStream_t>(s)

static int check_a(const float* A, int64_t m, int64_t n, int64_t lda) {
  if (A == nullptr || m < 1 || n < 1) return fail(CNMF_ERR_ARGUMENT, "A must be a non-empty device matrix");
  if (lda < n || (lda & 3) || ((uintptr_t)A & 15))
    return fail(CNMF_ERR_ARGUMENT, "A needs lda >= n, lda % 4 == 0 and a 16-byte aligned base");
  return CNMF_OK;
}

extern "C" {

int cnmf_abi_version(void) { return 1; }

const char* cnmf_last_error(void) { return last_error(); }

int cnmf_panel_ld(int s) { return panel_ld(s); }

int64_t cnmf_launch_count(void) { return launch_count(); }

void cnmf_set_pass_profiling(int on) { set_pass_profiling(on); }

void cnmf_set_pass_impl(int impl) { set_pass_impl(impl); }

int cnmf_pass_stats(double* total_ms, int64_t* launches, double* bytes) {
  return pass_stats(total_ms, launches, bytes);
}

uint64_t cnmf_child_seed(uint64_t seed, const char* tag) { return child_seed(seed, tag); }

int cnmf_gaussian_fill(uint64_t seed, int64_t rows, int64_t cols, int64_t chunk_rows, int dtype, void* out,
                       int64_t ld, void* stream) {
  return gaussian_fill(seed, rows, cols, chunk_rows, dtype, out, ld, STREAM(stream));
}

int cnmf_uniform_fill(uint64_t seed, int64_t rows, int64_t cols, double low, double high, int dtype, int transpose,
                      void* out, void* stream) {
  return uniform_fill(seed, rows, cols, low, high, dtype, transpose, out, STREAM(stream));
}

int cnmf_uniform_fill_at(uint64_t seed, int64_t start, int64_t rows, int64_t cols, double low, double high, int dtype,
                         int transpose, void* out, void* stream) {
  return uniform_fill_at(seed, start, rows, cols, low, high, dtype, transpose, out, STREAM(stream));
}

int cnmf_normal_fill_at(uint64_t seed, int64_t start, int64_t count, int dtype, void* out, int64_t* d_end,
                        void* stream) {
  return normal_fill_at(seed, start, count, dtype, out, d_end, STREAM(stream));
}

int cnmf_pass_forward(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int s, float* Y,
                      void* stream) {
  CNMF_TRY(check_a(A, m, n, lda));
  return pass_forward(A, m, n, lda, X, panel_ld(s), Y, STREAM(stream));
}

int cnmf_pass_transpose(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, int s, float* Z,
                        void* stream) {
  CNMF_TRY(check_a(A, m, n, lda));
  return pass_transpose(A, m, n, lda, W, panel_ld(s), Z, STREAM(stream));
}

size_t cnmf_compress_workspace(int64_t m, int64_t n, int s) { return compress_workspace(m, n, s); }

int cnmf_structured_compress(const float* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed,
                             int side, float* Q, void* ws, size_t ws_bytes, void* stream) {
  CNMF_TRY(check_a(A, m, n, lda));
  if (side != 0 && side != 1) return fail(CNMF_ERR_ARGUMENT, "side must be 0 (columns) or 1 (rows)");
  return structured_compress(A, m, n, lda, s, w, seed, side, Q, ws, ws_bytes, STREAM(stream), true);
}

int cnmf_structured_compress_async(const float* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed,
                                   int side, float* Q, void* ws, size_t ws_bytes, void* stream) {
  CNMF_TRY(check_a(A, m, n, lda));
  if (side != 0 && side != 1) return fail(CNMF_ERR_ARGUMENT, "side must be 0 (columns) or 1 (rows)");
  return structured_compress(A, m, n, lda, s, w, seed, side, Q, ws, ws_bytes, STREAM(stream), false);
}

int cnmf_pass_pair(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, const float* W,
                   float* Z, int s, void* stream) {
  const int S = panel_ld(s);
  if (S < 0) return fail(CNMF_ERR_ARGUMENT, "panel width must be <= 128");
  return pass_pair(A, m, n, lda, X, Y, W, Z, S, STREAM(stream));
}

int cnmf_compress_pair_async(const float* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed_left,
                             uint64_t seed_right, float* QL, float* QR, void* ws_left, void* ws_right,
                             size_t ws_bytes, void* stream) {
  return structured_compress_pair(A, m, n, lda, s, w, seed_left, seed_right, QL, QR, ws_left, ws_right, ws_bytes,
                                  STREAM(stream));
}

int cnmf_compress_check(const void* ws, int64_t m, int64_t n, int s, void* stream) {
  return compress_check(ws, m, n, s, STREAM(stream));
}

int cnmf_orthonormalize(float* P, int64_t rows, int s, double* R, void* ws, size_t ws_bytes, void* stream) {
  if (rows < s) return fail(CNMF_ERR_ARGUMENT, "panel must be at least as tall as it is wide");
  return orthonormalize(P, rows, s, R, ws, ws_bytes, STREAM(stream));
}

size_t cnmf_small_workspace(int s) { return small_workspace(s); }

int cnmf_status_reset(void* ws, int s, void* stream) { return status_reset(ws, s, STREAM(stream)); }

int cnmf_status_check(const void* ws, int s, void* stream) { return status_check(ws, s, "device", STREAM(stream)); }

int cnmf_orthonormalize_async(float* P, int64_t rows, int s, double* R, void* ws, size_t ws_bytes, void* stream) {
  if (rows < s) return fail(CNMF_ERR_ARGUMENT, "panel must be at least as tall as it is wide");
  return orthonormalize_async(P, rows, s, R, ws, ws_bytes, STREAM(stream));
}

int cnmf_cholesky_inverse_async(double* G, int s, int S, double* Rinv, double* R, void* ws, void* stream) {
  if (s < 1 || S < s) return fail(CNMF_ERR_ARGUMENT, "cholesky_inverse: bad widths");
  return cholesky_inverse_async(G, s, S, Rinv, R, ws, STREAM(stream));
}

int cnmf_cholesky_inverse(double* G, int s, int S, double* Rinv, double* R, void* stream) {
  if (s < 1 || S < s || panel_ld(s) != S) return fail(CNMF_ERR_ARGUMENT, "cholesky_inverse: bad widths");
  return cholesky_inverse(G, s, S, Rinv, R, STREAM(stream));
}

int cnmf_panel_apply(float* P, int64_t rows, int S, const double* T, void* stream) {
  if (rows < 1 || T == nullptr) return fail(CNMF_ERR_ARGUMENT, "panel_apply: empty panel or no transform");
  return panel_finalize(P, rows, S, T, nullptr, STREAM(stream));
}

size_t cnmf_spa_workspace(int64_t n, int s) { return spa_workspace(n, s); }

int cnmf_panel_to_f64(const float* src, int64_t rows, int S, double* dst, int64_t ld, void* stream) {
  return panel_to_f64(src, rows, S, dst, ld, STREAM(stream));
}

int cnmf_select_spa(double* W, int64_t n, int s, int64_t ld, int r, int64_t* picks, int* n_picks, void* ws,
                    size_t ws_bytes, void* stream) {
  return select_spa(W, n, s, ld, r, picks, n_picks, ws, ws_bytes, STREAM(stream));
}

int cnmf_select_xray(const double* W, int64_t n, int s, int64_t ld, int r, const double* mass, double nnls_tol,
                     int64_t* picks, int* n_picks, void* stream) {
  return select_xray(W, n, s, ld, r, mass, nnls_tol, picks, n_picks, STREAM(stream));
}

int cnmf_right_factor(const double* W, int64_t n, int s, int64_t ld, const int64_t* d_picks, int k, double tol,
                      double* Ht, int64_t* n_capped, void* stream) {
  if (k < 1 || k > 64) return fail(CNMF_ERR_ARGUMENT, "right factor supports 1 <= k <= 64");
  cudaStream_t st = STREAM(stream);
  keep_pool();
  double* scratch = nullptr;
  CNMF_CUDA(cudaMallocAsync((void**)&scratch, ((size_t)k * k + (size_t)n * k) * 8, st));
  int rc = right_factor_after_selection(W, n, s, ld, d_picks, k, tol, Ht, scratch, n_capped, st);
  cudaFreeAsync(scratch, st);
  return rc;
}

int cnmf_refit_norms(const double* W, int64_t n, int s, int64_t ld, const int64_t* d_picks, int k, const double* Ht,
                     double* out, void* stream) {
  return refit_norms(W, n, s, ld, d_picks, k, Ht, nullptr, nullptr, out, STREAM(stream));
}

int cnmf_nnls_gram(const double* gram, const double* target, int64_t k, int q, double tol, int max_exchanges,
                   double* H, int64_t* n_capped, void* stream) {
  return nnls_gram(gram, target, k, q, tol, max_exchanges, H, n_capped, STREAM(stream));
}

int cnmf_panel_cross(const float* P1, const float* P2, int64_t rows, int S, double* out, void* stream) {
  return panel_cross(P1, P2, rows, S, out, STREAM(stream));
}

int cnmf_residual_norms(const float* A, int64_t m, int64_t n, int64_t lda, const double* X, const int64_t* cols,
                        const double* Yt, int r, double* out, void* stream) {
  if (A == nullptr || m < 1 || n < 1 || lda < n) return fail(CNMF_ERR_ARGUMENT, "bad A");
  return residual_norms(A, m, n, lda, X, cols, Yt, r, out, STREAM(stream));
}

size_t cnmf_admm_workspace(int64_t m, int64_t n, int s, int r) { return admm_workspace(m, n, s, r); }

size_t cnmf_admm_full_workspace(int64_t m, int64_t n, int r) { return admm_full_workspace(m, n, r); }

int cnmf_admm_full_run(const float* A, int64_t m, int64_t n, int64_t lda, int r, double* u, double* du, double* vt,
                       double* dvt, double* xc, double* yct, double pu, double pv, double step, int max_iter,
                       double tol, double* trace, double* scores, int* iterations, int* done, int resume,
                       int step_limit, void* ws, size_t ws_bytes, void* stream) {
  CNMF_TRY(check_a(A, m, n, lda));
  if (max_iter < 0) return fail(CNMF_ERR_ARGUMENT, "max_iter must be >= 0");
  if (max_iter == 0) {
    if (iterations) *iterations = 0;
    if (done) *done = 1;
    return CNMF_OK;
  }
  return admm_full_run(A, m, n, lda, r, u, du, vt, dvt, xc, yct, pu, pv, step, max_iter, tol, trace, scores,
                       iterations, done, resume, step_limit, ws, ws_bytes, STREAM(stream));
}

int cnmf_admm_run(const double* core, const float* L, int64_t m, const float* Rt, int64_t n, int s, int r, double* u,
                  double* du, double* vt, double* dvt, double* xc, double* yc, double pu, double pv, double step,
                  int max_iter, double tol, double* trace, double* scores, int* iterations, int* done, int resume,
                  int step_limit, void* ws, size_t ws_bytes, void* stream) {
  if (max_iter < 0) return fail(CNMF_ERR_ARGUMENT, "max_iter must be >= 0");
  if (max_iter == 0) {
    if (iterations) *iterations = 0;
    if (done) *done = 1;
    return CNMF_OK;
  }
  int it = 0;
  int rc = admm_run(core, L, m, Rt, n, s, r, u, du, vt, dvt, xc, yc, pu, pv, step, max_iter, tol, trace, scores, &it,
                    ws, ws_bytes, resume, step_limit, STREAM(stream));
  if (iterations) *iterations = it < 0 ? -it - 1 : it;
  if (done) *done = it >= 0 ? 1 : 0;
  return rc;
}


/* ---- column-shard primitives (multi-GPU; distributed.py) ---------------- */
size_t cnmf_admm_shard_workspace(int s, int r) { return admm_shard_workspace(s, r); }
size_t cnmf_admm_shard_sums_offset(void) { return admm_shard_sums_offset(); }
int cnmf_admm_shard_begin(void* ws, int s, int r, const double* GL, const double* GR, int ld, void* stream) {
  return admm_shard_begin(ws, s, r, GL, GR, ld, STREAM(stream));
}
int cnmf_admm_shard_sweep(void* ws, const float* L, int64_t m, const float* Rt, int64_t n, int s, int r, double* u,
                          double* du, double* vt, double* dvt, double pu, double pv, double step, int update,
                          void* stream) {
  return admm_shard_sweep(ws, L, m, Rt, n, s, r, u, du, vt, dvt, pu, pv, step, update, STREAM(stream));
}
int cnmf_admm_shard_core(void* ws, const double* core, double* xc, double* yc, int s, int r, double pu, double pv,
                         double step, double tol, double* trace, double* scores, int k, int max_iter, int first,
                         int solve, void* stream) {
  return admm_shard_core(ws, core, xc, yc, s, r, pu, pv, step, tol, trace, scores, k, max_iter, first, solve,
                         STREAM(stream));
}
int cnmf_admm_shard_status(const void* ws, int* state, void* stream) {
  return admm_shard_status(ws, state, STREAM(stream));
}
int cnmf_shard_argmax(const double* v, int64_t n, const uint8_t* picked, const uint8_t* valid, double* out_v,
                      int64_t* out_i, void* stream) {
  return shard_argmax(v, n, picked, valid, out_v, out_i, STREAM(stream));
}
int cnmf_spa_shard_step(double* W, int64_t n, int s, int64_t ld, const double* v, const uint8_t* picked, double* sq,
                        void* stream) {
  return spa_shard_step(W, n, s, ld, v, picked, sq, STREAM(stream));
}
int cnmf_xray_shard_scores(const double* W, int64_t n, int s, int64_t ld, const double* rj, const double* denom,
                           double* score, void* stream) {
  return xray_shard_scores(W, n, s, ld, rj, denom, score, STREAM(stream));
}
int cnmf_col_mass(const double* W, int64_t n, int s, int64_t ld, const double* mass, double* denom, void* stream) {
  return col_mass_denoms(W, n, s, ld, mass, denom, STREAM(stream));
}
int cnmf_right_factor_given(const double* W, int64_t n, int s, int64_t ld, const double* P, int k, double tol,
                            double* Ht, int64_t* n_capped, void* stream) {
  return right_factor_given(W, n, s, ld, P, k, tol, Ht, n_capped, STREAM(stream));
}
int cnmf_refit_given(const double* W, int64_t n, int s, int64_t ld, const double* P, int k, const double* Ht,
                     double* R, double* sq, double* tot, void* stream) {
  return refit_given(W, n, s, ld, P, k, Ht, R, sq, tot, STREAM(stream));
}
/* ---- fp64 path (float64 inputs; BASELINE.json configs[0]) --------------- */
size_t cnmf_compress_f64_workspace(int64_t m, int64_t n, int s) { return compress_f64_workspace(m, n, s); }
int cnmf_structured_compress_f64(const double* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed,
                                 int side, double* Q, void* ws, size_t ws_bytes, void* stream) {
  return structured_compress_f64(A, m, n, lda, s, w, seed, side, Q, ws, ws_bytes, STREAM(stream));
}
int cnmf_pass_transpose_f64(const double* A, int64_t m, int64_t n, int64_t lda, const double* W, int s, double* Z,
                            void* stream) {
  return pass_transpose_f64(A, m, n, lda, W, s, Z, STREAM(stream));
}
int cnmf_residual_norms_f64(const double* A, int64_t m, int64_t n, int64_t lda, const double* X, const int64_t* cols,
                            const double* Yt, int r, double* out, void* stream) {
  return residual_norms_f64(A, m, n, lda, X, cols, Yt, r, out, STREAM(stream));
}
}  // extern "C"
