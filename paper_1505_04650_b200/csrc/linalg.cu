// Range finder driver and CholeskyQR machinery.
//
// Reference: compress.py:156-199 structured_compress, compress.py:202-227
// structured_compress_rows, compress.py:136-145 canonical_qr, tsqr.py:65-135.
//
// Every pass output is re-orthonormalised on the device by one CholeskyQR
// sweep (csrc/sweep.cu: fp64 Gram matrix, fixed-order reduction, one block
// factors G = R^T R -- with a shift when G is numerically singular -- into
// R^{-1}, and the grid applies it in place); the final basis gets a second,
// polishing sweep. The two range finders of the compressed NMF are
// interleaved so that one sweep launch serves both. All transforms are upper
// triangular, so the leading column spans -- and therefore the
// sign-canonical Q of the reference -- are those of the reference (its
// reorthogonalize flag changes nothing in exact arithmetic); numerically this
// is the stable variant.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "chol.cuh"
#include "common.cuh"
#include "pass.cuh"
#include "sweep.cuh"

namespace cnmf {

int panel_ld(int s);

int panel_finalize(float*, int64_t, int, const double*, double*, cudaStream_t);
int gaussian_fill_ws(uint64_t, int64_t, int64_t, int64_t, int, void*, int64_t, void*, size_t, cudaStream_t);
size_t gaussian_workspace(int64_t, int64_t, int64_t);

namespace {

__global__ void __launch_bounds__(512) chol_inv_kernel(const double* G, int s, int S, double* __restrict__ T,
                                                       double* __restrict__ Rout, int* __restrict__ info,
                                                       int pass_id) {
  extern __shared__ double a[];  // s x s (+ f[s], rowk[s])
  chol_small(G, s, S, T, Rout, info, pass_id, a);
}

__global__ void init_info(int* info) {
  info[0] = 0;
  info[1] = 1 << 30;
  info[4] = 0;  // counters of the fused finalize + factor (+ apply) kernel
  info[5] = 0;
  info[6] = 0;
}

}  // namespace

int chol_inv(const double* G, int s, int S, double* T, double* R, int* info, int pass_id, cudaStream_t st) {
  // s <= 32: 256-thread register-tile factorisation (chol_tile32), else the block version
  const size_t smem = std::max(((size_t)s * s + 2 * (size_t)s) * 8, (size_t)(32 * 33 + 128) * 8);
  CNMF_TRY(ensure_smem_attr((const void*)chol_inv_kernel, (128 * 128 + 256) * 8));
  chol_inv_kernel<<<1, s <= 32 ? 256 : 512, smem, st>>>(G, s, S, T, R, info, pass_id);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

static size_t small_bytes(int S) { return 2 * (size_t)S * S * 8 + 256; }
size_t small_workspace(int s) {
  const int S = panel_ld(s);
  return S < 0 ? 0 : small_bytes(S);
}

size_t compress_workspace(int64_t m, int64_t n, int s) {
  const int S = panel_ld(s);
  if (S < 0) return 0;
  return (size_t)std::max(m, n) * S * 4 + small_bytes(S) + gaussian_workspace(std::max(m, n), s, 4096) + 256;
}

struct Scratch {
  double* G;
  double* T;
  int* info;
  unsigned* counter;
};

static Scratch carve_small(void* base, int S) {
  char* p = (char*)base;
  Scratch sc;
  sc.G = (double*)p;
  sc.T = (double*)(p + (size_t)S * S * 8);
  sc.info = (int*)(p + 2 * (size_t)S * S * 8);
  sc.counter = (unsigned*)(sc.info + 4);
  return sc;
}

static int check_info(const int* d_info, const char* what, cudaStream_t st) {
  int h[2];
  CNMF_CUDA(cudaMemcpyAsync(h, d_info, sizeof(h), cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaStreamSynchronize(st));
  if (h[1] != (1 << 30)) {
    return fail(CNMF_ERR_NUMERIC, std::string("non-finite values after pass ") + std::to_string(h[1]) + " (" +
                                      what + ")");
  }
  return CNMF_OK;
}

// status of an asynchronous compression: reads the device info word it left
// in its workspace (synchronises the stream)
int compress_check(const void* ws, int64_t m, int64_t n, int s, cudaStream_t st) {
  const int S = panel_ld(s);
  if (S < 0) return fail(CNMF_ERR_ARGUMENT, "basis width must be <= 128");
  Scratch sc = carve_small((char*)ws + (size_t)std::max(m, n) * S * 4, S);
  return check_info(sc.info, "range finder", st);
}

// One range finder's device state (compress.py:156-227): the two panels
// (rows m and rows n; the output side uses Q), the pass output `cur` and the
// small CholeskyQR scratch.
struct Chain {
  const float* A;
  int64_t m, n, lda;
  int s, S, w, side;
  float *Pm, *Pn, *cur;
  int64_t cur_rows;
  Scratch sc;
  int pass_id;
};

// Validate, reset the status word and draw the reference's seeded test
// matrix (compress.py:125-127; rows = A.cols for the column basis, A.rows for
// the row basis) into the panel the first pass streams.
static int chain_begin(Chain& c, const float* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed,
                       int side, float* Q, void* ws, size_t ws_bytes, cudaStream_t st, cudaStream_t omega_st) {
  const int S = panel_ld(s);
  if (S < 0) return fail(CNMF_ERR_ARGUMENT, "basis width must be <= 128");
  if (s < 1 || w < 0) return fail(CNMF_ERR_ARGUMENT, "bad width or power exponent");
  if (s > std::min(m, n))
    return fail(CNMF_ERR_INFEASIBLE_RANK, "basis width " + std::to_string(s) + " exceeds min(m, n) = " +
                                              std::to_string(std::min(m, n)) + "; adjust_config first");
  if (ws_bytes < compress_workspace(m, n, s)) return fail(CNMF_ERR_ARGUMENT, "workspace too small");
  c.A = A;
  c.m = m;
  c.n = n;
  c.lda = lda;
  c.s = s;
  c.S = S;
  c.w = w;
  c.side = side;
  c.Pm = side == 0 ? Q : (float*)ws;
  c.Pn = side == 0 ? (float*)ws : Q;
  c.cur = nullptr;
  c.cur_rows = 0;
  c.pass_id = 0;
  c.sc = carve_small((char*)ws + (size_t)std::max(m, n) * S * 4, S);
  const size_t used = (size_t)std::max(m, n) * S * 4 + small_bytes(S);
  char* rng_ws = (char*)ws + used;
  const size_t rng_bytes = ws_bytes - used;
  init_info<<<1, 1, 0, st>>>(c.sc.info);
  CNMF_LAUNCH_CHECK();
  CNMF_CUDA(cudaMemsetAsync(c.sc.G, 0, (size_t)S * S * 8, st));
  float* omega = side == 0 ? c.Pn : c.Pm;
  const int64_t orows = side == 0 ? n : m;
  CNMF_CUDA(cudaMemsetAsync(omega, 0, (size_t)orows * S * 4, omega_st));
  return gaussian_fill_ws(child_seed(seed, "omega"), orows, s, 4096, CNMF_F32, omega, S, rng_ws, rng_bytes,
                          omega_st);
}

// The next of the 2w+1 passes over A: the first streams the test matrix, the
// others alternate transpose / forward (power iteration on A A^T or A^T A).
struct PassPlan {
  bool trans;
  const float* in;
  float* out;
};

static PassPlan chain_plan(const Chain& c) {
  if (c.cur == nullptr) return c.side == 0 ? PassPlan{false, c.Pn, c.Pm} : PassPlan{true, c.Pm, c.Pn};
  const bool to_n = (c.cur == c.Pm);  // next output has n rows: transpose pass
  return to_n ? PassPlan{true, c.cur, c.Pn} : PassPlan{false, c.cur, c.Pm};
}

static void chain_advance(Chain& c, const PassPlan& p) {
  if (c.cur != nullptr) ++c.pass_id;
  c.cur = p.out;
  c.cur_rows = (c.cur == c.Pm) ? c.m : c.n;
}

static int run_plan(const Chain& c, const PassPlan& p, cudaStream_t st) {
  return p.trans ? pass_transpose(c.A, c.m, c.n, c.lda, p.in, c.S, p.out, st)
                 : pass_forward(c.A, c.m, c.n, c.lda, p.in, c.S, p.out, st);
}

// the passes of one power step: with both range finders there is always one
// forward and one transpose pass, run as ONE paired launch
static int chains_pass(Chain* c, int nc, cudaStream_t st) {
  PassPlan p[2];
  for (int i = 0; i < nc; ++i) p[i] = chain_plan(c[i]);
  if (nc == 2 && p[0].trans != p[1].trans) {
    const int f = p[0].trans ? 1 : 0, t = 1 - f;
    CNMF_TRY(pass_pair(c[0].A, c[0].m, c[0].n, c[0].lda, p[f].in, p[f].out, p[t].in, p[t].out, c[0].S, st));
  } else {
    for (int i = 0; i < nc; ++i) CNMF_TRY(run_plan(c[i], p[i], st));
  }
  for (int i = 0; i < nc; ++i) chain_advance(c[i], p[i]);
  return CNMF_OK;
}

static SweepPanel chain_panel(const Chain& c) {
  return SweepPanel{c.cur, c.cur_rows, c.sc.G, c.sc.T, nullptr, c.sc.info, c.sc.counter, c.s, c.pass_id, 0};
}

// Every pass output P is orthonormalised with one explicit CholeskyQR sweep
// (Gram in fp64, R^{-1} applied in place); deferring the first,
// ill-conditioned R^{-1} (cond ~ sigma_1 / sigma_s) past the next pass would
// amplify the fp32 pass error by that condition number. The pass inputs need
// not be orthonormal to working precision -- any upper-triangular transform
// keeps the leading column spans, and the next output is orthonormalised
// again -- so the second (polishing) sweep runs once, on the final basis.
static int chains_run(Chain* c, int nc, cudaStream_t st) {
  SweepPanel p[2];
  const int passes = 2 * c[0].w + 1;
  for (int t = 0; t < passes; ++t) {
    CNMF_TRY(chains_pass(c, nc, st));
    for (int i = 0; i < nc; ++i) p[i] = chain_panel(c[i]);
    CNMF_TRY(panel_sweep(p, nc, c[0].S, st));
  }
  for (int i = 0; i < nc; ++i) p[i] = chain_panel(c[i]);
  return panel_sweep(p, nc, c[0].S, st);
}

int structured_compress(const float* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed, int side,
                        float* Q, void* ws, size_t ws_bytes, cudaStream_t st, bool check) {
  Chain c;
  CNMF_TRY(chain_begin(c, A, m, n, lda, s, w, seed, side, Q, ws, ws_bytes, st, st));
  CNMF_TRY(chains_run(&c, 1, st));
  if (!check) return CNMF_OK;
  return check_info(c.sc.info, side == 0 ? "column basis" : "row basis", st);
}

// Both range finders of the compressed NMF (nmf.py:120-135: column basis of
// A and row basis, independent seeds) interleaved on one stream: pass of the
// column chain, pass of the row chain, then ONE sweep launch that
// orthonormalises both outputs (their Gram passes, factorisations and
// applies overlap). Each chain is numerically exactly structured_compress.
static int side_stream(cudaStream_t* side, cudaEvent_t* fork, cudaEvent_t* join) {
  static cudaStream_t streams[64] = {};
  static cudaEvent_t forks[64] = {}, joins[64] = {};
  int dev = 0;
  CNMF_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(CNMF_ERR_CUDA, "device index out of range");
  if (streams[dev] == nullptr) {
    CNMF_CUDA(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
    CNMF_CUDA(cudaEventCreateWithFlags(&forks[dev], cudaEventDisableTiming));
    CNMF_CUDA(cudaEventCreateWithFlags(&joins[dev], cudaEventDisableTiming));
  }
  *side = streams[dev];
  *fork = forks[dev];
  *join = joins[dev];
  return CNMF_OK;
}

int structured_compress_pair(const float* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed_left,
                             uint64_t seed_right, float* QL, float* QR, void* wsL, void* wsR, size_t ws_bytes,
                             cudaStream_t st) {
  // the two seeded test matrices (small latency-bound grids) are drawn
  // concurrently: the row chain's on a side stream forked from and joined
  // back into `st` (two parallel branches inside a graph capture)
  cudaStream_t side;
  cudaEvent_t fork, join;
  CNMF_TRY(side_stream(&side, &fork, &join));
  CNMF_CUDA(cudaEventRecord(fork, st));
  CNMF_CUDA(cudaStreamWaitEvent(side, fork, 0));
  Chain c[2];
  int rc = chain_begin(c[0], A, m, n, lda, s, w, seed_left, 0, QL, wsL, ws_bytes, st, st);
  const int rc2 = chain_begin(c[1], A, m, n, lda, s, w, seed_right, 1, QR, wsR, ws_bytes, st, side);
  // always join (a capture must not be left forked)
  CNMF_CUDA(cudaEventRecord(join, side));
  CNMF_CUDA(cudaStreamWaitEvent(st, join, 0));
  CNMF_TRY(rc);
  CNMF_TRY(rc2);
  return chains_run(c, 2, st);
}

int cholesky_inverse(double* G, int s, int S, double* Rinv, double* R, cudaStream_t st) {
  keep_pool();
  int* info = nullptr;
  CNMF_CUDA(cudaMallocAsync((void**)&info, 64, st));
  init_info<<<1, 1, 0, st>>>(info);
  CNMF_LAUNCH_CHECK();
  const int rc = chol_inv(G, s, S, Rinv, R, info, 0, st);
  const int rc2 = rc == CNMF_OK ? check_info(info, "cholesky_inverse", st) : rc;
  cudaFreeAsync(info, st);
  return rc2;
}

int status_reset(void* ws, int s, cudaStream_t st);
int status_check(const void* ws, int s, const char* what, cudaStream_t st);
int orthonormalize_async(float* P, int64_t rows, int s, double* R, void* ws, size_t ws_bytes, cudaStream_t st);

int orthonormalize(float* P, int64_t rows, int s, double* R, void* ws, size_t ws_bytes, cudaStream_t st) {
  CNMF_TRY(status_reset(ws, s, st));
  CNMF_TRY(orthonormalize_async(P, rows, s, R, ws, ws_bytes, st));
  return status_check(ws, s, "orthonormalize", st);
}

// ---- asynchronous pieces for panels spread over several GPUs -------------
// The small workspace (small_bytes(S)) carries the Gram matrix, the
// transform, the last-block counters and the failure word; status_reset
// clears it once, the async calls only ever record failures in it, and
// status_check reads it (one synchronisation for a whole range finder).

int status_reset(void* ws, int s, cudaStream_t st) {
  const int S = panel_ld(s);
  if (S < 0) return fail(CNMF_ERR_ARGUMENT, "width must be <= 128");
  Scratch sc = carve_small(ws, S);
  init_info<<<1, 1, 0, st>>>(sc.info);
  CNMF_LAUNCH_CHECK();
  CNMF_CUDA(cudaMemsetAsync(sc.G, 0, (size_t)S * S * 8, st));
  return CNMF_OK;
}

int status_check(const void* ws, int s, const char* what, cudaStream_t st) {
  const int S = panel_ld(s);
  if (S < 0) return fail(CNMF_ERR_ARGUMENT, "width must be <= 128");
  return check_info(carve_small(const_cast<void*>(ws), S).info, what, st);
}

int orthonormalize_async(float* P, int64_t rows, int s, double* R, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int S = panel_ld(s);
  if (S < 0) return fail(CNMF_ERR_ARGUMENT, "width must be <= 128");
  if (ws_bytes < small_bytes(S)) return fail(CNMF_ERR_ARGUMENT, "workspace too small");
  Scratch sc = carve_small(ws, S);
  SweepPanel p{P, rows, sc.G, sc.T, nullptr, sc.info, sc.counter, s, 0, 0};
  CNMF_TRY(panel_sweep(&p, 1, S, st));
  p.R = R;  // CholeskyQR2: R of the second sweep
  return panel_sweep(&p, 1, S, st);
}

// Rinv = R^{-1} of G = R^T R (G consumed), failures recorded in ws
int cholesky_inverse_async(double* G, int s, int S, double* Rinv, double* R, void* ws, cudaStream_t st) {
  if (panel_ld(s) != S) return fail(CNMF_ERR_ARGUMENT, "cholesky_inverse: bad widths");
  return chol_inv(G, s, S, Rinv, R, carve_small(ws, S).info, 0, st);
}

}  // namespace cnmf
