// Extreme-column selection on the compressed matrix: SPA and XRAY.
//
// Reference: snmf.py:39-71 select_columns_spa, snmf.py:74-126
// select_columns_xray, snmf.py:129-137 snmf_right_factor.
//
// The reduced matrix (Q^T A, s x n) is stored transposed as an n x ld fp64
// panel, so every column of the reduced matrix is one contiguous row that a
// single warp owns. An SPA step is one kernel: every warp projects its
// columns off the previous pick (w -= v (v . w)), recomputes the squared norm
// and keeps a running (norm, index) maximum; the last block to finish reduces
// the per-block maxima (ties -> lowest index, as numpy.argmax), records the
// pick and normalises the picked column into the next projection vector.
// Across GPUs the same (norm, index) pair is what gets all-reduced.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace cnmf {

int nnls_gram(const double*, const double*, int64_t, int, double, int, double*, int64_t*, cudaStream_t,
              const double* H0 = nullptr, int q0 = 0, double* fstate = nullptr, size_t fstride = 0, int tld = 0);
size_t nnls_state_stride(int qmax);

namespace {

constexpr int kSelThreads = 256;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kMaxS = 128;

struct SpaState {
  double v[kMaxS];
  double floor;
  int t;
  int status;  // 0 ok, 1 rank deficient
  unsigned int counter;
  int pad;
};

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void better(double& bv, int64_t& bi, double ov, int64_t oi) {
  if (ov > bv || (ov == bv && oi < bi)) {
    bv = ov;
    bi = oi;
  }
}

// One SPA step. first: compute norms only (and the rank floor).
__global__ void __launch_bounds__(kSelThreads)
    spa_step(double* __restrict__ W, int64_t n, int s, int64_t ld, SpaState* st, uint8_t* __restrict__ picked,
             int64_t* __restrict__ picks, double* __restrict__ blk_v, int64_t* __restrict__ blk_i, int first) {
  if (st->status) return;
  __shared__ double sv[kMaxS];
  __shared__ double rv[kSelWarps];
  __shared__ int64_t ri[kSelWarps];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < s; i += blockDim.x) sv[i] = first ? 0.0 : st->v[i];
  __syncthreads();
  double bv = -1.0;
  int64_t bi = INT64_MAX;
  const int64_t gw = (int64_t)blockIdx.x * kSelWarps + warp, nw = (int64_t)gridDim.x * kSelWarps;
  for (int64_t c = gw; c < n; c += nw) {
    double* col = W + c * ld;
    double x[kMaxS / 32];
#pragma unroll
    for (int q = 0; q < kMaxS / 32; ++q) {
      const int i = lane + 32 * q;
      x[q] = (i < s) ? col[i] : 0.0;
    }
    if (!first) {
      double d = 0.0;
#pragma unroll
      for (int q = 0; q < kMaxS / 32; ++q) {
        const int i = lane + 32 * q;
        if (i < s) d += sv[i] * x[q];
      }
      d = wsum(d);
#pragma unroll
      for (int q = 0; q < kMaxS / 32; ++q) {
        const int i = lane + 32 * q;
        if (i < s) {
          x[q] -= sv[i] * d;
          col[i] = x[q];
        }
      }
    }
    double sq = 0.0;
#pragma unroll
    for (int q = 0; q < kMaxS / 32; ++q) sq += x[q] * x[q];
    sq = wsum(sq);
    if (picked[c]) sq = 0.0;
    better(bv, bi, sq, c);
  }
  if (lane == 0) {
    rv[warp] = bv;
    ri[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kSelWarps; ++w) better(bv, bi, rv[w], ri[w]);
    blk_v[blockIdx.x] = bv;
    blk_i[blockIdx.x] = bi;
    __threadfence();
    last = atomicAdd(&st->counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double gv = -1.0;
    int64_t gi = INT64_MAX;
    for (unsigned b = 0; b < gridDim.x; ++b) better(gv, gi, blk_v[b], blk_i[b]);
    st->counter = 0;
    if (first) {
      const double f = sqrt(gv) * 1e-14;
      st->floor = f * f;
    }
    if (!(gv > st->floor)) {
      st->status = 1;
    } else {
      picks[st->t] = gi;
      picked[gi] = 1;
      st->t += 1;
      rv[0] = gv;
      ri[0] = gi;
    }
  }
  __syncthreads();
  if (st->status) return;
  const double inv = 1.0 / sqrt(rv[0]);
  const double* col = W + ri[0] * ld;
  for (int i = threadIdx.x; i < s; i += blockDim.x) st->v[i] = col[i] * inv;
}

__global__ void f32_to_f64_panel(const float* __restrict__ src, int64_t rows, int S, double* __restrict__ dst,
                                 int64_t ld) {
  const int64_t total = rows * S;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / S, c = i - r * S;
    dst[r * ld + c] = (double)src[i];
  }
}

// gram[a][b] = W_{p_a} . W_{p_b};  target[c][k] = W_c . W_{p_k}
__global__ void __launch_bounds__(kSelThreads)
    gather_gram(const double* __restrict__ W, int64_t n, int s, int64_t ld, const double* __restrict__ Wp,
                const int64_t* __restrict__ picks, int k, double* __restrict__ gram, double* __restrict__ target,
                int a0, int tld) {
  // target columns [a0, k) are (re)computed, row stride tld: XRAY keeps the
  // targets of earlier picks (the picks grow by appending) and passes a0 = k - 1
  extern __shared__ double sc[];  // k x s picked columns: rows picks[a] of Wp (Wp = W, or a gathered copy)
  for (int i = threadIdx.x; i < k * s; i += blockDim.x) {
    const int a = i / s, j = i % s;
    sc[i] = Wp[(picks ? picks[a] : a) * ld + j];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
      const int a = e / k, b = e % k;
      double acc = 0.0;
      for (int j = 0; j < s; ++j) acc += sc[a * s + j] * sc[b * s + j];
      gram[e] = acc;
    }
  for (int64_t c = (int64_t)blockIdx.x * kSelWarps + warp; c < n; c += (int64_t)gridDim.x * kSelWarps) {
    double x[kMaxS / 32];
#pragma unroll
    for (int q = 0; q < kMaxS / 32; ++q) {
      const int i = lane + 32 * q;
      x[q] = (i < s) ? W[c * ld + i] : 0.0;
    }
    for (int a = a0; a < k; ++a) {
      double d = 0.0;
#pragma unroll
      for (int q = 0; q < kMaxS / 32; ++q) {
        const int i = lane + 32 * q;
        if (i < s) d += sc[a * s + i] * x[q];
      }
      d = wsum(d);
      if (lane == 0) target[c * tld + a] = d;
    }
  }
}

// res_c = W_c - sum_a H[c][a] W_{p_a}; out: residual squared norms (and the
// residual itself when R != null); picked columns report 0.
__global__ void __launch_bounds__(kSelThreads)
    refit_residual(const double* __restrict__ W, int64_t n, int s, int64_t ld, const double* __restrict__ Wp,
                   const int64_t* __restrict__ picks, int k, const double* __restrict__ H, double* __restrict__ R,
                   double* __restrict__ sq_out, double* __restrict__ tot) {
  extern __shared__ double sc[];
  for (int i = threadIdx.x; i < k * s; i += blockDim.x) {
    const int a = i / s, j = i % s;
    sc[i] = Wp[(picks ? picks[a] : a) * ld + j];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc_res = 0.0, acc_ref = 0.0;
  for (int64_t c = (int64_t)blockIdx.x * kSelWarps + warp; c < n; c += (int64_t)gridDim.x * kSelWarps) {
    double x[kMaxS / 32], w0[kMaxS / 32];
#pragma unroll
    for (int q = 0; q < kMaxS / 32; ++q) {
      const int i = lane + 32 * q;
      w0[q] = (i < s) ? W[c * ld + i] : 0.0;
      x[q] = w0[q];
    }
    for (int a = 0; a < k; ++a) {
      const double h = H[c * k + a];
#pragma unroll
      for (int q = 0; q < kMaxS / 32; ++q) {
        const int i = lane + 32 * q;
        if (i < s) x[q] -= h * sc[a * s + i];
      }
    }
    double sq = 0.0, rf = 0.0;
#pragma unroll
    for (int q = 0; q < kMaxS / 32; ++q) {
      sq += x[q] * x[q];
      rf += w0[q] * w0[q];
      const int i = lane + 32 * q;
      if (R != nullptr && i < s) R[c * ld + i] = x[q];
    }
    sq = wsum(sq);
    rf = wsum(rf);
    if (lane == 0) {
      if (sq_out) sq_out[c] = sq;
      acc_res += sq;
      acc_ref += rf;
    }
  }
  if (tot != nullptr && lane == 0) {
    atomicAdd(&tot[0], acc_res);
    atomicAdd(&tot[1], acc_ref);
  }
}

// XRAY pick: j = argmax residual norm (unpicked); then i = argmax over
// scorable unpicked columns of (R_j . W_c) / denom_c. One block reduces the
// residual norms, then all blocks score (two launches; see xray()).
__global__ void __launch_bounds__(kSelThreads)
    argmax_unpicked(const double* __restrict__ v, int64_t n, const uint8_t* __restrict__ picked,
                    const uint8_t* __restrict__ valid, double* __restrict__ blk_v, int64_t* __restrict__ blk_i) {
  __shared__ double rv[kSelWarps];
  __shared__ int64_t ri[kSelWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double bv = -DBL_MAX;
  int64_t bi = INT64_MAX;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    double x = v[c];
    if (picked[c]) x = (valid == nullptr) ? 0.0 : -DBL_MAX;
    if (valid != nullptr && !valid[c]) x = -DBL_MAX;
    better(bv, bi, x, c);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, ov, oi);
  }
  if (lane == 0) {
    rv[warp] = bv;
    ri[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kSelWarps; ++w) better(bv, bi, rv[w], ri[w]);
    blk_v[blockIdx.x] = bv;
    blk_i[blockIdx.x] = bi;
  }
}

// score_c = (R_j . W_c) / denom_c
__global__ void __launch_bounds__(kSelThreads)
    xray_scores(const double* __restrict__ W, const double* __restrict__ R, int64_t n, int s, int64_t ld,
                const int64_t* __restrict__ jsel, const double* __restrict__ denom, double* __restrict__ score) {
  __shared__ double rj[kMaxS];
  const int64_t j = jsel ? *jsel : 0;  // jsel = null: R is the residual column itself
  for (int i = threadIdx.x; i < s; i += blockDim.x) rj[i] = R[j * ld + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t c = (int64_t)blockIdx.x * kSelWarps + warp; c < n; c += (int64_t)gridDim.x * kSelWarps) {
    double d = 0.0;
    for (int i = lane; i < s; i += 32) d += rj[i] * W[c * ld + i];
    d = wsum(d);
    if (lane == 0) score[c] = d / denom[c];
  }
}

// denom_c = mass . W_c
__global__ void col_mass(const double* __restrict__ W, int64_t n, int s, int64_t ld, const double* __restrict__ mass,
                         double* __restrict__ denom) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  for (int64_t c = (int64_t)blockIdx.x * wpb + warp; c < n; c += (int64_t)gridDim.x * wpb) {
    double d = 0.0;
    for (int i = lane; i < s; i += 32) d += mass[i] * W[c * ld + i];
    d = wsum(d);
    if (lane == 0) denom[c] = d;
  }
}

}  // namespace

size_t spa_workspace(int64_t n, int s) {
  (void)s;
  return sizeof(SpaState) + 64 + (size_t)n + 64 + 4096 * 16 + (size_t)n * 8 * 4;
}

static unsigned sel_grid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kSelWarps * 4), 4 * kNumSMs));
}

// Runs SPA on a writable fp64 copy W (n x ld). picks: host array.
int select_spa(double* W, int64_t n, int s, int64_t ld, int r, int64_t* picks_host, int* n_picks, void* ws,
               size_t ws_bytes, cudaStream_t st) {
  if (s > kMaxS) return fail(CNMF_ERR_ARGUMENT, "SPA supports s <= 128");
  if (r < 1 || r > std::min<int64_t>(s, n))
    return fail(CNMF_ERR_ARGUMENT, "cannot pick " + std::to_string(r) + " columns from a " + std::to_string(s) + "x" +
                                       std::to_string(n) + " matrix");
  if (ws_bytes < spa_workspace(n, s)) return fail(CNMF_ERR_ARGUMENT, "workspace too small");
  char* p = (char*)ws;
  SpaState* state = (SpaState*)p;
  p += (sizeof(SpaState) + 63) & ~(size_t)63;
  uint8_t* picked = (uint8_t*)p;
  p += (n + 63) & ~(int64_t)63;
  int64_t* d_picks = (int64_t*)p;
  p += 4096 * 8;
  const unsigned grid = sel_grid(n);
  double* blk_v = (double*)p;
  int64_t* blk_i = (int64_t*)(p + grid * 8);
  CNMF_CUDA(cudaMemsetAsync(state, 0, sizeof(SpaState), st));
  CNMF_CUDA(cudaMemsetAsync(picked, 0, n, st));
  for (int t = 0; t < r; ++t) {
    spa_step<<<grid, kSelThreads, 0, st>>>(W, n, s, ld, state, picked, d_picks, blk_v, blk_i, t == 0);
    CNMF_LAUNCH_CHECK();
  }
  SpaState hs;
  CNMF_CUDA(cudaMemcpyAsync(&hs, state, sizeof(SpaState), cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaMemcpyAsync(picks_host, d_picks, sizeof(int64_t) * r, cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaStreamSynchronize(st));
  *n_picks = hs.t;
  if (hs.status)
    return fail(CNMF_ERR_RANK_DEFICIENCY,
                "only " + std::to_string(hs.t) + " numerically independent columns found");
  return CNMF_OK;
}

namespace {

// SPA on a column shard: project every column off v (v != null), store the
// residual squared norms (picked columns report 0)
__global__ void __launch_bounds__(kSelThreads)
    spa_project_norms(double* __restrict__ W, int64_t n, int s, int64_t ld, const double* __restrict__ v,
                      const uint8_t* __restrict__ picked, double* __restrict__ sq) {
  __shared__ double sv[kMaxS];
  for (int i = threadIdx.x; i < s; i += blockDim.x) sv[i] = v ? v[i] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t c = (int64_t)blockIdx.x * kSelWarps + warp; c < n; c += (int64_t)gridDim.x * kSelWarps) {
    double* col = W + c * ld;
    double x[kMaxS / 32];
#pragma unroll
    for (int q = 0; q < kMaxS / 32; ++q) {
      const int i = lane + 32 * q;
      x[q] = (i < s) ? col[i] : 0.0;
    }
    if (v != nullptr) {
      double d = 0.0;
#pragma unroll
      for (int q = 0; q < kMaxS / 32; ++q) {
        const int i = lane + 32 * q;
        if (i < s) d += sv[i] * x[q];
      }
      d = wsum(d);
#pragma unroll
      for (int q = 0; q < kMaxS / 32; ++q) {
        const int i = lane + 32 * q;
        if (i < s) {
          x[q] -= sv[i] * d;
          col[i] = x[q];
        }
      }
    }
    double q2 = 0.0;
#pragma unroll
    for (int q = 0; q < kMaxS / 32; ++q) q2 += x[q] * x[q];
    q2 = wsum(q2);
    if (lane == 0) sq[c] = picked[c] ? 0.0 : q2;
  }
}

// final stage of the two-stage argmax: (value, index) of the best block
__global__ void argmax_final(const double* __restrict__ blk_v, const int64_t* __restrict__ blk_i, int nb,
                             double* __restrict__ out_v, int64_t* __restrict__ out_i) {
  if (threadIdx.x != 0) return;
  double bv = -DBL_MAX;
  int64_t bi = INT64_MAX;
  for (int b = 0; b < nb; ++b) better(bv, bi, blk_v[b], blk_i[b]);
  *out_v = bv;
  *out_i = bi;
}

}  // namespace

// ---- column-shard primitives (multi-GPU SPA / XRAY, distributed.py) ------
// argmax over v[0..n) of the unpicked (and valid) entries; ties -> lowest
// index (numpy.argmax); picked entries count as 0 (valid == null, residual
// norms) or -inf (valid != null, scores). out_v / out_i: device scalars.
int shard_argmax(const double* v, int64_t n, const uint8_t* picked, const uint8_t* valid, double* out_v,
                 int64_t* out_i, cudaStream_t st) {
  const unsigned agrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kSelThreads), 4 * kNumSMs));
  void* scr = nullptr;
  CNMF_TRY(device_scratch("shard-argmax", (size_t)agrid * 16, &scr, st));
  double* bv = (double*)scr;
  int64_t* bi = (int64_t*)(bv + agrid);
  argmax_unpicked<<<agrid, kSelThreads, 0, st>>>(v, n, picked, valid, bv, bi);
  CNMF_LAUNCH_CHECK();
  argmax_final<<<1, 32, 0, st>>>(bv, bi, (int)agrid, out_v, out_i);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

int spa_shard_step(double* W, int64_t n, int s, int64_t ld, const double* v, const uint8_t* picked, double* sq,
                   cudaStream_t st) {
  if (s > kMaxS) return fail(CNMF_ERR_ARGUMENT, "SPA supports s <= 128");
  spa_project_norms<<<sel_grid(n), kSelThreads, 0, st>>>(W, n, s, ld, v, picked, sq);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

// XRAY on a column shard: scores of every local column against the
// residual column rj (an s-vector), denominators, NNLS right factor and
// residual refit against k picked columns given explicitly (P: k x ld fp64).
int xray_shard_scores(const double* W, int64_t n, int s, int64_t ld, const double* rj, const double* denom,
                      double* score, cudaStream_t st) {
  xray_scores<<<sel_grid(n), kSelThreads, 0, st>>>(W, rj, n, s, ld, nullptr, denom, score);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

int col_mass_denoms(const double* W, int64_t n, int s, int64_t ld, const double* mass, double* denom, cudaStream_t st) {
  col_mass<<<sel_grid(n), kSelThreads, 0, st>>>(W, n, s, ld, mass, denom);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

int right_factor_given(const double* W, int64_t n, int s, int64_t ld, const double* P, int k, double tol, double* Ht,
                       int64_t* n_capped, cudaStream_t st) {
  if (k < 1 || k > 64 || s > kMaxS) return fail(CNMF_ERR_ARGUMENT, "right factor: 1 <= k <= 64, s <= 128");
  void* scr = nullptr;
  CNMF_TRY(device_scratch("right-factor-given", ((size_t)k * k + (size_t)n * k) * 8, &scr, st));
  double* gram = (double*)scr;
  double* target = gram + (size_t)k * k;
  CNMF_TRY(ensure_smem_attr((const void*)gather_gram, 200 * 1024));
  gather_gram<<<sel_grid(n), kSelThreads, (size_t)k * s * 8, st>>>(W, n, s, ld, P, nullptr, k, gram, target, 0, k);
  CNMF_LAUNCH_CHECK();
  return nnls_gram(gram, target, n, k, tol, 0, Ht, n_capped, st);
}

int refit_given(const double* W, int64_t n, int s, int64_t ld, const double* P, int k, const double* Ht, double* R,
                double* sq, double* tot, cudaStream_t st) {
  CNMF_TRY(ensure_smem_attr((const void*)refit_residual, 200 * 1024));
  if (tot) CNMF_CUDA(cudaMemsetAsync(tot, 0, 16, st));
  refit_residual<<<sel_grid(n), kSelThreads, (size_t)std::max(k, 1) * s * 8, st>>>(W, n, s, ld, P, nullptr, k, Ht,
                                                                                    R, sq, tot);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

int panel_to_f64(const float* src, int64_t rows, int S, double* dst, int64_t ld, cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(rows * S, 256), 8 * kNumSMs);
  f32_to_f64_panel<<<grid, 256, 0, st>>>(src, rows, S, dst, ld);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

// NNLS coefficients of every column over the picked columns (snmf.py:129-137).
// Ht: n x k (coefficients transposed). scratch: k*k + n*k doubles.
int right_factor(const double* W, int64_t n, int s, int64_t ld, const int64_t* d_picks, int k, double tol,
                 double* Ht, double* scratch, int64_t* n_capped, cudaStream_t st, const double* H0 = nullptr,
                 int q0 = 0, double* fstate = nullptr, size_t fstride = 0, int tld = 0) {
  // tld > 0 (XRAY): the targets live at a fixed place in scratch with row
  // stride tld and those of the first k - 1 picks are already there
  double* gram = scratch;
  double* target = scratch + (tld > 0 ? (size_t)64 * 64 : (size_t)k * k);
  const size_t sm = (size_t)k * s * 8;
  CNMF_TRY(ensure_smem_attr((const void*)gather_gram, 200 * 1024));
  gather_gram<<<sel_grid(n), kSelThreads, sm, st>>>(W, n, s, ld, W, d_picks, k, gram, target, tld > 0 ? k - 1 : 0,
                                                    tld > 0 ? tld : k);
  CNMF_LAUNCH_CHECK();
  return nnls_gram(gram, target, n, k, tol, 0, Ht, n_capped, st, H0, q0, fstate, fstride, tld);
}

// residual norms ||W - W[:, picks] H||^2 and ||W||^2 into tot[0..1] (device)
int refit_norms(const double* W, int64_t n, int s, int64_t ld, const int64_t* d_picks, int k, const double* Ht,
                double* R, double* sq_out, double* tot, cudaStream_t st) {
  CNMF_TRY(ensure_smem_attr((const void*)refit_residual, 200 * 1024));
  if (tot) CNMF_CUDA(cudaMemsetAsync(tot, 0, 16, st));
  refit_residual<<<sel_grid(n), kSelThreads, (size_t)k * s * 8, st>>>(W, n, s, ld, W, d_picks, k, Ht, R, sq_out,
                                                                      tot);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

// The last XRAY run's final refit per device: the right factor that follows
// a selection (snmf.py:129-137 after snmf.py:74-126) is the same NNLS problem
// as XRAY's last refit, so it can start from that solution and only has to
// confirm the KKT conditions (configs[3]: 63 ms from h = 0, ~4 ms from here).
// A start only: the active-set iteration runs to the same tolerance on the
// caller's data whatever the cache holds, so a stale entry costs time, not
// correctness.
struct XrayLast {
  const double* W = nullptr;
  int64_t n = 0, ld = 0;
  int s = 0, k = 0;
  double tol = 0.0;
  std::vector<int64_t> picks;
  const double* H = nullptr;  // n x k (library scratch "xray-last-H")
};
static std::mutex g_xray_last_mu;
static std::map<int, XrayLast> g_xray_last;

// CNMF_XRAY_WARM=0: every refit from h = 0 like the reference (A/B)
static bool xray_warm() {
  const char* e = getenv("CNMF_XRAY_WARM");
  return !(e && e[0] == '0');
}

// XRAY (snmf.py:74-126). W: n x ld fp64 (the reduced matrix, transposed);
// mass: device s-vector; picks_host receives the picks.
int select_xray(const double* W, int64_t n, int s, int64_t ld, int r, const double* mass, double nnls_tol,
                int64_t* picks_host, int* n_picks, cudaStream_t st) {
  if (s > kMaxS || r > 64) return fail(CNMF_ERR_ARGUMENT, "XRAY supports s <= 128, r <= 64");
  if (r < 1 || r > std::min<int64_t>(s, n)) return fail(CNMF_ERR_ARGUMENT, "bad r for XRAY");
  const unsigned grid = sel_grid(n);
  const unsigned agrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kSelThreads), 4 * kNumSMs));
  // buffers
  size_t bytes = (size_t)n * ld * 8 /*R*/ + (size_t)n * 8 * 3 /*sq, denom, score*/ + (size_t)n * 2 /*flags*/ +
                 (size_t)64 * 64 * 8 + (size_t)n * 64 * 8 * 3 /*target, H, previous H*/ + 4096 * 16 + 64 * 8 + 1024;
  // per-column Cholesky factors of the NNLS passive sets, kept from one
  // refit to the next (the picks grow by appending, so a column's factor
  // stays valid): n x (33 + r (r + 1) / 2) doubles, 2.1 GB at configs[3];
  // skipped (factors rebuilt per refit) when it would not fit comfortably
  // (CNMF_XRAY_FACTORS=0 disables it)
  const size_t fstride = nnls_state_stride(r);
  size_t fbytes = (size_t)n * fstride * 8;
  {
    size_t free_b = 0, total_b = 0;
    const char* e = getenv("CNMF_XRAY_FACTORS");
    if ((e && e[0] == '0') || !xray_warm() || cudaMemGetInfo(&free_b, &total_b) != cudaSuccess ||
        fbytes + bytes > free_b / 2)
      fbytes = 0;
  }
  char* buf = nullptr;
  keep_pool();
  CNMF_CUDA(cudaMallocAsync((void**)&buf, bytes + fbytes + 256, st));
  char* p = buf;
  auto take = [&](size_t b) {
    char* q = p;
    p += (b + 255) & ~(size_t)255;
    return q;
  };
  double* R = (double*)take((size_t)n * ld * 8);
  double* sq = (double*)take((size_t)n * 8);
  double* denom = (double*)take((size_t)n * 8);
  double* score = (double*)take((size_t)n * 8);
  uint8_t* picked = (uint8_t*)take((size_t)n);
  uint8_t* scorable = (uint8_t*)take((size_t)n);
  double* scratch = (double*)take((size_t)64 * 64 * 8 + (size_t)n * 64 * 8);
  double* Ht = (double*)take((size_t)n * 64 * 8);
  double* Hprev = (double*)take((size_t)n * 64 * 8);
  double* blk_v = (double*)take(4096 * 8);
  int64_t* blk_i = (int64_t*)take(4096 * 8);
  int64_t* d_picks = (int64_t*)take(64 * 8);
  double* fstate = fbytes ? (double*)take(fbytes) : nullptr;
  CNMF_CUDA(cudaMemsetAsync(picked, 0, n, st));
  // denominators and the scorable mask (snmf.py:103-104)
  col_mass<<<grid, kSelThreads, 0, st>>>(W, n, s, ld, mass, denom);
  CNMF_LAUNCH_CHECK();
  std::vector<double> hden(n);
  CNMF_CUDA(cudaMemcpyAsync(hden.data(), denom, n * 8, cudaMemcpyDeviceToHost, st));
  // residual = W initially; sq = column norms
  CNMF_TRY(refit_norms(W, n, s, ld, d_picks, 0, Ht, R, sq, nullptr, st));
  std::vector<double> hsq(n);
  CNMF_CUDA(cudaMemcpyAsync(hsq.data(), sq, n * 8, cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaStreamSynchronize(st));
  double dmax = 0.0, smax = 0.0;
  for (int64_t c = 0; c < n; ++c) {
    dmax = std::max(dmax, std::fabs(hden[c]));
    smax = std::max(smax, hsq[c]);
  }
  const double thr = 1e-14 * std::max(dmax, 1.0);
  std::vector<uint8_t> hsc(n);
  for (int64_t c = 0; c < n; ++c) hsc[c] = hden[c] > thr;
  CNMF_CUDA(cudaMemcpyAsync(scorable, hsc.data(), n, cudaMemcpyHostToDevice, st));
  const double fl = std::sqrt(smax) * 1e-14, floor = fl * fl;
  std::vector<int64_t> hp;
  int status = CNMF_OK;
  auto argmax = [&](const double* v, const uint8_t* valid, double* bv, int64_t* bi) -> int {
    argmax_unpicked<<<agrid, kSelThreads, 0, st>>>(v, n, picked, valid, blk_v, blk_i);
    CNMF_LAUNCH_CHECK();
    std::vector<double> vv(agrid);
    std::vector<int64_t> ii(agrid);
    CNMF_CUDA(cudaMemcpyAsync(vv.data(), blk_v, agrid * 8, cudaMemcpyDeviceToHost, st));
    CNMF_CUDA(cudaMemcpyAsync(ii.data(), blk_i, agrid * 8, cudaMemcpyDeviceToHost, st));
    CNMF_CUDA(cudaStreamSynchronize(st));
    double gv = -DBL_MAX;
    int64_t gi = INT64_MAX;
    for (unsigned b = 0; b < agrid; ++b)
      if (vv[b] > gv || (vv[b] == gv && ii[b] < gi)) {
        gv = vv[b];
        gi = ii[b];
      }
    *bv = gv;
    *bi = gi;
    return CNMF_OK;
  };
  for (int t = 0; t < r; ++t) {
    double v;
    int64_t j;
    CNMF_TRY(argmax(sq, nullptr, &v, &j));
    if (!(v > floor)) {
      status = fail(CNMF_ERR_RANK_DEFICIENCY, "only " + std::to_string(hp.size()) +
                                                  " numerically independent columns found");
      break;
    }
    CNMF_CUDA(cudaMemcpyAsync(d_picks + t, &j, 8, cudaMemcpyHostToDevice, st));
    xray_scores<<<grid, kSelThreads, 0, st>>>(W, R, n, s, ld, d_picks + t, denom, score);
    CNMF_LAUNCH_CHECK();
    int64_t i;
    CNMF_TRY(argmax(score, scorable, &v, &i));
    if (!(v > -DBL_MAX) || !std::isfinite(v)) {
      status = fail(CNMF_ERR_RANK_DEFICIENCY, "no scorable columns left");
      break;
    }
    hp.push_back(i);
    CNMF_CUDA(cudaMemcpyAsync(d_picks, hp.data(), hp.size() * 8, cudaMemcpyHostToDevice, st));
    const uint8_t one = 1;
    CNMF_CUDA(cudaMemcpyAsync(picked + i, &one, 1, cudaMemcpyHostToDevice, st));
    int64_t capped = 0;
    // warm start from the previous refit (the picks only grew by one): the
    // same unique minimiser, a fraction of the exchanges (tools/xray_profile.py)
    CNMF_TRY(right_factor(W, n, s, ld, d_picks, (int)hp.size(), nnls_tol, Ht, scratch, &capped, st,
                          hp.size() > 1 && xray_warm() ? Hprev : nullptr, (int)hp.size() - 1, fstate, fstride, r));
    CNMF_TRY(refit_norms(W, n, s, ld, d_picks, (int)hp.size(), Ht, R, sq, nullptr, st));
    std::swap(Ht, Hprev);  // Hprev = this refit
  }
  if (status == CNMF_OK && (int)hp.size() == r && xray_warm()) {
    // keep the final refit (Hprev after the swap) for the right factor
    void* keep = nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        device_scratch("xray-last-H", (size_t)n * r * 8, &keep, st) == CNMF_OK &&
        cudaMemcpyAsync(keep, Hprev, (size_t)n * r * 8, cudaMemcpyDeviceToDevice, st) == cudaSuccess) {
      std::lock_guard<std::mutex> lk(g_xray_last_mu);
      XrayLast& e = g_xray_last[dev];
      e.W = W;
      e.n = n;
      e.ld = ld;
      e.s = s;
      e.k = r;
      e.tol = nnls_tol;
      e.picks = hp;
      e.H = (const double*)keep;
    }
  }
  CNMF_CUDA(cudaStreamSynchronize(st));
  CNMF_CUDA(cudaFreeAsync(buf, st));
  for (size_t a = 0; a < hp.size(); ++a) picks_host[a] = hp[a];
  *n_picks = (int)hp.size();
  return status;
}

// right_factor started from the last XRAY refit when it solved this very
// problem (same reduced matrix, picks in the same order, tolerance)
int right_factor_after_selection(const double* W, int64_t n, int s, int64_t ld, const int64_t* d_picks, int k,
                                 double tol, double* Ht, double* scratch, int64_t* n_capped, cudaStream_t st) {
  const double* H0 = nullptr;
  int dev = 0;
  if (xray_warm() && cudaGetDevice(&dev) == cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_xray_last_mu);
    auto it = g_xray_last.find(dev);
    if (it != g_xray_last.end() && it->second.W == W && it->second.n == n && it->second.ld == ld &&
        it->second.s == s && it->second.k == k && it->second.tol == tol) {
      std::vector<int64_t> hp(k);
      CNMF_CUDA(cudaMemcpyAsync(hp.data(), d_picks, (size_t)k * 8, cudaMemcpyDeviceToHost, st));
      CNMF_CUDA(cudaStreamSynchronize(st));
      if (hp == it->second.picks) H0 = it->second.H;
    }
  }
  return right_factor(W, n, s, ld, d_picks, k, tol, Ht, scratch, n_capped, st, H0, H0 ? k : 0);
}

}  // namespace cnmf

namespace cnmf {
namespace {

// out (a x b) = X^T Y for row-aligned fp64 matrices X (p x a), Y (p x b).
__global__ void gram_tn_f64_kernel(const double* __restrict__ X, int64_t p, int a, const double* __restrict__ Y, int b,
                                   double* __restrict__ out) {
  constexpr int T = 16;
  __shared__ double xs[32][T + 1];
  __shared__ double ys[32][T + 1];
  const int ty = threadIdx.y, tx = threadIdx.x;  // 16 x 16
  const int i0 = blockIdx.y * T, j0 = blockIdx.x * T;
  double acc = 0.0;
  for (int64_t k0 = (int64_t)blockIdx.z * 32; k0 < p; k0 += (int64_t)gridDim.z * 32) {
    for (int q = ty; q < 32; q += T) {
      const int64_t row = k0 + q;
      xs[q][tx] = (row < p && i0 + tx < a) ? X[row * a + i0 + tx] : 0.0;
      ys[q][tx] = (row < p && j0 + tx < b) ? Y[row * b + j0 + tx] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int q = 0; q < 32; ++q) acc = fma(xs[q][ty], ys[q][tx], acc);
    __syncthreads();
  }
  if (i0 + ty < a && j0 + tx < b) atomicAdd(&out[(int64_t)(i0 + ty) * b + j0 + tx], acc);
}

}  // namespace

int gram_tn_f64(const double* X, int64_t p, int a, const double* Y, int b, double* out, cudaStream_t st) {
  CNMF_CUDA(cudaMemsetAsync(out, 0, (size_t)a * b * 8, st));
  const int64_t tiles = ceil_div(a, 16) * ceil_div(b, 16);
  const int64_t z = std::max<int64_t>(1, std::min<int64_t>(ceil_div(p, 32), (4 * kNumSMs + tiles - 1) / tiles));
  gram_tn_f64_kernel<<<dim3((unsigned)ceil_div(b, 16), (unsigned)ceil_div(a, 16), (unsigned)z), dim3(16, 16), 0,
                       st>>>(X, p, a, Y, b, out);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

}  // namespace cnmf

extern "C" int cnmf_gram_f64(const double* X, int64_t p, int a, const double* Y, int b, double* out, void* stream) {
  if (p < 1 || a < 1 || b < 1) return cnmf::fail(CNMF_ERR_ARGUMENT, "gram_f64 needs positive sizes");
  return cnmf::gram_tn_f64(X, p, a, Y, b, out, reinterpret_cast<cudaStream_t>(stream));
}
