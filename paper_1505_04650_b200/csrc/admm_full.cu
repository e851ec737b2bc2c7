// The uncompressed ADMM NMF of nmf.py:306-377 (compressed=False: identity
// bases, a_comp = A itself) on the device, for r <= 32.
//
// Every iteration needs A yc^T (m x r) and A^T xc (n x r): the same skinny
// products as the range finder, so they run on the streaming pass kernels
// (csrc/tc_pass.cu, fp32 panels, 3xTF32) and A is read twice per iteration.
// Everything else is row-wise over the m x r and n x r iterates (fp64, the
// reference's precision) plus r x r Gram matrices and their ridge inverses,
// done by three grid-stride kernels per iteration whose last block to finish
// folds the block partials and runs the r x r step (no grid barrier):
//
//   pass_forward   Y  = A P(yc^T)                      (m x S fp32)
//   full_kkt       grad_left of the previous iteration = ||xc Gy - Y + du||
//                  (A yc^T of the previous yc is exactly this Y); its last
//                  block completes that iteration's KKT score (nmf.py:281-303)
//                  and decides tol / divergence (nmf.py:367-375)
//   full_left      xc = (Y + pu u - du) (Gy + pu I)^-1, u, du; Gx = xc^T xc;
//                  last block: Hx = (Gx + pv I)^-1
//   pass_transpose Z  = A^T P(xc)                      (n x S fp32)
//   full_right     yc^T = (Z + pv v^T - dv^T) Hx, v, dv; Gy = yc yc^T, grad/
//                  feasibility/complementarity of the right side; last block:
//                  Hy = (Gy + pu I)^-1 and the objective ||A - xc yc||^2 =
//                  ||A||^2 - 2 <yc^T, Z> + <Gx, Gy> (nmf.py:362)
//
// Kernels after the stop decision return immediately (the passes still run;
// their outputs are not read).
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "pass.cuh"

namespace cnmf {
namespace {

constexpr int kR = 32;        // lanes = columns of the iterates (r <= 32)
constexpr int kThreads = 256;  // 8 warps, one row per warp at a time
constexpr int kB = 4;          // rows whose loads a warp keeps in flight together

struct FullCtrl {
  unsigned ticket[3];  // last-block detection of full_kkt / full_left / full_right
  int done;            // 1 once the run has stopped
  int iters;           // iterations completed (reference's `iterations`)
  int diverged;        // iteration index that diverged, -1 if none
  int k;               // iterations whose updates have run
  int pad;
  double nA2;          // ||A||_F^2
  double part[5];      // feas_left, comp_left, grad_right, feas_right, comp_right of iteration k - 1
  double acc[8];       // block-partial sums of the running kernels
};

struct FullMats {
  double Gy[kR * kR];  // yc yc^T of the latest right update (finalised)
  double Gx[kR * kR];  // xc^T xc of the latest left update (finalised)
  double Hy[kR * kR];  // (Gy + pu I)^-1
  double Hx[kR * kR];  // (Gx + pv I)^-1
  double accG[kR * kR];  // block partials of the Gram being accumulated
};

struct FullArgs {
  int64_t m, n;
  int r, S;
  double pu, pv, step, tol;
  int max_iter;
  double *u, *du, *vt, *dvt, *xc, *yct;
  float *Pyc, *Pxc, *Y, *Z;
  double *trace, *scores;
  FullCtrl* ctrl;
  FullMats* mats;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// x (one value per lane) times the r x r matrix H in shared memory: lane j
// returns sum_l x_l H[l][j]
__device__ __forceinline__ double row_times(double x, const double* H, int r, int lane) {
  double acc = 0.0;
  for (int l = 0; l < r; ++l) acc = fma(__shfl_sync(0xffffffffu, x, l), H[l * kR + lane], acc);
  return acc;
}

// lane j accumulates row j of x^T x (g[l] += x_j x_l)
__device__ __forceinline__ void gram_acc(double (&g)[kR], double x, int r) {
#pragma unroll
  for (int l = 0; l < kR; ++l) {
    const double xl = __shfl_sync(0xffffffffu, x, l);
    if (l < r) g[l] = fma(x, xl, g[l]);
  }
}

// the block's warps add their Gram rows into blk (r x r, stride kR) in turn:
// plain shared-memory adds, no atomics
__device__ __forceinline__ void block_gram(double* blk, const double (&g)[kR], int r, int lane, int warp) {
  for (int w = 0; w < kThreads / 32; ++w) {
    if (warp == w && lane < r)
#pragma unroll
      for (int l = 0; l < kR; ++l)
        if (l < r) blk[lane * kR + l] += g[l];
    __syncthreads();
  }
}

// (G + ridge I)^-1 of an SPD r x r matrix by Gauss-Jordan in shared memory
// (one block; the ridge keeps every pivot >= ridge > 0)
__device__ void ridge_inverse(const double* G, double ridge, int r, double* H, double* w) {
  // w: r x 2r work matrix [G + ridge I | I]
  const int tid = threadIdx.x;
  const int W = 2 * r;
  for (int idx = tid; idx < r * W; idx += blockDim.x) {
    const int i = idx / W, j = idx - i * W;
    w[idx] = j < r ? G[i * kR + j] + (i == j ? ridge : 0.0) : (j - r == i ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    const double inv = 1.0 / w[k * W + k];
    __syncthreads();
    // scale row k, then eliminate column k from the other rows
    for (int j = tid; j < W; j += blockDim.x) w[k * W + j] *= inv;
    __syncthreads();
    for (int idx = tid; idx < r * W; idx += blockDim.x) {
      const int i = idx / W, j = idx - i * W;
      if (i != k) {
        const double f = w[i * W + k];
        if (j != k) w[idx] = fma(-f, w[k * W + j], w[idx]);
      }
    }
    __syncthreads();
    for (int i = tid; i < r; i += blockDim.x)
      if (i != k) w[i * W + k] = 0.0;
    __syncthreads();
  }
  for (int idx = tid; idx < kR * kR; idx += blockDim.x) {
    const int i = idx / kR, j = idx - i * kR;
    H[idx] = (i < r && j < r) ? w[i * W + r + j] : 0.0;
  }
  __syncthreads();
}

// block partials -> global accumulators; returns true in the last block
// (which then sees every block's contribution)
__device__ bool fold_block(double* sblk, int nvals, double* gacc, unsigned* ticket) {
  __syncthreads();
  for (int i = threadIdx.x; i < nvals; i += blockDim.x)
    if (sblk[i] != 0.0) atomicAdd(gacc + i, sblk[i]);
  __threadfence();
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    if (threadIdx.x == 0) *ticket = 0;
  }
  return last;
}

__device__ __forceinline__ bool stopped(const FullCtrl* c) { return *(volatile const int*)&c->done; }

// ---------------------------------------------------------------------------
// grad_left of iteration k - 1 and the stop decision
__global__ void __launch_bounds__(kThreads) full_kkt(FullArgs a) {
  FullCtrl* c = a.ctrl;
  if (stopped(c)) return;
  __shared__ double Gy[kR * kR];
  __shared__ double sum[1];
  for (int i = threadIdx.x; i < kR * kR; i += blockDim.x) Gy[i] = a.mats->Gy[i];
  if (threadIdx.x == 0) sum[0] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = a.r;
  double g2 = 0.0;
  const int64_t stride = (int64_t)gridDim.x * 8;
  for (int64_t i0 = (int64_t)blockIdx.x * 8 + warp; i0 < a.m; i0 += kB * stride) {
    double x4[kB], y4[kB], d4[kB];  // loads of kB rows in flight together
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int64_t i = i0 + q * stride;
      const bool ok = lane < r && i < a.m;
      x4[q] = ok ? a.xc[i * r + lane] : 0.0;
      y4[q] = ok ? (double)a.Y[i * a.S + lane] : 0.0;
      d4[q] = ok ? a.du[i * r + lane] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const double t = row_times(x4[q], Gy, r, lane);
      const double g = t - y4[q] + d4[q];  // zero for padding lanes and rows past m
      g2 = fma(g, g, g2);
    }
  }
  g2 = warp_sum(g2);
  if (lane == 0) atomicAdd(&sum[0], g2);
  if (!fold_block(sum, 1, c->acc + 0, &c->ticket[0])) return;
  if (threadIdx.x == 0) {
    const int k = c->k - 1;  // the iteration being scored
    volatile double* acc = c->acc;
    double score = sqrt(acc[0]);
    for (int q = 0; q < 5; ++q) score = fmax(score, c->part[q]);
    c->acc[0] = 0.0;
    a.scores[k] = score;
    if (score < a.tol) {
      c->done = 1;
      c->iters = k + 1;
    } else if (k >= 50 && score > 10.0 * a.scores[k - 50]) {
      c->done = 1;
      c->iters = k + 1;
      c->diverged = k;
    } else if (k + 1 >= a.max_iter) {
      c->done = 1;
      c->iters = k + 1;
    }
  }
}

// xc, u, du, Gx; last block: Hx
__global__ void __launch_bounds__(kThreads) full_left(FullArgs a) {
  FullCtrl* c = a.ctrl;
  if (stopped(c)) return;
  __shared__ double Hy[kR * kR];
  __shared__ double blk[kR * kR + 2];
  __shared__ double work[kR * 2 * kR];
  for (int i = threadIdx.x; i < kR * kR; i += blockDim.x) {
    Hy[i] = a.mats->Hy[i];
    blk[i] = 0.0;
  }
  if (threadIdx.x < 2) blk[kR * kR + threadIdx.x] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = a.r;
  double g[kR];
#pragma unroll
  for (int l = 0; l < kR; ++l) g[l] = 0.0;
  double feas = 0.0, comp = 0.0;
  const int64_t stride = (int64_t)gridDim.x * 8;
  const bool on = lane < r;
  for (int64_t i0 = (int64_t)blockIdx.x * 8 + warp; i0 < a.m; i0 += kB * stride) {
    double y4[kB], u4[kB], d4[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int64_t i = i0 + q * stride;
      const bool ok = on && i < a.m;
      y4[q] = ok ? (double)a.Y[i * a.S + lane] : 0.0;
      u4[q] = ok ? a.u[i * r + lane] : 0.0;
      d4[q] = ok ? a.du[i * r + lane] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int64_t i = i0 + q * stride;
      if (i >= a.m) break;  // warp-uniform
      const double rhs = y4[q] + a.pu * u4[q] - d4[q];
      const double x = row_times(rhs, Hy, r, lane);
      gram_acc(g, on ? x : 0.0, r);
      a.Pxc[i * a.S + lane] = on ? (float)x : 0.f;
      if (on) {
        const double du0 = d4[q];
        const double un = fmax(x + du0 / a.pu, 0.0);
        const double dun = du0 + a.step * a.pu * (x - un);
        a.xc[i * r + lane] = x;
        a.u[i * r + lane] = un;
        a.du[i * r + lane] = dun;
        feas = fma(x - un, x - un, feas);
        const double p = fmax(dun, 0.0);
        comp += (dun * un) * (dun * un) + p * p;  // neg(u) = 0: u is a projection
      }
    }
  }
  block_gram(blk, g, r, lane, warp);
  feas = warp_sum(feas);
  comp = warp_sum(comp);
  if (lane == 0) {
    atomicAdd(&blk[kR * kR], feas);
    atomicAdd(&blk[kR * kR + 1], comp);
  }
  // Gram partials into accG, the two sums into acc[1..2]
  __syncthreads();
  for (int i = threadIdx.x; i < kR * kR; i += blockDim.x)
    if (blk[i] != 0.0) atomicAdd(&a.mats->accG[i], blk[i]);
  if (threadIdx.x < 2 && blk[kR * kR + threadIdx.x] != 0.0) atomicAdd(&c->acc[1 + threadIdx.x], blk[kR * kR + threadIdx.x]);
  __shared__ double none[1];
  if (threadIdx.x == 0) none[0] = 0.0;
  if (!fold_block(none, 1, c->acc + 7, &c->ticket[1])) return;
  for (int i = threadIdx.x; i < kR * kR; i += blockDim.x) {
    a.mats->Gx[i] = __ldcg(&a.mats->accG[i]);
    a.mats->accG[i] = 0.0;
  }
  __syncthreads();
  ridge_inverse(a.mats->Gx, a.pv, r, a.mats->Hx, work);
  if (threadIdx.x == 0) {
    volatile double* acc = c->acc;
    c->part[0] = sqrt(acc[1]);
    c->part[1] = sqrt(acc[2]);
    c->acc[1] = c->acc[2] = 0.0;
  }
}

// yc^T, v, dv, Gy, right-side KKT terms; last block: Hy and the objective
__global__ void __launch_bounds__(kThreads) full_right(FullArgs a, int init) {
  FullCtrl* c = a.ctrl;
  if (stopped(c)) return;
  __shared__ double Hx[kR * kR];
  __shared__ double Gx[kR * kR];
  __shared__ double blk[kR * kR + 4];
  __shared__ double work[kR * 2 * kR];
  for (int i = threadIdx.x; i < kR * kR; i += blockDim.x) {
    Hx[i] = a.mats->Hx[i];
    Gx[i] = a.mats->Gx[i];
    blk[i] = 0.0;
  }
  if (threadIdx.x < 4) blk[kR * kR + threadIdx.x] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = a.r;
  const bool on = lane < r;
  double g[kR];
#pragma unroll
  for (int l = 0; l < kR; ++l) g[l] = 0.0;
  double yz = 0.0, grad = 0.0, feas = 0.0, comp = 0.0;
  const int64_t stride = (int64_t)gridDim.x * 8;
  for (int64_t j0 = (int64_t)blockIdx.x * 8 + warp; j0 < a.n; j0 += kB * stride) {
    double z4[kB], v4[kB], d4[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int64_t j = j0 + q * stride;
      const bool ok = on && j < a.n;
      z4[q] = ok && !init ? (double)a.Z[j * a.S + lane] : 0.0;
      v4[q] = ok ? a.vt[j * r + lane] : 0.0;
      d4[q] = ok && !init ? a.dvt[j * r + lane] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int64_t j = j0 + q * stride;
      if (j >= a.n) break;  // warp-uniform
      double y;
      if (init) {  // the start: yc = v (identity right basis, nmf.py:342)
        y = v4[q];
        if (on) a.yct[j * r + lane] = y;
      } else {
        const double z = z4[q];
        const double rhs = z + a.pv * v4[q] - d4[q];
        y = row_times(rhs, Hx, r, lane);
        const double t = row_times(y, Gx, r, lane);  // (yc^T Gx)_j
        if (on) {
          const double dv0 = d4[q];
          const double vn = fmax(y + dv0 / a.pv, 0.0);
          const double dvn = dv0 + a.step * a.pv * (y - vn);
          a.yct[j * r + lane] = y;
          a.vt[j * r + lane] = vn;
          a.dvt[j * r + lane] = dvn;
          yz = fma(y, z, yz);
          const double gr = t - z + dvn;
          grad = fma(gr, gr, grad);
          feas = fma(y - vn, y - vn, feas);
          const double p = fmax(dvn, 0.0);
          comp += (dvn * vn) * (dvn * vn) + p * p;
        }
      }
      gram_acc(g, on ? y : 0.0, r);
      a.Pyc[j * a.S + lane] = on ? (float)y : 0.f;
    }
  }
  block_gram(blk, g, r, lane, warp);
  const double sums[4] = {warp_sum(yz), warp_sum(grad), warp_sum(feas), warp_sum(comp)};
  if (lane == 0)
    for (int q = 0; q < 4; ++q) atomicAdd(&blk[kR * kR + q], sums[q]);
  __syncthreads();
  for (int i = threadIdx.x; i < kR * kR; i += blockDim.x)
    if (blk[i] != 0.0) atomicAdd(&a.mats->accG[i], blk[i]);
  if (threadIdx.x < 4 && blk[kR * kR + threadIdx.x] != 0.0)
    atomicAdd(&c->acc[3 + threadIdx.x], blk[kR * kR + threadIdx.x]);
  __shared__ double none[1];
  if (threadIdx.x == 0) none[0] = 0.0;
  if (!fold_block(none, 1, c->acc + 7, &c->ticket[2])) return;
  for (int i = threadIdx.x; i < kR * kR; i += blockDim.x) {
    a.mats->Gy[i] = __ldcg(&a.mats->accG[i]);
    a.mats->accG[i] = 0.0;
  }
  __syncthreads();
  ridge_inverse(a.mats->Gy, a.pu, r, a.mats->Hy, work);
  if (threadIdx.x == 0) {
    volatile double* acc = c->acc;
    if (!init) {
      double gg = 0.0;
      for (int i = 0; i < r; ++i)
        for (int l = 0; l < r; ++l) gg = fma(a.mats->Gx[i * kR + l], a.mats->Gy[i * kR + l], gg);
      // the expansion cancels for well-fitted data (absolute error ~1e-7 ||A||^2,
      // DESIGN.md): a squared norm is never negative
      a.trace[c->k] = fmax(c->nA2 - 2.0 * acc[3] + gg, 0.0);
      c->part[2] = sqrt(acc[4]);
      c->part[3] = sqrt(acc[5]);
      c->part[4] = sqrt(acc[6]);
      c->k += 1;
    }
    for (int q = 3; q < 7; ++q) c->acc[q] = 0.0;
  }
}

// ||A||_F^2 in fp64
__global__ void __launch_bounds__(kThreads) full_norm(const float* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                                       FullCtrl* c) {
  double s = 0.0;
  const int64_t total = m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    const double v = A[i * lda + j];
    s = fma(v, v, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) atomicAdd(&c->nA2, s);
}

__global__ void full_init_ctrl(FullCtrl* c) {
  c->ticket[0] = c->ticket[1] = c->ticket[2] = 0;
  c->done = 0;
  c->iters = 0;
  c->diverged = -1;
  c->k = 0;
  c->nA2 = 0.0;
  for (int q = 0; q < 5; ++q) c->part[q] = 0.0;
  for (int q = 0; q < 8; ++q) c->acc[q] = 0.0;
}

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

}  // namespace

size_t admm_full_workspace(int64_t m, int64_t n, int r) {
  (void)r;
  const int S = 32;
  return align256(sizeof(FullCtrl)) + align256(sizeof(FullMats)) + 2 * align256((size_t)m * S * 4) +
         2 * align256((size_t)n * S * 4);
}

int admm_full_run(const float* A, int64_t m, int64_t n, int64_t lda, int r, double* u, double* du, double* vt,
                  double* dvt, double* xc, double* yct, double pu, double pv, double step, int max_iter, double tol,
                  double* trace, double* scores, int* iterations, int* done, int resume, int step_limit, void* ws,
                  size_t ws_bytes, cudaStream_t st) {
  if (r < 1 || r > kR) return fail(CNMF_ERR_ARGUMENT, "the uncompressed device ADMM supports 1 <= r <= 32");
  if (!(pu > 0) || !(pv > 0)) return fail(CNMF_ERR_ARGUMENT, "penalties must be positive");
  if (ws_bytes < admm_full_workspace(m, n, r)) return fail(CNMF_ERR_ARGUMENT, "workspace too small");
  const int S = 32;
  char* p = (char*)ws;
  FullArgs a;
  a.ctrl = (FullCtrl*)p;
  p += align256(sizeof(FullCtrl));
  a.mats = (FullMats*)p;
  p += align256(sizeof(FullMats));
  a.Pxc = (float*)p;
  p += align256((size_t)m * S * 4);
  a.Y = (float*)p;
  p += align256((size_t)m * S * 4);
  a.Pyc = (float*)p;
  p += align256((size_t)n * S * 4);
  a.Z = (float*)p;
  a.m = m;
  a.n = n;
  a.r = r;
  a.S = S;
  a.pu = pu;
  a.pv = pv;
  a.step = step;
  a.tol = tol;
  a.max_iter = max_iter;
  a.u = u;
  a.du = du;
  a.vt = vt;
  a.dvt = dvt;
  a.xc = xc;
  a.yct = yct;
  a.trace = trace;
  a.scores = scores;
  // one block per SM (210 registers per thread: one resident block), each
  // warp >= 4 rows (one batch of kB loads); every block adds one r x r Gram
  // partial to the same r^2 global words
  const unsigned gl = (unsigned)std::max<int64_t>(1, std::min<int64_t>(kNumSMs, ceil_div(m, 32)));
  const unsigned gr = (unsigned)std::max<int64_t>(1, std::min<int64_t>(kNumSMs, ceil_div(n, 32)));
  if (!resume) {
    full_init_ctrl<<<1, 1, 0, st>>>(a.ctrl);
    CNMF_LAUNCH_CHECK();
    CNMF_CUDA(cudaMemsetAsync(a.mats, 0, sizeof(FullMats), st));
    CNMF_CUDA(cudaMemsetAsync(du, 0, (size_t)m * r * 8, st));
    CNMF_CUDA(cudaMemsetAsync(dvt, 0, (size_t)n * r * 8, st));
    CNMF_CUDA(cudaMemsetAsync(xc, 0, (size_t)m * r * 8, st));
    full_norm<<<2 * kNumSMs, kThreads, 0, st>>>(A, m, n, lda, a.ctrl);
    CNMF_LAUNCH_CHECK();
    full_right<<<gr, kThreads, 0, st>>>(a, 1);  // yc = v, Gy, Hy, P(yc^T)
    CNMF_LAUNCH_CHECK();
  }
  FullCtrl hc;
  auto sync_ctrl = [&]() -> int {
    CNMF_CUDA(cudaMemcpyAsync(&hc, a.ctrl, sizeof(FullCtrl), cudaMemcpyDeviceToHost, st));
    CNMF_CUDA(cudaStreamSynchronize(st));
    return CNMF_OK;
  };
  // one iteration on stream s: Y = A yc^T, the previous iteration's score,
  // then the updates (which return at once after a stop)
  auto iteration = [&](cudaStream_t s, bool score) -> int {
    CNMF_TRY(pass_forward(A, m, n, lda, a.Pyc, S, a.Y, s));
    if (score) {
      full_kkt<<<gl, kThreads, 0, s>>>(a);
      CNMF_LAUNCH_CHECK();
    }
    full_left<<<gl, kThreads, 0, s>>>(a);
    CNMF_LAUNCH_CHECK();
    CNMF_TRY(pass_transpose(A, m, n, lda, a.Pxc, S, a.Z, s));
    full_right<<<gr, kThreads, 0, s>>>(a, 0);
    CNMF_LAUNCH_CHECK();
    return CNMF_OK;
  };
  CNMF_TRY(sync_ctrl());
  int k = hc.k;
  int steps = 0;
  // a run to completion replays 8 iterations per CUDA graph launch (the
  // kernels read the iteration index from the control block), checking the
  // stop flag between launches
  constexpr int kChunk = 8;
  if (step_limit == 0 && !hc.done && k == 0 && max_iter > 2 * kChunk) {  // the first iteration has no score
    CNMF_TRY(iteration(st, false));
    ++k;
  }
  if (step_limit == 0 && !hc.done && k > 0 && max_iter - k >= 2 * kChunk) {
    cudaStream_t cs;
    CNMF_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    CNMF_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    int rc = CNMF_OK;
    for (int g = 0; g < kChunk && rc == CNMF_OK; ++g) rc = iteration(cs, true);
    const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
    if (rc == CNMF_OK && ce == cudaSuccess) {
      CNMF_CUDA(cudaGraphInstantiate(&exec, graph, 0));
      while (!hc.done && max_iter - k >= kChunk) {
        CNMF_CUDA(cudaGraphLaunch(exec, st));
        k += kChunk;
        CNMF_TRY(sync_ctrl());
      }
      cudaGraphExecDestroy(exec);
    }
    if (graph) cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
    CNMF_TRY(rc);
    if (ce != cudaSuccess) return fail(CNMF_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    if (!hc.done) k = hc.k;
  }
  while (!hc.done) {
    if (k >= max_iter) {  // only the last score is still owed
      CNMF_TRY(pass_forward(A, m, n, lda, a.Pyc, S, a.Y, st));
      full_kkt<<<gl, kThreads, 0, st>>>(a);
      CNMF_LAUNCH_CHECK();
      CNMF_TRY(sync_ctrl());
      break;
    }
    CNMF_TRY(iteration(st, k > 0));
    ++k;
    ++steps;
    const bool pause = step_limit > 0 && steps >= step_limit;
    if (pause || (k & 7) == 0) {
      CNMF_TRY(sync_ctrl());
      k = hc.done ? k : hc.k;
      if (pause) break;
    }
  }
  if (done) *done = hc.done;
  if (iterations) *iterations = hc.done ? hc.iters : hc.k;
  if (hc.diverged >= 0) {
    if (iterations) *iterations = hc.diverged + 1;
    return fail(CNMF_ERR_DIVERGENCE, "KKT residual grew 10x over 50 iterations at iteration " +
                                         std::to_string(hc.diverged));
  }
  return CNMF_OK;
}

}  // namespace cnmf
