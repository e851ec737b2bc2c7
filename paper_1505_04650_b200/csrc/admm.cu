// Compressed ADMM NMF (reference nmf.py:306-377, KKT residual nmf.py:281-303).
//
// Per iteration two launches:
//   core kernel (one CTA): finishes the previous iteration's KKT score from
//     the reduced partials and applies the stopping / divergence rules on the
//     device, then solves the two r x r ridge systems for Xc and Yc
//     (Cholesky by one warp, triangular solves by all threads) and records
//     the compressed objective ||L^T A R^T - Xc Yc||^2;
//   split kernel (all SMs): one fused sweep over the rows of L and of R^T
//     that forms L Xc (resp. Yc R), projects onto the nonnegative orthant,
//     takes the dual step and accumulates every reduction the next core step
//     needs (L^T U, L^T dU, V R^T, dV R^T, feasibility and complementarity
//     sums) — U, V, dU, dV are each read and written exactly once.
// The state is fp64 (the method is sensitive to roundoff over hundreds of
// iterations); the bases are the fp32 panels produced by the compression.
// Batches of iterations are captured once into a CUDA graph and replayed;
// a device flag turns the remaining kernels into no-ops after convergence, so
// the iteration count is exactly the reference's.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace cnmf {
int64_t launch_count();
namespace {

constexpr int kAdmmMax = 64;  // s, r <= 64
constexpr int kTile = 64;     // rows per split-kernel tile
constexpr int kSplitThreads = 256;

struct Ctrl {
  int k;         // next iteration index
  int done;
  int iters;     // iterations completed when done
  int diverged;  // iteration index (0-based) that tripped the divergence rule, or -1
};

// reduced partials written by the split kernel for one iteration
struct Acc {
  double LtU[kAdmmMax * kAdmmMax];   // s x r : L^T U
  double LtDU[kAdmmMax * kAdmmMax];  // s x r : L^T dU
  double RtV[kAdmmMax * kAdmmMax];   // s x r : R V^T   (= (V R^T)^T)
  double RtDV[kAdmmMax * kAdmmMax];  // s x r : R dV^T
  double scal[4];                    // feasL^2, compL^2, feasR^2, compR^2
};

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Cholesky of the r x r SPD matrix M (row-major, stride r) in place (lower
// factor in the lower triangle) by warp 0.
__device__ void warp_cholesky(double* M, int r) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < r; ++k) {
    const double d = sqrt(M[k * r + k]);
    __syncwarp();
    for (int i = k + 1 + lane; i < r; i += 32) M[i * r + k] /= d;
    if (lane == 0) M[k * r + k] = d;
    __syncwarp();
    for (int i = k + 1 + lane; i < r; i += 32) {
      const double lik = M[i * r + k];
      for (int j = k + 1; j <= i; ++j) M[i * r + j] -= lik * M[j * r + k];
    }
    __syncwarp();
  }
}

// x = M^{-1} b for a lower Cholesky factor (row-major, stride r), in place.
__device__ void chol_solve_vec(const double* L, int r, double* x, int stride) {
  for (int i = 0; i < r; ++i) {
    double v = x[i * stride];
    for (int j = 0; j < i; ++j) v -= L[i * r + j] * x[j * stride];
    x[i * stride] = v / L[i * r + i];
  }
  for (int i = r - 1; i >= 0; --i) {
    double v = x[i * stride];
    for (int j = i + 1; j < r; ++j) v -= L[j * r + i] * x[j * stride];
    x[i * stride] = v / L[i * r + i];
  }
}

__global__ void __launch_bounds__(512)
    admm_core(const double* __restrict__ core, int s, int r, double pu, double pv, int max_iter, double tol,
              Ctrl* ctrl, Acc* acc, double* __restrict__ xc_g, double* __restrict__ yc_g, double* __restrict__ trace,
              double* __restrict__ scores) {
  extern __shared__ double sm[];
  double* C = sm;                    // s x s core
  double* xc = C + s * s;            // s x r
  double* yc = xc + s * r;           // r x s
  double* W = yc + r * s;            // s x s scratch (E) / r x s rhs
  double* M = W + s * s;             // r x r
  __shared__ double red[16][6];
  __shared__ int s_stop;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (ctrl->done) return;
  const int k = ctrl->k;
  for (int i = tid; i < s * s; i += nt) C[i] = core[i];
  for (int i = tid; i < s * r; i += nt) {
    xc[i] = xc_g[i];
    yc[i] = yc_g[i];
  }
  if (tid == 0) s_stop = 0;
  __syncthreads();
  if (k == 0) {
    // yc = V R^T (nmf.py:342)
    for (int i = tid; i < r * s; i += nt) {
      const int a = i / s, j = i % s;
      yc[i] = acc->RtV[j * r + a];
    }
    __syncthreads();
  } else {
    // ---- KKT score of iteration k-1 (nmf.py:281-303, 365-374) ----
    // E = xc yc - C
    for (int i = tid; i < s * s; i += nt) {
      const int a = i / s, b = i % s;
      double v = -C[i];
      for (int q = 0; q < r; ++q) v += xc[a * r + q] * yc[q * s + b];
      W[i] = v;
    }
    __syncthreads();
    double g1 = 0.0, g2 = 0.0;
    // grad_left = E yc^T + L^T dU  (s x r)
    for (int i = tid; i < s * r; i += nt) {
      const int a = i / r, q = i % r;
      double v = acc->LtDU[a * r + q];
      for (int b = 0; b < s; ++b) v += W[a * s + b] * yc[q * s + b];
      g1 += v * v;
    }
    // grad_right = xc^T E + dV R^T  (r x s)
    for (int i = tid; i < r * s; i += nt) {
      const int q = i / s, b = i % s;
      double v = acc->RtDV[b * r + q];
      for (int a = 0; a < s; ++a) v += xc[a * r + q] * W[a * s + b];
      g2 += v * v;
    }
    g1 = wsum(g1);
    g2 = wsum(g2);
    if (lane == 0) {
      red[warp][0] = g1;
      red[warp][1] = g2;
    }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < nt / 32; ++w) {
        a += red[w][0];
        b += red[w][1];
      }
      const double score = fmax(fmax(fmax(sqrt(a), sqrt(b)), fmax(sqrt(acc->scal[0]), sqrt(acc->scal[2]))),
                                fmax(sqrt(acc->scal[1]), sqrt(acc->scal[3])));
      scores[k - 1] = score;
      if (score < tol) {
        s_stop = 1;
      } else if (k - 1 >= 50 && score > 10.0 * scores[k - 1 - 50]) {
        s_stop = 1;
        ctrl->diverged = k - 1;
      } else if (k >= max_iter) {
        s_stop = 1;
      }
      if (s_stop) {
        ctrl->done = 1;
        ctrl->iters = k;
      }
    }
    __syncthreads();
    if (s_stop) return;
  }
  // ---- Xc: solve (yc yc^T + pu I) xc^T = rhs^T, rhs = C yc^T + pu L^T U - L^T dU
  for (int i = tid; i < r * r; i += nt) {
    const int a = i / r, b = i % r;
    double v = (a == b) ? pu : 0.0;
    for (int j = 0; j < s; ++j) v += yc[a * s + j] * yc[b * s + j];
    M[i] = v;
  }
  for (int i = tid; i < s * r; i += nt) {
    const int a = i / r, q = i % r;
    double v = pu * acc->LtU[a * r + q] - acc->LtDU[a * r + q];
    for (int b = 0; b < s; ++b) v += C[a * s + b] * yc[q * s + b];
    xc[i] = v;  // rhs, solved in place row by row
  }
  __syncthreads();
  if (warp == 0) warp_cholesky(M, r);
  __syncthreads();
  for (int a = tid; a < s; a += nt) chol_solve_vec(M, r, xc + a * r, 1);
  __syncthreads();
  // ---- Yc: solve (xc^T xc + pv I) yc = xc^T C + pv V R^T - dV R^T
  for (int i = tid; i < r * r; i += nt) {
    const int a = i / r, b = i % r;
    double v = (a == b) ? pv : 0.0;
    for (int j = 0; j < s; ++j) v += xc[j * r + a] * xc[j * r + b];
    M[i] = v;
  }
  for (int i = tid; i < r * s; i += nt) {
    const int q = i / s, b = i % s;
    double v = pv * acc->RtV[b * r + q] - acc->RtDV[b * r + q];
    for (int a = 0; a < s; ++a) v += xc[a * r + q] * C[a * s + b];
    yc[i] = v;
  }
  __syncthreads();
  if (warp == 0) warp_cholesky(M, r);
  __syncthreads();
  for (int b = tid; b < s; b += nt) chol_solve_vec(M, r, yc + b, s);
  __syncthreads();
  // ---- objective trace ||C - xc yc||^2 (nmf.py:360)
  double t = 0.0;
  for (int i = tid; i < s * s; i += nt) {
    const int a = i / s, b = i % s;
    double v = C[i];
    for (int q = 0; q < r; ++q) v -= xc[a * r + q] * yc[q * s + b];
    t += v * v;
  }
  t = wsum(t);
  if (lane == 0) red[warp][0] = t;
  for (int i = tid; i < s * r; i += nt) {
    xc_g[i] = xc[i];
    yc_g[i] = yc[i];
  }
  // reset the partials for this iteration's split sweep
  double* z = (double*)acc;
  for (int i = tid; i < (int)(sizeof(Acc) / 8); i += nt) z[i] = 0.0;
  __syncthreads();
  if (tid == 0) {
    double a = 0.0;
    for (int w = 0; w < nt / 32; ++w) a += red[w][0];
    trace[k] = a;
    ctrl->k = k + 1;
  }
}

// One side of the split/dual sweep. For the left side P = L (m x S panel),
// X = xc (s x r); for the right side P = R^T (n x S panel), X = yc^T.
// mode 0: accumulate P^T U only (initial projection); mode 1: full update.
struct SideArgs {
  const float* P;
  int64_t rows;
  int S;
  double* U;
  double* D;
  double pen;
  double* accU;   // s x r
  double* accD;   // s x r
  double* scal;   // [feas, comp]
  int transposeX; // X read as yc (r x s) transposed
};

__device__ void split_side(const SideArgs& a, const double* Xg, int s, int r, double step, int mode, int bid,
                           int nblk, double* sm) {
  double* X = sm;                          // s x r (padded to 64 x 64)
  double* Pt = X + kAdmmMax * kAdmmMax;    // kTile x 64
  double* Ut = Pt + kTile * kAdmmMax;      // kTile x 64
  double* Dt = Ut + kTile * kAdmmMax;      // kTile x 64
  __shared__ double red[kSplitThreads / 32][2];
  const int tid = threadIdx.x;
  const int rp = (r + 3) & ~3, sp = (s + 3) & ~3;
  for (int i = tid; i < kAdmmMax * kAdmmMax; i += kSplitThreads) {
    const int j = i / kAdmmMax, b = i % kAdmmMax;
    double v = 0.0;
    if (j < s && b < r) v = a.transposeX ? Xg[b * s + j] : Xg[j * r + b];
    X[i] = v;
  }
  // accumulator block owned by this thread: rows 4*bj.., cols 4*bb..
  const int nbb = rp / 4;
  const int nbj = sp / 4;
  const int myb = tid;
  const bool own = myb < nbj * nbb;
  const int bj = own ? myb / nbb : 0, bb = own ? myb % nbb : 0;
  double au[4][4], ad[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      au[x][y] = 0.0;
      ad[x][y] = 0.0;
    }
  double feas = 0.0, comp = 0.0;
  const double invpen = 1.0 / a.pen, sp_ = step * a.pen;
  for (int64_t t0 = (int64_t)bid * kTile; t0 < a.rows; t0 += (int64_t)nblk * kTile) {
    const int nr = (int)min64(kTile, a.rows - t0);
    __syncthreads();
    for (int i = tid; i < kTile * kAdmmMax; i += kSplitThreads) {
      const int rr = i / kAdmmMax, c = i % kAdmmMax;
      const bool in = rr < nr;
      Pt[i] = (in && c < s) ? (double)a.P[(t0 + rr) * a.S + c] : 0.0;
      if (mode == 0) {
        Ut[i] = (in && c < r) ? a.U[(t0 + rr) * r + c] : 0.0;
        Dt[i] = 0.0;
      } else {
        Dt[i] = (in && c < r) ? a.D[(t0 + rr) * r + c] : 0.0;
      }
    }
    __syncthreads();
    if (mode == 1) {
      // lx = P X ; u = max(lx + d/pen, 0) ; d += step*pen*(lx - u)
      for (int i = tid; i < kTile * r; i += kSplitThreads) {
        const int rr = i / r, b = i % r;
        if (rr >= nr) continue;
        double lx = 0.0;
        for (int j = 0; j < s; ++j) lx += Pt[rr * kAdmmMax + j] * X[j * kAdmmMax + b];
        const double d0 = Dt[rr * kAdmmMax + b];
        const double u = fmax(lx + d0 * invpen, 0.0);
        const double d1 = d0 + sp_ * (lx - u);
        Ut[rr * kAdmmMax + b] = u;
        Dt[rr * kAdmmMax + b] = d1;
        a.U[(t0 + rr) * r + b] = u;
        a.D[(t0 + rr) * r + b] = d1;
        const double fe = lx - u;
        feas += fe * fe;
        const double du = d1 * u;
        comp += du * du + (d1 > 0.0 ? d1 * d1 : 0.0) + (u < 0.0 ? u * u : 0.0);
      }
      __syncthreads();
    }
    if (own) {
      for (int rr = 0; rr < nr; ++rr) {
        double pv[4], uv[4], dv[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          pv[x] = Pt[rr * kAdmmMax + 4 * bj + x];
          uv[x] = Ut[rr * kAdmmMax + 4 * bb + x];
          dv[x] = Dt[rr * kAdmmMax + 4 * bb + x];
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) {
            au[x][y] = fma(pv[x], uv[y], au[x][y]);
            ad[x][y] = fma(pv[x], dv[y], ad[x][y]);
          }
      }
    }
  }
  if (own) {
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int j = 4 * bj + x, b = 4 * bb + y;
        if (j < s && b < r) {
          atomicAdd(&a.accU[j * r + b], au[x][y]);
          if (mode == 1) atomicAdd(&a.accD[j * r + b], ad[x][y]);
        }
      }
  }
  if (mode == 1) {
    feas = wsum(feas);
    comp = wsum(comp);
    const int lane = tid & 31, warp = tid >> 5;
    if (lane == 0) {
      red[warp][0] = feas;
      red[warp][1] = comp;
    }
    __syncthreads();
    if (tid == 0) {
      double f = 0.0, c = 0.0;
      for (int w = 0; w < kSplitThreads / 32; ++w) {
        f += red[w][0];
        c += red[w][1];
      }
      atomicAdd(&a.scal[0], f);
      atomicAdd(&a.scal[1], c);
    }
  }
}

__global__ void __launch_bounds__(kSplitThreads)
    admm_split(SideArgs left, SideArgs right, const double* __restrict__ xc, const double* __restrict__ yc, int s,
               int r, double step, int mode, int nblk_left, const Ctrl* ctrl) {
  extern __shared__ double sm[];
  if (mode == 1 && ctrl->done) return;
  if ((int)blockIdx.x < nblk_left)
    split_side(left, xc, s, r, step, mode, blockIdx.x, nblk_left, sm);
  else
    split_side(right, yc, s, r, step, mode, blockIdx.x - nblk_left, gridDim.x - nblk_left, sm);
}

__global__ void init_ctrl(Ctrl* c) {
  c->k = 0;
  c->done = 0;
  c->iters = 0;
  c->diverged = -1;
}

}  // namespace

size_t admm_workspace(int64_t m, int64_t n, int s, int r) {
  (void)m;
  (void)n;
  (void)s;
  (void)r;
  return sizeof(Ctrl) + 256 + sizeof(Acc) + 256;
}

int admm_run(const double* core, const float* L, int64_t m, const float* Rt, int64_t n, int s, int r, double* u,
             double* du, double* vt, double* dvt, double* xc, double* yc, double pu, double pv, double step,
             int max_iter, double tol, double* trace, double* scores, int* iterations, void* ws, size_t ws_bytes,
             int resume, int step_limit, cudaStream_t st) {
  if (s < 1 || s > kAdmmMax || r < 1 || r > kAdmmMax)
    return fail(CNMF_ERR_ARGUMENT, "ADMM supports 1 <= r, s <= 64");
  if (!(pu > 0) || !(pv > 0)) return fail(CNMF_ERR_ARGUMENT, "penalties must be positive");
  if (ws_bytes < admm_workspace(m, n, s, r)) return fail(CNMF_ERR_ARGUMENT, "workspace too small");
  int S = s <= 32 ? 32 : 64;
  Ctrl* ctrl = (Ctrl*)ws;
  Acc* acc = (Acc*)((char*)ws + 256);
  const size_t core_smem = (size_t)(2 * s * s + 2 * s * r + r * r) * 8;
  const size_t split_smem = (size_t)(kAdmmMax * kAdmmMax + 3 * kTile * kAdmmMax) * 8;
  static bool attr = false;
  if (!attr) {
    CNMF_CUDA(cudaFuncSetAttribute(admm_core, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CNMF_CUDA(cudaFuncSetAttribute(admm_split, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)split_smem));
    attr = true;
  }
  const int64_t tl = ceil_div(m, kTile), tr = ceil_div(n, kTile);
  int nbl = (int)std::max<int64_t>(1, std::min<int64_t>(tl, std::max<int64_t>(1, kNumSMs * tl / (tl + tr))));
  int nbr = (int)std::max<int64_t>(1, std::min<int64_t>(tr, kNumSMs - std::min(nbl, kNumSMs - 1)));
  SideArgs left{L, m, S, u, du, pu, acc->LtU, acc->LtDU, acc->scal, 0};
  SideArgs right{Rt, n, S, vt, dvt, pv, acc->RtV, acc->RtDV, acc->scal + 2, 1};
  if (!resume) {
    init_ctrl<<<1, 1, 0, st>>>(ctrl);
    CNMF_LAUNCH_CHECK();
    CNMF_CUDA(cudaMemsetAsync(acc, 0, sizeof(Acc), st));
    CNMF_CUDA(cudaMemsetAsync(du, 0, (size_t)m * r * 8, st));
    CNMF_CUDA(cudaMemsetAsync(dvt, 0, (size_t)n * r * 8, st));
    CNMF_CUDA(cudaMemsetAsync(xc, 0, (size_t)s * r * 8, st));
    CNMF_CUDA(cudaMemsetAsync(yc, 0, (size_t)s * r * 8, st));
    // initial projections L^T U0 and R V0^T
    admm_split<<<nbl + nbr, kSplitThreads, split_smem, st>>>(left, right, xc, yc, s, r, step, 0, nbl, ctrl);
    CNMF_LAUNCH_CHECK();
  }
  auto one_iter = [&]() -> int {
    admm_core<<<1, 512, core_smem, st>>>(core, s, r, pu, pv, max_iter, tol, ctrl, acc, xc, yc, trace, scores);
    CNMF_LAUNCH_CHECK();
    admm_split<<<nbl + nbr, kSplitThreads, split_smem, st>>>(left, right, xc, yc, s, r, step, 1, nbl, ctrl);
    CNMF_LAUNCH_CHECK();
    return CNMF_OK;
  };
  Ctrl hc;
  if (step_limit > 0) {
    for (int i = 0; i < step_limit; ++i) CNMF_TRY(one_iter());
  } else {
    // capture a batch of iterations once, replay until the device says done
    const int batch = 25;
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    cudaStream_t cap;
    CNMF_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    CNMF_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    cudaStream_t saved = st;
    st = cap;
    const int64_t before = launch_count();
    for (int i = 0; i < batch; ++i) {
      int rc = one_iter();
      if (rc != CNMF_OK) {
        cudaStreamEndCapture(cap, &graph);
        return rc;
      }
    }
    st = saved;
    count_launches(before - launch_count());  // captured, not launched
    CNMF_CUDA(cudaStreamEndCapture(cap, &graph));
    CNMF_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    for (int done = 0; !done;) {
      for (int b = 0; b < 4; ++b) {
        CNMF_CUDA(cudaGraphLaunch(exec, st));
        count_launches(2 * batch);
      }
      CNMF_CUDA(cudaMemcpyAsync(&hc, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
      CNMF_CUDA(cudaStreamSynchronize(st));
      done = hc.done;
    }
    CNMF_CUDA(cudaGraphExecDestroy(exec));
    CNMF_CUDA(cudaGraphDestroy(graph));
    CNMF_CUDA(cudaStreamDestroy(cap));
  }
  CNMF_CUDA(cudaMemcpyAsync(&hc, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaStreamSynchronize(st));
  if (iterations) *iterations = hc.done ? hc.iters : -hc.k - 1;  // negative: still running
  if (hc.diverged >= 0) {
    if (iterations) *iterations = hc.diverged + 1;
    return fail(CNMF_ERR_DIVERGENCE, "KKT residual grew 10x over 50 iterations at iteration " +
                                         std::to_string(hc.diverged));
  }
  return CNMF_OK;
}

}  // namespace cnmf
