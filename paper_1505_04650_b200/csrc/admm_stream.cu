// Compressed ADMM NMF for problems whose per-CTA state does not fit the
// persistent kernel (csrc/admm.cu keeps s x s / s x r fp64 matrices and the
// row slices in shared memory: r > 32 with s > 32, or very tall sides).
//
// Reference: nmf.py:306-377 (the loop), nmf.py:281-303 (KKT score); the same
// arithmetic as oracle/cnmf_oracle.py admm_compressed.
//
// One iteration = three launches, all state in HBM:
//   core_step  (1 block)   KKT score of the previous iteration from the
//                          reduced sums, convergence / divergence rule, then
//                          xc = (core yc^T + pu L^T U - L^T dU)(yc yc^T + pu I)^-1
//                          yc = (xc^T xc + pv I)^-1 (xc^T core + pv V R^T - dV R^T)
//   row_sweep  (grid)      every row of both sides: x = max(P z + dx / p, 0),
//                          dx += step p (P z - x), and the block partials of
//                          P^T x, P^T dx and the four KKT sums
//   reduce     (grid)      fixed-order sums of the block partials
// so every reduction is deterministic. Streaming bytes per iteration:
// U, dU, V, dV read and written (fp64) + L, R read (fp32).
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace cnmf {
namespace {

constexpr int kT = 256;   // threads per block
constexpr int kTR = 32;   // rows per tile
constexpr int kMaxD = 64; // s, r <= 64

struct SCtrl {
  int k;         // next iteration index
  int done;
  int iters;
  int diverged;  // 0-based iteration that tripped the divergence rule, or -1
};

struct SSide {
  const float* P;  // rows x ldp panel (L or R^T)
  int64_t rows;
  int ldp;
  double* x;   // rows x r (U or V^T)
  double* dx;  // rows x r (dU or dV^T)
  double pen;
};

// per-side reduced sums: [P^T x (s x r) | P^T dx (s x r) | 4 KKT sums]
__host__ __device__ inline int sums_len(int s, int r) { return 2 * s * r + 4; }

// ---------------------------------------------------------------------------
// row sweep: blocks [0, nbl) take left rows, [nbl, grid) right rows
// ---------------------------------------------------------------------------
template <int SP>
__global__ void __launch_bounds__(kT) row_sweep(SSide L, SSide R, int nbl, const double* __restrict__ Zl,
                                                 const double* __restrict__ Zr, int s, int r, double step, int update,
                                                 double* __restrict__ part, const SCtrl* ctrl) {
  if (update && ctrl->done) return;
  extern __shared__ __align__(16) unsigned char sm[];
  double* Z = (double*)sm;                  // SP x kMaxD (rows c, cols k; zero padded)
  double* Xt = Z + SP * kMaxD;              // kTR x kMaxD
  double* Dt = Xt + kTR * kMaxD;            // kTR x kMaxD
  float* Pt = (float*)(Dt + kTR * kMaxD);   // kTR x SP
  __shared__ double red[4][kT / 32];
  const bool left = (int)blockIdx.x < nbl;
  const SSide sd = left ? L : R;
  const int b = left ? (int)blockIdx.x : (int)blockIdx.x - nbl;
  const int nb = left ? nbl : (int)gridDim.x - nbl;
  const int64_t r0 = sd.rows * b / nb, r1 = sd.rows * (b + 1) / nb;
  const int tid = threadIdx.x, sr = s * r;
  const double* Zs = left ? Zl : Zr;
  for (int i = tid; i < SP * kMaxD; i += kT) {
    const int c = i / kMaxD, k = i % kMaxD;
    Z[i] = (update && c < s && k < r) ? Zs[c * r + k] : 0.0;
  }
  for (int i = tid; i < 2 * kTR * kMaxD; i += kT) Xt[i] = 0.0;  // padding columns stay zero
  // lane j of a half-warp owns the columns k = j + 16 q (q < 4): consecutive
  // lanes touch consecutive doubles in Z, Xt, Dt and in x, dx (no bank
  // conflicts; a 4-consecutive-column split put 4 lanes on each bank)
  const int j16 = tid & 15, cg = tid >> 4;  // reduction tile: rows 4 cg .. 4 cg + 3 of P^T
  const bool red_on = 4 * cg < s;
  double au[16], ad[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) au[q] = ad[q] = 0.0;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int64_t t0 = r0; t0 < r1; t0 += kTR) {
    const int nr = (int)min64(kTR, r1 - t0);
    __syncthreads();
    for (int i = tid; i < kTR * SP; i += kT) {
      const int row = i / SP, c = i % SP;
      Pt[i] = (row < nr && c < s) ? sd.P[(t0 + row) * sd.ldp + c] : 0.f;
    }
    __syncthreads();
    // ---- update: thread = (row, lane j), columns j + 16 q ----
#pragma unroll 1
    for (int row = tid >> 4; row < kTR; row += kT / 16) {
      double lx[4] = {0.0, 0.0, 0.0, 0.0};
      if (update && row < nr) {
#pragma unroll 4
        for (int c = 0; c < s; ++c) {
          const double p = (double)Pt[row * SP + c];
#pragma unroll
          for (int q = 0; q < 4; ++q) lx[q] = fma(p, Z[c * kMaxD + j16 + 16 * q], lx[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = j16 + 16 * q;
        double xn = 0.0, dxn = 0.0;
        if (row < nr && k < r) {
          const int64_t gi = (t0 + row) * r + k;
          const double xo = sd.x[gi], dxo = sd.dx[gi];
          if (update) {
            xn = fmax(lx[q] + dxo / sd.pen, 0.0);
            dxn = dxo + step * sd.pen * (lx[q] - xn);
            sd.x[gi] = xn;
            sd.dx[gi] = dxn;
            const double dl = lx[q] - xn, dp = dxn * xn, dpos = fmax(dxn, 0.0), xneg = fmax(-xn, 0.0);
            s0 += dl * dl;
            s1 += dp * dp;
            s2 += dpos * dpos;
            s3 += xneg * xneg;
          } else {
            xn = xo;
            dxn = dxo;
          }
        }
        Xt[row * kMaxD + k] = xn;
        Dt[row * kMaxD + k] = dxn;
      }
    }
    __syncthreads();
    // ---- partials P^T x, P^T dx: 4 rows of P^T x 4 strided columns ----
    if (red_on) {
      for (int row = 0; row < nr; ++row) {
        const float4 p4 = *(const float4*)(Pt + row * SP + 4 * cg);
        const double pc[4] = {p4.x, p4.y, p4.z, p4.w};
        double xv[4], dv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          xv[q] = Xt[row * kMaxD + j16 + 16 * q];
          dv[q] = Dt[row * kMaxD + j16 + 16 * q];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            au[a * 4 + q] = fma(pc[a], xv[q], au[a * 4 + q]);
            ad[a * 4 + q] = fma(pc[a], dv[q], ad[a * 4 + q]);
          }
      }
    }
  }
  double* out = part + (size_t)blockIdx.x * sums_len(s, r);
  if (red_on) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = 4 * cg + a, k = j16 + 16 * q;
        if (c < s && k < r) {
          out[c * r + k] = au[a * 4 + q];
          out[sr + c * r + k] = ad[a * 4 + q];
        }
      }
  }
  // KKT sums: warp shuffles, then the warps in order
  double v[4] = {s0, s1, s2, s3};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
    if ((tid & 31) == 0) red[j][tid >> 5] = v[j];
  }
  __syncthreads();
  if (tid < 4) {
    double acc = 0.0;
    for (int w = 0; w < kT / 32; ++w) acc += red[tid][w];
    out[2 * sr + tid] = acc;
  }
}

// fixed-order sums of the block partials of each side: sums[side][e]
__global__ void __launch_bounds__(kT) reduce_parts(const double* __restrict__ part, int nbl, int nbr, int len,
                                                    double* __restrict__ sums, const SCtrl* ctrl, int update) {
  if (update && ctrl->done) return;
  const int e = blockIdx.x * kT + threadIdx.x;
  const int side = blockIdx.y;
  if (e >= len) return;
  const int b0 = side ? nbl : 0, nb = side ? nbr : nbl;
  double acc = 0.0;
  for (int j0 = 0; j0 < nb; j0 += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (j0 + j < nb) ? part[(size_t)(b0 + j0 + j) * len + e] : 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j];
  }
  sums[side * len + e] = acc;
}

// sum_j a[j * sa] * b[j * sb] with four interleaved partial sums (the
// single-block core step is bound by the fp64 FMA latency of one long chain)
__device__ __forceinline__ double dot4(const double* a, int sa, const double* b, int sb, int len) {
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
  int j = 0;
  for (; j + 4 <= len; j += 4) {
    v0 = fma(a[j * sa], b[j * sb], v0);
    v1 = fma(a[(j + 1) * sa], b[(j + 1) * sb], v1);
    v2 = fma(a[(j + 2) * sa], b[(j + 2) * sb], v2);
    v3 = fma(a[(j + 3) * sa], b[(j + 3) * sb], v3);
  }
  for (; j < len; ++j) v0 = fma(a[j * sa], b[j * sb], v0);
  return (v0 + v1) + (v2 + v3);
}

// In-place inverse of an SPD r x r matrix (ld kMaxD + 1) by Gauss-Jordan
// without pivoting (the ridge term keeps the pivots >= the penalty).
__device__ void spd_inverse(double* M, double* piv, int r) {
  const int tid = threadIdx.x;
  constexpr int LD = kMaxD + 1;
  double* colk = piv + kMaxD;
  for (int k = 0; k < r; ++k) {
    __syncthreads();
    const double inv = 1.0 / M[k * LD + k];
    for (int j = tid; j < r; j += kT) {
      piv[j] = M[k * LD + j] * inv;  // scaled pivot row
      colk[j] = M[j * LD + k];       // column k before this step overwrites it
    }
    __syncthreads();
    for (int i = tid; i < r * r; i += kT) {
      const int a = i / r, c = i % r;
      if (a == k) {
        M[a * LD + c] = (c == k) ? inv : piv[c];
      } else {
        const double f = colk[a];
        M[a * LD + c] = (c == k) ? -f * inv : fma(-f, piv[c], M[a * LD + c]);
      }
    }
  }
  __syncthreads();
}

// KKT of the iteration just swept (k > 0), the stopping / divergence rule,
// then the two ridge solves of iteration k (nmf.py:341-350).
__global__ void __launch_bounds__(kT) core_step(const double* __restrict__ core, const double* __restrict__ sums,
                                                 double* __restrict__ xc, double* __restrict__ yc, double* Zl,
                                                 double* Zr, int s, int r, double pu, double pv, double tol,
                                                 double* trace, double* scores, SCtrl* ctrl, int k, int max_iter,
                                                 int first, int solve) {
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int LD = kMaxD + 1;
  double* A = (double*)sm;      // 64 x 65 scratch (s x s or s x r)
  double* B = A + kMaxD * LD;   // 64 x 65
  double* M = B + kMaxD * LD;   // r x r
  double* piv = M + kMaxD * LD; // 2 x 64
  // the small operands staged in shared memory (every loop below reads them
  // many times): core (s x s), xc (s x r), yc (r x s)
  double* coreS = piv + 2 * kMaxD;
  double* xcS = coreS + s * s;
  double* ycS = xcS + s * r;
  __shared__ double red[6][kT / 32];
  __shared__ int s_stop;
  const int tid = threadIdx.x, sr = s * r, len = sums_len(s, r);
  const double* sl = sums;        // left: L^T U | L^T dU | sums
  const double* srt = sums + len; // right: R V^T | R dV^T (as s x r) | sums
  if (tid == 0) s_stop = 0;
  for (int i = tid; i < s * s; i += kT) coreS[i] = core[i];
  for (int i = tid; i < s * r; i += kT) xcS[i] = xc[i];
  for (int i = tid; i < r * s; i += kT) ycS[i] = yc[i];
  __syncthreads();
  if (first) {
    // yc = V R^T (nmf.py:338): the reduced right sums of the initial state
    for (int i = tid; i < r * s; i += kT) {
      const int a = i / s, c = i % s;
      yc[i] = srt[c * r + a];
      ycS[i] = srt[c * r + a];
    }
    __syncthreads();
  } else if (k > 0) {
    // ---- KKT score of iteration k - 1 (nmf.py:281-303) ----
    // A = E = xc yc - core (s x s)
    for (int i = tid; i < s * s; i += kT) {
      const int a = i / s, c = i % s;
      double e = -coreS[i];
      e += dot4(xcS + a * r, 1, ycS + c, s, r);
      A[a * LD + c] = e;
    }
    __syncthreads();
    double t1 = 0.0, t2 = 0.0, obj = 0.0;
    for (int i = tid; i < s * s; i += kT) obj += A[(i / s) * LD + i % s] * A[(i / s) * LD + i % s];
    for (int i = tid; i < s * r; i += kT) {  // (E yc^T + L^T dU)[a][j]
      const int a = i / r, j = i % r;
      double v = sl[sr + a * r + j];
      v += dot4(A + a * LD, 1, ycS + j * s, 1, s);
      t1 += v * v;
    }
    for (int i = tid; i < r * s; i += kT) {  // (xc^T E + dV R^T)[j][c]
      const int j = i / s, c = i % s;
      double v = srt[sr + c * r + j];
      v += dot4(xcS + j, r, A + c, LD, s);
      t2 += v * v;
    }
    double vals[3] = {t1, t2, obj};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) vals[q] += __shfl_xor_sync(0xffffffffu, vals[q], o);
      if ((tid & 31) == 0) red[q][tid >> 5] = vals[q];
    }
    __syncthreads();
    if (tid == 0) {
      double a1 = 0, a2 = 0, ob = 0;
      for (int w = 0; w < kT / 32; ++w) {
        a1 += red[0][w];
        a2 += red[1][w];
        ob += red[2][w];
      }
      const double sc = fmax(fmax(fmax(sqrt(a1), sqrt(a2)), fmax(sqrt(sl[2 * sr]), sqrt(srt[2 * sr]))),
                             fmax(sqrt(sl[2 * sr + 1] + sl[2 * sr + 2] + sl[2 * sr + 3]),
                                  sqrt(srt[2 * sr + 1] + srt[2 * sr + 2] + srt[2 * sr + 3])));
      const int it = k - 1;
      trace[it] = ob;
      scores[it] = sc;
      ctrl->k = k;
      if (sc < tol || k >= max_iter) {
        ctrl->done = 1;
        ctrl->iters = k;
        s_stop = 1;
      } else if (it >= 50 && sc > 10.0 * scores[it - 50]) {
        ctrl->diverged = it;
        ctrl->done = 1;
        ctrl->iters = k;
        s_stop = 1;
      }
    }
    __syncthreads();
    if (s_stop) return;
  }
  if (!solve || k >= max_iter) return;
  // ---- xc = (core yc^T + pu L^T U - L^T dU) (yc yc^T + pu I)^-1 ----
  for (int i = tid; i < r * r; i += kT) {
    const int a = i / r, c = i % r;
    double v = (a == c) ? pu : 0.0;
    v += dot4(ycS + a * s, 1, ycS + c * s, 1, s);
    M[a * LD + c] = v;
  }
  for (int i = tid; i < s * r; i += kT) {  // rhs (s x r) in A
    const int a = i / r, c = i % r;
    double v = pu * sl[a * r + c] - sl[sr + a * r + c];
    v += dot4(coreS + a * s, 1, ycS + c * s, 1, s);
    A[a * LD + c] = v;
  }
  spd_inverse(M, piv, r);
  for (int i = tid; i < s * r; i += kT) {
    const int a = i / r, c = i % r;
    double v = 0.0;
    v += dot4(A + a * LD, 1, M + c, LD, r);
    xc[i] = v;
    xcS[i] = v;
    Zl[i] = v;
  }
  __syncthreads();
  // ---- yc = (xc^T xc + pv I)^-1 (xc^T core + pv V R^T - dV R^T) ----
  for (int i = tid; i < r * r; i += kT) {
    const int a = i / r, c = i % r;
    double v = (a == c) ? pv : 0.0;
    v += dot4(xcS + a, r, xcS + c, r, s);
    M[a * LD + c] = v;
  }
  for (int i = tid; i < r * s; i += kT) {  // rhs2 (r x s) in B
    const int a = i / s, c = i % s;
    double v = pv * srt[c * r + a] - srt[sr + c * r + a];
    v += dot4(xcS + a, r, coreS + c, s, s);
    B[a * LD + c] = v;
  }
  spd_inverse(M, piv, r);
  for (int i = tid; i < r * s; i += kT) {
    const int a = i / s, c = i % s;
    double v = 0.0;
    v += dot4(M + a * LD, 1, B + c, LD, r);
    yc[i] = v;
    Zr[c * r + a] = v;  // Z for the right rows: yc^T (s x r)
  }
}

__global__ void init_sctrl(SCtrl* c) {
  c->k = 0;
  c->done = 0;
  c->iters = 0;
  c->diverged = -1;
}

}  // namespace

int admm_stream_run(const double* core, const float* L, int64_t m, const float* Rt, int64_t n, int s, int r, double* u,
                    double* du, double* vt, double* dvt, double* xc, double* yc, double pu, double pv, double step,
                    int max_iter, double tol, double* trace, double* scores, int* iterations, void* ws, int resume,
                    int step_limit, cudaStream_t st) {
  const int S = s <= 32 ? 32 : 64;
  SCtrl* ctrl = (SCtrl*)ws;
  int dev = 0, sms = 0;
  CNMF_CUDA(cudaGetDevice(&dev));
  CNMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // row blocks: two per SM, split between the sides by row count
  const int total = 2 * sms;
  const int nbl = (int)std::max<int64_t>(1, std::min<int64_t>(total - 1, (total * m + (m + n) / 2) / (m + n)));
  const int nbr = total - nbl;
  const int len = sums_len(s, r);
  // library scratch: block partials, reduced sums, Z operands
  static double* scratch = nullptr;
  static size_t cap = 0;
  const size_t need = ((size_t)total * len + 2 * (size_t)len + 2 * kMaxD * kMaxD) * 8;
  if (cap < need) {
    CNMF_CUDA(cudaStreamSynchronize(st));
    if (scratch) cudaFree(scratch);
    scratch = nullptr;
    cap = 0;
    CNMF_CUDA(cudaMalloc(&scratch, need));
    cap = need;
  }
  double* part = scratch;
  double* sums = part + (size_t)total * len;
  double* Zl = sums + 2 * len;
  double* Zr = Zl + kMaxD * kMaxD;
  const size_t sweep_smem = ((size_t)S * kMaxD + 2 * kTR * kMaxD) * 8 + (size_t)kTR * S * 4;
  const size_t core_smem = (3 * (size_t)kMaxD * (kMaxD + 1) + 2 * kMaxD + (size_t)s * s + 2 * (size_t)s * r) * 8;
  static bool attr = false;
  if (!attr) {
    CNMF_CUDA(cudaFuncSetAttribute(row_sweep<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(((size_t)32 * kMaxD + 2 * kTR * kMaxD) * 8 + (size_t)kTR * 32 * 4)));
    CNMF_CUDA(cudaFuncSetAttribute(row_sweep<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(((size_t)64 * kMaxD + 2 * kTR * kMaxD) * 8 + (size_t)kTR * 64 * 4)));
    CNMF_CUDA(cudaFuncSetAttribute(core_step, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)((3 * kMaxD * (kMaxD + 1) + 2 * kMaxD + 3 * kMaxD * kMaxD) * 8)));
    attr = true;
  }
  const SSide sl{L, m, S, u, du, pu}, sr{Rt, n, S, vt, dvt, pv};
  auto sweep = [&](int update) -> int {
    if (S == 32)
      row_sweep<32><<<total, kT, sweep_smem, st>>>(sl, sr, nbl, Zl, Zr, s, r, step, update, part, ctrl);
    else
      row_sweep<64><<<total, kT, sweep_smem, st>>>(sl, sr, nbl, Zl, Zr, s, r, step, update, part, ctrl);
    CNMF_LAUNCH_CHECK();
    reduce_parts<<<dim3((unsigned)ceil_div(len, kT), 2), kT, 0, st>>>(part, nbl, nbr, len, sums, ctrl, update);
    CNMF_LAUNCH_CHECK();
    return CNMF_OK;
  };
  int k0 = 0;
  if (!resume) {
    init_sctrl<<<1, 1, 0, st>>>(ctrl);
    CNMF_LAUNCH_CHECK();
    CNMF_CUDA(cudaMemsetAsync(du, 0, (size_t)m * r * 8, st));
    CNMF_CUDA(cudaMemsetAsync(dvt, 0, (size_t)n * r * 8, st));
    CNMF_TRY(sweep(0));  // L^T U and V R^T of the start
  } else {
    SCtrl h;
    CNMF_CUDA(cudaMemcpyAsync(&h, ctrl, sizeof h, cudaMemcpyDeviceToHost, st));
    CNMF_CUDA(cudaStreamSynchronize(st));
    if (h.done) {
      if (iterations) *iterations = h.iters;
      return CNMF_OK;
    }
    k0 = h.k;
  }
  const int k1 = step_limit > 0 ? std::min(max_iter, k0 + step_limit) : max_iter;
  for (int k = k0; k < k1; ++k) {
    core_step<<<1, kT, core_smem, st>>>(core, sums, xc, yc, Zl, Zr, s, r, pu, pv, tol, trace, scores, ctrl, k,
                                        max_iter, k == 0 && !resume, 1);
    CNMF_LAUNCH_CHECK();
    CNMF_TRY(sweep(1));
  }
  // score of the last swept iteration (and the stop decision)
  core_step<<<1, kT, core_smem, st>>>(core, sums, xc, yc, Zl, Zr, s, r, pu, pv, tol, trace, scores, ctrl, k1,
                                      max_iter, 0, 0);
  CNMF_LAUNCH_CHECK();
  SCtrl h;
  CNMF_CUDA(cudaMemcpyAsync(&h, ctrl, sizeof h, cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaStreamSynchronize(st));
  if (iterations) *iterations = h.done ? h.iters : -h.k - 1;
  if (h.diverged >= 0) {
    if (iterations) *iterations = h.diverged + 1;
    return fail(CNMF_ERR_DIVERGENCE, "KKT residual grew 10x over 50 iterations at iteration " +
                                         std::to_string(h.diverged));
  }
  return CNMF_OK;
}

}  // namespace cnmf
