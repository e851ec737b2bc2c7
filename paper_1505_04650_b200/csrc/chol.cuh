// Cholesky factor + inverse of a small fp64 Gram matrix by one thread block
// (shared by the stand-alone kernel and the fused finalize + factor kernel).
#pragma once

#include "common.cuh"

namespace cnmf {

// G (upper triangle valid, S x S) = R^T R; T = R^{-1} written S x S (zero
// outside the leading s x s block). Symmetric Gaussian elimination of G held
// in place, LU-style: after step k the upper triangle holds D L^T and the
// strict lower triangle the accumulated row operations E = L^{-1}; scaling
// row k by d_k^{-1/2} at the end yields R (upper) and R^{-T} (lower) at once,
// so the factor and its inverse cost s parallel rank-1 steps (two barriers
// each) instead of two serial triangular sweeps.
// info[0] |= 1 when a shift was needed, info[1] = min(pass id) whose Gram
// matrix was not finite or not factorable. One block.
// the Gram buffer is consumed here and handed back zeroed for the next sweep
static __device__ __forceinline__ void G_rw_zero(const double* G, int idx) { const_cast<double*>(G)[idx] = 0.0; }

// `a` = shared scratch of (s * s + 2 s) doubles; every thread of the block
// calls this. G is read through L2 (it was accumulated with atomics by other
// blocks of the calling grid in the fused finalize).
static __device__ __noinline__ void chol_block(const double* G, int s, int S, double* __restrict__ T,
                                        double* __restrict__ Rout, int* __restrict__ info, int pass_id,
                                        double* a) {
  double* f = a + s * s;
  double* rowk = f + s;
  __shared__ double s_maxd;
  __shared__ int s_fail, s_nonfinite;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) {
    s_maxd = 0.0;
    s_fail = 0;
    s_nonfinite = 0;
  }
  __syncthreads();
  for (int idx = tid; idx < s * s; idx += nt) {
    const int i = idx / s, j = idx - i * s;
    const double v = (i <= j) ? __ldcg(G + i * S + j) : __ldcg(G + j * S + i);
    if (!isfinite(v)) s_nonfinite = 1;
    if (i == j) atomicMax((unsigned long long*)&s_maxd, __double_as_longlong(fmax(v, 0.0)));
  }
  __syncthreads();
  if (s_nonfinite || !(s_maxd > 0.0)) {
    if (tid == 0) atomicMin(&info[1], pass_id);
    __syncthreads();
    for (int idx = tid; idx < S * S; idx += nt) {
      T[idx] = 0.0;
      G_rw_zero(G, idx);
    }
    return;
  }
  const double thr = 1e-15 * s_maxd;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const double shift = attempt ? 1e-12 * s_maxd : 0.0;
    for (int idx = tid; idx < s * s; idx += nt) {
      const int i = idx / s, j = idx - i * s;
      a[idx] = ((i <= j) ? __ldcg(G + i * S + j) : __ldcg(G + j * S + i)) + (i == j ? shift : 0.0);
    }
    if (tid == 0 && attempt) info[0] |= 1;
    __syncthreads();
    for (int k = 0; k < s; ++k) {
      const double d = a[k * s + k];
      if (!(d > thr)) break;  // uniform: every thread reads the same value
      for (int i = tid; i < s; i += nt) {
        rowk[i] = a[k * s + i];
        f[i] = (i > k) ? a[i * s + k] / d : 0.0;
      }
      __syncthreads();
      const int rows = s - k - 1;
      for (int idx = tid; idx < rows * s; idx += nt) {
        const int i = k + 1 + idx / s, j = idx % s;
        a[i * s + j] = (j == k) ? -f[i] : a[i * s + j] - f[i] * rowk[j];
      }
      __syncthreads();
    }
    // a pivot below the threshold aborted the sweep (checked uniformly)
    bool ok = true;
    for (int k = 0; k < s; ++k)
      if (!(a[k * s + k] > thr)) ok = false;
    if (ok) {
      s_fail = 0;
      break;
    }
    s_fail = 1;
    __syncthreads();
  }
  if (s_fail) {
    if (tid == 0) atomicMin(&info[1], pass_id);
    for (int idx = tid; idx < S * S; idx += nt) {
      T[idx] = 0.0;
      G_rw_zero(G, idx);
    }
    return;
  }
  __syncthreads();
  for (int idx = tid; idx < S * S; idx += nt) G_rw_zero(G, idx);
  for (int idx = tid; idx < S * S; idx += nt) {
    const int i = idx / S, j = idx - i * S;
    double t = 0.0, r = 0.0;
    if (i < s && j < s) {
      // T[i][j] = R^{-T}[j][i]: row j of E scaled by d_j^{-1/2}
      if (i <= j) {
        const double dj = sqrt(a[j * s + j]);
        t = (i == j) ? 1.0 / dj : a[j * s + i] / dj;
        const double di = sqrt(a[i * s + i]);
        r = (i == j) ? di : a[i * s + j] / di;
      }
    }
    T[idx] = t;
    if (Rout != nullptr) Rout[idx] = r;
  }
}

}  // namespace cnmf

namespace cnmf {

// The same factorisation for s <= 32 by one warp, entirely in registers:
// lane j holds column j of the working matrix (col[i] = a[i][j]); step k
// broadcasts the pivot column k from lane k with shuffles. About 30x faster
// than the block version, which needs two block barriers per step.
// 1/d to ~1 ulp: fp32 reciprocal seed + two Newton steps in fp64 (a short,
// branch-free chain; the generic fp64 division sits on the critical path of
// every elimination step otherwise)
static __device__ __forceinline__ double rcp64(double d) {
  double x = (double)__frcp_rn((float)d);
  x = x * fma(-d, x, 2.0);
  x = x * fma(-d, x, 2.0);
  return fma(x, fma(-d, x, 1.0), x);
}

// The same factorisation for s <= 32 by 256 threads: thread t owns the four
// entries a[i][j], j = t & 31, i = (t >> 5) + 8 q, in registers; step k
// publishes row k and column k through a double-buffered shared-memory
// strip (one barrier per step). A small runtime loop keeps the instruction
// footprint tiny (a fully unrolled one-warp version is instruction-fetch
// bound: every instruction executes once).
static __device__ __forceinline__ bool elim_tile32(double (&a)[4], int i0, int j, int s, double thr, double* buf) {
  bool ok = true;
  for (int k = 0; k < s; ++k) {
    double* colk = buf + (k & 1) * 64;  // a[.][k]
    double* rowk = colk + 32;           // a[k][.]
    if (j == k)
#pragma unroll
      for (int q = 0; q < 4; ++q) colk[i0 + 8 * q] = a[q];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + 8 * q == k) rowk[j] = a[q];
    __syncthreads();
    const double d = rowk[k];
    ok = ok && (d > thr);  // uniform: every thread reads the same pivot
    const double inv = rcp64(d > thr ? d : 1.0);
    const double rkj = rowk[j];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + 8 * q;
      if (i > k) {
        const double f = colk[i] * inv;
        a[q] = (j == k) ? -f : fma(-f, rkj, a[q]);
      }
    }
  }
  return ok;
}

// `buf`: shared scratch of >= 32 * 33 + 128 doubles. Every thread of a
// 256-thread block calls this.
#ifdef CHOL_TIMING
__device__ long long g_chol_t[8];
#define CT(i) if (threadIdx.x == 0) g_chol_t[i] = clock64()
#else
#define CT(i)
#endif
static __device__ __noinline__ void chol_tile32(const double* G, int s, int S, double* __restrict__ T,
                                                double* __restrict__ Rout, int* __restrict__ info, int pass_id,
                                                double* buf) {
  __shared__ double s_maxd;
  __shared__ int s_bad;
  const int t = threadIdx.x, j = t & 31, i0 = t >> 5;
  CT(0);
  if (t == 0) {
    s_maxd = 0.0;
    s_bad = 0;
  }
  __syncthreads();
  double g[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = i0 + 8 * q;
    double v = (i == j) ? 1.0 : 0.0;
    if (i < s && j < s) v = (i <= j) ? __ldcg(G + i * S + j) : __ldcg(G + j * S + i);
    g[q] = v;
    if (!isfinite(v)) s_bad = 1;
    if (i == j && j < s) atomicMax((unsigned long long*)&s_maxd, __double_as_longlong(fmax(v, 0.0)));
  }
  __syncthreads();
  CT(1);
  const double maxd = s_maxd;
  bool ok = !s_bad && maxd > 0.0;
  double a[4];
  if (ok) {
    const double thr = 1e-15 * maxd;
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] = g[q];
    ok = elim_tile32(a, i0, j, s, thr, buf + 32 * 33);
    if (!ok) {  // numerically singular Gram matrix: retry with a small diagonal shift
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) a[q] = g[q] + ((i0 + 8 * q == j && j < s) ? 1e-12 * maxd : 0.0);
      if (t == 0) atomicOr(&info[0], 1);
      ok = elim_tile32(a, i0, j, s, thr, buf + 32 * 33);
    }
  }
  CT(2);
  // the Gram buffer is handed back zeroed for the next sweep
  for (int idx = t; idx < S * S; idx += blockDim.x) G_rw_zero(G, idx);
  if (!ok) {
    if (t == 0) atomicMin(&info[1], pass_id);
    for (int idx = t; idx < S * S; idx += blockDim.x) T[idx] = 0.0;
    return;
  }
  // full matrix to shared memory (padded rows), then T = R^{-1} and R:
  // T[i][c] = a[c][i] / sqrt(d_c) (c > i), R[i][c] = a[i][c] / sqrt(d_i) (i < c)
#pragma unroll
  for (int q = 0; q < 4; ++q) buf[(i0 + 8 * q) * 33 + j] = a[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = i0 + 8 * q;  // output row i, column c = j
    const int c = j;
    double tv = 0.0, rv = 0.0;
    if (i < s && c < s) {
      if (i == c) {
        const double sq = sqrt(buf[i * 33 + i]);
        tv = rcp64(sq);
        rv = sq;
      } else if (c > i) {
        tv = buf[c * 33 + i] * rcp64(sqrt(buf[c * 33 + c]));
        rv = buf[i * 33 + c] * rcp64(sqrt(buf[i * 33 + i]));
      }
    }
    if (c < S && i < S) {
      T[i * S + c] = tv;
      if (Rout != nullptr) Rout[i * S + c] = rv;
    }
  }
  for (int idx = 32 * S + t; idx < S * S; idx += blockDim.x) T[idx] = 0.0;  // rows >= 32 when S > 32
  CT(3);
}

// Dispatch: every thread of the block calls this.
static __device__ __forceinline__ void chol_small(const double* G, int s, int S, double* T, double* Rout, int* info,
                                                  int pass_id, double* a) {
  if (s <= 32 && blockDim.x == 256) {
    chol_tile32(G, s, S, T, Rout, info, pass_id, a);
  } else {
    chol_block(G, s, S, T, Rout, info, pass_id, a);
  }
}

}  // namespace cnmf
