// Batched active-set NNLS on shared Gram products, one warp per target column.
//
// Reference: nnls.py:21-111 (nnls_solve), nnls.py:122-148 (_solve_passive),
// nnls.py:151-168 (_step_back). The reference advances all columns in
// lockstep and solves each passive-set system with LU on the masked q x q
// matrix; here every warp walks its own column through the same sequence of
// exchanges (entering index = first argmax of the negative gradient over the
// active set, step-back to the first blocking bound, release threshold
// 1e-14 * max(|h|, 1), forced release of the tightest blocker) and solves the
// passive system with a Cholesky factor kept in insertion order and extended
// by one row per entering index (O(p^2) per exchange instead of O(p^3)).
// Singular passive systems fall back to the reference's ridge
// 1e-12 * trace(C^T C).
#include <algorithm>
#include <cfloat>

#include "common.cuh"

namespace cnmf {
namespace {

constexpr int kQMax = 64;

struct WarpScratch {
  double* L;    // lower factor, packed by rows (entry (i, j), j <= i, at i (i + 1) / 2 + j), insertion order
  int* order;   // passive indices in insertion order
  int ld;       // unused (packed storage: half the shared memory per warp, twice the warps per SM)
};

__device__ __forceinline__ int tri(int i, int j) { return ((i * (i + 1)) >> 1) + j; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// value of the distributed vector (lane holds entries lane, lane+32) at index i
__device__ __forceinline__ double vget(const double (&x)[2], int i) {
  return __shfl_sync(0xffffffffu, x[i >> 5], i & 31);
}

// Extend the factor by index a at position p. Returns false if singular.
__device__ bool chol_add(const double* G, int q, WarpScratch ws, int p, int a, double ridge) {
  const int lane = threadIdx.x & 31;
  // b_i = G[order[i]][a] for i < p (row a of the symmetric Gram)
  double b[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = lane + 32 * h;
    b[h] = (i < p) ? G[a * q + ws.order[i]] : 0.0;
  }
  // forward substitution L y = b (column-oriented)
  for (int j = 0; j < p; ++j) {
    const double yj = vget(b, j) / ws.L[tri(j, j)];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      if (i == j) b[h] = yj;
      else if (i > j && i < p) b[h] -= ws.L[tri(i, j)] * yj;
    }
  }
  double yy = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = lane + 32 * h;
    if (i < p) {
      yy += b[h] * b[h];
      ws.L[tri(p, i)] = b[h];
    }
  }
  yy = warp_sum(yy);
  const double gaa = G[a * q + a] + ridge;
  const double d = gaa - yy;
  __syncwarp();
  if (!(d > 1e-13 * fabs(gaa)) || !isfinite(d)) return false;
  if (lane == 0) {
    ws.L[tri(p, p)] = sqrt(d);
    ws.order[p] = a;
  }
  __syncwarp();
  return true;
}

// Rebuild the factor for the passive set in `ws.order[0..p)` (order kept).
__device__ bool chol_rebuild(const double* G, int q, WarpScratch ws, int p, double ridge) {
  for (int k = 0; k < p; ++k)
    if (!chol_add(G, q, ws, k, ws.order[k], ridge)) return false;
  return true;
}

// z = G_PP^{-1} t_P scattered to full length (zero off P).
__device__ void chol_solve(const double (&t)[2], int q, WarpScratch ws, int p, double (&z)[2]) {
  const int lane = threadIdx.x & 31;
  double w[2];
  // gather t at the passive indices (position-ordered)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = lane + 32 * h;
    const int oi = (i < p) ? ws.order[i] : 0;
    const double v0 = __shfl_sync(0xffffffffu, t[0], oi & 31);
    const double v1 = __shfl_sync(0xffffffffu, t[1], oi & 31);
    w[h] = (i < p) ? ((oi < 32) ? v0 : v1) : 0.0;
  }
  // forward L u = t_P
  for (int j = 0; j < p; ++j) {
    const double uj = vget(w, j) / ws.L[tri(j, j)];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      if (i == j) w[h] = uj;
      else if (i > j && i < p) w[h] -= ws.L[tri(i, j)] * uj;
    }
  }
  // backward L^T v = u
  for (int j = p - 1; j >= 0; --j) {
    const double vj = vget(w, j) / ws.L[tri(j, j)];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      if (i == j) w[h] = vj;
      else if (i < j) w[h] -= ws.L[tri(j, i)] * vj;
    }
  }
  // scatter back to index space: z[order[i]] = w[i]
  z[0] = 0.0;
  z[1] = 0.0;
  for (int i = 0; i < p; ++i) {
    const double v = vget(w, i);
    const int oi = ws.order[i];
    if ((oi & 31) == lane) z[oi >> 5] = v;
  }
}

// H0 (optional, k x q0 with q0 < q): a feasible start -- the solution of the
// same targets over the first q0 design columns (XRAY's previous refit: the
// picks grow by appending). Its support becomes the initial passive set and
// the iteration proceeds from it exactly as from any feasible iterate; the
// minimiser is unique when the design has full column rank, so only the
// exchange path (not the answer) changes.
__global__ void nnls_kernel(const double* __restrict__ gram_g, const double* __restrict__ target, int64_t k, int q,
                            double tol, int cap, double ridge, double* __restrict__ H,
                            unsigned long long* __restrict__ n_capped, const double* __restrict__ H0, int q0) {
  extern __shared__ double smem[];
  double* G = smem;  // q x q
  const int wpb = blockDim.x / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < q * q; i += blockDim.x) G[i] = gram_g[i];
  WarpScratch ws;
  const int tsz = (q * (q + 1) / 2 + 1) & ~1;  // packed factor, 16-byte multiple
  ws.ld = 0;
  ws.L = G + q * q + (size_t)warp * tsz;
  ws.order = (int*)(G + q * q + (size_t)wpb * tsz) + warp * kQMax;
  __syncthreads();

  for (int64_t col = (int64_t)blockIdx.x * wpb + warp; col < k; col += (int64_t)gridDim.x * wpb) {
    double t[2], h[2], grad[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = lane + 32 * e;
      t[e] = (i < q) ? target[col * q + i] : 0.0;
      h[e] = 0.0;
      grad[e] = t[e];
    }
    uint64_t pas = 0;
    int p = 0, swaps = 0;
    bool capped = false;
    bool factored = true;  // factor of order[0..p) is valid
    bool ridged = false;
    bool warm = false;     // run the feasibility loop on the start before the first entering index
    if (H0 != nullptr) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = lane + 32 * e;
        h[e] = (i < q0) ? fmax(H0[col * q0 + i], 0.0) : 0.0;
      }
      pas = (uint64_t)__ballot_sync(0xffffffffu, h[0] > 0.0) |
            ((uint64_t)__ballot_sync(0xffffffffu, h[1] > 0.0) << 32);
      p = __popcll(pas);
      if (p > 0) {
        if (lane == 0) {
          int np = 0;
          for (int i = 0; i < q; ++i)
            if ((pas >> i) & 1ull) ws.order[np++] = i;
        }
        __syncwarp();
        ridged = !chol_rebuild(G, q, ws, p, 0.0);
        if (ridged) chol_rebuild(G, q, ws, p, ridge);
        warm = true;
      }
    }
    for (;;) {
      if (!warm) {
      // entering index: first argmax of grad over the active set
      double bv = -DBL_MAX;
      int bi = q;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = lane + 32 * e;
        if (i < q && !((pas >> i) & 1ull)) {
          if (grad[e] > bv || (grad[e] == bv && i < bi)) {
            bv = grad[e];
            bi = i;
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (bi >= q || !(bv > tol)) break;
      pas |= 1ull << bi;
      ++swaps;
      if (swaps > cap) {
        capped = true;
        break;
      }
      // extend the factor (or rebuild with the ridge when singular)
      if (factored && !ridged && chol_add(G, q, ws, p, bi, 0.0)) {
        ++p;
      } else {
        if (lane == 0) ws.order[p] = bi;
        __syncwarp();
        ++p;
        ridged = !chol_rebuild(G, q, ws, p, 0.0);
        if (ridged) chol_rebuild(G, q, ws, p, ridge);
        factored = true;
      }
      }  // !warm
      warm = false;
      for (;;) {
        double z[2];
        chol_solve(t, q, ws, p, z);
        bool feas = true;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = lane + 32 * e;
          if (i < q && ((pas >> i) & 1ull) && !(z[e] > 0.0)) feas = false;
        }
        feas = __all_sync(0xffffffffu, feas);
        if (feas) {
          h[0] = z[0];
          h[1] = z[1];
          break;
        }
        // step back towards z (nnls.py:151-168)
        double amin = DBL_MAX;
        int imin = q;
        uint64_t blk = 0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = lane + 32 * e;
          if (i < q && ((pas >> i) & 1ull) && z[e] <= 0.0) {
            const double den = h[e] - z[e];
            const double ratio = den > 0.0 ? h[e] / den : 0.0;
            if (ratio < amin || (ratio == amin && i < imin)) {
              amin = ratio;
              imin = i;
            }
          }
        }
        blk = __ballot_sync(0xffffffffu, (lane < q) && ((pas >> lane) & 1ull) && z[0] <= 0.0);
        blk |= (uint64_t)__ballot_sync(0xffffffffu, (lane + 32 < q) && ((pas >> (lane + 32)) & 1ull) && z[1] <= 0.0)
               << 32;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, amin, o);
          const int oi = __shfl_xor_sync(0xffffffffu, imin, o);
          if (ov < amin || (ov == amin && oi < imin)) {
            amin = ov;
            imin = oi;
          }
        }
        const double alpha = (blk != 0) ? amin : 0.0;
        double mx = 0.0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          h[e] = h[e] + alpha * (z[e] - h[e]);
          const int i = lane + 32 * e;
          if (i < q) mx = fmax(mx, fabs(h[e]));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const double scale = fmax(mx, 1.0);
        uint64_t rel = 0;
        rel = __ballot_sync(0xffffffffu, ((blk >> lane) & 1ull) && h[0] <= 1e-14 * scale);
        rel |= (uint64_t)__ballot_sync(0xffffffffu, ((blk >> (lane + 32)) & 1ull) && h[1] <= 1e-14 * scale) << 32;
        if (rel == 0) rel = 1ull << imin;
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if ((rel >> (lane + 32 * e)) & 1ull) h[e] = 0.0;
        pas &= ~rel;
        // compact the insertion order and rebuild the factor
        if (lane == 0) {
          int np = 0;
          for (int i = 0; i < p; ++i)
            if (!((rel >> ws.order[i]) & 1ull)) ws.order[np++] = ws.order[i];
        }
        __syncwarp();
        p = __popcll(pas);
        ridged = !chol_rebuild(G, q, ws, p, 0.0);
        if (ridged) chol_rebuild(G, q, ws, p, ridge);
        ++swaps;
        if (swaps > cap) {
          capped = true;
          break;
        }
      }
      if (capped) break;
      // grad = t - G h   (G symmetric: read row j for coalescing)
#pragma unroll
      for (int e = 0; e < 2; ++e) grad[e] = t[e];
      for (int j = 0; j < q; ++j) {
        const double hj = vget(h, j);
        if (hj == 0.0) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = lane + 32 * e;
          if (i < q) grad[e] -= G[j * q + i] * hj;
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = lane + 32 * e;
      if (i < q) H[col * q + i] = fmax(h[e], 0.0);
    }
    if (capped && lane == 0) atomicAdd(n_capped, 1ull);
  }
}

}  // namespace

int nnls_gram(const double* gram, const double* target, int64_t k, int q, double tol, int max_exchanges, double* H,
              int64_t* n_capped, cudaStream_t st, const double* H0, int q0) {
  if (q < 1 || q > kQMax) return fail(CNMF_ERR_ARGUMENT, "nnls: 1 <= q <= 64 required");
  if (!(tol > 0)) return fail(CNMF_ERR_ARGUMENT, "tol must be positive");
  if (k == 0) return CNMF_OK;
  const int cap = max_exchanges > 0 ? max_exchanges : 3 * q;
  // ridge = 1e-12 * trace(gram) (nnls.py:66)
  double* hg = new double[(size_t)q * q];
  CNMF_CUDA(cudaMemcpyAsync(hg, gram, (size_t)q * q * 8, cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaStreamSynchronize(st));
  double tr = 0.0;
  for (int i = 0; i < q; ++i) tr += hg[i * q + i];
  delete[] hg;
  const double ridge = 1e-12 * tr;
  const size_t tsz = (size_t)((q * (q + 1) / 2 + 1) & ~1);
  const size_t per_warp = tsz * 8 + kQMax * 4;
  int wpb = (int)std::min<size_t>(32, (220 * 1024 - (size_t)q * q * 8) / per_warp);
  wpb = std::max(1, wpb);
  const size_t smem = (size_t)q * q * 8 + (size_t)wpb * per_warp;
  CNMF_TRY(ensure_smem_attr((const void*)nnls_kernel, 227 * 1024));
  unsigned long long* d_cap = nullptr;
  keep_pool();
  CNMF_CUDA(cudaMallocAsync((void**)&d_cap, 8, st));
  CNMF_CUDA(cudaMemsetAsync(d_cap, 0, 8, st));
  const int64_t blocks = std::min<int64_t>(ceil_div(k, wpb), 16 * kNumSMs);
  nnls_kernel<<<(unsigned)blocks, 32 * wpb, smem, st>>>(gram, target, k, q, tol, cap, ridge, H, d_cap,
                                                        (H0 != nullptr && q0 > 0 && q0 < q) ? H0 : nullptr, q0);
  CNMF_LAUNCH_CHECK();
  unsigned long long hcap = 0;
  CNMF_CUDA(cudaMemcpyAsync(&hcap, d_cap, 8, cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaFreeAsync(d_cap, st));
  CNMF_CUDA(cudaStreamSynchronize(st));
  if (n_capped) *n_capped = (int64_t)hcap;
  return CNMF_OK;
}

}  // namespace cnmf
