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
//
// The factor lives packed in shared memory with reciprocal diagonals (every
// substitution step multiplies); a removal rebuilds it by a left-looking
// column Cholesky (O(p) dependent steps, bit-identical to p row insertions).
// XRAY's refits are warm: a column starts from its previous solution, and,
// when the caller keeps per-column factor states (fstate), from its previous
// factor too -- then neither a rebuild nor the first passive-set solve is
// needed. Columns are handed to the warps one at a time (their exchange
// counts vary by an order of magnitude).
#include <algorithm>
#include <cfloat>
#include <cstdio>

#include "common.cuh"

namespace cnmf {
namespace {

#ifdef CNMF_NNLS_STATS
// per-launch event counts (tools builds only): columns, entering indices,
// solves, removals (rebuilds), warm loads, warm rebuilds
__device__ unsigned long long g_nnls_stats[8];
#define NNLS_STAT(i)                                                  \
  do {                                                                \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_nnls_stats[i], 1ull);   \
  } while (0)
__device__ unsigned long long g_nnls_cyc[8];  // cycles: 0 rebuild, 1 add, 2 solve, 3 gradient, 4 load, 5 save, 6 total
#define NNLS_T0 const long long nnls_t0_ = clock64()
#define NNLS_T1(i)                                                                             \
  do {                                                                                         \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_nnls_cyc[i], (unsigned long long)(clock64() - nnls_t0_)); \
  } while (0)
#else
#define NNLS_STAT(i) \
  do {               \
  } while (0)
#define NNLS_T0 \
  do {          \
  } while (0)
#define NNLS_T1(i) \
  do {             \
  } while (0)
#endif

constexpr int kQMax = 64;
// per-column factor state (doubles): [0] passive count or -1, [1, 33) the
// insertion order (64 ints), [33, ...) the packed factor
constexpr int kStateHead = 1 + kQMax / 2;

struct WarpScratch {
  double* L;    // lower factor, packed by rows (entry (i, j), j <= i, at i (i + 1) / 2 + j), insertion order;
                // the diagonal slots hold 1 / L[j][j] (the diagonal is only ever a divisor: the
                // substitutions multiply, which takes the division out of their dependent chains)
  int* order;   // passive indices in insertion order
  int ld;       // unused (packed storage: half the shared memory per warp, twice the warps per SM)
};

__device__ __forceinline__ int tri(int i, int j) { return ((i * (i + 1)) >> 1) + j; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Vectors of length q <= 64 are distributed over the warp: a lane holds
// entries lane and lane + 32 in two named registers (never a dynamically
// indexed array: that is demoted to local memory, which put a store and a
// load on every substitution step).

// One step of a column-oriented substitution on a vector distributed over the
// warp (entries lane, lane + 32): entry j becomes xj = x_j * dinv, entries
// i in (j, hi) lose l_i * xj. Branch-free (the two loads are predicated), so
// a step is ~a dozen instructions with no reconvergence points.
#define NNLS_FWD_STEP(x0, x1, j, hi, L0, L1, dinv)                                         \
  do {                                                                                     \
    const double xj_ = __shfl_sync(0xffffffffu, ((j) >> 5) ? (x1) : (x0), (j)&31) * (dinv); \
    const double l0_ = (lane > (j) && lane < (hi)) ? (L0)[j] : 0.0;                        \
    const double l1_ = (lane + 32 > (j) && lane + 32 < (hi)) ? (L1)[j] : 0.0;              \
    (x0) = (lane == (j)) ? xj_ : (x0) - l0_ * xj_;                                         \
    (x1) = (lane + 32 == (j)) ? xj_ : (x1) - l1_ * xj_;                                    \
  } while (0)

// Extend the factor by index a at position p. Returns false if singular.
// (The helpers are not inlined: the kernel calls them from several places
// and its code footprint decides how often the warps wait for instruction
// fetches -- ncu: "no instruction" was the top stall with everything inlined.)
__device__ __noinline__ bool chol_add(const double* G, int q, WarpScratch ws, int p, int a, double ridge) {
  const int lane = threadIdx.x & 31;
  // b_i = G[order[i]][a] for i < p (row a of the symmetric Gram)
  double b0 = (lane < p) ? G[a * q + ws.order[lane]] : 0.0;
  double b1 = (lane + 32 < p) ? G[a * q + ws.order[lane + 32]] : 0.0;
  const double* L0 = ws.L + tri(lane, 0);
  const double* L1 = ws.L + tri(lane + 32, 0);
  // forward substitution L y = b (column-oriented)
  int dj = 0;  // tri(j, j)
#pragma unroll 2
  for (int j = 0; j < p; ++j) {
    NNLS_FWD_STEP(b0, b1, j, p, L0, L1, ws.L[dj]);
    dj += j + 2;
  }
  double yy = 0.0;
  if (lane < p) {
    yy += b0 * b0;
    ws.L[tri(p, lane)] = b0;
  }
  if (lane + 32 < p) {
    yy += b1 * b1;
    ws.L[tri(p, lane + 32)] = b1;
  }
  yy = warp_sum(yy);
  const double gaa = G[a * q + a] + ridge;
  const double d = gaa - yy;
  __syncwarp();
  if (!(d > 1e-13 * fabs(gaa)) || !isfinite(d)) return false;
  if (lane == 0) {
    ws.L[tri(p, p)] = 1.0 / sqrt(d);
    ws.order[p] = a;
  }
  __syncwarp();
  return true;
}

// Rebuild the factor for the passive set in `ws.order[0..p)` (order kept):
// a left-looking Cholesky by columns. Lane l owns rows l and l + 32; column j
// is one dependent FMA chain of length j per row (all rows in parallel), a
// warp-wide sum for the diagonal, one reciprocal square root -- O(p)
// dependent steps where p successive chol_add calls (a forward substitution
// each) take O(p^2). Every entry goes through exactly the operations chol_add
// would apply, in the same order (L[r][c] = (G[r][c] - sum_{t<c} L[c][t] L[r][t])
// * (1 / L[c][c]) with t ascending; the diagonal from the same lane-distributed
// sum of squares), so the factor is bit-identical to the incremental one.
__device__ __noinline__ bool chol_rebuild(const double* G, int q, WarpScratch ws, int p, double ridge) {
  const int lane = threadIdx.x & 31;
  int ord[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) ord[h] = (lane + 32 * h < p) ? ws.order[lane + 32 * h] : 0;
  for (int j = 0; j < p; ++j) {
    const int oj = ws.order[j];
    const double* Lj = ws.L + tri(j, 0);
    // diagonal: d = G[oj][oj] + ridge - sum_{t<j} L[j][t]^2 (chol_add's sum: position t on lane t % 32)
    double yy = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = lane + 32 * h;
      if (t < j) {
        const double v = Lj[t];
        yy += v * v;
      }
    }
    yy = warp_sum(yy);
    const double gaa = G[oj * q + oj] + ridge;
    const double d = gaa - yy;
    if (!(d > 1e-13 * fabs(gaa)) || !isfinite(d)) return false;
    const double rjj = 1.0 / sqrt(d);
    // column j below the diagonal
    double acc[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) acc[h] = G[ord[h] * q + oj];
    const double* L0 = ws.L + tri(lane, 0);
    const double* L1 = ws.L + tri(lane + 32, 0);
    const bool on0 = lane > j && lane < p, on1 = lane + 32 > j && lane + 32 < p;
    if (on1 && on0) {
      for (int t = 0; t < j; ++t) {
        const double ljt = Lj[t];
        acc[0] -= L0[t] * ljt;
        acc[1] -= L1[t] * ljt;
      }
    } else if (on1) {
      for (int t = 0; t < j; ++t) acc[1] -= L1[t] * Lj[t];
    } else if (on0) {
      for (int t = 0; t < j; ++t) acc[0] -= L0[t] * Lj[t];
    }
    if (on0) ws.L[tri(lane, j)] = acc[0] * rjj;
    if (on1) ws.L[tri(lane + 32, j)] = acc[1] * rjj;
    if (lane == 0) ws.L[tri(j, j)] = rjj;
    __syncwarp();
  }
  return true;
}

// z = G_PP^{-1} t_P scattered to full length (zero off P); (z0, z1) = entries lane, lane + 32.
__device__ __noinline__ double2 chol_solve(double t0, double t1, WarpScratch ws, int p) {
  const int lane = threadIdx.x & 31;
  // gather t at the passive indices (position-ordered)
  const int o0 = (lane < p) ? ws.order[lane] : 0, o1 = (lane + 32 < p) ? ws.order[lane + 32] : 0;
  const double a0 = __shfl_sync(0xffffffffu, t0, o0 & 31), a1 = __shfl_sync(0xffffffffu, t1, o0 & 31);
  const double c0 = __shfl_sync(0xffffffffu, t0, o1 & 31), c1 = __shfl_sync(0xffffffffu, t1, o1 & 31);
  double w0 = (lane < p) ? ((o0 < 32) ? a0 : a1) : 0.0;
  double w1 = (lane + 32 < p) ? ((o1 < 32) ? c0 : c1) : 0.0;
  const double* L0 = ws.L + tri(lane, 0);
  const double* L1 = ws.L + tri(lane + 32, 0);
  // forward L u = t_P
  int dj = 0;  // tri(j, j)
#pragma unroll 2
  for (int j = 0; j < p; ++j) {
    NNLS_FWD_STEP(w0, w1, j, p, L0, L1, ws.L[dj]);
    dj += j + 2;
  }
  // backward L^T v = u: entry j becomes vj, entries i < j lose L[j][i] vj (row j: contiguous)
#pragma unroll 2
  for (int j = p - 1; j >= 0; --j) {
    const double* Lj = ws.L + tri(j, 0);
    const double vj = __shfl_sync(0xffffffffu, (j >> 5) ? w1 : w0, j & 31) * Lj[j];
    const double l0 = (lane < j) ? Lj[lane] : 0.0;
    const double l1 = (lane + 32 < j) ? Lj[lane + 32] : 0.0;
    w0 = (lane == j) ? vj : w0 - l0 * vj;
    w1 = (lane + 32 == j) ? vj : w1 - l1 * vj;
  }
  // scatter back to index space: z[order[i]] = w[i]
  double z0 = 0.0, z1 = 0.0;
#pragma unroll 2
  for (int i = 0; i < p; ++i) {
    const double v = __shfl_sync(0xffffffffu, (i >> 5) ? w1 : w0, i & 31);
    const int oi = ws.order[i];
    z0 = (oi == lane) ? v : z0;
    z1 = (oi == lane + 32) ? v : z1;
  }
  return make_double2(z0, z1);
}

// grad = t - G h (G symmetric: row j is read contiguously)
__device__ __noinline__ double2 nnls_gradient(const double* G, int q, double t0, double t1, double h0, double h1) {
  const int lane = threadIdx.x & 31;
  double g0 = t0, g1 = t1;
  for (int j = 0; j < q; ++j) {
    const double hj = __shfl_sync(0xffffffffu, (j >> 5) ? h1 : h0, j & 31);
    if (hj == 0.0) continue;
    if (lane < q) g0 -= G[j * q + lane] * hj;
    if (lane + 32 < q) g1 -= G[j * q + lane + 32] * hj;
  }
  return make_double2(g0, g1);
}

// H0 (optional, k x q0 with q0 <= q): a feasible start -- the solution of the
// same targets over the first q0 design columns (XRAY's previous refit: the
// picks grow by appending; q0 = q: the right factor after a selection). Its support becomes the initial passive set and
// the iteration proceeds from it exactly as from any feasible iterate; the
// minimiser is unique when the design has full column rank, so only the
// exchange path (not the answer) changes.
__global__ void __launch_bounds__(1024) nnls_kernel(const double* __restrict__ gram_g, const double* __restrict__ target, int64_t k, int q,
                            double tol, int cap, double ridge, double* __restrict__ H,
                            unsigned long long* __restrict__ n_capped, const double* __restrict__ H0, int q0,
                            double* __restrict__ fstate, size_t fstride, unsigned long long* next_col, int tld) {
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

  // columns are handed out one at a time (their exchange counts vary widely:
  // a static split leaves most warps of a block waiting for its slowest)
  for (;;) {
    long long c0 = 0;
    if (lane == 0) c0 = (long long)atomicAdd(next_col, 1ull);
    const int64_t col = __shfl_sync(0xffffffffu, c0, 0);
    if (col >= k) break;
    double t[2], h[2], grad[2];
#ifdef CNMF_NNLS_STATS
    const long long col_t0 = clock64();
#endif
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = lane + 32 * e;
      t[e] = (i < q) ? target[col * tld + i] : 0.0;
      h[e] = 0.0;
      grad[e] = t[e];
    }
    NNLS_STAT(0);
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
        // the factor this column's previous refit ended with (its passive
        // set is the support of H0), when the caller keeps factor states
        bool loaded = false;
        if (fstate != nullptr) {
          const double* fs = fstate + (size_t)col * fstride;
          if ((int)fs[0] == p) {
            const int* fo = (const int*)(fs + 1);
            for (int i = lane; i < p; i += 32) ws.order[i] = fo[i];
            const int nl = tri(p, 0);
            for (int i = lane; i < nl; i += 32) ws.L[i] = fs[kStateHead + i];
            __syncwarp();
            loaded = true;
            NNLS_STAT(4);
          }
        }
        // with the previous factor the passive-set solve would reproduce H0
        // (same system, same operations): go straight to the gradient
        warm = !loaded;
        if (!loaded) {
          NNLS_STAT(5);
          if (lane == 0) {
            int np = 0;
            for (int i = 0; i < q; ++i)
              if ((pas >> i) & 1ull) ws.order[np++] = i;
          }
          __syncwarp();
          ridged = !chol_rebuild(G, q, ws, p, 0.0);
          if (ridged) chol_rebuild(G, q, ws, p, ridge);
        }
        if (loaded) {
          // grad = t - G h at the start
          const double2 gg = nnls_gradient(G, q, t[0], t[1], h[0], h[1]);
          grad[0] = gg.x;
          grad[1] = gg.y;
        }
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
      NNLS_STAT(1);
      ++swaps;
      if (swaps > cap) {
        capped = true;
        break;
      }
      // extend the factor (or rebuild with the ridge when singular)
      bool added;
      {
        NNLS_T0;
        added = factored && !ridged && chol_add(G, q, ws, p, bi, 0.0);
        NNLS_T1(1);
      }
      if (added) {
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
        NNLS_STAT(2);
        {
          NNLS_T0;
          const double2 zz = chol_solve(t[0], t[1], ws, p);
          z[0] = zz.x;
          z[1] = zz.y;
          NNLS_T1(2);
        }
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
        NNLS_STAT(3);
        if (lane == 0) {
          int np = 0;
          for (int i = 0; i < p; ++i)
            if (!((rel >> ws.order[i]) & 1ull)) ws.order[np++] = ws.order[i];
        }
        __syncwarp();
        p = __popcll(pas);
        {
          NNLS_T0;
          ridged = !chol_rebuild(G, q, ws, p, 0.0);
          if (ridged) chol_rebuild(G, q, ws, p, ridge);
          NNLS_T1(0);
        }
        ++swaps;
        if (swaps > cap) {
          capped = true;
          break;
        }
      }
      if (capped) break;
      // grad = t - G h   (G symmetric: read row j for coalescing)
      {
        NNLS_T0;
        const double2 gg = nnls_gradient(G, q, t[0], t[1], h[0], h[1]);
        grad[0] = gg.x;
        grad[1] = gg.y;
        NNLS_T1(3);
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = lane + 32 * e;
      if (i < q) H[col * q + i] = fmax(h[e], 0.0);
    }
    if (capped && lane == 0) atomicAdd(n_capped, 1ull);
    if (fstate != nullptr) {
      // keep the factor for the next refit's warm start (valid when it is
      // the ridge-free factor of the final passive set)
      double* fs = fstate + (size_t)col * fstride;
      const bool keep = !capped && !ridged && factored && p > 0 && (size_t)(kStateHead + tri(p, 0)) <= fstride;
      if (keep) {
        int* fo = (int*)(fs + 1);
        for (int i = lane; i < p; i += 32) fo[i] = ws.order[i];
        const int nl = tri(p, 0);
        for (int i = lane; i < nl; i += 32) fs[kStateHead + i] = ws.L[i];
      }
      if (lane == 0) fs[0] = keep ? (double)p : -1.0;
      __syncwarp();
    }
#ifdef CNMF_NNLS_STATS
    if (lane == 0) atomicAdd(&g_nnls_cyc[6], (unsigned long long)(clock64() - col_t0));
#endif
  }
}

}  // namespace

size_t nnls_state_stride(int qmax) { return (size_t)kStateHead + (size_t)((qmax * (qmax + 1) / 2 + 1) & ~1); }

int nnls_gram(const double* gram, const double* target, int64_t k, int q, double tol, int max_exchanges, double* H,
              int64_t* n_capped, cudaStream_t st, const double* H0, int q0, double* fstate, size_t fstride, int tld) {
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
  CNMF_CUDA(cudaMallocAsync((void**)&d_cap, 16, st));
  CNMF_CUDA(cudaMemsetAsync(d_cap, 0, 16, st));
  const int64_t blocks = std::min<int64_t>(ceil_div(k, wpb), 2 * device_sms());
  nnls_kernel<<<(unsigned)blocks, 32 * wpb, smem, st>>>(gram, target, k, q, tol, cap, ridge, H, d_cap,
                                                        (H0 != nullptr && q0 > 0 && q0 <= q) ? H0 : nullptr, q0,
                                                        fstate, fstride, d_cap + 1, tld > 0 ? tld : q);
  CNMF_LAUNCH_CHECK();
  unsigned long long hcap = 0;
  CNMF_CUDA(cudaMemcpyAsync(&hcap, d_cap, 8, cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaFreeAsync(d_cap, st));
  CNMF_CUDA(cudaStreamSynchronize(st));
  if (n_capped) *n_capped = (int64_t)hcap;
#ifdef CNMF_NNLS_STATS
  {
    unsigned long long hs[8], z8[8] = {0};
    cudaMemcpyFromSymbol(hs, g_nnls_stats, sizeof hs);
    cudaMemcpyToSymbol(g_nnls_stats, z8, sizeof z8);
    unsigned long long hc[8];
    cudaMemcpyFromSymbol(hc, g_nnls_cyc, sizeof hc);
    cudaMemcpyToSymbol(g_nnls_cyc, z8, sizeof z8);
    fprintf(stderr, "[nnls q=%d] kcycles per column: rebuild %.1f add %.1f solve %.1f grad %.1f total %.1f\n", q,
            hc[0] / 1e3 / hs[0], hc[1] / 1e3 / hs[0], hc[2] / 1e3 / hs[0], hc[3] / 1e3 / hs[0], hc[6] / 1e3 / hs[0]);
    fprintf(stderr, "[nnls q=%d] columns %llu enter %llu solves %llu removals %llu loads %llu warm-rebuilds %llu\n", q,
            hs[0], hs[1], hs[2], hs[3], hs[4], hs[5]);
  }
#endif
  return CNMF_OK;
}

}  // namespace cnmf
