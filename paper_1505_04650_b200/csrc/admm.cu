// Compressed ADMM NMF (reference nmf.py:306-377, KKT residual nmf.py:281-303).
//
// The whole iteration loop is ONE persistent cooperative kernel (one CTA per
// SM) with a single grid-wide barrier per iteration:
//
//   split(k)  every CTA owns a contiguous slice of the rows of L (m x s) or of
//             R^T (n x s): it forms L Xc_k (resp. Yc_k R), projects onto the
//             nonnegative orthant, takes the dual step and accumulates every
//             reduction the next step needs (L^T U, L^T dU, R V^T, R dV^T,
//             feasibility and complementarity sums) into acc[k % 3];
//   barrier
//   score(k)  every CTA redundantly finishes the six KKT residuals from
//             acc[k % 3] and applies the reference's stopping and divergence
//             rules — all CTAs reach the same decision without a broadcast;
//   core(k+1) every CTA redundantly solves the two r x r ridge systems for
//             Xc_{k+1}, Yc_{k+1} (block Gauss-Jordan inverses) in shared
//             memory, so the next split needs no global round trip.
//
// When a CTA's slice fits in shared memory (configs[1]: ~100 rows per CTA),
// its rows of the basis, U and dU stay resident there for the whole run: an
// iteration then touches global memory only for the reduced partials.
// acc is triple-buffered: a buffer is zeroed (by CTA 0, during split k) two
// barriers after its last reader, so one barrier per iteration suffices;
// reads of the reduced partials bypass L1 (ld.global.cg).
// Sizes are compile-time (s <= SP, r <= RP, zero padded: exact) so every
// small product is an unrolled register-blocked loop.
// The state is fp64 (the method is sensitive to roundoff over hundreds of
// iterations); the bases are the fp32 panels produced by the compression.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace cnmf {
namespace {

constexpr int kMax = 64;      // s, r <= 64
constexpr int kTile = 32;     // rows per streamed split tile
constexpr int kThreads = 256;
constexpr size_t kSmemCap = 227 * 1024 - 512;  // B200 opt-in maximum less the static red[]

struct Ctrl {
  int k;         // next iteration index (resume point)
  int done;
  int iters;     // iterations completed when done
  int diverged;  // iteration index (0-based) that tripped the divergence rule, or -1
  unsigned int bar_count;  // grid_barrier arrivals in this launch
  unsigned int bar_gen;
};

// reduced partials of one split sweep (stride kMax so every SP/RP fits)
struct Acc {
  double LtU[kMax * kMax];   // s x r : L^T U
  double RtV[kMax * kMax];   // s x r : R V^T   (= (V R^T)^T)
  double scal[4];            // feasL^2, compL^2, feasR^2, compR^2
};

// State every CTA keeps redundantly, saved here between launches. The dual
// projections L^T dU and R dV^T are linear in dU, dV, so they follow from the
// dual step dU_k = dU_{k-1} + step pu (L Xc_k - U_k) without a reduction:
//   L^T dU_k = L^T dU_{k-1} + step pu (G_L Xc_k - L^T U_k),  G_L = L^T L
// (the same for the right side with G_R = R R^T), which halves the per-row
// products and the cross-CTA atomics of every split.
struct Rep {
  double GL[kMax * kMax];  // s x s : L^T L (fp64 of the fp32 panel)
  double GR[kMax * kMax];  // s x s : R R^T
  double DL[kMax * kMax];  // s x r : L^T dU
  double DR[kMax * kMax];  // s x r : R dV^T
};

// What the helper CTA publishes for window k (between barriers k and k + 1),
// double-buffered by the parity of k: the ridge inverse and the right-hand
// side parts of core(k + 1) that depend only on (xc_k, yc_k), and that state
// itself for the scorer CTA.
struct Pub {
  double Minv[kMax * kMax];  // r x r : (yc_k yc_k^T + pu I)^{-1}
  double P1[kMax * kMax];    // s x r : C yc_k^T - TL
  double TL[kMax * kMax];    // s x r : L^T dU_{k-1} + step pu G_L xc_k
  double TR[kMax * kMax];    // s x r : R dV_{k-1}^T + step pv G_R yc_k^T
  double xc[kMax * kMax];    // s x r
  double yc[kMax * kMax];    // r x s
};

struct Side {
  const float* P;  // panel (rows x S)
  int64_t rows;
  int S;
  double* U;       // rows x r
  double* D;       // rows x r
  double pen;
};

struct Params {
  const double* core;
  Side left, right;
  int s, r;
  double pu, pv, step, tol;
  int max_iter;
  int step_limit;  // > 0: stop after this many splits (resume later)
  int fresh;
  int nblk_left;
  int64_t rows_left, rows_right;  // rows per CTA slice
  double* xc_g;
  double* yc_g;
  double* trace;
  double* scores;
  Ctrl* ctrl;
  Acc* acc;  // [3]
  Rep* rep;
  Pub* pub;  // [2]
  unsigned long long* prof;  // optional: per-iteration phase timestamps (CTA 0)
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void stamp(const Params& p, int k, int slot) {
  if (p.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0 && k < 256) p.prof[k * 8 + slot] = gtime();
}

__device__ unsigned long long* g_prof_ptr;  // CTA 0 phase stamps (profiling only)
__device__ int g_prof_k;
__device__ __forceinline__ void sstamp(int slot) {
  if (g_prof_ptr != nullptr && blockIdx.x == 0 && threadIdx.x == 0 && g_prof_k < 256)
    g_prof_ptr[g_prof_k * 8 + slot] = gtime();
}

__device__ __forceinline__ double ld(const double* p) { return __ldcg(p); }

// D (8 x 8) += A (8 x 4, row g, column t) B (4 x 8, row t, column g) on the
// fp64 tensor cores; the accumulator holds row g, columns 2 t, 2 t + 1
// (g = lane / 4, t = lane % 4)
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Grid barrier on a counter that only grows within a launch (the host zeroes
// it before every launch): barrier i of the launch completes when the count
// reaches (i + 1) * gridDim.x, so arrival is one atomic and the release is
// seen by the waiters directly (no second "generation" atomic).
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ void grid_barrier(Ctrl* c, unsigned int& epoch) {
  __syncthreads();
  epoch += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&c->bar_count, 1u);
    while ((int)(ld_acquire(&c->bar_count) - epoch) < 0) {
    }
  }
  __syncthreads();
}

// out(i, j) = sum_k a(i, k) b(k, j) for an MO x NO output (MO, NO multiples
// of 16): a 16 x 16 thread grid, each thread a (MO/16) x (NO/16) register
// block (i = ti + 16 a, j = tj + 16 b), so per k it loads MO/16 + NO/16
// operands for (MO/16)(NO/16) FMAs. Operands are read through accessors;
// callers use odd leading dimensions, so transposed reads are conflict-free.
template <int MO, int NO, int K, class FA, class FB, class FO>
__device__ __forceinline__ void bgemm(FA a, FB b, FO o) {
  static_assert(MO % 16 == 0 && NO % 16 == 0, "bgemm tiles");
  constexpr int BI = MO / 16, BJ = NO / 16;
  const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;
  double acc[BI][BJ];
#pragma unroll
  for (int x = 0; x < BI; ++x)
#pragma unroll
    for (int y = 0; y < BJ; ++y) acc[x][y] = 0.0;
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    double av[BI], bv[BJ];
#pragma unroll
    for (int x = 0; x < BI; ++x) av[x] = a(ti + 16 * x, k);
#pragma unroll
    for (int y = 0; y < BJ; ++y) bv[y] = b(k, tj + 16 * y);
#pragma unroll
    for (int x = 0; x < BI; ++x)
#pragma unroll
      for (int y = 0; y < BJ; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
  }
#pragma unroll
  for (int x = 0; x < BI; ++x)
#pragma unroll
    for (int y = 0; y < BJ; ++y) o(ti + 16 * x, tj + 16 * y, acc[x][y]);
}

// Gauss-Jordan inverse of the leading r x r block of the RP x RP SPD matrix
// M by the whole block, ping-ponging between M and T so that each pivot step
// reads only the previous matrix: one barrier per pivot. The padded block is
// pen*I and is inverted on the diagonal. The result ends in M.
template <int RP>
__device__ void gj_inverse(double* M, double* T, int r) {
  constexpr int LR = RP + 1;
  const int tid = threadIdx.x;
  double* src = M;
  double* dst = T;
  for (int k = 0; k < r; ++k) {
    const double inv = 1.0 / src[k * LR + k];
#pragma unroll
    for (int t = 0; t < (RP * RP + kThreads - 1) / kThreads; ++t) {
      const int idx = tid + t * kThreads;
      if (idx < RP * RP) {
        const int i = idx / RP, j = idx % RP;
        if (i < r && j < r) {
          const double nk = ((j == k) ? 1.0 : src[k * LR + j]) * inv;
          dst[i * LR + j] = (i == k) ? nk : ((j == k) ? 0.0 : src[i * LR + j]) - src[i * LR + k] * nk;
        }
      }
    }
    __syncthreads();
    double* tmp = src;
    src = dst;
    dst = tmp;
  }
  if (src != M) {
    for (int idx = tid; idx < r * RP; idx += kThreads) {
      const int i = idx / RP, j = idx % RP;
      if (j < r) M[i * LR + j] = src[i * LR + j];
    }
  }
  for (int i = r + tid; i < RP; i += kThreads) M[i * LR + i] = 1.0 / M[i * LR + i];
  __syncthreads();
}

// The same inverse with the matrix in registers (RP <= 32): warp w owns rows
// w + 8 t, lane j column j. Pivot k's row is published to shared memory by
// its owner warp, column k reaches the row owners by a shuffle from lane k,
// one barrier per pivot. The pivot loop is unrolled so every register index
// is a compile-time constant: a dynamically indexed read would demote the
// row array to local memory (measured: 750 -> 370 cycles per pivot).
template <int RP>
__device__ void gj_inverse_reg(double* M, double* strip, int r) {
  static_assert(RP <= 32 && RP % 8 == 0, "one column per lane, RP / 8 rows per warp");
  constexpr int LR = RP + 1, RT = RP / 8;
  const int w = threadIdx.x >> 5, j = threadIdx.x & 31;
  double a[RT];
#pragma unroll
  for (int t = 0; t < RT; ++t) a[t] = (j < RP) ? M[(w + 8 * t) * LR + j] : 0.0;
#pragma unroll
  for (int k = 0; k < RP; ++k) {
    if (k >= r) break;  // uniform
    double* prow = strip + (k & 1) * 32;
    if (w == (k & 7) && j < RP) prow[j] = a[k >> 3];
    double colk[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) colk[t] = __shfl_sync(0xffffffffu, a[t], k);
    __syncthreads();
    const double inv = 1.0 / prow[k];
    const double nk = ((j == k) ? 1.0 : prow[j]) * inv;
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int i = w + 8 * t;
      if (i < r && j < r) a[t] = (i == k) ? nk : ((j == k) ? 0.0 : a[t]) - colk[t] * nk;
    }
  }
#pragma unroll
  for (int t = 0; t < RT; ++t) {
    const int i = w + 8 * t;
    if (j < RP) M[i * LR + j] = (i >= r && i == j) ? 1.0 / a[t] : a[t];
  }
  __syncthreads();
}

// Gauss-Jordan inverse of the leading r x r block by ONE warp (RP <= 32):
// lane i owns row i in shared memory; per pivot the pivot row is broadcast
// into registers and each lane updates its own row, so the only
// synchronisation is __syncwarp. The other warps stay free for independent
// work meanwhile.
template <int RP>
__device__ void gj_warp(double* M, int r) {
  static_assert(RP <= 32, "one row per lane");
  constexpr int LR = RP + 1;
  const int i = threadIdx.x & 31;
  double row[RP];
#pragma unroll
  for (int j = 0; j < RP; ++j) row[j] = (i < RP) ? M[i * LR + j] : 0.0;
  for (int k = 0; k < r; ++k) {
    double f = 0.0;
#pragma unroll
    for (int j = 0; j < RP; ++j) f = (j == k) ? row[j] : f;  // row_i[k] without dynamic indexing
    const double inv = 1.0 / __shfl_sync(0xffffffffu, f, k);
#pragma unroll
    for (int j = 0; j < RP; ++j) {
      const double nk = ((j == k) ? 1.0 : __shfl_sync(0xffffffffu, row[j], k)) * inv;
      row[j] = (i == k) ? nk : ((j == k) ? 0.0 : row[j]) - f * nk;
    }
  }
  if (i < RP) {
#pragma unroll
    for (int j = 0; j < RP; ++j) M[i * LR + j] = (j >= r && i == j) ? 1.0 / row[j] : row[j];
  }
  __syncwarp();
}

// out(i, j) = sum_k a(i, k) b(k, j) by threads [first, kThreads) (plain
// strided loop; used for work that overlaps a one-warp inverse).
template <int MO, int NO, int K, class FA, class FB, class FO>
__device__ __forceinline__ void sgemm_part(int first, FA a, FB b, FO o) {
  for (int idx = threadIdx.x - first; idx < MO * NO; idx += kThreads - first) {
    const int i = idx / NO, j = idx % NO;
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int k = 0; k < K; k += 2) {
      v0 = fma(a(i, k), b(k, j), v0);
      v1 = fma(a(i, k + 1), b(k + 1, j), v1);
    }
    o(i, j, v0 + v1);
  }
}

template <int SP, int RP>
struct Smem {
  static constexpr int LS = SP + 1, LR = RP + 1;  // odd strides: conflict-free columns
  double* C;   // SP x SP
  double* xc;  // SP x RP
  double* yc;  // RP x SP
  double* X;   // SP x RP  split operand (xc or yc^T)
  double* W;   // SP x SP  scratch
  double* M;   // RP x RP
  double* T;   // RP x RP  Gauss-Jordan ping-pong buffer
  // staged reductions and published parts (speculative layout only)
  double *LU, *RV;      // SP x RP : L^T U, R V^T of the last split
  double *Minv, *P1;    // RP x RP, SP x RP
  double *TL, *TR;      // SP x RP
  double* GL;  // SP x SP  L^T L      (Rep)
  double* GR;  // SP x SP  R R^T
  double* DL;  // SP x RP  L^T dU
  double* DR;  // SP x RP  R dV^T
  double* fold;  // 256 x 16: row-group folding of the split accumulators
  double* Pt;  // rows x (SP + 2) (resident slice or one tile; the padding
               // shifts consecutive rows by 16 B so paired row reads do not
               // share banks)
  double *Ut0, *Ut1;  // rows x r (row stride r); two buffers when the score
  double *Dt0, *Dt1;  // runs a split behind (selected, never indexed: an
                      // indexed member array would move the struct to the stack)
  __device__ double* Ut(int b) const { return b ? Ut1 : Ut0; }
  __device__ double* Dt(int b) const { return b ? Dt1 : Dt0; }
  static constexpr int kCommon = 2 * SP * LS + 2 * SP * LR + RP * LS + 2 * RP * LR;
  static constexpr int kStage = 5 * SP * LR + RP * LR > kThreads * 16 ? 5 * SP * LR + RP * LR : kThreads * 16;
  static constexpr int kGram = 2 * SP * LS + 2 * SP * LR;
  // spec: the fold (split) and the staged reductions (core) are never live
  // together, and the Gram / dual state (helper CTAs) and the resident slice
  // (split CTAs) never share a CTA
  __device__ Smem(double* base, int rows, bool spec, int r) {
    C = base;
    xc = C + SP * LS;
    yc = xc + SP * LR;
    X = yc + RP * LS;
    W = X + SP * LR;
    M = W + SP * LS;
    T = M + RP * LR;
    double* q = T + RP * LR;
    if (spec) {
      LU = q;
      RV = LU + SP * LR;
      Minv = RV + SP * LR;
      P1 = Minv + RP * LR;
      TL = P1 + SP * LR;
      TR = TL + SP * LR;
      fold = q;
      q += kStage;
    } else {
      LU = RV = Minv = P1 = TL = TR = nullptr;
    }
    GL = q;
    GR = GL + SP * LS;
    DL = GR + SP * LS;
    DR = DL + SP * LR;
    if (!spec) {
      fold = DR + SP * LR;
      Pt = fold + kThreads * 16;
    } else {
      Pt = q;
    }
    Ut0 = Pt + (size_t)rows * (SP + 2);
    Dt0 = Ut0 + (size_t)rows * r;
    Ut1 = spec ? Dt0 + (size_t)rows * r : Ut0;
    Dt1 = spec ? Ut1 + (size_t)rows * r : Dt0;
  }
  static size_t bytes(int rows, bool spec, int r) {
    const size_t slice = (size_t)rows * (SP + 2 + (spec ? 4 : 2) * r);
    if (spec) return ((size_t)kCommon + kStage + std::max<size_t>(slice, kGram)) * 8;
    return ((size_t)kCommon + kGram + kThreads * 16 + slice) * 8;
  }
};

// KKT score of the state (xc, yc) with the split reductions `a` (nmf.py:281-303).
template <int SP, int RP>
__device__ double kkt_score(const Smem<SP, RP>& sm, const Acc* a, double* red, double* objective) {
  constexpr int LS = SP + 1, LR = RP + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* xc = sm.xc;
  const double* yc = sm.yc;
  double* W = sm.W;
  const double* C = sm.C;
  // E = xc yc - C
  double e2 = 0.0;
  bgemm<SP, SP, RP>([&](int i, int k) { return xc[i * LR + k]; }, [&](int k, int j) { return yc[k * LS + j]; },
                    [&](int i, int j, double v) {
                      const double e = v - C[i * LS + j];
                      W[i * LS + j] = e;
                      e2 += e * e;
                    });
  __syncthreads();
  double g1 = 0.0, g2 = 0.0;
  // E yc^T + L^T dU   and   xc^T E + dV R^T
  bgemm<SP, RP, SP>([&](int i, int k) { return W[i * LS + k]; }, [&](int k, int j) { return yc[j * LS + k]; },
                    [&](int i, int j, double v) {
                      const double t = v + sm.DL[i * LR + j];
                      g1 += t * t;
                    });
  bgemm<RP, SP, SP>([&](int i, int k) { return xc[k * LR + i]; }, [&](int k, int j) { return W[k * LS + j]; },
                    [&](int i, int j, double v) {
                      const double t = v + sm.DR[j * LR + i];
                      g2 += t * t;
                    });
  g1 = wsum(g1);
  g2 = wsum(g2);
  e2 = wsum(e2);
  if (lane == 0) {
    red[3 * warp] = g1;
    red[3 * warp + 1] = g2;
    red[3 * warp + 2] = e2;
  }
  __syncthreads();
  double t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    t1 += red[3 * w];
    t2 += red[3 * w + 1];
    t3 += red[3 * w + 2];
  }
  *objective = t3;
  __syncthreads();
  return fmax(fmax(fmax(sqrt(t1), sqrt(t2)), fmax(sqrt(ld(&a->scal[0])), sqrt(ld(&a->scal[2])))),
              fmax(sqrt(ld(&a->scal[1])), sqrt(ld(&a->scal[3]))));
}

// Xc, Yc of the next iteration from the current yc and the split reductions
// (nmf.py:350-353). For RP <= 32 each r x r inverse runs on warp 0 while the
// other warps form the matching right-hand side.
template <int SP, int RP>
__device__ void core_step(const Smem<SP, RP>& sm, const Acc* a, int s, int r, double pu, double pv) {
  constexpr int LS = SP + 1, LR = RP + 1;
  double* xc = sm.xc;
  double* yc = sm.yc;
  double* W = sm.W;
  const double* C = sm.C;
  double* M = sm.M;
  // Xc = rhs (yc yc^T + pu I)^{-1},  rhs = C yc^T + pu L^T U - L^T dU:
  // one product [yc; C] yc^T gives the ridge matrix and the right-hand side
  bgemm<RP + SP, RP, SP>(
      [&](int i, int k) { return i < RP ? yc[i * LS + k] : C[(i - RP) * LS + k]; },
      [&](int k, int j) { return yc[j * LS + k]; },
      [&](int i, int j, double v) {
        if (i < RP) {
          M[i * LR + j] = v + (i == j ? pu : 0.0);
        } else {
          const int q = i - RP;
          W[q * LS + j] = v + pu * ld(&a->LtU[q * kMax + j]) - sm.DL[q * LR + j];
        }
      });
  __syncthreads();
  if constexpr (RP <= 32)
    gj_inverse_reg<RP>(M, sm.T, r);  // its first barrier also orders the products above
  else
    gj_inverse<RP>(M, sm.T, r);
  sstamp(6);
  bgemm<SP, RP, RP>([&](int i, int k) { return W[i * LS + k]; }, [&](int k, int j) { return M[k * LR + j]; },
                    [&](int i, int j, double v) { xc[i * LR + j] = (i < s && j < r) ? v : 0.0; });
  __syncthreads();
  // Yc = (xc^T xc + pv I)^{-1} (xc^T C + pv V R^T - dV R^T): one product
  // xc^T [xc | C]
  bgemm<RP, RP + SP, SP>(
      [&](int i, int k) { return xc[k * LR + i]; },
      [&](int k, int j) { return j < RP ? xc[k * LR + j] : C[k * LS + (j - RP)]; },
      [&](int i, int j, double v) {
        if (j < RP) {
          M[i * LR + j] = v + (i == j ? pv : 0.0);
        } else {
          const int q = j - RP;
          W[i * LS + q] = v + pv * ld(&a->RtV[q * kMax + i]) - sm.DR[q * LR + i];
        }
      });
  __syncthreads();
  if constexpr (RP <= 32)
    gj_inverse_reg<RP>(M, sm.T, r);
  else
    gj_inverse<RP>(M, sm.T, r);
  sstamp(7);
  bgemm<RP, SP, RP>([&](int i, int k) { return M[i * LR + k]; }, [&](int k, int j) { return W[k * LS + j]; },
                    [&](int i, int j, double v) { yc[i * LS + j] = (i < r && j < s) ? v : 0.0; });
  __syncthreads();
}

// Dual projections of iteration k from those of k - 1 (see Rep): xc, yc are
// the state split k used, `a` its reductions. Every CTA runs the same
// instructions on the same data, so the replicated copies stay identical.
template <int SP, int RP>
__device__ void dual_update(const Smem<SP, RP>& sm, const Acc* a, int s, int r, double spl, double spr) {
  constexpr int LS = SP + 1, LR = RP + 1;
  bgemm<SP, RP, SP>([&](int i, int k) { return sm.GL[i * LS + k]; }, [&](int k, int j) { return sm.xc[k * LR + j]; },
                    [&](int i, int j, double v) {
                      if (i < s && j < r) sm.DL[i * LR + j] += spl * (v - ld(&a->LtU[i * kMax + j]));
                    });
  bgemm<SP, RP, SP>([&](int i, int k) { return sm.GR[i * LS + k]; }, [&](int k, int j) { return sm.yc[j * LS + k]; },
                    [&](int i, int j, double v) {
                      if (i < s && j < r) sm.DR[i * LR + j] += spr * (v - ld(&a->RtV[i * kMax + j]));
                    });
  __syncthreads();
}

// Role of a CTA in the speculative schedule.
enum Role { kWorker = 0, kHelper = 1, kScorer = 2 };

// After barrier k: the reductions of split k, and the parts of core(k + 1)
// the helper published for this window, into shared memory (one round of
// L2 loads), zero padded.
template <int SP, int RP>
__device__ void stage(const Smem<SP, RP>& sm, const Acc* a, const Pub* pb, int role, int s, int r) {
  constexpr int LS = SP + 1, LR = RP + 1;
  // batches of 4 entries per thread, every load of a batch issued before
  // the first store (one L2 round trip per batch, not per entry)
  constexpr int NT = (SP * RP + kThreads - 1) / kThreads, NB = NT < 4 ? NT : 4;
#pragma unroll 1
  for (int t0 = 0; t0 < NT; t0 += NB) {
    double v[NB][6];
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int idx = threadIdx.x + (t0 + t) * kThreads;
      const int i = idx / RP, j = idx % RP;
      const bool in = idx < SP * RP && i < s && j < r;
      const int g = i * kMax + j;
      v[t][0] = in ? ld(&a->LtU[g]) : 0.0;
      v[t][1] = in ? ld(&a->RtV[g]) : 0.0;
      v[t][2] = in && role != kHelper ? ld(role == kWorker ? &pb->P1[g] : &pb->TL[g]) : 0.0;
      v[t][3] = in && role != kHelper ? ld(&pb->TR[g]) : 0.0;
      v[t][4] = in && role == kScorer ? ld(&pb->xc[g]) : 0.0;
      v[t][5] = in && role == kScorer ? ld(&pb->yc[j * kMax + i]) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int idx = threadIdx.x + (t0 + t) * kThreads;
      if (idx >= SP * RP) continue;
      const int i = idx / RP, j = idx % RP, o = i * LR + j;
      sm.LU[o] = v[t][0];
      sm.RV[o] = v[t][1];
      if (role == kWorker) sm.P1[o] = v[t][2];
      if (role == kScorer) {
        sm.TL[o] = v[t][2];
        sm.xc[o] = v[t][4];
        sm.yc[j * LS + i] = v[t][5];
      }
      if (role != kHelper) sm.TR[o] = v[t][3];
    }
  }
  if (role == kWorker) {
    constexpr int NM = (RP * RP + kThreads - 1) / kThreads, NC = NM < 8 ? NM : 8;
#pragma unroll 1
    for (int t0 = 0; t0 < NM; t0 += NC) {
      double v[NC];
#pragma unroll
      for (int t = 0; t < NC; ++t) {
        const int idx = threadIdx.x + (t0 + t) * kThreads;
        v[t] = idx < RP * RP ? ld(&pb->Minv[(idx / RP) * kMax + idx % RP]) : 0.0;
      }
#pragma unroll
      for (int t = 0; t < NC; ++t) {
        const int idx = threadIdx.x + (t0 + t) * kThreads;
        if (idx < RP * RP) sm.Minv[(idx / RP) * LR + idx % RP] = v[t];
      }
    }
  }
  __syncthreads();
}

// dual projections of split k from the published parts:
// L^T dU_k = TL - step pu L^T U_k (the same expression on every CTA that needs it)
template <int SP, int RP>
__device__ void duals_from_published(const Smem<SP, RP>& sm, double spl, double spr) {
  for (int idx = threadIdx.x; idx < SP * (RP + 1); idx += kThreads) {
    sm.DL[idx] = fma(-spl, sm.LU[idx], sm.TL[idx]);
    sm.DR[idx] = fma(-spr, sm.RV[idx], sm.TR[idx]);
  }
  __syncthreads();
}

// core(k + 1) given the published inverse and right-hand side parts
// (nmf.py:350-353): xc = (P1 + (pu + step pu) L^T U) Minv, then the
// yc solve as in core_step with R dV^T = TR - step pv R V^T folded in.
template <int SP, int RP>
__device__ void fast_core(const Smem<SP, RP>& sm, int s, int r, double pv, double cl, double cr) {
  constexpr int LS = SP + 1, LR = RP + 1;
  double* xc = sm.xc;
  double* M = sm.M;
  double* W = sm.W;
  bgemm<SP, RP, RP>([&](int i, int k) { return fma(cl, sm.LU[i * LR + k], sm.P1[i * LR + k]); },
                    [&](int k, int j) { return sm.Minv[k * LR + j]; },
                    [&](int i, int j, double v) { xc[i * LR + j] = (i < s && j < r) ? v : 0.0; });
  __syncthreads();
  sstamp(6);
  bgemm<RP, RP + SP, SP>(
      [&](int i, int k) { return xc[k * LR + i]; },
      [&](int k, int j) { return j < RP ? xc[k * LR + j] : sm.C[k * LS + (j - RP)]; },
      [&](int i, int j, double v) {
        if (j < RP) {
          M[i * LR + j] = v + (i == j ? pv : 0.0);
        } else {
          const int q = j - RP;
          W[i * LS + q] = v + fma(cr, sm.RV[q * LR + i], -sm.TR[q * LR + i]);
        }
      });
  __syncthreads();
  if constexpr (RP <= 32)
    gj_inverse_reg<RP>(M, sm.T, r);
  else
    gj_inverse<RP>(M, sm.T, r);
  sstamp(7);
  bgemm<RP, SP, RP>([&](int i, int k) { return M[i * LR + k]; }, [&](int k, int j) { return W[k * LS + j]; },
                    [&](int i, int j, double v) { sm.yc[i * LS + j] = (i < r && j < s) ? v : 0.0; });
  __syncthreads();
}

// Helper CTA: from the new state (xc_k, yc_k) and the duals of split k - 1
// (DL, DR), the parts of core(k + 1) that do not depend on split k, into its
// own shared memory and into `out` for the other CTAs.
template <int SP, int RP>
__device__ void precompute(const Smem<SP, RP>& sm, int s, int r, double pu, double spl, double spr, Pub* out) {
  constexpr int LS = SP + 1, LR = RP + 1;
  const double* yc = sm.yc;
  double* M = sm.M;
  bgemm<RP + SP, RP, SP>(
      [&](int i, int k) { return i < RP ? yc[i * LS + k] : sm.C[(i - RP) * LS + k]; },
      [&](int k, int j) { return yc[j * LS + k]; },
      [&](int i, int j, double v) {
        if (i < RP)
          M[i * LR + j] = v + (i == j ? pu : 0.0);
        else
          sm.P1[(i - RP) * LR + j] = v;
      });
  bgemm<SP, RP, SP>([&](int i, int k) { return sm.GL[i * LS + k]; }, [&](int k, int j) { return sm.xc[k * LR + j]; },
                    [&](int i, int j, double v) {
                      sm.TL[i * LR + j] = (i < s && j < r) ? fma(spl, v, sm.DL[i * LR + j]) : 0.0;
                    });
  bgemm<SP, RP, SP>([&](int i, int k) { return sm.GR[i * LS + k]; }, [&](int k, int j) { return yc[j * LS + k]; },
                    [&](int i, int j, double v) {
                      sm.TR[i * LR + j] = (i < s && j < r) ? fma(spr, v, sm.DR[i * LR + j]) : 0.0;
                    });
  __syncthreads();
  if constexpr (RP <= 32)
    gj_inverse_reg<RP>(M, sm.T, r);
  else
    gj_inverse<RP>(M, sm.T, r);
  for (int idx = threadIdx.x; idx < SP * RP; idx += kThreads) {
    const int i = idx / RP, j = idx % RP;
    const int g = i * kMax + j, o = i * LR + j;
    const bool in = i < s && j < r;
    const double p1 = in ? sm.P1[o] - sm.TL[o] : 0.0;
    sm.P1[o] = p1;
    out->P1[g] = p1;
    out->TL[g] = sm.TL[o];
    out->TR[g] = sm.TR[o];
    out->xc[g] = sm.xc[o];
    out->yc[j * kMax + i] = sm.yc[j * LS + i];
  }
  for (int idx = threadIdx.x; idx < RP * RP; idx += kThreads) {
    const int i = idx / RP, j = idx % RP;
    const double v = M[i * LR + j];
    sm.Minv[i * LR + j] = v;
    out->Minv[i * kMax + j] = v;
  }
  __syncthreads();
}

// Split sweep of one CTA over its contiguous slice [r0, r1) of a side.
// mode 0: initial projection: load U0 into buffer wb, accumulate P^T U0 and
// the Gram matrix P^T P (into gram); mode 1: full update reading dU from
// buffer wb ^ 1 and writing U, dU into buffer wb (one buffer without the
// speculative score: wb ^ 1 aliases wb).
// RES: the slice lives in shared memory (loaded when `load`).
template <int SP, int RP, bool RES>
__device__ void split_side(const Side& a, const Smem<SP, RP>& sm, bool right, int s, int r, double step, int mode,
                           int64_t r0, int64_t r1, bool load, int wb, double* accU, double* gram, double* scal,
                           double* red) {
  const int tid = threadIdx.x;
  constexpr int NBJ = SP / 4, NBB = RP / 4, NBLK = NBJ * NBB;
  constexpr int GROUPS = NBLK >= kThreads ? 1 : kThreads / NBLK;
  constexpr int NG = (SP * SP + kThreads - 1) / kThreads;
  const int grp = tid / NBLK, myb = tid - grp * NBLK;
  const bool own = grp < GROUPS;
  const int bj = own ? myb / NBB : 0, bb = own ? myb % NBB : 0;
  double* Uw = sm.Ut(wb);
  double* Dw = sm.Dt(wb);
  double* Dr = sm.Dt(wb ^ 1);
  double au[4][4], g[NG];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) au[x][y] = 0.0;
#pragma unroll
  for (int t = 0; t < NG; ++t) g[t] = 0.0;
  double feas = 0.0, comp = 0.0;
  const double invpen = 1.0 / a.pen, sp_ = step * a.pen;
  constexpr int LS = SP + 1, LR = RP + 1;
  // split operand X (SP x RP): xc, or yc^T for the right side
  if (mode == 1) {
    for (int i = tid; i < SP * RP; i += kThreads) {
      const int j = i / RP, b = i % RP;
      sm.X[j * LR + b] = right ? sm.yc[b * LS + j] : sm.xc[j * LR + b];
    }
  }
  const int64_t span = RES ? (r1 - r0) : kTile;
  for (int64_t t0 = r0; t0 < r1; t0 += span) {
    const int nr = (int)min64(span, r1 - t0);
    __syncthreads();
    if (!RES || load) {
      for (int i = tid; i < nr * SP; i += kThreads) {
        const int rr = i / SP, c = i % SP;
        sm.Pt[rr * (SP + 2) + c] = (c < s) ? (double)a.P[(t0 + rr) * a.S + c] : 0.0;
      }
      for (int i = tid; i < nr * r; i += kThreads) {
        if (mode == 0) {
          Uw[i] = a.U[t0 * r + i];
          Dw[i] = 0.0;
        } else {
          Dr[i] = a.D[t0 * r + i];
        }
      }
      __syncthreads();
    }
    if (mode == 0) {
#pragma unroll
      for (int t = 0; t < NG; ++t) {
        const int e = tid + t * kThreads, j = e / SP, l = e % SP;
        if (e < SP * SP)
          for (int rr = 0; rr < nr; ++rr) g[t] = fma(sm.Pt[rr * (SP + 2) + j], sm.Pt[rr * (SP + 2) + l], g[t]);
      }
    }
    if (RES && mode == 1) {
      // Resident slice: both products on the fp64 tensor cores (DMMA m8n8k4).
      // lx = P X (nr x r, K = s): warp w owns the 8-row tiles w, w + 8, ...,
      // all r / 8 column tiles of each; then u = max(lx + d/pen, 0),
      // d += step*pen*(lx - u) (nmf.py:354-357) on the accumulator fragments.
      const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
      constexpr int NT = RP / 8, KS = SP / 4, NW = kThreads / 32;
      const int nmt = (nr + 7) >> 3, nnt = min(NT, (r + 7) >> 3);
      for (int mt0 = warp; mt0 < nmt; mt0 += 2 * NW) {
        // two row tiles (mt0, mt0 + 8) at a time: 2 x r / 8 independent accumulators
        double dd[2][NT][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) dd[h][ni][0] = dd[h][ni][1] = 0.0;
        const bool two = mt0 + NW < nmt;
        int rrs[2];
        const double* pa[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          rrs[h] = 8 * (mt0 + h * NW) + g;  // rows >= nr compute on the last row and are dropped
          pa[h] = sm.Pt + min(rrs[h], nr - 1) * (SP + 2) + tq;
        }
        const double* xb = sm.X + tq * LR + g;
        // even and odd k steps accumulate separately: a dependent DMMA waits
        // ~300 cycles for its predecessor, so the chains are kept short and
        // 4 x r / 8 of them are in flight per warp
        double de[2][NT][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) de[h][ni][0] = de[h][ni][1] = 0.0;
        static_assert(KS % 2 == 0, "k steps in pairs");
#pragma unroll
        for (int ks = 0; ks < KS; ks += 2) {
          const double a0 = pa[0][4 * ks], a1 = pa[1][4 * ks];
          const double a2 = pa[0][4 * ks + 4], a3 = pa[1][4 * ks + 4];
          double bv[NT], bw[NT];
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            bv[ni] = xb[4 * ks * LR + 8 * ni];
            bw[ni] = xb[(4 * ks + 4) * LR + 8 * ni];
          }
#pragma unroll
          for (int ni = 0; ni < NT; ++ni)
            if (ni < nnt) {
              dmma(dd[0][ni], a0, bv[ni]);
              dmma(de[0][ni], a2, bw[ni]);
              if (two) {
                dmma(dd[1][ni], a1, bv[ni]);
                dmma(de[1][ni], a3, bw[ni]);
              }
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            dd[h][ni][0] += de[h][ni][0];
            dd[h][ni][1] += de[h][ni][1];
          }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int rr = rrs[h];
          if (rr >= nr || (h == 1 && !two)) continue;
#pragma unroll
          for (int ni = 0; ni < NT; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int b = 8 * ni + 2 * tq + e;
              if (b >= r) continue;
              const int i = rr * r + b;
              const double lx = dd[h][ni][e];
              const double d0 = Dr[i];
              const double u = fmax(lx + d0 * invpen, 0.0);
              const double d1 = d0 + sp_ * (lx - u);
              Uw[i] = u;
              Dw[i] = d1;
              const double fe = lx - u;
              feas += fe * fe;
              const double du = d1 * u;
              comp += du * du + (d1 > 0.0 ? d1 * d1 : 0.0);  // u >= 0: neg(u) = 0
            }
        }
      }
      __syncthreads();
      sstamp(4);
      // L^T U (s x r, K = the slice's rows): warp w takes k steps w % 4, w % 4 + 4,
      // ... and the row-tile half w / 4 (SP / 16 row tiles x all column tiles:
      // independent accumulators, short chains); the four K partials meet in
      // shared memory and one atomic per entry goes to the grid sums
      static_assert(kThreads == 256 && SP % 16 == 0, "8 warps: 4 K slices x 2 row-tile halves");
      constexpr int MH = SP / 16;  // row tiles per half
      {
        const int kq = warp & 3, half = warp >> 2;
        const int nkt = (nr + 3) >> 2;
        double dt[MH][NT][2];
#pragma unroll
        for (int mi = 0; mi < MH; ++mi)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) dt[mi][ni][0] = dt[mi][ni][1] = 0.0;
        const double* pa = sm.Pt + tq * (SP + 2) + 8 * MH * half + g;  // A[c][row] = Pt[row][c]
        for (int ks = kq; ks < nkt; ks += 4) {
          const int ra = 4 * ks + tq;
          const bool ron = ra < nr;
          double av[MH], bv[NT];
#pragma unroll
          for (int mi = 0; mi < MH; ++mi) av[mi] = ron ? pa[4 * ks * (SP + 2) + 8 * mi] : 0.0;
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) bv[ni] = (ron && 8 * ni + g < r) ? Uw[ra * r + 8 * ni + g] : 0.0;
#pragma unroll
          for (int mi = 0; mi < MH; ++mi)
#pragma unroll
            for (int ni = 0; ni < NT; ++ni)
              if (ni < nnt) dmma(dt[mi][ni], av[mi], bv[ni]);
        }
        if constexpr (4 * SP * RP <= kThreads * 16) {
          // partial kq of entry (c, b) at fold[kq][c * RP + b]
          double* fd = sm.fold + kq * (SP * RP);
#pragma unroll
          for (int mi = 0; mi < MH; ++mi)
#pragma unroll
            for (int ni = 0; ni < NT; ++ni)
#pragma unroll
              for (int e = 0; e < 2; ++e)
                fd[(8 * (MH * half + mi) + g) * RP + 8 * ni + 2 * tq + e] = dt[mi][ni][e];
        } else {
          // (the fold buffer holds 4 partials only up to 32 x 32: larger cores add them atomically)
#pragma unroll
          for (int mi = 0; mi < MH; ++mi)
#pragma unroll
            for (int ni = 0; ni < NT; ++ni)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int j = 8 * (MH * half + mi) + g, b = 8 * ni + 2 * tq + e;
                if (j < s && b < r) atomicAdd(&accU[j * kMax + b], dt[mi][ni][e]);
              }
        }
      }
      if constexpr (4 * SP * RP <= kThreads * 16) {
        __syncthreads();
        for (int i = tid; i < s * r; i += kThreads) {
          const int j = i / r, b = i - j * r;
          const double* f0 = sm.fold + j * RP + b;
          atomicAdd(&accU[j * kMax + b], (f0[0] + f0[SP * RP]) + (f0[2 * SP * RP] + f0[3 * SP * RP]));
        }
      }
    } else if (mode == 1) {
      // lx = P X ; u = max(lx + d/pen, 0) ; d += step*pen*(lx - u)   (nmf.py:354-357)
      // 16 threads across b (BJ values each), 16 row groups of BR rows
      constexpr int BJ = RP / 16, BR = (8 / BJ) > 0 ? 8 / BJ : 1;
      const int tb = tid & 15, tr = tid >> 4;
      for (int rbase = 0; rbase < nr; rbase += 16 * BR) {
        double acc[BR][BJ];
#pragma unroll
        for (int x = 0; x < BR; ++x)
#pragma unroll
          for (int y = 0; y < BJ; ++y) acc[x][y] = 0.0;
        int rows[BR];
#pragma unroll
        for (int x = 0; x < BR; ++x) rows[x] = min(rbase + tr + 16 * x, nr - 1);
#pragma unroll 4
        for (int j = 0; j < SP; ++j) {
          double pv[BR], xv[BJ];
#pragma unroll
          for (int x = 0; x < BR; ++x) pv[x] = sm.Pt[rows[x] * (SP + 2) + j];
#pragma unroll
          for (int y = 0; y < BJ; ++y) xv[y] = sm.X[j * LR + tb + 16 * y];
#pragma unroll
          for (int x = 0; x < BR; ++x)
#pragma unroll
            for (int y = 0; y < BJ; ++y) acc[x][y] = fma(pv[x], xv[y], acc[x][y]);
        }
#pragma unroll
        for (int x = 0; x < BR; ++x) {
          const int rr = rbase + tr + 16 * x;
          if (rr >= nr) continue;
#pragma unroll
          for (int y = 0; y < BJ; ++y) {
            const int b = tb + 16 * y;
            if (b >= r) continue;
            const int i = rr * r + b;
            const double lx = acc[x][y];
            const double d0 = Dr[i];
            const double u = fmax(lx + d0 * invpen, 0.0);
            const double d1 = d0 + sp_ * (lx - u);
            Uw[i] = u;
            Dw[i] = d1;
            if (!RES) {
              a.U[(t0 + rr) * r + b] = u;
              a.D[(t0 + rr) * r + b] = d1;
            }
            const double fe = lx - u;
            feas += fe * fe;
            const double du = d1 * u;
            comp += du * du + (d1 > 0.0 ? d1 * d1 : 0.0);  // u >= 0: neg(u) = 0
          }
        }
      }
      __syncthreads();
      sstamp(4);
    }
    if (own && !(RES && mode == 1)) {
      for (int rr = grp; rr < nr; rr += GROUPS) {
        double pv[4], uv[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          pv[x] = sm.Pt[rr * (SP + 2) + 4 * bj + x];
          uv[x] = (4 * bb + x < r) ? Uw[rr * r + 4 * bb + x] : 0.0;
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) au[x][y] = fma(pv[x], uv[y], au[x][y]);
      }
    }
  }
  if (mode == 1) {
    __syncthreads();
    sstamp(5);
  }
  if (mode == 0) {
#pragma unroll
    for (int t = 0; t < NG; ++t) {
      const int e = tid + t * kThreads, j = e / SP, l = e % SP;
      if (e < SP * SP && j < s && l < s) atomicAdd(&gram[j * kMax + l], g[t]);
    }
  }
  // fold the row groups through shared memory, then one atomic per
  // accumulator entry per CTA; the fold is laid out entry-major so that the
  // lanes of a warp (consecutive blocks) touch consecutive words -- the
  // block-major layout put all 32 lanes on one bank (32-way conflicts)
  double* fold = sm.fold;  // GROUPS x NBLK x 16 <= kThreads x 16 doubles
  const bool folded = !(RES && mode == 1);  // the DMMA path added its tiles to the grid sums already
  if (GROUPS > 1 && folded) {
    __syncthreads();
    if (own)
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) fold[(x * 4 + y) * (GROUPS * NBLK) + grp * NBLK + myb] = au[x][y];
    __syncthreads();
  }
  if (own && grp == 0 && folded) {
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        double v = au[x][y];
        if (GROUPS > 1) {
          v = 0.0;
          for (int q = 0; q < GROUPS; ++q) v += fold[(x * 4 + y) * (GROUPS * NBLK) + q * NBLK + myb];
        }
        const int j = 4 * bj + x, b = 4 * bb + y;
        if (j < s && b < r) atomicAdd(&accU[j * kMax + b], v);
      }
  }
  if (mode == 1) {
    feas = wsum(feas);
    comp = wsum(comp);
    const int lane = tid & 31, warp = tid >> 5;
    if (lane == 0) {
      red[2 * warp] = feas;
      red[2 * warp + 1] = comp;
    }
    __syncthreads();
    if (tid == 0) {
      double f = 0.0, c = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) {
        f += red[2 * w];
        c += red[2 * w + 1];
      }
      atomicAdd(&scal[0], f);
      atomicAdd(&scal[1], c);
    }
  }
  __syncthreads();
}

template <int SP, int RP, bool RES>
__device__ void split(const Params& p, const Smem<SP, RP>& sm, int mode, bool load, int wb, Acc* acc, double* red) {
  const int b = blockIdx.x;
  if (b < p.nblk_left) {
    const int64_t r0 = min64((int64_t)b * p.rows_left, p.left.rows), r1 = min64(r0 + p.rows_left, p.left.rows);
    split_side<SP, RP, RES>(p.left, sm, false, p.s, p.r, p.step, mode, r0, r1, load, wb, acc->LtU, p.rep->GL,
                            acc->scal, red);
  } else {
    const int64_t bb = b - p.nblk_left;
    const int64_t r0 = min64(bb * p.rows_right, p.right.rows), r1 = min64(r0 + p.rows_right, p.right.rows);
    split_side<SP, RP, RES>(p.right, sm, true, p.s, p.r, p.step, mode, r0, r1, load, wb, acc->RtV, p.rep->GR,
                            acc->scal + 2, red);
  }
}

// write buffer `wb` of the resident slice of U and dU back to global memory
template <int SP, int RP>
__device__ void write_back(const Params& p, const Smem<SP, RP>& sm, int wb) {
  const int b = blockIdx.x;
  const Side& a = b < p.nblk_left ? p.left : p.right;
  const int64_t per = b < p.nblk_left ? p.rows_left : p.rows_right;
  const int64_t bb = b < p.nblk_left ? b : b - p.nblk_left;
  const int64_t r0 = min64(bb * per, a.rows), r1 = min64(r0 + per, a.rows);
  const int r = p.r;
  for (int64_t i = threadIdx.x; i < (r1 - r0) * r; i += kThreads) {
    a.U[r0 * r + i] = sm.Ut(wb)[i];
    a.D[r0 * r + i] = sm.Dt(wb)[i];
  }
}

// save the replicated state of iteration k (the xc, yc split k used and the
// dual projections after it); the next launch resumes at k + 1
template <int SP, int RP>
__device__ void save_state(const Params& p, const Smem<SP, RP>& sm, int k) {
  constexpr int LS = SP + 1, LR = RP + 1;
  const int s = p.s, r = p.r;
  for (int i = threadIdx.x; i < s * r; i += kThreads) {
    const int a = i / r, b = i - a * r;
    p.xc_g[i] = sm.xc[a * LR + b];
    p.yc_g[b * s + a] = sm.yc[b * LS + a];
    p.rep->DL[a * kMax + b] = sm.DL[a * LR + b];
    p.rep->DR[a * kMax + b] = sm.DR[a * LR + b];
  }
  if (threadIdx.x == 0) p.ctrl->k = k + 1;
}

// clear the used part of a partials buffer
__device__ void zero_acc(Acc* a, int s, int r) {
  for (int i = threadIdx.x; i < s * kMax; i += blockDim.x) {
    if ((i % kMax) < r) {
      a->LtU[i] = 0.0;
      a->RtV[i] = 0.0;
    }
  }
  if (threadIdx.x < 4) a->scal[threadIdx.x] = 0.0;
}

// Synchronous schedule: every CTA splits, scores and solves the core.
// RES: slices resident in shared memory; else streamed in tiles.
template <int SP, int RP, bool RES>
__global__ void __launch_bounds__(kThreads, 1) admm_persistent(const Params p) {
  extern __shared__ double smraw[];
  __shared__ double red[3 * kThreads / 32];
  const int s = p.s, r = p.r, tid = threadIdx.x;
  const Smem<SP, RP> sm(smraw, RES ? (int)max(p.rows_left, p.rows_right) : kTile, false, p.r);
  Ctrl* c = p.ctrl;
  if (c->done) return;
  unsigned int epoch = 0;
  const bool writer = blockIdx.x == 0;  // writes scores, trace, ctrl and the saved state
  if (blockIdx.x == 0 && tid == 0) g_prof_ptr = p.prof;
  constexpr int LS = SP + 1, LR = RP + 1;
  const double spl = p.step * p.pu, spr = p.step * p.pv;
  for (int i = tid; i < SP * SP; i += kThreads) {
    const int a = i / SP, b = i % SP;
    sm.C[a * LS + b] = (a < s && b < s) ? p.core[a * s + b] : 0.0;
  }
  for (int i = tid; i < SP * RP; i += kThreads) {
    const int a = i / RP, b = i % RP;
    sm.xc[a * LR + b] = 0.0;
    sm.yc[b * LS + a] = 0.0;
    sm.DL[a * LR + b] = 0.0;
    sm.DR[a * LR + b] = 0.0;
  }
  __syncthreads();
  int k = c->k;
  if (p.fresh) {
    // initial projections L^T U0 and R V0^T into acc[2] (nmf.py:337-343),
    // Gram matrices into rep
    split<SP, RP, RES>(p, sm, 0, true, 0, &p.acc[2], red);
    grid_barrier(c, epoch);
    for (int i = tid; i < r * s; i += kThreads) {  // yc = V0 R^T
      const int q = i / s, j = i - q * s;
      sm.yc[q * LS + j] = ld(&p.acc[2].RtV[j * kMax + q]);
    }
  }
  for (int i = tid; i < SP * SP; i += kThreads) {
    const int a = i / SP, b = i % SP;
    const bool in = a < s && b < s;
    sm.GL[a * LS + b] = in ? ld(&p.rep->GL[a * kMax + b]) : 0.0;
    sm.GR[a * LS + b] = in ? ld(&p.rep->GR[a * kMax + b]) : 0.0;
  }
  if (p.fresh) {
    __syncthreads();
    core_step<SP, RP>(sm, &p.acc[2], s, r, p.pu, p.pv);
    k = 0;
  } else {
    for (int i = tid; i < s * r; i += kThreads) {
      const int a = i / r, b = i - a * r;
      sm.xc[a * LR + b] = p.xc_g[i];
      sm.yc[b * LS + a] = p.yc_g[b * s + a];
      sm.DL[a * LR + b] = p.rep->DL[a * kMax + b];
      sm.DR[a * LR + b] = p.rep->DR[a * kMax + b];
    }
    __syncthreads();
    // finish the iteration the previous launch stopped after
    const Acc* a = &p.acc[(k - 1) % 3];
    double obj;
    const double score = kkt_score<SP, RP>(sm, a, red, &obj);
    const bool conv = score < p.tol;
    const bool div = !conv && k - 1 >= 50 && score > 10.0 * ld(&p.scores[k - 1 - 50]);
    const bool cap = k >= p.max_iter;
    if (writer && tid == 0) {
      p.scores[k - 1] = score;
      p.trace[k - 1] = obj;
      if (conv || div || cap) {
        if (div) c->diverged = k - 1;
        c->done = 1;
        c->iters = k;
      }
    }
    if (conv || div || cap) return;
    core_step<SP, RP>(sm, a, s, r, p.pu, p.pv);
  }
  int splits = 0;
  bool load = !p.fresh;  // fresh runs loaded the slice in the projection sweep
  for (;;) {
    // split(k) into acc[k % 3]; CTA 0 clears the buffer split(k+1) will use
    stamp(p, k, 0);
    if (blockIdx.x == 0 && tid == 0) g_prof_k = k;
    if (blockIdx.x == 0) zero_acc(&p.acc[(k + 1) % 3], s, r);
    split<SP, RP, RES>(p, sm, 1, load, 0, &p.acc[k % 3], red);
    load = false;
    ++splits;
    stamp(p, k, 1);
    grid_barrier(c, epoch);
    stamp(p, k, 2);
    const Acc* a = &p.acc[k % 3];
    dual_update<SP, RP>(sm, a, s, r, spl, spr);
    if (p.step_limit > 0 && splits >= p.step_limit) {
      // hand the state to the next launch (which scores iteration k first)
      if (RES) write_back<SP, RP>(p, sm, 0);
      if (writer) save_state<SP, RP>(p, sm, k);
      return;
    }
    const bool cap = k + 1 >= p.max_iter;
    double obj;
    const double score = kkt_score<SP, RP>(sm, a, red, &obj);
    stamp(p, k, 3);
    const bool conv = score < p.tol;
    // scores[k - 50] was written by the writer CTA at least 50 barriers ago
    const bool div = !conv && k >= 50 && score > 10.0 * ld(&p.scores[k - 50]);
    if (writer && tid == 0) {
      p.scores[k] = score;
      p.trace[k] = obj;  // ||C - xc_k yc_k||^2 (nmf.py:360)
      if (conv || div || cap) {
        if (div) c->diverged = k;
        c->done = 1;
        c->iters = k + 1;
      }
    }
    if (conv || div || cap) {
      if (RES) write_back<SP, RP>(p, sm, 0);
      if (writer) save_state<SP, RP>(p, sm, k);
      return;
    }
    core_step<SP, RP>(sm, a, s, r, p.pu, p.pv);
    ++k;
  }
}

// Speculative schedule (slices resident): CTAs [0, nsplit) split; CTA
// nsplit (helper) precomputes, for each window k between barriers k and
// k + 1, everything of core(k + 2) that depends only on (xc_{k+1}, yc_{k+1})
// -- the first ridge inverse, C yc^T, the dual-projection carry -- and
// publishes it with the new state; CTA nsplit + 1 (scorer) scores split k
// from the published state while the others run core(k + 1) and split
// k + 1. The critical path per iteration is then: stage the reductions,
// xc = W Minv, one ridge solve, yc, split.
//
// The score of k only decides whether to stop: if it stops, the scorer marks
// ctrl.done (iters = k + 1) before arriving at barrier k + 1; the others see
// it after that barrier and write back U, dU of iteration k, which split
// k + 1 left untouched in the other buffer. A run with an iteration cap
// ends at the cap without the extra barrier. Results equal the synchronous
// schedule's up to the order of the (nondeterministic) atomic reductions.
template <int SP, int RP>
__global__ void __launch_bounds__(kThreads, 1) admm_spec(const Params p) {
  extern __shared__ double smraw[];
  __shared__ double red[3 * kThreads / 32];
  __shared__ int flag;
  const int s = p.s, r = p.r, tid = threadIdx.x;
  const Smem<SP, RP> sm(smraw, (int)max(p.rows_left, p.rows_right), true, p.r);
  Ctrl* c = p.ctrl;
  if (c->done) return;
  unsigned int epoch = 0;
  const int nsplit = gridDim.x - 2;
  const int role = blockIdx.x < nsplit ? kWorker : blockIdx.x == nsplit ? kHelper : kScorer;
  if (blockIdx.x == 0 && tid == 0) g_prof_ptr = p.prof;
  constexpr int LS = SP + 1, LR = RP + 1;
  const double spl = p.step * p.pu, spr = p.step * p.pv, cl = p.pu + spl, cr = p.pv + spr;
  for (int i = tid; i < SP * SP; i += kThreads) {
    const int a = i / SP, b = i % SP;
    sm.C[a * LS + b] = (a < s && b < s) ? p.core[a * s + b] : 0.0;
  }
  for (int i = tid; i < SP * RP; i += kThreads) {
    const int a = i / RP, b = i % RP;
    sm.xc[a * LR + b] = 0.0;
    sm.yc[b * LS + a] = 0.0;
    if (role != kWorker) {
      sm.DL[a * LR + b] = 0.0;
      sm.DR[a * LR + b] = 0.0;
    }
  }
  __syncthreads();
  int k = c->k;
  bool stopped = false;
  if (p.fresh) {
    if (role == kWorker) split<SP, RP, true>(p, sm, 0, true, 1, &p.acc[2], red);
    grid_barrier(c, epoch);
    if (role == kHelper) {
      for (int i = tid; i < r * s; i += kThreads) {  // yc = V0 R^T
        const int q = i / s, j = i - q * s;
        sm.yc[q * LS + j] = ld(&p.acc[2].RtV[j * kMax + q]);
      }
    }
    k = 0;
  } else if (role != kWorker) {
    for (int i = tid; i < s * r; i += kThreads) {
      const int a = i / r, b = i - a * r;
      sm.xc[a * LR + b] = p.xc_g[i];
      sm.yc[b * LS + a] = p.yc_g[b * s + a];
      sm.DL[a * LR + b] = p.rep->DL[a * kMax + b];
      sm.DR[a * LR + b] = p.rep->DR[a * kMax + b];
    }
    __syncthreads();
    if (role == kScorer) {
      // finish the iteration the previous launch stopped after
      double obj;
      const double score = kkt_score<SP, RP>(sm, &p.acc[(k - 1) % 3], red, &obj);
      const bool conv = score < p.tol;
      const bool div = !conv && k - 1 >= 50 && score > 10.0 * ld(&p.scores[k - 1 - 50]);
      stopped = conv || div || k >= p.max_iter;
      if (tid == 0) {
        p.scores[k - 1] = score;
        p.trace[k - 1] = obj;
        if (stopped) {
          if (div) c->diverged = k - 1;
          c->iters = k;
          c->done = k;  // done carries the iteration count: one word to read
        }
      }
    }
  }
  if (role == kHelper) {
    for (int i = tid; i < SP * SP; i += kThreads) {
      const int a = i / SP, b = i % SP;
      const bool in = a < s && b < s;
      sm.GL[a * LS + b] = in ? ld(&p.rep->GL[a * kMax + b]) : 0.0;
      sm.GR[a * LS + b] = in ? ld(&p.rep->GR[a * kMax + b]) : 0.0;
    }
    __syncthreads();
    core_step<SP, RP>(sm, &p.acc[p.fresh ? 2 : (k - 1) % 3], s, r, p.pu, p.pv);
    precompute<SP, RP>(sm, s, r, p.pu, spl, spr, &p.pub[k & 1]);
  }
  grid_barrier(c, epoch);  // Pub[k & 1] holds (xc_k, yc_k)
  if (stopped) return;
  if (role != kScorer) {
    if (tid == 0) flag = *(volatile int*)&c->done;
    __syncthreads();
    if (flag) return;  // the prologue's score stopped the run
  }
  if (role == kWorker) {
    const Pub* pb = &p.pub[k & 1];
    for (int i = tid; i < SP * RP; i += kThreads) {
      const int a = i / RP, b = i % RP;
      const bool in = a < s && b < r;
      sm.xc[a * LR + b] = in ? ld(&pb->xc[a * kMax + b]) : 0.0;
      sm.yc[b * LS + a] = in ? ld(&pb->yc[b * kMax + a]) : 0.0;
    }
  }
  int splits = 0;
  bool load = !p.fresh;
  for (;;) {
    const int wb = k & 1;
    stamp(p, k, 0);
    if (role == kWorker) {
      if (blockIdx.x == 0 && tid == 0) g_prof_k = k;
      if (blockIdx.x == 0) zero_acc(&p.acc[(k + 1) % 3], s, r);
      split<SP, RP, true>(p, sm, 1, load, wb, &p.acc[k % 3], red);
    }
    load = false;
    ++splits;
    stamp(p, k, 1);
    grid_barrier(c, epoch);
    stamp(p, k, 2);
    const Acc* a = &p.acc[k % 3];
    stage<SP, RP>(sm, a, &p.pub[k & 1], role, s, r);
    if (role != kScorer) {
      // done == k: the scorer stopped at k - 1 (k iterations) and split k was
      // speculative (a stop at k may already be visible to a CTA that left
      // the barrier late; it is acted on after barrier k + 1)
      if (tid == 0) {
        const int d = *(volatile int*)&c->done;
        flag = d != 0 && d == k;
      }
      __syncthreads();
      if (flag) {
        if (role == kWorker) write_back<SP, RP>(p, sm, wb ^ 1);
        return;
      }
    }
    stamp(p, k, 3);
    const bool cap = k + 1 >= p.max_iter;
    const bool pause = p.step_limit > 0 && splits >= p.step_limit;
    if (role == kScorer) {
      duals_from_published<SP, RP>(sm, spl, spr);
      if (pause) {
        // hand the state to the next launch (which scores iteration k first)
        save_state<SP, RP>(p, sm, k);
        return;
      }
      double obj;
      const double score = kkt_score<SP, RP>(sm, a, red, &obj);
      const bool conv = score < p.tol;
      const bool div = !conv && k >= 50 && score > 10.0 * ld(&p.scores[k - 50]);
      const bool stop = conv || div || cap;
      if (stop) save_state<SP, RP>(p, sm, k);
      if (tid == 0) {
        p.scores[k] = score;
        p.trace[k] = obj;  // ||C - xc_k yc_k||^2 (nmf.py:360)
        if (stop) {
          if (div) c->diverged = k;
          c->iters = k + 1;
          c->done = k + 1;
        }
      }
      if (stop) {
        if (!cap) grid_barrier(c, epoch);  // the others are in split k + 1
        return;
      }
      ++k;
      continue;
    }
    if (pause || cap) {
      if (role == kWorker) write_back<SP, RP>(p, sm, wb);
      return;
    }
    if (role == kHelper) duals_from_published<SP, RP>(sm, spl, spr);
    fast_core<SP, RP>(sm, s, r, p.pv, cl, cr);
    if (role == kHelper) precompute<SP, RP>(sm, s, r, p.pu, spl, spr, &p.pub[(k + 1) & 1]);
    ++k;
  }
}

__global__ void init_ctrl(Ctrl* c) {
  c->k = 0;
  c->done = 0;
  c->iters = 0;
  c->diverged = -1;
  c->bar_count = 0;
  c->bar_gen = 0;
}

template <class K>
int launch(K kernel, Params& p, int grid, size_t smem, cudaStream_t st) {
  CNMF_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap));
  int per_sm = 0;
  CNMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem));
  if (per_sm < 1) return fail(CNMF_ERR_CUDA, "ADMM kernel does not fit on an SM");
  void* args[] = {(void*)&p};
  CNMF_CUDA(cudaLaunchCooperativeKernel((void*)kernel, dim3(grid), dim3(kThreads), args, smem, st));
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

// split CTAs between the two sides by row count
void plan(Params& p, int nsplit, int64_t m, int64_t n) {
  const int nbl = (int)std::max<int64_t>(1, std::min<int64_t>(nsplit - 1, (nsplit * m + (m + n) / 2) / (m + n)));
  const int nbr = std::max(1, nsplit - nbl);
  p.nblk_left = nbl;
  p.rows_left = ceil_div(m, nbl);
  p.rows_right = ceil_div(n, nbr);
}

// One CTA per SM. Prefer the speculative schedule (slices resident, two
// helper CTAs), then resident slices, then streamed tiles
// (CNMF_ADMM_SPEC=0 disables the speculative schedule).
template <int SP, int RP>
int dispatch(Params& p, int sms, int64_t want, int64_t m, int64_t n, cudaStream_t st) {
  const char* e = getenv("CNMF_ADMM_SPEC");
  const bool spec_ok = !(e && e[0] == '0') && sms >= 4;
  auto rows = [&]() { return (int)std::min<int64_t>(std::max(p.rows_left, p.rows_right), 1 << 20); };
  if (spec_ok) {
    const int nsplit = (int)std::max<int64_t>(2, std::min<int64_t>(want, sms - 2));
    plan(p, nsplit, m, n);
    const size_t b2 = Smem<SP, RP>::bytes(rows(), true, p.r);
    if (b2 <= kSmemCap) return launch(admm_spec<SP, RP>, p, nsplit + 2, b2, st);
  }
  plan(p, (int)want, m, n);
  const size_t b1 = Smem<SP, RP>::bytes(rows(), false, p.r);
  if (b1 <= kSmemCap) return launch(admm_persistent<SP, RP, true>, p, (int)want, b1, st);
  return launch(admm_persistent<SP, RP, false>, p, (int)want, Smem<SP, RP>::bytes(kTile, false, p.r), st);
}

}  // namespace

size_t admm_workspace(int64_t m, int64_t n, int s, int r) {
  (void)m;
  (void)n;
  (void)s;
  (void)r;
  return 256 + 3 * sizeof(Acc) + sizeof(Rep) + 2 * sizeof(Pub) + 256;
}

int admm_stream_run(const double* core, const float* L, int64_t m, const float* Rt, int64_t n, int s, int r, double* u,
                    double* du, double* vt, double* dvt, double* xc, double* yc, double pu, double pv, double step,
                    int max_iter, double tol, double* trace, double* scores, int* iterations, void* ws, int resume,
                    int step_limit, cudaStream_t st);

int admm_run(const double* core, const float* L, int64_t m, const float* Rt, int64_t n, int s, int r, double* u,
             double* du, double* vt, double* dvt, double* xc, double* yc, double pu, double pv, double step,
             int max_iter, double tol, double* trace, double* scores, int* iterations, void* ws, size_t ws_bytes,
             int resume, int step_limit, cudaStream_t st) {
  if (s < 1 || s > kMax || r < 1 || r > kMax) return fail(CNMF_ERR_ARGUMENT, "ADMM supports 1 <= r, s <= 64");
  if (!(pu > 0) || !(pv > 0)) return fail(CNMF_ERR_ARGUMENT, "penalties must be positive");
  if (ws_bytes < admm_workspace(m, n, s, r)) return fail(CNMF_ERR_ARGUMENT, "workspace too small");
  const int S = s <= 32 ? 32 : 64;
  Ctrl* ctrl = (Ctrl*)ws;
  Acc* acc = (Acc*)((char*)ws + 256);
  Rep* rep = (Rep*)(acc + 3);
  Pub* pub = (Pub*)(rep + 1);
  int dev = 0, sms = 0;
  CNMF_CUDA(cudaGetDevice(&dev));
  CNMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t want = std::max<int64_t>(2, std::min<int64_t>((int64_t)sms, ceil_div(m, 8) + ceil_div(n, 8)));
  if (!resume) {
    init_ctrl<<<1, 1, 0, st>>>(ctrl);
    CNMF_LAUNCH_CHECK();
    CNMF_CUDA(cudaMemsetAsync(acc, 0, 3 * sizeof(Acc) + sizeof(Rep), st));
    CNMF_CUDA(cudaMemsetAsync(du, 0, (size_t)m * r * 8, st));
    CNMF_CUDA(cudaMemsetAsync(dvt, 0, (size_t)n * r * 8, st));
  }
  CNMF_CUDA(cudaMemsetAsync(&ctrl->bar_count, 0, sizeof(unsigned int), st));  // grid_barrier epochs
  Params p;
  p.core = core;
  p.left = Side{L, m, S, u, du, pu};
  p.right = Side{Rt, n, S, vt, dvt, pv};
  p.s = s;
  p.r = r;
  p.pu = pu;
  p.pv = pv;
  p.step = step;
  p.tol = tol;
  p.max_iter = max_iter;
  p.step_limit = step_limit;
  p.fresh = !resume;
  p.xc_g = xc;
  p.yc_g = yc;
  p.trace = trace;
  p.scores = scores;
  p.ctrl = ctrl;
  p.acc = acc;
  p.rep = rep;
  p.pub = pub;
  p.prof = nullptr;
  if (const char* e = getenv("CNMF_ADMM_PROFILE")) {
    static unsigned long long* buf = nullptr;
    if (!buf) cudaMalloc(&buf, 256 * 8 * 8);
    p.prof = buf;
    (void)e;
  }
  // the persistent kernel keeps its s x s / s x r state per CTA in shared
  // memory; where that cannot fit (s > 32 with r > 32) the three-launch
  // streaming iteration runs instead (csrc/admm_stream.cu; CNMF_ADMM_STREAM=1
  // forces it)
  const char* fe = getenv("CNMF_ADMM_STREAM");
  if ((fe && fe[0] == '1') || (s > 32 && r > 32))
    return admm_stream_run(core, L, m, Rt, n, s, r, u, du, vt, dvt, xc, yc, pu, pv, step, max_iter, tol, trace,
                           scores, iterations, ws, resume, step_limit, st);
  int rc;
  if (s <= 32 && r <= 16)
    rc = dispatch<32, 16>(p, sms, want, m, n, st);
  else if (s <= 32 && r <= 32)
    rc = dispatch<32, 32>(p, sms, want, m, n, st);
  else if (r <= 16)
    rc = dispatch<64, 16>(p, sms, want, m, n, st);
  else if (r <= 32)
    rc = dispatch<64, 32>(p, sms, want, m, n, st);
  else
    rc = dispatch<64, 64>(p, sms, want, m, n, st);
  CNMF_TRY(rc);
  if (p.prof) {
    unsigned long long h[256 * 8];
    cudaMemcpyAsync(h, p.prof, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double acc8[8] = {0};
    int n = 0;
    for (int k = 5; k < 105 && k + 1 < 256; ++k) {
      const unsigned long long* t = h + k * 8;
      const unsigned long long next0 = h[(k + 1) * 8];
      if (!next0 || !t[3]) break;
      acc8[0] += t[4] - t[0];  // lx + update
      acc8[1] += t[5] - t[4];  // accumulate
      acc8[2] += t[1] - t[5];  // fold + atomics
      acc8[3] += t[2] - t[1];  // barrier
      acc8[4] += t[3] - t[2];  // score
      acc8[5] += t[6] - t[3];  // core up to first inverse done
      acc8[6] += t[7] - t[6];  // to second inverse done
      acc8[7] += next0 - t[7];  // rest
      ++n;
    }
    if (n)
      fprintf(stderr,
              "[admm profile] ns/iter: lx %.0f acc %.0f fold %.0f | barrier %.0f | score %.0f | core: inv1 %.0f "
              "inv2 %.0f tail %.0f\n",
              acc8[0] / n, acc8[1] / n, acc8[2] / n, acc8[3] / n, acc8[4] / n, acc8[5] / n, acc8[6] / n,
              acc8[7] / n);
  }
  Ctrl hc;
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
