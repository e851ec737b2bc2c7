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

int panel_cross(const float* P1, const float* P2, int64_t rows, int S, double* out, cudaStream_t st);

namespace {

constexpr int kT = 256;   // threads per block
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
// row sweep: blocks [0, nbl) take left rows, [nbl, grid) right rows, one
// block per SM, 64-row tiles, on the fp64 tensor cores (DMMA, mma.sync
// m8n8k4.f64: measured 37 TFLOP/s on B200 vs 34 for DFMA, with a fraction of
// the issue slots and shared-memory traffic). Two warp groups work on
// consecutive tiles (double-buffered P and x tiles, named barriers):
//
//   update group     loads a tile (P rows -> fp64 Pr, old x, dx by cp.async),
//     (warps 0..7)   forms P z (64 rows x 64 columns, K = s) -- warp w owns a
//                    16 x 32 block, 2 x 4 DMMA tiles -- updates its (x, dx)
//                    pairs in HBM, adds the KKT sums and leaves the new x in
//                    the tile buffer;
//   reduction group  accumulates the block partial P^T x (64 x 64, K = the
//     (warps 8..15)  tile's rows) in DMMA accumulators that persist across
//                    tiles, while the update group works on the next tile.
// Per k step a warp loads 6 fragments (LDS.64) for 8 DMMA; row strides of
// 68 doubles (544 B) put the 4 rows a half warp touches on 4 distinct 32-byte
// bank groups, so every fragment load is conflict-free.
// ---------------------------------------------------------------------------
constexpr int kRT = 64;      // rows per tile
constexpr int kLD = 68;      // row stride (doubles) of Z, the P and the x tiles
constexpr int kSW = 2 * kT;  // threads of the row sweep (two warp groups)

template <int SP>
constexpr size_t sweep_smem() {
  // Z + Pr[2] + Xs[2] + Ds
  return ((size_t)kMaxD * kLD + 5 * (size_t)kRT * kLD) * 8;
}

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// named barriers: 1 = update group internal, 2 + b = tile buffer b filled,
// 4 + b = tile buffer b consumed by the reduction group
constexpr int kBarU = 1, kBarFull = 2, kBarEmpty = 4;

// D (8 x 8) += A (8 x 4, row g, column t) B (4 x 8, row t, column g); the
// accumulator holds row g, columns 2 t, 2 t + 1 (g = lane / 4, t = lane % 4)
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int SP>
__global__ void __launch_bounds__(kSW, 1) row_sweep(SSide L, SSide R, int nbl, const double* __restrict__ Zl,
                                                     const double* __restrict__ Zr, int s, int r, double step,
                                                     int update, double* __restrict__ part, const SCtrl* ctrl) {
  if (update && ctrl->done) return;
  extern __shared__ __align__(16) unsigned char sm[];
  double* Z = (double*)sm;               // [kMaxD][kLD]: Z[c][k], zero outside c < s, k < r
  double* PrB = Z + kMaxD * kLD;         // [2][kRT][kLD]: panel rows (fp64), zero for c >= s and rows >= nr
  double* XsB = PrB + 2 * kRT * kLD;     // [2][kRT][kLD]: old x, then the updated x (zero outside the tile)
  double* Ds = XsB + 2 * kRT * kLD;      // [kRT][kLD]: old dx
  __shared__ double red[4][kT / 32];
  const bool left = (int)blockIdx.x < nbl;
  const SSide sd = left ? L : R;
  const int b = left ? (int)blockIdx.x : (int)blockIdx.x - nbl;
  const int nb = left ? nbl : (int)gridDim.x - nbl;
  const int64_t r0 = sd.rows * b / nb, r1 = sd.rows * (b + 1) / nb;
  const int64_t ntile = (r1 - r0 + kRT - 1) / kRT;
  const int sr = s * r;
  const double* Zs = left ? Zl : Zr;
  for (int i = threadIdx.x; i < kMaxD * kMaxD; i += kSW) {
    const int c = i / kMaxD, k = i % kMaxD;
    Z[c * kLD + k] = (update && c < s && k < r) ? Zs[c * r + k] : 0.0;
  }
  if (SP < kMaxD)  // columns the panel does not have
    for (int i = threadIdx.x; i < 2 * kRT * (kMaxD - SP); i += kSW)
      PrB[(i / (kMaxD - SP)) * kLD + SP + i % (kMaxD - SP)] = 0.0;
  __syncthreads();
  const bool ugroup = threadIdx.x < kT;
  const int tid = threadIdx.x & (kT - 1);
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;  // 16-row (or 16-c) block wm, 32-column block wn
  double* out = part + (size_t)blockIdx.x * sums_len(s, r);
  constexpr int KS = SP / 4;  // k steps over c (Pr columns >= s and Z rows >= s are zero)

  if (ugroup) {
    // ======================= update group =======================
    // x = max(P z + dx / p, 0) with dx / p as dx * (1 / p): one rounding
    // more than the reference's division (<= 1 ulp), ~30 instructions less
    const double inv_pen = 1.0 / sd.pen, step_pen = step * sd.pen;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    constexpr int PF = kRT * (SP / 4) / kT;  // float4 j of this thread: element tid + j kT of the tile
    float4 pf[PF];
    auto load_p = [&](int64_t t0n) {
      const int nrn = (int)min64(kRT, r1 - t0n);
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        const int i = tid + j * kT, row = i / (SP / 4), c4 = 4 * (i % (SP / 4));
        pf[j] = (row < nrn) ? __ldg((const float4*)(sd.P + (t0n + row) * sd.ldp + c4)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    if (ntile > 0) load_p(r0);
    const int hi4 = tid >> 4, kg = tid & 15;  // cp.async mapping: 16 rows x 16 columns per pass
    for (int64_t t = 0; t < ntile; ++t) {
      const int buf = (int)(t & 1);
      const int64_t t0 = r0 + t * kRT;
      const int nr = (int)min64(kRT, r1 - t0);
      double* Pr = PrB + buf * kRT * kLD;
      double* Xs = XsB + buf * kRT * kLD;
      if (t >= 2) nbar_sync(kBarEmpty + buf, kSW);  // the reduction group is done with buffer buf
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        const int i = tid + j * kT, row = i / (SP / 4), c4 = 4 * (i % (SP / 4));
        double* d = Pr + row * kLD + c4;
        *(double2*)d = make_double2(c4 + 0 < s ? (double)pf[j].x : 0.0, c4 + 1 < s ? (double)pf[j].y : 0.0);
        *(double2*)(d + 2) = make_double2(c4 + 2 < s ? (double)pf[j].z : 0.0, c4 + 3 < s ? (double)pf[j].w : 0.0);
      }
      // the tile's old (x, dx) land in Xs, Ds while P z is formed
      for (int row = hi4; row < nr; row += kT / 16)
        for (int k = kg; k < r; k += 16) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(Xs + row * kLD + k)),
                       "l"(sd.x + (t0 + row) * r + k)
                       : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(Ds + row * kLD + k)),
                       "l"(sd.dx + (t0 + row) * r + k)
                       : "memory");
        }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (t + 1 < ntile) load_p(t0 + kRT);  // next tile's P rows: in flight during this tile
      nbar_sync(kBarU, kT);                 // Pr complete
      double acc[2][4][2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      if (update) {
        const double* pa = Pr + (16 * wm + g) * kLD + tq;  // A[row][c]: rows 16 wm + 8 mi + g
        const double* zb = Z + tq * kLD + 32 * wn + g;     // B[c][k]: k = 32 wn + 8 ni + g
#pragma unroll 4
        for (int ks = 0; ks < KS; ++ks) {
          const double a0 = pa[4 * ks], a1 = pa[8 * kLD + 4 * ks];
          double bv[4];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) bv[ni] = zb[4 * ks * kLD + 8 * ni];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            dmma(acc[0][ni], a0, bv[ni]);
            dmma(acc[1][ni], a1, bv[ni]);
          }
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      nbar_sync(kBarU, kT);  // every thread's cp.async data visible
      // (x, dx) update, KKT sums, the new x into Xs (in place: every thread
      // reads and writes only its own elements: row 16 wm + 8 mi + g,
      // columns 32 wn + 8 ni + 2 tq + e)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int row = 16 * wm + 8 * mi + g;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int k = 32 * wn + 8 * ni + 2 * tq + e;
            double xn = 0.0;
            if (row < nr && k < r) {
              const double xo = Xs[row * kLD + k];
              if (update) {
                const double pz = acc[mi][ni][e];
                const double dxo = Ds[row * kLD + k];
                const double x = fmax(pz + dxo * inv_pen, 0.0);
                const double dx = dxo + step_pen * (pz - x);
                const int64_t gi = (t0 + row) * r + k;
                sd.x[gi] = x;
                sd.dx[gi] = dx;
                const double dl = pz - x, dp = dx * x, dpos = fmax(dx, 0.0), xneg = fmax(-x, 0.0);
                s0 += dl * dl;
                s1 += dp * dp;
                s2 += dpos * dpos;
                s3 += xneg * xneg;
                xn = x;
              } else {
                xn = xo;
              }
            }
            Xs[row * kLD + k] = xn;
          }
      }
      nbar_sync(kBarU, kT);              // Ds read and the tile buffers written by the whole group
      nbar_arrive(kBarFull + buf, kSW);  // tile buffer buf ready for the reduction group
    }
    // KKT sums: warp shuffles, then the update group's warps in order
    double v[4] = {s0, s1, s2, s3};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
      if (lane == 0) red[j][warp] = v[j];
    }
    nbar_sync(kBarU, kT);
    if (tid < 4) {
      double a = 0.0;
      for (int w = 0; w < kT / 32; ++w) a += red[tid][w];
      out[2 * sr + tid] = a;
    }
  } else {
    // ======================= reduction group =======================
    // P^T x: A[c][row] = Pr[row][c] (c = 16 wm + 8 mi + g), B[row][k] = Xs[row][k]
    double au[2][4][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) au[mi][ni][0] = au[mi][ni][1] = 0.0;
    const bool con = 16 * wm < s;
    for (int64_t t = 0; t < ntile; ++t) {
      const int buf = (int)(t & 1);
      nbar_sync(kBarFull + buf, kSW);
      if (con) {
        const double* pa = PrB + buf * kRT * kLD + tq * kLD + 16 * wm + g;
        const double* xb = XsB + buf * kRT * kLD + tq * kLD + 32 * wn + g;
#pragma unroll 4
        for (int ks = 0; ks < kRT / 4; ++ks) {  // rows >= nr are zero in Pr and Xs
          const double a0 = pa[4 * ks * kLD], a1 = pa[4 * ks * kLD + 8];
          double bv[4];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) bv[ni] = xb[4 * ks * kLD + 8 * ni];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            dmma(au[0][ni], a0, bv[ni]);
            dmma(au[1][ni], a1, bv[ni]);
          }
        }
      }
      if (t + 2 < ntile) nbar_arrive(kBarEmpty + buf, kSW);  // the update group refills buffer buf
    }
    if (con) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 16 * wm + 8 * mi + g, k = 32 * wn + 8 * ni + 2 * tq + e;
            if (c < s && k < r) out[c * r + k] = au[mi][ni][e];
          }
    }
  }
}

// resident row-sweep blocks on the device (one wave; the occupancy of the
// larger instantiation)
int sweep_blocks(int sms) {
  static int occ = 0;
  if (occ == 0) {
    int o = 0;
    ensure_smem_attr((const void*)row_sweep<64>, (int)sweep_smem<64>());
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, row_sweep<64>, kSW, sweep_smem<64>()) != cudaSuccess || o < 1)
      o = 1;
    occ = o;
  }
  return occ * sms;
}

// fixed-order sums of the block partials of each side: sums[side][e]
__global__ void __launch_bounds__(kT) reduce_parts(const double* __restrict__ part, int nbl, int nbr, int len,
                                                    double* __restrict__ sums, const SCtrl* ctrl, int update) {
  if (update && ctrl->done) return;
  const int e = blockIdx.x * kT + threadIdx.x;
  const int side = blockIdx.y;
  if (e >= len) return;
  const int b0 = side ? nbl : 0, nb = side ? nbr : nbl;
  const int sr = (len - 4) / 2;
  if (e >= sr && e < 2 * sr) {  // the dual projections come from the core step's recurrence
    sums[side * len + e] = 0.0;
    return;
  }
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

// ---------------------------------------------------------------------------
// core step: one block of kCT threads; every small product is a register-
// tiled shared-memory GEMM (2 x 4 outputs per thread, operands broadcast
// within a warp), the two r x r ridge systems are inverted by Gauss-Jordan
// ---------------------------------------------------------------------------
constexpr int kCT = 512;

// C(m, n) = sum_k A[m * am + k * ak] * B[k * bk + n] for m < M, n < N <= 64,
// M <= 64; out(m, n, value) consumes every result. Thread t owns rows
// m = t / 16 + 32 p (p < 2) and columns n = t % 16 + 16 q (q < 4): a warp
// reads 2 distinct A values (broadcast) and 16 consecutive B values per k
// (conflict-free), with 8 independent FMA chains per thread.
template <class F>
__device__ __forceinline__ void small_gemm(int M, int N, int K, const double* A, int am, int ak, const double* B,
                                           int bk, F out) {
  static_assert(kCT == 512, "thread mapping covers 64 x 64");
  const int tm = threadIdx.x >> 4, tn = threadIdx.x & 15;
  if (tm >= M || tn >= N) return;
  const int m1 = tm + 32 < M ? tm + 32 : tm;  // clamped reads; results masked below
  int nn[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) nn[q] = tn + 16 * q < N ? tn + 16 * q : tn;
  double c[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    const double a0 = A[tm * am + k * ak], a1 = A[m1 * am + k * ak];
    double bv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) bv[q] = B[k * bk + nn[q]];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      c[0][q] = fma(a0, bv[q], c[0][q]);
      c[1][q] = fma(a1, bv[q], c[1][q]);
    }
  }
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (tm + 32 * p < M && tn + 16 * q < N) out(tm + 32 * p, tn + 16 * q, c[p][q]);
}

// In-place inverse of an SPD r x r matrix (ld r) by Gauss-Jordan without
// pivoting (the ridge term keeps the pivots >= the penalty). Thread t owns
// row t / 8 and columns t % 8 + 8 j (no integer division in the r elimination
// steps; the 1-D version spent ~40 % of the core step's instructions on it).
__device__ void spd_inverse(double* M, double* piv, int r) {
  static_assert(kCT == 512, "64 rows x 8 column lanes");
  const int tid = threadIdx.x, a = tid >> 3, c8 = tid & 7;
  double* colk = piv + kMaxD;
  for (int k = 0; k < r; ++k) {
    __syncthreads();
    const double inv = 1.0 / M[k * r + k];
    if (tid < r) {
      piv[tid] = M[k * r + tid] * inv;  // scaled pivot row
      colk[tid] = M[tid * r + k];       // column k before this step overwrites it
    }
    __syncthreads();
    if (a < r) {
      const double f = colk[a];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = c8 + 8 * j;
        if (c < r) {
          double* e = M + a * r + c;
          if (a == k)
            *e = (c == k) ? inv : piv[c];
          else
            *e = (c == k) ? -f * inv : fma(-f, piv[c], *e);
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, double* red, int slot) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[slot * (kCT / 32) + (threadIdx.x >> 5)] = v;
  return v;
}

// KKT of the iteration just swept (k > 0), the stopping / divergence rule,
// then the two ridge solves of iteration k (nmf.py:341-350).
// The dual projections follow from the dual step without a reduction (the
// persistent kernel's recurrence, csrc/admm.cu):
//   L^T dU_k = L^T dU_{k-1} + step pu (G_L xc_k - L^T U_k),   G_L = L^T L,
//   R dV_k^T = R dV_{k-1}^T + step pv (G_R yc_k^T - R V_k^T), G_R = R R^T,
// so the row sweep reduces L^T U and R V^T only. DL, DR (s x r) carry the
// projections between launches; `first` zeroes them (dU, dV start at 0).
__global__ void __launch_bounds__(kCT) core_step(const double* __restrict__ core, const double* __restrict__ sums,
                                                  double* __restrict__ xc, double* __restrict__ yc, double* Zl,
                                                  double* Zr, const double* __restrict__ GL,
                                                  const double* __restrict__ GR, int ldg, double* __restrict__ DL,
                                                  double* __restrict__ DR, int s, int r, double pu, double pv,
                                                  double step, double tol, double* trace, double* scores, SCtrl* ctrl,
                                                  int k, int max_iter, int first, int solve) {
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char sm[];
  double* E = (double*)sm;         // s x s: E = xc yc - core, later the rhs (s x r)
  double* B = E + s * s;           // rhs2 (r x s)
  double* M = B + r * s;           // r x r
  double* piv = M + r * r;         // 2 x 64
  double* coreS = piv + 2 * kMaxD; // s x s
  double* xcS = coreS + s * s;     // s x r
  double* ycS = xcS + s * r;       // r x s
  double* ycT = ycS + r * s;       // s x r (yc transposed: conflict-free B operand)
  __shared__ double red[3 * (kCT / 32)];
  __shared__ int s_stop;
  const int tid = threadIdx.x, sr = s * r, len = sums_len(s, r);
  const double* sl = sums;         // left: L^T U | L^T dU | sums
  const double* srt = sums + len;  // right: R V^T | R dV^T (as s x r) | sums
  if (tid == 0) s_stop = 0;
  for (int i = tid; i < s * s; i += kCT) coreS[i] = core[i];
  for (int i = tid; i < s * r; i += kCT) xcS[i] = xc[i];
  for (int i = tid; i < r * s; i += kCT) {
    ycS[i] = yc[i];
    ycT[(i % s) * r + i / s] = yc[i];
  }
  __syncthreads();
  if (first) {
    // yc = V R^T (nmf.py:338): the reduced right sums of the initial state
    for (int i = tid; i < r * s; i += kCT) {
      const int a = i / s, c = i % s;
      yc[i] = srt[c * r + a];
      ycS[i] = srt[c * r + a];
      ycT[c * r + a] = srt[c * r + a];
    }
    for (int i = tid; i < sr; i += kCT) DL[i] = DR[i] = 0.0;
    __syncthreads();
  } else if (k > 0) {
    // dual projections after the sweep of iteration k - 1 (xc, yc of k - 1)
    small_gemm(s, r, s, GL, ldg, 1, xcS, r, [&](int a, int j, double v) {
      DL[a * r + j] += step * pu * (v - sl[a * r + j]);
    });
    small_gemm(s, r, s, GR, ldg, 1, ycT, r, [&](int c, int j, double v) {
      DR[c * r + j] += step * pv * (v - srt[c * r + j]);
    });
    __syncthreads();
    // ---- KKT score of iteration k - 1 (nmf.py:281-303) ----
    double obj = 0.0, t1 = 0.0, t2 = 0.0;
    small_gemm(s, s, r, xcS, r, 1, ycS, s, [&](int a, int c, double v) {
      const double e = v - coreS[a * s + c];
      E[a * s + c] = e;
      obj += e * e;
    });
    __syncthreads();
    small_gemm(s, r, s, E, s, 1, ycT, r, [&](int a, int j, double v) {  // (E yc^T + L^T dU)[a][j]
      const double w = v + DL[a * r + j];
      t1 += w * w;
    });
    small_gemm(r, s, s, xcS, 1, r, E, s, [&](int j, int c, double v) {  // (xc^T E + dV R^T)[j][c]
      const double w = v + DR[c * r + j];
      t2 += w * w;
    });
    block_sum(t1, red, 0);
    block_sum(t2, red, 1);
    block_sum(obj, red, 2);
    __syncthreads();
    if (tid == 0) {
      double a1 = 0, a2 = 0, ob = 0;
      for (int w = 0; w < kCT / 32; ++w) {
        a1 += red[w];
        a2 += red[(kCT / 32) + w];
        ob += red[2 * (kCT / 32) + w];
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
  small_gemm(r, r, s, ycS, s, 1, ycT, r, [&](int a, int c, double v) { M[a * r + c] = v + (a == c ? pu : 0.0); });
  small_gemm(s, r, s, coreS, s, 1, ycT, r, [&](int a, int c, double v) {  // rhs (s x r) in E
    E[a * r + c] = v + (pu * sl[a * r + c] - DL[a * r + c]);
  });
  spd_inverse(M, piv, r);
  small_gemm(s, r, r, E, r, 1, M, r, [&](int a, int c, double v) {
    xc[a * r + c] = v;
    xcS[a * r + c] = v;
    Zl[a * r + c] = v;
  });
  __syncthreads();
  // ---- yc = (xc^T xc + pv I)^-1 (xc^T core + pv V R^T - dV R^T) ----
  small_gemm(r, r, s, xcS, 1, r, xcS, r, [&](int a, int c, double v) { M[a * r + c] = v + (a == c ? pv : 0.0); });
  small_gemm(r, s, s, xcS, 1, r, coreS, s, [&](int a, int c, double v) {  // rhs2 (r x s) in B
    B[a * s + c] = v + (pv * srt[c * r + a] - DR[c * r + a]);
  });
  spd_inverse(M, piv, r);
  small_gemm(r, s, r, M, r, 1, B, s, [&](int a, int c, double v) {
    yc[a * s + c] = v;
    Zr[c * r + a] = v;  // Z for the right rows: yc^T (s x r)
  });
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
  // row blocks: as many as are resident at once, split between the sides by row count
  const int total = sweep_blocks(sms);
  const int nbl = (int)std::max<int64_t>(1, std::min<int64_t>(total - 1, (total * m + (m + n) / 2) / (m + n)));
  const int nbr = total - nbl;
  const int len = sums_len(s, r);
  // library scratch: block partials, reduced sums, Z operands
  const size_t need = ((size_t)total * len + 2 * (size_t)len + 6 * kMaxD * kMaxD) * 8;
  void* scr = nullptr;
  CNMF_TRY(device_scratch("admm-stream", need, &scr, st));
  double* scratch = (double*)scr;
  double* part = scratch;
  double* sums = part + (size_t)total * len;
  double* Zl = sums + 2 * len;
  double* Zr = Zl + kMaxD * kMaxD;
  double* GL = Zr + kMaxD * kMaxD;  // L^T L and R R^T (S x S), for the dual-projection recurrence
  double* GR = GL + kMaxD * kMaxD;
  double* DL = GR + kMaxD * kMaxD;  // L^T dU, R dV^T (s x r)
  double* DR = DL + kMaxD * kMaxD;
  const size_t core_smem = (2 * (size_t)s * s + 4 * (size_t)s * r + (size_t)r * r + 2 * kMaxD) * 8;
  CNMF_TRY(ensure_smem_attr((const void*)row_sweep<32>, (int)sweep_smem<32>()));
  CNMF_TRY(ensure_smem_attr((const void*)row_sweep<64>, (int)sweep_smem<64>()));
  CNMF_TRY(ensure_smem_attr((const void*)core_step, (int)((7 * kMaxD * kMaxD + 2 * kMaxD) * 8)));
  const SSide sl{L, m, S, u, du, pu}, sr{Rt, n, S, vt, dvt, pv};
  auto sweep = [&](int update) -> int {
    if (S == 32)
      row_sweep<32><<<total, kSW, sweep_smem<32>(), st>>>(sl, sr, nbl, Zl, Zr, s, r, step, update, part, ctrl);
    else
      row_sweep<64><<<total, kSW, sweep_smem<64>(), st>>>(sl, sr, nbl, Zl, Zr, s, r, step, update, part, ctrl);
    CNMF_LAUNCH_CHECK();
    reduce_parts<<<dim3((unsigned)ceil_div(len, kT), 2), kT, 0, st>>>(part, nbl, nbr, len, sums, ctrl, update);
    CNMF_LAUNCH_CHECK();
    return CNMF_OK;
  };
  int k0 = 0;
  if (!resume) {
    init_sctrl<<<1, 1, 0, st>>>(ctrl);
    CNMF_LAUNCH_CHECK();
    CNMF_TRY(panel_cross(L, L, m, S, GL, st));
    CNMF_TRY(panel_cross(Rt, Rt, n, S, GR, st));
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
    core_step<<<1, kCT, core_smem, st>>>(core, sums, xc, yc, Zl, Zr, GL, GR, S, DL, DR, s, r, pu, pv, step, tol,
                                        trace, scores, ctrl, k,
                                        max_iter, k == 0 && !resume, 1);
    CNMF_LAUNCH_CHECK();
    CNMF_TRY(sweep(1));
  }
  // score of the last swept iteration (and the stop decision)
  core_step<<<1, kCT, core_smem, st>>>(core, sums, xc, yc, Zl, Zr, GL, GR, S, DL, DR, s, r, pu, pv, step, tol, trace,
                                      scores, ctrl, k1,
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

// ---------------------------------------------------------------------------
// Column-sharded ADMM (paper_1505_04650_b200/distributed.py): the same
// kernels driven one phase at a time by the host, so that the reduced sums of
// every rank's row blocks can be all-reduced (NCCL) between the sweep and the
// replicated core step. Workspace (doubles): [ctrl 8 | Zl 64 x 64 | Zr 64 x 64 |
// sums 2 x sums_len(s, r)]; the sums are [left: L^T U | L^T dU | 4 KKT sums,
// right: R V^T | R dV^T | 4 KKT sums] (s x r blocks, row-major).
// ---------------------------------------------------------------------------
size_t admm_shard_workspace(int s, int r) { return (8 + 6 * (size_t)kMaxD * kMaxD + 2 * (size_t)sums_len(s, r)) * 8; }
size_t admm_shard_sums_offset() { return (8 + 2 * (size_t)kMaxD * kMaxD) * 8; }

struct ShardWs {
  SCtrl* ctrl;
  double* Zl;
  double* Zr;
  double* sums;
  double *GL, *GR, *DL, *DR;
};

static ShardWs shard_ws(void* ws, int s, int r) {
  double* p = (double*)ws;
  double* g = p + 8 + 2 * kMaxD * kMaxD + 2 * (size_t)sums_len(s, r);
  return ShardWs{(SCtrl*)p, p + 8, p + 8 + kMaxD * kMaxD, p + 8 + 2 * kMaxD * kMaxD,
                 g, g + kMaxD * kMaxD, g + 2 * kMaxD * kMaxD, g + 3 * kMaxD * kMaxD};
}

// GL = L^T L over all rows of L, GR = R R^T over all columns of R (ld x ld
// fp64, ld = the panel width): the dual-projection recurrence's Gram
// matrices, all-reduced by the caller for a sharded R
int admm_shard_begin(void* ws, int s, int r, const double* GL, const double* GR, int ld, cudaStream_t st) {
  if (s < 1 || r < 1 || s > kMaxD || r > kMaxD || ld < s || ld > kMaxD)
    return fail(CNMF_ERR_ARGUMENT, "sharded ADMM: 1 <= r, s <= ld <= 64");
  const ShardWs w = shard_ws(ws, s, r);
  init_sctrl<<<1, 1, 0, st>>>(w.ctrl);
  CNMF_LAUNCH_CHECK();
  CNMF_CUDA(cudaMemcpyAsync(w.GL, GL, (size_t)ld * ld * 8, cudaMemcpyDeviceToDevice, st));
  CNMF_CUDA(cudaMemcpyAsync(w.GR, GR, (size_t)ld * ld * 8, cudaMemcpyDeviceToDevice, st));
  return CNMF_OK;
}

int admm_shard_sweep(void* ws, const float* L, int64_t m, const float* Rt, int64_t n, int s, int r, double* u,
                     double* du, double* vt, double* dvt, double pu, double pv, double step, int update,
                     cudaStream_t st) {
  if (s < 1 || r < 1 || s > kMaxD || r > kMaxD) return fail(CNMF_ERR_ARGUMENT, "sharded ADMM: 1 <= r, s <= 64");
  const ShardWs w = shard_ws(ws, s, r);
  const int S = s <= 32 ? 32 : 64;
  const int total = sweep_blocks(device_sms());
  const int64_t rows = std::max<int64_t>(m + n, 1);
  const int nbl = (int)std::max<int64_t>(1, std::min<int64_t>(total - 1, (total * m + rows / 2) / rows));
  const int nbr = total - nbl;
  const int len = sums_len(s, r);
  void* part = nullptr;
  CNMF_TRY(device_scratch("admm-shard-part", (size_t)total * len * 8, &part, st));
  CNMF_TRY(ensure_smem_attr((const void*)row_sweep<32>, (int)sweep_smem<32>()));
  CNMF_TRY(ensure_smem_attr((const void*)row_sweep<64>, (int)sweep_smem<64>()));
  const SSide sl{L, m, S, u, du, pu}, sr{Rt, n, S, vt, dvt, pv};
  if (S == 32)
    row_sweep<32><<<total, kSW, sweep_smem<32>(), st>>>(sl, sr, nbl, w.Zl, w.Zr, s, r, step, update, (double*)part,
                                                        w.ctrl);
  else
    row_sweep<64><<<total, kSW, sweep_smem<64>(), st>>>(sl, sr, nbl, w.Zl, w.Zr, s, r, step, update, (double*)part,
                                                        w.ctrl);
  CNMF_LAUNCH_CHECK();
  reduce_parts<<<dim3((unsigned)ceil_div(len, kT), 2), kT, 0, st>>>((double*)part, nbl, nbr, len, w.sums, w.ctrl,
                                                                    update);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

int admm_shard_core(void* ws, const double* core, double* xc, double* yc, int s, int r, double pu, double pv,
                    double step, double tol, double* trace, double* scores, int k, int max_iter, int first, int solve,
                    cudaStream_t st) {
  const ShardWs w = shard_ws(ws, s, r);
  const int S = s <= 32 ? 32 : 64;
  const size_t core_smem = (2 * (size_t)s * s + 4 * (size_t)s * r + (size_t)r * r + 2 * kMaxD) * 8;
  CNMF_TRY(ensure_smem_attr((const void*)core_step, (int)((7 * kMaxD * kMaxD + 2 * kMaxD) * 8)));
  core_step<<<1, kCT, core_smem, st>>>(core, w.sums, xc, yc, w.Zl, w.Zr, w.GL, w.GR, S, w.DL, w.DR, s, r, pu, pv,
                                      step, tol, trace, scores, w.ctrl, k,
                                      max_iter, first, solve);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

// state[0..3] = (next iteration, done, iterations, diverged iteration or -1)
int admm_shard_status(const void* ws, int* state, cudaStream_t st) {
  CNMF_CUDA(cudaMemcpyAsync(state, ws, sizeof(SCtrl), cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaStreamSynchronize(st));
  return CNMF_OK;
}

}  // namespace cnmf
