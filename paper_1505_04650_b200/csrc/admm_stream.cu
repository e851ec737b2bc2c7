// Compressed ADMM NMF for problems whose per-CTA state does not fit the
// persistent kernel (csrc/admm.cu keeps s x s / s x r fp64 matrices and the
// row slices in shared memory: r > 32 with s > 32, or very tall sides).
//
// Reference: nmf.py:306-377 (the loop), nmf.py:281-303 (KKT score); the same
// arithmetic as oracle/cnmf_oracle.py admm_compressed.
//
// All state in HBM; the kernels of one iteration:
//   core step              KKT score of the previous iteration from the
//                          reduced sums, convergence / divergence rule, then
//                          xc = (core yc^T + pu L^T U - L^T dU)(yc yc^T + pu I)^-1
//                          yc = (xc^T xc + pv I)^-1 (xc^T core + pv V R^T - dV R^T)
//   row_sweep  (grid)      every row of a side: x = max(P z + dx / p, 0),
//                          dx += step p (P z - x), and the block partials of
//                          P^T x and the four KKT sums
//   reduce_parts (grid)    fixed-order sums of the block partials
// so every reduction is deterministic. On one GPU (admm_stream_run) the core
// step is split into core_x (xc + the score, between two sweeps) and core_y
// (yc + the next iteration's operands, concurrent with the left sweep); the
// column-sharded driver (admm_shard_*) runs it as one kernel, core_step,
// between the host's all-reduces. Streaming bytes per iteration: dU, dV read
// and written, U, V written (fp64) + L, R read (fp32).
#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>

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
// named barriers: 1 = update group internal, 6 = reduction group internal,
// 2 + b = tile buffer b updated (update -> reduction group),
// 4 + b = tile buffer b filled (reduction -> update group)
constexpr int kBarU = 1, kBarFull = 2, kBarEmpty = 4, kBarR = 6;

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

  // 16-byte copies when every row of x, dx starts 16-byte aligned (r even)
  const bool vec = (r & 1) == 0;

  if (ugroup) {
    // ======================= update group =======================
    // x = max(P z + dx / p, 0) with dx / p as dx * (1 / p): one rounding
    // more than the reference's division (<= 1 ulp), ~30 instructions less
    const double inv_pen = 1.0 / sd.pen, step_pen = step * sd.pen;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int64_t t = 0; t < ntile; ++t) {
      const int buf = (int)(t & 1);
      const int64_t t0 = r0 + t * kRT;
      const int nr = (int)min64(kRT, r1 - t0);
      const double* Pr = PrB + buf * kRT * kLD;
      double* Xs = XsB + buf * kRT * kLD;
      nbar_sync(kBarEmpty + buf, kSW);  // Pr[buf] and the old x in Xs[buf] are in place
      // the tile's old dx lands in Ds while P z is formed (the previous
      // tile's update is done with Ds: barrier kBarU below)
      if (update) {
        if (vec) {
          const int h = r >> 1;  // 16-byte chunks per row
          for (int i = tid; i < nr * h; i += kT) {
            const int row = i / h, c2 = i - row * h;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(Ds + row * kLD + 2 * c2)),
                         "l"(sd.dx + (t0 + row) * r + 2 * c2)
                         : "memory");
          }
        } else {
          for (int i = tid; i < nr * r; i += kT) {
            const int row = i / r, k = i - row * r;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(Ds + row * kLD + k)),
                         "l"(sd.dx + (t0 + row) * r + k)
                         : "memory");
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      double acc[2][4][2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      if (update) {
        const double* pa = Pr + (16 * wm + g) * kLD + tq;  // A[row][c]: rows 16 wm + 8 mi + g
        const double* zb = Z + tq * kLD + 32 * wn + g;     // B[c][k]: k = 32 wn + 8 ni + g
        const int nn = min(4, (r - 32 * wn + 7) >> 3);     // 8-column tiles this warp needs
        const int ksn = min(KS, (s + 3) >> 2);  // k steps that hold columns c < s
#pragma unroll 4
        for (int ks = 0; ks < ksn; ++ks) {
          const double a0 = pa[4 * ks], a1 = pa[8 * kLD + 4 * ks];
          double bv[4];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) bv[ni] = zb[4 * ks * kLD + 8 * ni];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
            if (ni < nn) {
              dmma(acc[0][ni], a0, bv[ni]);
              dmma(acc[1][ni], a1, bv[ni]);
            }
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      nbar_sync(kBarU, kT);  // every thread's dx visible
      // (x, dx) update, KKT sums, the new x into Xs (in place: every thread
      // reads and writes only its own elements: row 16 wm + 8 mi + g,
      // columns 32 wn + 8 ni + 2 tq + {0, 1})
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int row = 16 * wm + 8 * mi + g;
        const bool ron = row < nr;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          const int k = 32 * wn + 8 * ni + 2 * tq;
          double* xs = Xs + row * kLD + k;
          double xn[2] = {0.0, 0.0};
          if (update) {
            const double2 dxo2 = *(const double2*)(Ds + row * kLD + k);
            const double dxo[2] = {dxo2.x, dxo2.y};
            double dxn[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const bool on = ron && k + e < r;
              const double pz = acc[mi][ni][e];
              const double v = pz + dxo[e] * inv_pen;
              const double x = v > 0.0 ? v : 0.0;
              const double dx = dxo[e] + step_pen * (pz - x);
              const double dl = pz - x, dp = dx * x, dpos = dx > 0.0 ? dx : 0.0;
              s0 += on ? dl * dl : 0.0;
              s1 += on ? dp * dp : 0.0;
              s2 += on ? dpos * dpos : 0.0;  // x >= 0, so the negative part of x is 0
              xn[e] = on ? x : 0.0;
              dxn[e] = dx;
            }
            const int64_t gi = (t0 + row) * r + k;
            if (vec && ron && k + 1 < r) {
              *(double2*)(sd.x + gi) = make_double2(xn[0], xn[1]);
              *(double2*)(sd.dx + gi) = make_double2(dxn[0], dxn[1]);
            } else if (ron) {
#pragma unroll
              for (int e = 0; e < 2; ++e)
                if (k + e < r) {
                  sd.x[gi + e] = xn[e];
                  sd.dx[gi + e] = dxn[e];
                }
            }
          } else {
            const double2 xo = *(const double2*)xs;
            xn[0] = ron && k < r ? xo.x : 0.0;
            xn[1] = ron && k + 1 < r ? xo.y : 0.0;
          }
          *(double2*)xs = make_double2(xn[0], xn[1]);
        }
      }
      nbar_sync(kBarU, kT);              // Ds read and Xs[buf] written by the whole group
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
    // fills tile buffers (P rows -> fp64 Pr, old x by cp.async) two tiles
    // ahead, and reduces P^T x: A[c][row] = Pr[row][c] (c = 16 wm + 8 mi + g),
    // B[row][k] = Xs[row][k]
    // a tile's panel rows are fetched into registers (fill_load) before the
    // reduction of the tile two back, whose buffer they go to, and stored
    // after it (fill_store): the loads' HBM latency hides under the DMMAs
    constexpr int PF = kRT * (SP / 4) / kT;
    float4 pf[PF];
    auto fill_load = [&](int64_t t) {
      const int64_t t0 = r0 + t * kRT;
      const int nr = (int)min64(kRT, r1 - t0);
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        const int i = tid + j * kT, row = i / (SP / 4), c4 = 4 * (i % (SP / 4));
        pf[j] = (row < nr) ? __ldg((const float4*)(sd.P + (t0 + row) * sd.ldp + c4)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto fill_store = [&](int64_t t) {
      const int buf = (int)(t & 1);
      const int64_t t0 = r0 + t * kRT;
      const int nr = (int)min64(kRT, r1 - t0);
      double* Pr = PrB + buf * kRT * kLD;
      double* Xs = XsB + buf * kRT * kLD;
      // the old x is needed only by the start-up sweep (update = 0: P^T x of
      // the initial splits); an update sweep overwrites every entry of Xs
      if (update) {
      } else if (vec) {
        const int h = r >> 1;
        for (int i = tid; i < nr * h; i += kT) {
          const int row = i / h, c2 = i - row * h;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(Xs + row * kLD + 2 * c2)),
                       "l"(sd.x + (t0 + row) * r + 2 * c2)
                       : "memory");
        }
      } else {
        for (int i = tid; i < nr * r; i += kT) {
          const int row = i / r, k = i - row * r;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(Xs + row * kLD + k)),
                       "l"(sd.x + (t0 + row) * r + k)
                       : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        const int i = tid + j * kT, row = i / (SP / 4), c4 = 4 * (i % (SP / 4));
        double* d = Pr + row * kLD + c4;
        *(double2*)d = make_double2(c4 + 0 < s ? (double)pf[j].x : 0.0, c4 + 1 < s ? (double)pf[j].y : 0.0);
        *(double2*)(d + 2) = make_double2(c4 + 2 < s ? (double)pf[j].z : 0.0, c4 + 3 < s ? (double)pf[j].w : 0.0);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      nbar_arrive(kBarEmpty + buf, kSW);  // the bar.arrive orders the group's smem writes before the update group
    };
    double au[2][4][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) au[mi][ni][0] = au[mi][ni][1] = 0.0;
    const bool con = 16 * wm < s;
    const int nn = min(4, (r - 32 * wn + 7) >> 3);
    for (int64_t t = 0; t < ntile && t < 2; ++t) {
      fill_load(t);
      fill_store(t);
    }
    for (int64_t t = 0; t < ntile; ++t) {
      const int buf = (int)(t & 1);
      if (t + 2 < ntile) fill_load(t + 2);
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
          for (int ni = 0; ni < 4; ++ni)
            if (ni < nn) {
              dmma(au[0][ni], a0, bv[ni]);
              dmma(au[1][ni], a1, bv[ni]);
            }
        }
      }
      if (t + 2 < ntile) {
        nbar_sync(kBarR, kT);  // every reduction warp is done reading buffer buf
        fill_store(t + 2);
      }
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

// fixed-order sums of the block partials of each side: sums[side][e]. A block
// covers kRE elements x kRS segments of the side's blocks; a segment is summed
// in block order and the segments are combined in segment order, so the
// result does not depend on scheduling.
constexpr int kRS = 4, kRE = kT / kRS;
__global__ void __launch_bounds__(kT) reduce_parts(const double* __restrict__ part, int nbl, int nbr, int len,
                                                    double* __restrict__ sums, const SCtrl* ctrl, int update) {
  if (update && ctrl->done) return;
  __shared__ double seg[kRS][kRE];
  const int el = threadIdx.x % kRE, sg = threadIdx.x / kRE;
  const int e = blockIdx.x * kRE + el;
  const int side = blockIdx.y;
  const int b0 = side ? nbl : 0, nb = side ? nbr : nbl;
  const int sr = (len - 4) / 2;
  const bool dual = e >= sr && e < 2 * sr;  // the dual projections come from the core step's recurrence
  double acc = 0.0;
  if (e < len && !dual) {
    const int per = (nb + kRS - 1) / kRS, j1 = min(nb, (sg + 1) * per);
    for (int j0 = sg * per; j0 < j1; j0 += 8) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (j0 + j < j1) ? part[(size_t)(b0 + j0 + j) * len + e] : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += v[j];
    }
  }
  seg[sg][el] = acc;
  __syncthreads();
  if (sg == 0 && e < len) {
    double t = seg[0][el];
#pragma unroll
    for (int j = 1; j < kRS; ++j) t += seg[j][el];
    sums[side * len + e] = dual ? 0.0 : t;
  }
}

// ---------------------------------------------------------------------------
// core step: one block of kCT threads; every small product is a register-
// tiled shared-memory GEMM (2 x 4 outputs per thread, operands broadcast
// within a warp), the two r x r ridge systems are inverted by Gauss-Jordan
// ---------------------------------------------------------------------------
constexpr int kCT = 512;

// C(m, n) = sum_k A[m * am + k * ak] * B[k * bk + n * bn] for m < M, n < N,
// M, N <= 64; out(m, n, value) consumes every result exactly once. On the
// fp64 tensor cores: warp w owns the 2 x 2 block of 8 x 8 output tiles at
// rows 16 (w / 4), columns 16 (w % 4); per k step of 4 a lane loads two A and
// two B elements (the next step's loads are issued before this step's four
// DMMA). Rows >= M and columns >= N are computed on clamped (valid) data and
// dropped at the output; only the k tail is masked. ~4.5k cycles for
// 60 x 50 x 60 (tools/gemm_probe.cu), 2.2x the one-tile-per-load version.
template <class F>
__device__ __forceinline__ void small_gemm(int M, int N, int K, const double* A, int am, int ak, const double* B,
                                           int bk, int bn, F out) {
  static_assert(kCT == 512, "16 warps x (16 x 16) cover 64 x 64");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int bm_ = warp >> 2, bn_ = warp & 3;
  if (16 * bm_ >= M || 16 * bn_ >= N) return;
  const int m0 = min(16 * bm_ + g, M - 1), m1 = min(16 * bm_ + 8 + g, M - 1);
  const int n0 = min(16 * bn_ + g, N - 1), n1 = min(16 * bn_ + 8 + g, N - 1);
  const double* a0p = A + m0 * am + tq * ak;
  const double* a1p = A + m1 * am + tq * ak;
  const double* b0p = B + tq * bk + n0 * bn;
  const double* b1p = B + tq * bk + n1 * bn;
  double c[2][2][2] = {};
  const int K4 = K & ~3;
  if (K4 > 0) {
    double x0 = a0p[0], x1 = a1p[0], y0 = b0p[0], y1 = b1p[0];
    for (int k0 = 4; k0 < K4; k0 += 4) {
      const double nx0 = a0p[k0 * ak], nx1 = a1p[k0 * ak], ny0 = b0p[k0 * bk], ny1 = b1p[k0 * bk];
      dmma(c[0][0], x0, y0);
      dmma(c[0][1], x0, y1);
      dmma(c[1][0], x1, y0);
      dmma(c[1][1], x1, y1);
      x0 = nx0;
      x1 = nx1;
      y0 = ny0;
      y1 = ny1;
    }
    dmma(c[0][0], x0, y0);
    dmma(c[0][1], x0, y1);
    dmma(c[1][0], x1, y0);
    dmma(c[1][1], x1, y1);
  }
  if (K4 < K) {  // tail: k = K4 + tq may pass K
    const bool kon = K4 + tq < K;
    const double x0 = kon ? a0p[K4 * ak] : 0.0, x1 = kon ? a1p[K4 * ak] : 0.0;
    const double y0 = kon ? b0p[K4 * bk] : 0.0, y1 = kon ? b1p[K4 * bk] : 0.0;
    dmma(c[0][0], x0, y0);
    dmma(c[0][1], x0, y1);
    dmma(c[1][0], x1, y0);
    dmma(c[1][1], x1, y1);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = 16 * bm_ + 8 * i + g, n = 16 * bn_ + 8 * j + 2 * tq + e;
        if (m < M && n < N) out(m, n, c[i][j][e]);
      }
}

// In-place inverse of an SPD r x r matrix (ld r, r <= 64) by Gauss-Jordan
// without pivoting (the ridge term keeps the pivots >= the penalty). Thread t
// of the first 64 * TPR owns row t / TPR, columns EPT (t % TPR) .. + EPT - 1
// (EPT = 64 / TPR) in registers. Per elimination step the owners of the
// pivot row publish it (scaled) and the reciprocal pivot in a double-buffered
// shared row, one named barrier, and every thread updates its entries
// branch-free (a divergent branch per entry serialised every DFMA behind its
// predecessor); the pivot-column entry of a row comes from the lane holding
// it by shuffle, picked out of the registers by a select tree.
constexpr int kPivLD = 72;  // per buffer: 64 pivot-row entries + the reciprocal pivot at [64]
constexpr int kPivDoubles = 2 * kPivLD;  // two pivot-row buffers
// (a version passing the pivot rows through an mbarrier-guarded ring, so that
// only the next pivot row's owners sit on the critical path, measured the
// same ~1.2k cycles per step and deadlocked when called twice per launch)
#ifndef CNMF_GJ_TPR
#define CNMF_GJ_TPR 2
#endif

__device__ void spd_inverse(double* M, double* piv, int r) {
  constexpr int TPR = CNMF_GJ_TPR, EPT = 64 / TPR, NT = 64 * TPR;
  static_assert(kCT >= NT && (TPR & (TPR - 1)) == 0 && TPR <= 32, "threads per row");
  __syncthreads();  // M complete
  const int t = threadIdx.x;
  if (t < NT) {
    const int a = t / TPR, q = t % TPR, cb = EPT * q, lane = t & 31;
    double m[EPT];
#pragma unroll
    for (int j = 0; j < EPT; ++j) m[j] = (a < r && cb + j < r) ? M[a * r + cb + j] : 0.0;
    double fk = m[0];  // this thread's entry in the next pivot column (column 0 first)
    for (int k = 0; k < r; ++k) {
      double* pv = piv + (k & 1) * kPivLD;
      const double f = __shfl_sync(0xffffffffu, fk, (lane & ~(TPR - 1)) | (k / EPT));  // row a, column k
      if (a == k) {
        const double inv = 1.0 / f;
#pragma unroll
        for (int j = 0; j < EPT; j += 2) *(double2*)(pv + cb + j) = make_double2(m[j] * inv, m[j + 1] * inv);
        if (q == 0) pv[64] = inv;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
      const double inv = pv[64];
      //   row k:      m = piv (column k: inv)
      //   other rows: m = m - f piv (column k: -f inv)
      const bool own = (a == k);
      const double coef = own ? 0.0 : -f, ck = own ? inv : -f * inv;
      const int kc = k - cb;  // the pivot column, relative to this thread's entries
      double2 p2[EPT / 2];
#pragma unroll
      for (int j = 0; j < EPT / 2; ++j) p2[j] = *(const double2*)(pv + cb + 2 * j);
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const double pj = (j & 1) ? p2[j >> 1].y : p2[j >> 1].x;
        const double v = fma(coef, pj, own ? pj : m[j]);
        m[j] = (j == kc) ? ck : v;
      }
      // this thread's entry in the next pivot column: a select tree
      const int kn = k + 1 - cb;
      double tr[EPT];
#pragma unroll
      for (int j = 0; j < EPT; ++j) tr[j] = m[j];
#pragma unroll
      for (int w = EPT / 2; w >= 1; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) tr[j] = (kn & w) ? tr[j + w] : tr[j];
      fk = tr[0];
    }
#pragma unroll
    for (int j = 0; j < EPT; ++j)
      if (a < r && cb + j < r) M[a * r + cb + j] = m[j];
  }
  __syncthreads();
}

#ifdef CNMF_CORE_TRACE
// phase timestamps of the last core step (tools/core_trace.py; A/B builds only)
__device__ long long g_core_trace[16];
#define CORE_MARK(i)                                   \
  do {                                                 \
    __syncthreads();                                   \
    if (threadIdx.x == 0) g_core_trace[i] = clock64(); \
  } while (0)
// (the product build's barriers are explicit: CORE_MARK adds one only here)
#else
#define CORE_MARK(i) \
  do {               \
  } while (0)
#endif

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
#ifdef CNMF_CORE_TRACE
  if (threadIdx.x == 0) g_core_trace[0] = clock64();
#endif
  extern __shared__ __align__(16) unsigned char sm[];
  double* E = (double*)sm;         // s x s: E = xc yc - core, later the rhs (s x r)
  double* B = E + s * s;           // rhs2 (r x s)
  double* M = B + ((r * s + s * s) & 1) + r * s;  // r x r (even offset: piv below stays 16-byte aligned)
  double* piv = M + ((r * r + 1) & ~1);  // pivot ring + mbarriers (kPivDoubles), 16-byte aligned
  double* coreS = piv + kPivDoubles; // s x s
  double* xcS = coreS + s * s;     // s x r
  double* ycS = xcS + s * r;       // r x s
  double* G = E;                   // s x s: G_L, then G_R, staged for the dual projections (E is free then)
  __shared__ double red[3 * (kCT / 32)];
  __shared__ int s_stop;
  const int tid = threadIdx.x, sr = s * r, len = sums_len(s, r);
  const double* sl = sums;         // left: L^T U | L^T dU | sums
  const double* srt = sums + len;  // right: R V^T | R dV^T (as s x r) | sums
  if (tid == 0) s_stop = 0;
  for (int i = tid; i < s * s; i += kCT) coreS[i] = core[i];
  for (int i = tid; i < s * r; i += kCT) xcS[i] = xc[i];
  for (int i = tid; i < r * s; i += kCT) ycS[i] = yc[i];
  if (!first && k > 0)  // G_L (ld ldg) compacted to s x s
    for (int i = tid; i < s * s; i += kCT) G[i] = GL[(i / s) * ldg + i % s];
  __syncthreads();
  CORE_MARK(1);
  if (first) {
    // yc = V R^T (nmf.py:338): the reduced right sums of the initial state
    for (int i = tid; i < r * s; i += kCT) {
      const int a = i / s, c = i % s;
      yc[i] = srt[c * r + a];
      ycS[i] = srt[c * r + a];
    }
    for (int i = tid; i < sr; i += kCT) DL[i] = DR[i] = 0.0;
    __syncthreads();
  } else if (k > 0) {
    // dual projections after the sweep of iteration k - 1 (xc, yc of k - 1)
    small_gemm(s, r, s, G, s, 1, xcS, r, 1, [&](int a, int j, double v) {
      DL[a * r + j] += step * pu * (v - sl[a * r + j]);
    });
    __syncthreads();
    for (int i = tid; i < s * s; i += kCT) G[i] = GR[(i / s) * ldg + i % s];
    __syncthreads();
    small_gemm(s, r, s, G, s, 1, ycS, 1, s, [&](int c, int j, double v) {
      DR[c * r + j] += step * pv * (v - srt[c * r + j]);
    });
    __syncthreads();
    CORE_MARK(2);
    // ---- KKT score of iteration k - 1 (nmf.py:281-303) ----
    double obj = 0.0, t1 = 0.0, t2 = 0.0;
    small_gemm(s, s, r, xcS, r, 1, ycS, s, 1, [&](int a, int c, double v) {
      const double e = v - coreS[a * s + c];
      E[a * s + c] = e;
      obj += e * e;
    });
    __syncthreads();
    small_gemm(s, r, s, E, s, 1, ycS, 1, s, [&](int a, int j, double v) {  // (E yc^T + L^T dU)[a][j]
      const double w = v + DL[a * r + j];
      t1 += w * w;
    });
    small_gemm(r, s, s, xcS, 1, r, E, s, 1, [&](int j, int c, double v) {  // (xc^T E + dV R^T)[j][c]
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
  CORE_MARK(3);
  if (!solve || k >= max_iter) return;
  // ---- xc = (core yc^T + pu L^T U - L^T dU) (yc yc^T + pu I)^-1 ----
  small_gemm(r, r, s, ycS, s, 1, ycS, 1, s, [&](int a, int c, double v) { M[a * r + c] = v + (a == c ? pu : 0.0); });
  small_gemm(s, r, s, coreS, s, 1, ycS, 1, s, [&](int a, int c, double v) {  // rhs (s x r) in E
    E[a * r + c] = v + (pu * sl[a * r + c] - DL[a * r + c]);
  });
  CORE_MARK(4);
  spd_inverse(M, piv, r);
  CORE_MARK(5);
  small_gemm(s, r, r, E, r, 1, M, r, 1, [&](int a, int c, double v) {
    xc[a * r + c] = v;
    xcS[a * r + c] = v;
    Zl[a * r + c] = v;
  });
  __syncthreads();
  // ---- yc = (xc^T xc + pv I)^-1 (xc^T core + pv V R^T - dV R^T) ----
  small_gemm(r, r, s, xcS, 1, r, xcS, r, 1, [&](int a, int c, double v) { M[a * r + c] = v + (a == c ? pv : 0.0); });
  small_gemm(r, s, s, xcS, 1, r, coreS, s, 1, [&](int a, int c, double v) {  // rhs2 (r x s) in B
    B[a * s + c] = v + (pv * srt[c * r + a] - DR[c * r + a]);
  });
  CORE_MARK(6);
  spd_inverse(M, piv, r);
  CORE_MARK(7);
  small_gemm(r, s, r, M, r, 1, B, s, 1, [&](int a, int c, double v) {
    yc[a * s + c] = v;
    Zr[c * r + a] = v;  // Z for the right rows: yc^T (s x r)
  });
  CORE_MARK(8);
}

#ifdef CNMF_CORE_TRACE
}  // namespace
extern "C" int cnmf_debug_core_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, g_core_trace, sizeof(long long) * 16) == cudaSuccess ? 0 : -1;
}
namespace {
#endif

// ---------------------------------------------------------------------------
// Single-GPU driver: the core step split so that only what the next sweep
// needs sits between two sweeps (the column-sharded driver below keeps the
// one-kernel core_step, its sums being all-reduced by the host in between).
//
//   core_x(k)  2 CTAs after the sweeps of iteration k - 1:
//     CTA 0    xc_k = (P1 + pu L^T U - L^T dU) Minv: one product, Minv =
//              (yc yc^T + pu I)^-1, P1 = core yc^T and G_L xc_{k-1} having
//              been prepared by core_y(k - 1) while the sweeps ran;
//     CTA 1    KKT score of iteration k - 1 and the stopping rule;
//   core_y(k)  1 CTA on a side stream, concurrent with the left sweep of
//              iteration k (which needs xc_k only): yc_k, then Minv, P1,
//              G_L xc_k, G_R yc_k^T for core_x(k + 1);
//   left sweep(k) -> right sweep(k) (after core_y(k)) -> reduce.
// xc_k is published in scratch (xcn, Zl) and copied to the caller's xc by
// core_y(k), which runs only when the score CTA did not stop the run, so xc,
// yc stay those of the last completed iteration. L^T dU and R dV^T are
// double-buffered by the parity of k (iteration k reads k - 1's, writes its
// own), so recomputing an iteration's core_x on resume is idempotent.
// ---------------------------------------------------------------------------
struct CoreBufs {
  double *Zl, *Zr;    // s x r operands of the sweeps: xc, yc^T
  double *GL, *GR;    // ldg x ldg Gram matrices of the panels
  double *DL, *DR;    // [2][kMaxD * kMaxD]: L^T dU, R dV^T (s x r) by iteration parity
  double *Minv;       // r x r
  double *P1;         // s x r: core yc^T
  double *GLx, *GRy;  // s x r: G_L xc, G_R yc^T
  double *xcn;        // s x r: xc of the iteration being swept
};
constexpr int kCoreBufDoubles = 13 * kMaxD * kMaxD;

__global__ void __launch_bounds__(kCT) core_x(const double* __restrict__ core, const double* __restrict__ sums,
                                               const double* __restrict__ xc, const double* __restrict__ yc,
                                               CoreBufs cb, int s, int r, double pu, double pv, double step,
                                               double tol, double* trace, double* scores, SCtrl* ctrl, int k,
                                               int max_iter, int solve) {
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ double red[3 * (kCT / 32)];
  const int tid = threadIdx.x, sr = s * r, len = sums_len(s, r);
  const double* sl = sums;         // left: L^T U | - | sums
  const double* srt = sums + len;  // right: R V^T (as s x r) | - | sums
  const double* DLo = cb.DL + ((k + 1) & 1) * kMaxD * kMaxD;
  const double* DRo = cb.DR + ((k + 1) & 1) * kMaxD * kMaxD;
  double* DLn = cb.DL + (k & 1) * kMaxD * kMaxD;
  double* DRn = cb.DR + (k & 1) * kMaxD * kMaxD;
  if (blockIdx.x == 0) {
    // ---- xc = (core yc^T + pu L^T U - L^T dU) (yc yc^T + pu I)^-1 (nmf.py:342-343) ----
    if (!solve || k >= max_iter) return;
    double* rhs = (double*)sm;  // s x r
    double* Mi = rhs + sr;      // r x r
    for (int i = tid; i < r * r; i += kCT) Mi[i] = cb.Minv[i];
    for (int i = tid; i < sr; i += kCT) {
      const double dl = k > 0 ? DLo[i] + step * pu * (cb.GLx[i] - sl[i]) : 0.0;
      DLn[i] = dl;
      rhs[i] = cb.P1[i] + (pu * sl[i] - dl);
    }
    __syncthreads();
    small_gemm(s, r, r, rhs, r, 1, Mi, r, 1, [&](int a, int c, double v) {
      cb.xcn[a * r + c] = v;
      cb.Zl[a * r + c] = v;
    });
    return;
  }
  // ---- KKT score of iteration k - 1 (nmf.py:281-303) and the stopping rule ----
  if (k == 0) return;
  double* E = (double*)sm;      // s x s: xc yc - core
  double* coreS = E + s * s;    // s x s
  double* xcS = coreS + s * s;  // s x r
  double* ycS = xcS + sr;       // r x s
  for (int i = tid; i < s * s; i += kCT) coreS[i] = core[i];
  for (int i = tid; i < sr; i += kCT) {
    xcS[i] = xc[i];
    ycS[i] = yc[i];
    DRn[i] = DRo[i] + step * pv * (cb.GRy[i] - srt[i]);
  }
  __syncthreads();
  double obj = 0.0, t1 = 0.0, t2 = 0.0;
  small_gemm(s, s, r, xcS, r, 1, ycS, s, 1, [&](int a, int c, double v) {
    const double e = v - coreS[a * s + c];
    E[a * s + c] = e;
    obj += e * e;
  });
  __syncthreads();
  small_gemm(s, r, s, E, s, 1, ycS, 1, s, [&](int a, int j, double v) {  // (E yc^T + L^T dU)[a][j]
    const double w = v + (DLo[a * r + j] + step * pu * (cb.GLx[a * r + j] - sl[a * r + j]));
    t1 += w * w;
  });
  small_gemm(r, s, s, xcS, 1, r, E, s, 1, [&](int j, int c, double v) {  // (xc^T E + dV R^T)[j][c]
    const double w = v + DRn[c * r + j];
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
    } else if (it >= 50 && sc > 10.0 * scores[it - 50]) {
      ctrl->diverged = it;
      ctrl->done = 1;
      ctrl->iters = k;
    }
  }
}

__global__ void __launch_bounds__(kCT) core_y(const double* __restrict__ core, const double* __restrict__ sums,
                                               double* __restrict__ xc, double* __restrict__ yc, CoreBufs cb, int ldg,
                                               int s, int r, double pu, double pv, const SCtrl* ctrl, int k,
                                               int first) {
  if (ctrl->done) return;
  extern __shared__ __align__(16) unsigned char sm[];
  double* G = (double*)sm;         // s x s: G_L, then G_R
  double* B = G + s * s;           // rhs2 (r x s)
  double* M = B + ((r * s + s * s) & 1) + r * s;  // r x r (even offset: piv below stays 16-byte aligned)
  double* piv = M + ((r * r + 1) & ~1);
  double* coreS = piv + kPivDoubles;  // s x s
  double* xcS = coreS + s * s;        // s x r
  double* ycS = xcS + s * r;          // r x s
  const int tid = threadIdx.x, sr = s * r, len = sums_len(s, r);
  const double* srt = sums + len;
  for (int i = tid; i < s * s; i += kCT) {
    coreS[i] = core[i];
    G[i] = cb.GL[(i / s) * ldg + i % s];
  }
  if (first) {
    // yc = V R^T (nmf.py:338): the reduced right sums of the initial state;
    // dU = dV = 0
    for (int i = tid; i < sr; i += kCT) {
      const int a = i / s, c = i % s;
      const double v = srt[c * r + a];
      yc[i] = v;
      ycS[i] = v;
      cb.Zr[c * r + a] = v;
      xcS[i] = xc[i];
    }
    for (int i = tid; i < 2 * kMaxD * kMaxD; i += kCT) cb.DL[i] = cb.DR[i] = 0.0;
    __syncthreads();
  } else {
    const double* DRn = cb.DR + (k & 1) * kMaxD * kMaxD;
    for (int i = tid; i < sr; i += kCT) {
      const double v = cb.xcn[i];
      xc[i] = v;
      xcS[i] = v;
    }
    __syncthreads();
    // ---- yc = (xc^T xc + pv I)^-1 (xc^T core + pv V R^T - dV R^T) (nmf.py:344-345) ----
    small_gemm(r, r, s, xcS, 1, r, xcS, r, 1, [&](int a, int c, double v) { M[a * r + c] = v + (a == c ? pv : 0.0); });
    small_gemm(r, s, s, xcS, 1, r, coreS, s, 1, [&](int a, int c, double v) {  // rhs2 (r x s) in B
      B[a * s + c] = v + (pv * srt[c * r + a] - DRn[c * r + a]);
    });
    spd_inverse(M, piv, r);
    small_gemm(r, s, r, M, r, 1, B, s, 1, [&](int a, int c, double v) {
      yc[a * s + c] = v;
      ycS[a * s + c] = v;
      cb.Zr[c * r + a] = v;  // Z for the right rows: yc^T (s x r)
    });
    __syncthreads();
  }
  // ---- for core_x(k + 1), while the sweeps run ----
  small_gemm(s, r, s, G, s, 1, xcS, r, 1, [&](int a, int j, double v) { cb.GLx[a * r + j] = v; });
  small_gemm(r, r, s, ycS, s, 1, ycS, 1, s, [&](int a, int c, double v) { M[a * r + c] = v + (a == c ? pu : 0.0); });
  small_gemm(s, r, s, coreS, s, 1, ycS, 1, s, [&](int a, int c, double v) { cb.P1[a * r + c] = v; });
  __syncthreads();
  for (int i = tid; i < s * s; i += kCT) G[i] = cb.GR[(i / s) * ldg + i % s];
  spd_inverse(M, piv, r);  // (barriers on entry and exit)
  for (int i = tid; i < r * r; i += kCT) cb.Minv[i] = M[i];
  small_gemm(s, r, s, G, s, 1, ycS, 1, s, [&](int c, int j, double v) { cb.GRy[c * r + j] = v; });
}

__global__ void init_sctrl(SCtrl* c) {
  c->k = 0;
  c->done = 0;
  c->iters = 0;
  c->diverged = -1;
}

}  // namespace

namespace {
// side stream and fork / join events of the streaming driver, one set per device
int stream_side(cudaStream_t* side, cudaEvent_t* fork, cudaEvent_t* join) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  static cudaEvent_t forks[64] = {}, joins[64] = {};
  int dev = 0;
  CNMF_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(CNMF_ERR_CUDA, "device index out of range");
  std::lock_guard<std::mutex> lk(mu);
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
}  // namespace

int admm_stream_run(const double* core, const float* L, int64_t m, const float* Rt, int64_t n, int s, int r, double* u,
                    double* du, double* vt, double* dvt, double* xc, double* yc, double pu, double pv, double step,
                    int max_iter, double tol, double* trace, double* scores, int* iterations, void* ws, int resume,
                    int step_limit, cudaStream_t st) {
  const int S = s <= 32 ? 32 : 64;
  SCtrl* ctrl = (SCtrl*)ws;
  const int sms = device_sms();
  // row blocks: as many as are resident at once. The start-up sweep splits
  // them between the sides by row count; an iteration sweeps the left rows on
  // all but two SMs (core_y runs beside it), then the right rows on all.
  const int total = sweep_blocks(sms);
  const int nbl = (int)std::max<int64_t>(1, std::min<int64_t>(total - 1, (total * m + (m + n) / 2) / (m + n)));
  const int nbr = total - nbl;
  const int gl = std::max(1, total - 2), gr = total;
  const int len = sums_len(s, r);
  // library scratch: block partials, reduced sums, the core kernels' buffers
  const size_t need = ((size_t)(gl + gr) * len + 2 * (size_t)len + kCoreBufDoubles) * 8;
  void* scr = nullptr;
  CNMF_TRY(device_scratch("admm-stream", need, &scr, st));
  double* scratch = (double*)scr;
  double* part = scratch;
  double* sums = part + (size_t)(gl + gr) * len;
  double* cbp = sums + 2 * len;
  constexpr int D2 = kMaxD * kMaxD;
  const CoreBufs cb{cbp,          cbp + D2,     cbp + 2 * D2,  cbp + 3 * D2,  cbp + 4 * D2, cbp + 6 * D2,
                    cbp + 8 * D2, cbp + 9 * D2, cbp + 10 * D2, cbp + 11 * D2, cbp + 12 * D2};
  const size_t corey_smem = (2 * (size_t)s * s + 3 * (size_t)s * r + (size_t)r * r + 3 + kPivDoubles) * 8;
  const size_t corex_smem = (2 * (size_t)s * s + 2 * (size_t)s * r + (size_t)r * r) * 8;
  CNMF_TRY(ensure_smem_attr((const void*)row_sweep<32>, (int)sweep_smem<32>()));
  CNMF_TRY(ensure_smem_attr((const void*)row_sweep<64>, (int)sweep_smem<64>()));
  CNMF_TRY(ensure_smem_attr((const void*)core_y, (int)((6 * D2 + 3 + kPivDoubles) * 8)));
  CNMF_TRY(ensure_smem_attr((const void*)core_x, (int)(5 * D2 * 8)));
  cudaStream_t side;
  cudaEvent_t fork, join;
  CNMF_TRY(stream_side(&side, &fork, &join));
  const SSide sl{L, m, S, u, du, pu}, sr{Rt, n, S, vt, dvt, pv};
  // grid blocks, the first nl of them on the left rows, partials from part + off
  auto sweep = [&](int grid, int nl, size_t off, int update) -> int {
    if (S == 32)
      row_sweep<32><<<grid, kSW, sweep_smem<32>(), st>>>(sl, sr, nl, cb.Zl, cb.Zr, s, r, step, update, part + off, ctrl);
    else
      row_sweep<64><<<grid, kSW, sweep_smem<64>(), st>>>(sl, sr, nl, cb.Zl, cb.Zr, s, r, step, update, part + off, ctrl);
    CNMF_LAUNCH_CHECK();
    return CNMF_OK;
  };
  auto reduce = [&](int nl, int nr, int update) -> int {
    reduce_parts<<<dim3((unsigned)ceil_div(len, kRE), 2), kT, 0, st>>>(part, nl, nr, len, sums, ctrl, update);
    CNMF_LAUNCH_CHECK();
    return CNMF_OK;
  };
  int k0 = 0;
  if (!resume) {
    init_sctrl<<<1, 1, 0, st>>>(ctrl);
    CNMF_LAUNCH_CHECK();
    CNMF_TRY(panel_cross(L, L, m, S, cb.GL, st));
    CNMF_TRY(panel_cross(Rt, Rt, n, S, cb.GR, st));
    CNMF_CUDA(cudaMemsetAsync(du, 0, (size_t)m * r * 8, st));
    CNMF_CUDA(cudaMemsetAsync(dvt, 0, (size_t)n * r * 8, st));
    CNMF_TRY(sweep(total, nbl, 0, 0));  // L^T U and V R^T of the start
    CNMF_TRY(reduce(nbl, nbr, 0));
    core_y<<<1, kCT, corey_smem, st>>>(core, sums, xc, yc, cb, S, s, r, pu, pv, ctrl, 0, 1);
    CNMF_LAUNCH_CHECK();
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
    core_x<<<2, kCT, corex_smem, st>>>(core, sums, xc, yc, cb, s, r, pu, pv, step, tol, trace, scores, ctrl, k,
                                       max_iter, 1);
    CNMF_LAUNCH_CHECK();
    CNMF_CUDA(cudaEventRecord(fork, st));
    CNMF_CUDA(cudaStreamWaitEvent(side, fork, 0));
    core_y<<<1, kCT, corey_smem, side>>>(core, sums, xc, yc, cb, S, s, r, pu, pv, ctrl, k, 0);
    const cudaError_t ey = cudaGetLastError();
    CNMF_CUDA(cudaEventRecord(join, side));
    const int rl = ey == cudaSuccess ? sweep(gl, gl, 0, 1) : CNMF_OK;  // left rows: needs xc_k only
    CNMF_CUDA(cudaStreamWaitEvent(st, join, 0));                       // always join the side stream
    if (ey != cudaSuccess) return fail(CNMF_ERR_CUDA, std::string("core_y launch: ") + cudaGetErrorString(ey));
    CNMF_TRY(rl);
    CNMF_TRY(sweep(gr, 0, (size_t)gl * len, 1));  // right rows: yc_k
    CNMF_TRY(reduce(gl, gr, 1));
  }
  // score of the last swept iteration (and the stop decision)
  core_x<<<2, kCT, corex_smem, st>>>(core, sums, xc, yc, cb, s, r, pu, pv, step, tol, trace, scores, ctrl, k1, max_iter,
                                     0);
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
  reduce_parts<<<dim3((unsigned)ceil_div(len, kRE), 2), kT, 0, st>>>((double*)part, nbl, nbr, len, w.sums, w.ctrl,
                                                                    update);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

int admm_shard_core(void* ws, const double* core, double* xc, double* yc, int s, int r, double pu, double pv,
                    double step, double tol, double* trace, double* scores, int k, int max_iter, int first, int solve,
                    cudaStream_t st) {
  const ShardWs w = shard_ws(ws, s, r);
  const int S = s <= 32 ? 32 : 64;
  const size_t core_smem = (2 * (size_t)s * s + 3 * (size_t)s * r + (size_t)r * r + 3 + kPivDoubles) * 8;
  CNMF_TRY(ensure_smem_attr((const void*)core_step, (int)((6 * kMaxD * kMaxD + 3 + kPivDoubles) * 8)));
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
