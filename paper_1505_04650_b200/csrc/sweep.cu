// CholeskyQR sweeps over one or two tall-skinny panels per cooperative launch.
//
// Reference: compress.py:136-145 canonical_qr (the Q factor with diag(R) > 0)
// applied after every pass of structured_compress (compress.py:186-198) and
// structured_compress_rows (compress.py:202-227); tsqr.py:65-135.
//
// One sweep: every block accumulates the fp64 Gram matrix of its 64-row
// tiles (fp32 products are exact in fp64) and stores the partial; partials
// are summed in a fixed order (groups of 16 blocks, then the group sums, each
// by the group's last-arriving block), so G is bit-reproducible for a given
// panel; the block completing the last group factors
// G = R^T R (chol.cuh) into T = R^{-1}; the panel's blocks wait for T
// (cooperative launch: all blocks are resident) and apply it to the tiles
// they still hold in shared memory.
// The two range finders of the compressed NMF sweep their panels in the same
// launch, so their Gram passes, factorisations and applies overlap and a
// power step costs one sweep instead of two.
#include <algorithm>

#include "chol.cuh"
#include "sweep.cuh"

namespace cnmf {
namespace {

#ifndef SWEEP_X
#define SWEEP_X 0  // probe-only variants (tools/sweep_probe.cu); 0 in the library
#endif
constexpr int kSweepThreads = 256;
#ifdef SWEEP_TRACE
__device__ unsigned long long g_sw_t[512][12];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SWT(k) do { if (threadIdx.x == 0) g_sw_t[blockIdx.x][k] = gtime(); } while (0)
#else
#define SWT(k) do {} while (0)
#endif
constexpr int kTR = 64;  // panel rows per tile

constexpr int kGroup = 16;  // blocks per first-level Gram reduction group

struct SweepSet {
  SweepPanel p[2];
  int np;
  double* part;      // [grid][NBLK * 16] per-block Gram partials, then [2][groups][NBLK * 16] group sums
  unsigned* gcount;  // [2][64] group arrival counters (zero between launches)
};

template <int S>
constexpr size_t sweep_smem() {
  constexpr int NB = S / 4, NBLK = NB * (NB + 1) / 2;
  constexpr int GROUPS = (NBLK >= kSweepThreads) ? 1 : kSweepThreads / NBLK;
  constexpr size_t fin = (size_t)(S * S + 2 * kTR * S) * 4 + (GROUPS > 1 ? (size_t)GROUPS * NBLK * 16 * 8 : 0);
  constexpr size_t chol = ((size_t)S * S + 2 * (size_t)S + 32 * 33 + 128) * 8;
  return fin > chol ? fin : chol;
}

template <int S>
__global__ void __launch_bounds__(kSweepThreads, 2) sweep_kernel(const __grid_constant__ SweepSet set) {
  constexpr int NB = S / 4;                  // 4-wide blocks per side
  constexpr int NBLK = NB * (NB + 1) / 2;    // upper-triangular 4x4 blocks
  constexpr int BPT = (NBLK + kSweepThreads - 1) / kSweepThreads;
  constexpr int GROUPS = (NBLK >= kSweepThreads) ? 1 : kSweepThreads / NBLK;  // row groups
  extern __shared__ __align__(16) float fsm[];
  float* sT = fsm;               // S x S
  float* sIn = sT + S * S;       // kTR x S
  float* sOut = sIn + kTR * S;   // kTR x S
  const int tid = threadIdx.x;
  const int which = (set.np > 1 && (int)blockIdx.x >= set.p[0].blocks) ? 1 : 0;
  const SweepPanel pp = set.p[which];
  const int b = (int)blockIdx.x - (which ? set.p[0].blocks : 0), nb = pp.blocks;
  float* __restrict__ P = pp.P;
  const int64_t rows = pp.rows;
  SWT(0);

  // ---- Gram: thread (grp, bidx) accumulates 4x4 block(s) over row group grp
  const int grp = tid / (GROUPS > 1 ? NBLK : kSweepThreads);
  const int bidx = tid - grp * (GROUPS > 1 ? NBLK : kSweepThreads);
  int bi[BPT], bj[BPT];
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    int k = bidx + q * kSweepThreads;
    bi[q] = -1;
    bj[q] = -1;
    if (k < NBLK && grp < GROUPS) {
      int i = 0;
      while (k >= NB - i) {
        k -= NB - i;
        ++i;
      }
      bi[q] = i;
      bj[q] = i + k;
    }
  }
  double g[BPT][16];
#pragma unroll
  for (int q = 0; q < BPT; ++q)
#pragma unroll
    for (int e = 0; e < 16; ++e) g[q][e] = 0.0;
  for (int64_t t0 = (int64_t)b * kTR; t0 < rows; t0 += (int64_t)nb * kTR) {
    __syncthreads();
    const int nr = (int)min64(kTR, rows - t0);
    for (int i = tid; i < kTR * S / 4; i += kSweepThreads) {
      const int r = (i * 4) / S;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nr) v = __ldcg((const float4*)(P + t0 * S) + i);
      *(float4*)(sIn + 4 * i) = v;
    }
    __syncthreads();
    SWT(8);
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      if (bi[q] < 0 || SWEEP_X == 3) continue;
      for (int r = grp; r < nr; r += GROUPS) {
        const float4 x = *(const float4*)(sIn + r * S + 4 * bi[q]);
        const float4 y = *(const float4*)(sIn + r * S + 4 * bj[q]);
        const double xs[4] = {x.x, x.y, x.z, x.w};
        const double ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) g[q][a * 4 + c] = fma(xs[a], ys[c], g[q][a * 4 + c]);
      }
    }
  }
  SWT(9);
  if (GROUPS > 1) {
    // fold the row groups in shared memory: one partial per block
    // entry-major [16][GROUPS][NBLK]: a warp's 32 threads touch consecutive
    // doubles (a block-major layout put all 32 on one bank: 32-way conflicts)
    double* red = (double*)(sOut + kTR * S);
    __syncthreads();
    if (bi[0] >= 0)
#pragma unroll
      for (int e = 0; e < 16; ++e) red[(e * GROUPS + grp) * NBLK + bidx] = g[0][e];
    __syncthreads();
    if (grp == 0 && bi[0] >= 0)
      for (int q = 1; q < GROUPS; ++q)
#pragma unroll
        for (int e = 0; e < 16; ++e) g[0][e] += red[(e * GROUPS + q) * NBLK + bidx];
  }
  SWT(1);
  if (SWEEP_X == 5) {  // probe: Gram only
    if (tid == 0 && g[0][0] == 12345.0) pp.G[0] = 1.0;
    return;
  }
  // ---- deterministic reduction of the block partials (fixed order, no
  // floating-point atomics): groups of kGroup blocks, then the group sums;
  // the block completing the last group factors G and publishes T
  constexpr int NE = NBLK * 16;
  const int nblk_total = set.p[0].blocks + (set.np > 1 ? set.p[1].blocks : 0);
  const int b0 = which ? set.p[0].blocks : 0;  // first block of this panel
  const int ngroups = (nb + kGroup - 1) / kGroup;
  double* gsum = set.part + (size_t)nblk_total * NE + (size_t)which * 64 * NE;
  if (grp == 0) {
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      if (bi[q] < 0) continue;
      double* dst = set.part + (size_t)blockIdx.x * NE + (size_t)(bidx + q * kSweepThreads) * 16;
#pragma unroll
      for (int e = 0; e < 16; ++e) __stcg(dst + e, g[q][e]);
    }
  }
  __shared__ int s_role;  // 0: done, 1: group reducer, 2: group reducer that also factors
  __threadfence();
  __syncthreads();
  SWT(2);
  const int grp_id = b / kGroup, g0 = grp_id * kGroup, g1 = min(nb, g0 + kGroup);
  if (tid == 0) s_role = atomicAdd(set.gcount + which * 64 + grp_id, 1u) == (unsigned)(g1 - g0) - 1 ? 1 : 0;
  __syncthreads();
  if (s_role) {
    __threadfence();
    // the group's partials are loaded together (independent L2 reads), then
    // added in block order: a load-add loop would serialise 16 L2 round trips
    for (int e = tid; e < NE; e += kSweepThreads) {
      double v[kGroup];
#pragma unroll
      for (int j = 0; j < kGroup; ++j) v[j] = (g0 + j < g1) ? __ldcg(set.part + (size_t)(b0 + g0 + j) * NE + e) : 0.0;
      double acc = v[0];
#pragma unroll
      for (int j = 1; j < kGroup; ++j) acc += v[j];
      __stcg(gsum + (size_t)grp_id * NE + e, acc);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      set.gcount[which * 64 + grp_id] = 0u;
      if (atomicAdd(pp.counter, 1u) == (unsigned)ngroups - 1) s_role = 2;
    }
    __syncthreads();
  }
  SWT(3);
  const bool s_last = s_role == 2;
  if (s_last) {
    __threadfence();
    for (int e = tid; e < NE; e += kSweepThreads) {
      double acc = 0.0;
      for (int j0 = 0; j0 < ngroups; j0 += 8) {  // 8 independent loads, then in-order adds
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = (j0 + j < ngroups) ? __ldcg(gsum + (size_t)(j0 + j) * NE + e) : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += v[j];
      }
      int k = e >> 4, i = 0;  // 4x4 block k -> (bi, bj)
      while (k >= NB - i) {
        k -= NB - i;
        ++i;
      }
      const int ia = 4 * i + ((e >> 2) & 3), jb = 4 * (i + k) + (e & 3);
      if (ia <= jb) pp.G[ia * S + jb] = acc;
    }
    __threadfence();
    __syncthreads();
    SWT(4);
#if SWEEP_X == 1  // probe: no factorisation (T = I)
    for (int i = tid; i < S * S; i += kSweepThreads) pp.T[i] = (i / S == i % S) ? 1.0 : 0.0;
#else
    chol_small(pp.G, pp.s, S, pp.T, pp.R, pp.info, pp.pass_id, reinterpret_cast<double*>(fsm));
#endif
    __threadfence();
    __syncthreads();
    SWT(5);
    if (tid == 0) atomicExch(pp.counter + 1, 1u);  // R^{-1} published
  } else {
    if (tid == 0) {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(pp.counter + 1) : "memory");
      } while (v == 0u);
    }
    __syncthreads();
  }

  SWT(6);
  if (SWEEP_X == 2) return;  // probe: no apply (counters left dirty; timing only)
  // ---- P <- P R^{-1}: a block that owned a single tile still holds it in sIn
  for (int i = tid; i < S * S; i += kSweepThreads) sT[i] = (float)__ldcg(pp.T + i);
  const bool kept = !s_last && (int64_t)nb * kTR >= rows;
  for (int64_t t0 = (int64_t)b * kTR; t0 < rows; t0 += (int64_t)nb * kTR) {
    const int nr = (int)min64(kTR, rows - t0);
    if (!kept) {
      __syncthreads();
      for (int i = tid; i < kTR * S / 4; i += kSweepThreads) {
        const int r = (i * 4) / S;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < nr) v = __ldcg((const float4*)(P + t0 * S) + i);
        *(float4*)(sIn + 4 * i) = v;
      }
    }
    __syncthreads();
    if constexpr (S <= 64) {
      // thread = one row x CPT consecutive columns: the row in registers, T
      // rows read as float4 (T is upper triangular, so the j > c terms add
      // exact zeros: the same sums, in the same order, as a j <= c loop)
      constexpr int CPT = kTR * S / kSweepThreads, TPR = S / CPT;
      const int r = tid / TPR, c0 = (tid % TPR) * CPT;
      float rowv[S], acc[CPT];
#pragma unroll
      for (int k = 0; k < S / 4; ++k) {
        const float4 v = *(const float4*)(sIn + r * S + 4 * k);
        rowv[4 * k] = v.x;
        rowv[4 * k + 1] = v.y;
        rowv[4 * k + 2] = v.z;
        rowv[4 * k + 3] = v.w;
      }
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) acc[cc] = 0.f;
#pragma unroll
      for (int j = 0; j < S; ++j) {
#pragma unroll
        for (int cc = 0; cc < CPT; cc += 4) {
          const float4 t4 = *(const float4*)(sT + j * S + c0 + cc);
          acc[cc] = fmaf(rowv[j], t4.x, acc[cc]);
          acc[cc + 1] = fmaf(rowv[j], t4.y, acc[cc + 1]);
          acc[cc + 2] = fmaf(rowv[j], t4.z, acc[cc + 2]);
          acc[cc + 3] = fmaf(rowv[j], t4.w, acc[cc + 3]);
        }
      }
#pragma unroll
      for (int cc = 0; cc < CPT; cc += 4)
        *(float4*)(sOut + r * S + c0 + cc) = make_float4(acc[cc], acc[cc + 1], acc[cc + 2], acc[cc + 3]);
    } else {
      for (int i = tid; i < kTR * S; i += kSweepThreads) {
        const int r = i / S, c = i % S;
        float acc = 0.f;
        for (int j = 0; j <= c; ++j) acc = fmaf(sIn[r * S + j], sT[j * S + c], acc);
        sOut[i] = acc;
      }
    }
    __syncthreads();
    for (int i = tid; i < kTR * S / 4; i += kSweepThreads) {
      const int r = (i * 4) / S;
      if (r < nr) *(float4*)(P + t0 * S + 4 * (int64_t)i) = *(const float4*)(sOut + 4 * i);
    }
  }
  __syncthreads();
  SWT(7);
  if (tid == 0 && atomicAdd(pp.counter + 2, 1u) == (unsigned)nb - 1) {
    pp.counter[0] = 0u;
    pp.counter[1] = 0u;
    pp.counter[2] = 0u;
  }
}

template <int S>
int launch_sweep(SweepPanel* panels, int np, cudaStream_t st) {
  constexpr size_t smem = sweep_smem<S>();
  constexpr int NB = S / 4, NE = NB * (NB + 1) / 2 * 16;
  static int per_sm = 0;
  // partial-sum scratch (sized for a full wave; one buffer: sweeps on a
  // stream run in order) and the group counters
  static double* part = nullptr;
  static unsigned* gcount = nullptr;
  if (per_sm == 0) {
    CNMF_CUDA(cudaFuncSetAttribute(sweep_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CNMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<S>, kSweepThreads, smem));
    per_sm = std::max(per_sm, 1);
    cudaStreamCaptureStatus cs;
    CNMF_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return fail(CNMF_ERR_CUDA, "sweep scratch must be allocated by an eager call before graph capture");
    CNMF_CUDA(cudaMalloc(&part, ((size_t)per_sm * kNumSMs + 2 * 64) * NE * sizeof(double)));
    CNMF_CUDA(cudaMalloc(&gcount, 2 * 64 * sizeof(unsigned)));
    CNMF_CUDA(cudaMemset(gcount, 0, 2 * 64 * sizeof(unsigned)));
  }
  // one wave (cooperative): blocks split between the panels by row count,
  // at most one per 64-row tile
  const int64_t cap = (int64_t)per_sm * kNumSMs;
  int64_t tiles[2] = {0, 0}, total = 0;
  for (int i = 0; i < np; ++i) {
    tiles[i] = std::max<int64_t>(1, ceil_div(panels[i].rows, kTR));
    total += tiles[i];
  }
  SweepSet set{};
  set.np = np;
  set.part = part;
  set.gcount = gcount;
  int64_t used = 0;
  for (int i = 0; i < np; ++i) {
    int64_t want = total <= cap ? tiles[i] : std::max<int64_t>(1, tiles[i] * cap / total);
    if (i == np - 1) want = std::min<int64_t>(want, cap - used);
    set.p[i] = panels[i];
    set.p[i].blocks = (int)std::max<int64_t>(1, want);
    used += set.p[i].blocks;
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)used);
  lc.blockDim = dim3(kSweepThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  CNMF_CUDA(cudaLaunchKernelEx(&lc, sweep_kernel<S>, set));
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

}  // namespace

int panel_sweep(SweepPanel* panels, int np, int S, cudaStream_t st) {
  if (np < 1 || np > 2) return fail(CNMF_ERR_ARGUMENT, "panel_sweep: one or two panels");
  switch (S) {
    case 32: return launch_sweep<32>(panels, np, st);
    case 64: return launch_sweep<64>(panels, np, st);
    case 128: return launch_sweep<128>(panels, np, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "panel width must be 32, 64 or 128");
}

}  // namespace cnmf
