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

constexpr int kSweepThreads = 256;
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
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      if (bi[q] < 0) continue;
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
  if (GROUPS > 1) {
    // fold the row groups in shared memory: one partial per block
    double* red = (double*)(sOut + kTR * S);  // GROUPS x NBLK x 16
    __syncthreads();
    if (bi[0] >= 0)
#pragma unroll
      for (int e = 0; e < 16; ++e) red[(grp * NBLK + bidx) * 16 + e] = g[0][e];
    __syncthreads();
    if (grp == 0 && bi[0] >= 0)
      for (int q = 1; q < GROUPS; ++q)
#pragma unroll
        for (int e = 0; e < 16; ++e) g[0][e] += red[(q * NBLK + bidx) * 16 + e];
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
  const int grp_id = b / kGroup, g0 = grp_id * kGroup, g1 = min(nb, g0 + kGroup);
  if (tid == 0) s_role = atomicAdd(set.gcount + which * 64 + grp_id, 1u) == (unsigned)(g1 - g0) - 1 ? 1 : 0;
  __syncthreads();
  if (s_role) {
    __threadfence();
    for (int e = tid; e < NE; e += kSweepThreads) {
      double acc = 0.0;
      for (int j = g0; j < g1; ++j) acc += __ldcg(set.part + (size_t)(b0 + j) * NE + e);
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
  const bool s_last = s_role == 2;
  if (s_last) {
    __threadfence();
    for (int e = tid; e < NE; e += kSweepThreads) {
      double acc = 0.0;
      for (int j = 0; j < ngroups; ++j) acc += __ldcg(gsum + (size_t)j * NE + e);
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
    chol_small(pp.G, pp.s, S, pp.T, pp.R, pp.info, pp.pass_id, reinterpret_cast<double*>(fsm));
    __threadfence();
    __syncthreads();
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
    for (int i = tid; i < kTR * S; i += kSweepThreads) {
      const int r = i / S, c = i % S;
      float acc = 0.f;
      for (int j = 0; j <= c; ++j) acc = fmaf(sIn[r * S + j], sT[j * S + c], acc);
      sOut[i] = acc;
    }
    __syncthreads();
    for (int i = tid; i < kTR * S / 4; i += kSweepThreads) {
      const int r = (i * 4) / S;
      if (r < nr) *(float4*)(P + t0 * S + 4 * (int64_t)i) = *(const float4*)(sOut + 4 * i);
    }
  }
  __syncthreads();
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
