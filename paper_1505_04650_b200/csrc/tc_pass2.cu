// Streaming passes over A on the 5th-generation tensor cores, version 2:
// 256-row units (two 128-row TMEM sub-tiles share one split of the panel
// tile) and one S-wide accumulator per sub-tile.
//
//   A X ~= A_hi X_hi + A_hi X_lo + A_lo X_hi   (3xTF32, v_hi = rn_tf32(v),
//                                              v_lo = v - v_hi exact; the
//                                              tensor core truncates v_lo)
//
// Forward pass  Y = A X   (M = rows of A, K = columns of A, N = S)
// Transpose     Z = A^T W (M = columns of A, K = rows of A, N = S)
//
// What changed against tc_pass.cu (measured there with ncu at configs[4]'s
// S = 64: ~3100 warp instructions and ~750 shared-memory wavefronts per
// 16 KB tile, issue 62 % busy, no single pipe saturated):
//   * a unit is 256 output rows x 32 k: the raw panel tile is TMA-loaded,
//     split into the K-major SW128 [hi; lo] B operand and read by the
//     tensor core for BOTH sub-tiles -- the panel load/split (8 + 8 + 16 KB
//     of shared-memory traffic per unit at S = 64) is amortised over 32 KB
//     of A instead of 16 KB;
//   * the three products of a sub-tile accumulate into one S-wide TMEM
//     accumulator (three N = S MMAs), so the epilogue drains S columns per
//     row instead of 2S and adds no hi/lo halves;
//   * the stage is released after the split arithmetic has consumed every
//     loaded value (register dependence), so the generic-proxy reads are
//     complete before the next TMA write without a proxy fence.
// Warp roles (one CTA per SM): warp 0 TMA producer, warp 1 MMA issuer (one
// elected thread), warps 2..9 splitters (lane quarter w & 3, K half of the
// tile, both sub-tiles; panel K chunk w - 2), warps 10.. epilogue (lane
// quarter, 32-column group; one row in each sub-tile per thread).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "pass.cuh"

namespace cnmf {
namespace {

constexpr int BMT = 128;  // rows per sub-tile (TMEM lanes)
constexpr int NSUB = 2;   // sub-tiles per unit: a unit is 256 output rows
constexpr int BKT = 32;   // K per stage (one 128B swizzle atom of fp32)
constexpr int NSPL = 8;   // splitter warps (2 per TMEM lane quarter; 8 panel K chunks)
#ifndef CNMF_PASS_KB
#define CNMF_PASS_KB 2
#endif
#ifdef CNMF_PASS_ACC64
using acc_t = double;
#else
using acc_t = float;
#endif
#ifndef CNMF_PASS_NACC
#define CNMF_PASS_NACC 2
#endif
#ifndef CNMF_PASS_AST64
#define CNMF_PASS_AST64 4
#endif

// mbarrier wait with a suspend-time hint: a waiting warp sleeps in the
// try_wait until the phase completes instead of re-polling (the epilogue and
// producer warps spend most of a pass waiting; their polling loops were 15 %
// of the issued instructions)
__device__ __forceinline__ void mbar_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.b32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(pred));
  return pred;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 8 consecutive fp32 columns per warp
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 16 / 32 consecutive fp32 columns per warp: one TMEM round trip
// for what eight x8 loads (each followed by its own wait) fetched
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 16 consecutive 32-bit columns per warp
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}

// SM100 shared-memory matrix descriptor, 128B swizzle.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// kind::tf32 instruction descriptor: D fp32, A/B tf32, K-major A and B, M = 128.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BMT >> 4) << 24);
}

// Round to the nearest tf32 value (10 explicit mantissa bits, ties away from
// zero). The tensor core truncates the low 13 bits of an fp32 operand, so
// both split halves are pre-rounded: hi = rn(v), lo = rn(v - hi) (v - hi is
// exact in fp32), which keeps the split error unbiased and <= 2^-22 |v| --
// truncating would bias every product of nonnegative data toward zero.
__device__ __forceinline__ float tf32_rn(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Slot index + phase parity of a ring of N mbarrier-guarded buffers.
template <int N>
struct Ring {
  int i = 0;
  uint32_t ph = 0;
  bool wrapped = false;  // every slot has been handed out at least once
  __device__ __forceinline__ void next() {
    if (++i == N) {
      i = 0;
      ph ^= 1;
      wrapped = true;
    }
  }
};


// Accumulator layout: 1 = one S-wide accumulator per sub-tile, fed per K
// tile with the small products (A_hi X_lo, A_lo X_hi over all k steps)
// first and the large ones (A_hi X_hi) on top; 2 = [A_hi X_hi | A_hi X_lo +
// A_lo X_hi] (2S columns, large and small accumulate apart). KB = K tiles
// the tensor core accumulates before the epilogue drains into fp32
// registers. Measured (tools/pass_accuracy.py at K = 16384, S = 64: rms
// error relative to |A||X|; projector distances to the reference basis,
// tests/test_gpu_fullsize.py, the reference's own band under one fp32
// rounding of A in brackets; 20000 x 100000 forward/transpose TB/s):
//   tc_pass.cu (128-row units, split, KB 2): rms 2.6e-9; c1 2000 x 1000
//     8.6e-5 [6.4e-5], c4 4000 x 2000 5.8e-5 [4.3e-5]; S=64 3.72/3.86
//   ACC 1 / KB 1 (default): rms 2.2e-9; c1 7.0e-5, c4 5.3e-5;
//     S=64 4.15/4.42, S=32 5.84/5.95
//   ACC 2 / KB 2: rms 2.6e-9; c1 1.24-1.29e-4, c4 6.2e-5; S=64 3.73 (two
//     2S-wide sub-tile accumulators fill half of TMEM: single-buffered)
//   ACC 1 / KB 2: rms 4.6e-9; c4 1.2e-4 (over the 1e-4 bound)
//   ACC 1 / KB 2 with the products interleaved per k step: rms 5.6e-9
#ifndef CNMF_PASS2_ACC32
#define CNMF_PASS2_ACC32 1
#endif
#ifndef CNMF_PASS2_ACC64
#define CNMF_PASS2_ACC64 1
#endif
#ifndef CNMF_PASS2_KB32
#define CNMF_PASS2_KB32 1
#endif
#ifndef CNMF_PASS2_KB64
#define CNMF_PASS2_KB64 1
#endif

// TMA load with an L2 eviction policy (createpolicy): A is streamed once per
// pass and must not push the panels out of L2 -- without the hint the
// panel rows were re-read from DRAM, 101 GB per 80 GB pass at configs[4]
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const void* tmap, uint64_t* bar, int c0, int c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

#ifndef REBAL_LOW
#define REBAL_LOW 64
#endif
#ifndef REBAL_SPL
#define REBAL_SPL 96
#endif
#ifndef REBAL_EPI
#define REBAL_EPI 112
#endif

template <int S>
struct TcCfg2 {
  static constexpr int ABYTES = NSUB * BMT * BKT * 4;  // 32 KB raw A (256 rows x 32 k)
  static constexpr int BRAW = BKT * S * 4;             // raw fp32 panel tile [32 k][S]
  static constexpr int STAGE = ABYTES + BRAW;
  static constexpr int BSPL = BKT * 2 * S * 4;         // split K-major SW128 panel slot [hi; lo]
  static constexpr int ACC = S == 64 ? CNMF_PASS2_ACC64 : CNMF_PASS2_ACC32;
  static constexpr int AW = ACC * S;                   // accumulator columns per sub-tile
  static constexpr int ACC_COLS = NSUB * AW;           // per accumulator buffer: sub-tile j at j AW
  static constexpr int NACC = (ACC_COLS * 2 + NSUB * 2 * BKT * 2 <= 512) ? 2 : 1;  // buffers (1: S = 64, split)
  static constexpr int ASLOT = NSUB * 2 * BKT;         // TMEM A ring slot: [sub-tile][hi | lo] x 32 k
  static constexpr int A_COL0 = NACC * ACC_COLS;
  static constexpr int AST = (512 - A_COL0) / ASLOT;   // TMEM A ring = split panel ring = MMA-done ring
  static constexpr int ST = (227 * 1024 - 1024 - AST * BSPL) / STAGE;
  static constexpr int KB = S == 64 ? CNMF_PASS2_KB64 : CNMF_PASS2_KB32;  // K tiles per tensor-core accumulation block
  static constexpr int NEPI = 4 * (S / 32);
  // warp roles: 0 TMA, 1 MMA, then NSPL splitters, then NEPI epilogue warps.
  // S = 64 (18 warps) would cap every thread at 96 registers (16K registers
  // per SM sub-partition, 5 warps each) and the epilogue's 64 running sums
  // spilled (10 % of the instructions were spill traffic, ncu); there the
  // roles are warpgroup-aligned instead -- warpgroup 0 = TMA, MMA and two
  // idle warps, 1-2 splitters, 3-4 epilogue -- and setmaxnreg moves
  // registers from warpgroup 0 to the epilogue.
  static constexpr bool REBAL = (S == 64);
  static constexpr int SPL0 = REBAL ? 4 : 2;
  static constexpr int EPI0 = SPL0 + NSPL;
  static constexpr int THREADS = 32 * (EPI0 + NEPI);
  static constexpr int REG_LOW = REBAL_LOW, REG_SPL = REBAL_SPL, REG_EPI = REBAL_EPI;  // after setmaxnreg (REBAL only)
  static_assert(!REBAL || REG_LOW + 2 * REG_SPL + 2 * REG_EPI <= 5 * 96, "register file per sub-partition");
  // registers: each SM sub-partition holds 16K of them for its ceil(warps / 4) warps
  static constexpr int MAXREG = (16384 / (((THREADS / 32) + 3) / 4 * 32)) & ~7;
  static constexpr size_t SMEM = (size_t)ST * STAGE + (size_t)AST * BSPL + 512;
  static_assert(AST >= 2, "TMEM A ring");
  static_assert(ST >= 3, "stage ring depth");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(A_COL0 + AST * ASLOT <= 512, "TMEM budget");
};

constexpr int kWarpTma = 0, kWarpMma = 1;

struct PassSide {
  float* out;
  int64_t P;        // output rows
  int64_t nblocks;  // 256-row output units
  int nt;           // K tiles per output unit
  int trans;
  double* sumsq;    // forward side only, may be null: += sum of A^2 over the side's tiles
};
// The (side, output tile, K tile) walk of one CTA's units: [lo0, hi0) of
// side 0, then [lo1, hi1) of side 1 (unit indices local to each side; plain
// scalars, no indexed arrays, so nothing lands in local memory).
template <bool SINGLE>
struct WalkT;

// two sides: side 0's units, then side 1's
template <>
struct WalkT<false> {
  int p;
  int ob, u;
  int kt;
  int lo0, hi0, lo1, hi1;
  __device__ __forceinline__ void start(int a0, int a1, int b0, int b1, const PassSide& s0,
                                        const PassSide& s1) {
    lo0 = a0;
    hi0 = a1;
    lo1 = b0;
    hi1 = b1;
    p = lo0 < hi0 ? 0 : 1;
    u = p ? lo1 : lo0;
    const int nt = p ? s1.nt : s0.nt;
    ob = u / nt;
    kt = (int)(u - ob * nt);
  }
  __device__ __forceinline__ bool last() const { return u == (p ? hi1 : hi0) - 1; }  // last unit in range
  __device__ __forceinline__ bool owned(int nt) const {                               // whole tile in range
    const int t0 = ob * nt;
    return t0 >= (p ? lo1 : lo0) && t0 + nt <= (p ? hi1 : hi0);
  }
  // units left in the current output tile within this CTA's range
  __device__ __forceinline__ int tile_left(int nt) const {
    const int r = (p ? hi1 : hi0) - u, t = nt - kt;
    return r < t ? r : t;
  }
  // advance by len units that stay inside the current tile (len <= tile_left)
  __device__ __forceinline__ void skip(int len, const PassSide& s0, const PassSide& s1) {
    u += len;
    kt += len;
    const int nt = p ? s1.nt : s0.nt;
    if (p == 0 && u == hi0) {
      p = 1;
      u = lo1;
      ob = u / s1.nt;
      kt = (int)(u - ob * s1.nt);
    } else if (kt == nt) {
      kt = 0;
      ++ob;
    }
  }
  __device__ __forceinline__ void next(const PassSide& s0, const PassSide& s1) {
    ++u;
    if (p == 0 && u == hi0) {
      p = 1;
      u = lo1;
      ob = u / s1.nt;
      kt = (int)(u - ob * s1.nt);
    } else if (++kt == (p ? s1.nt : s0.nt)) {
      kt = 0;
      ++ob;
    }
  }
};

// one side (the common launch): no side switch, so the walk state and every
// side-dependent operand fold to side 0 at compile time
template <>
struct WalkT<true> {
  static constexpr int p = 0;
  int ob, u, kt;
  int lo0, hi0;
  __device__ __forceinline__ void start(int a0, int a1, int, int, const PassSide& s0, const PassSide&) {
    lo0 = a0;
    hi0 = a1;
    u = lo0;
    ob = u / s0.nt;
    kt = u - ob * s0.nt;
  }
  __device__ __forceinline__ bool owned(int nt) const {
    const int t0 = ob * nt;
    return t0 >= lo0 && t0 + nt <= hi0;
  }
  __device__ __forceinline__ int tile_left(int nt) const {
    const int r = hi0 - u, t = nt - kt;
    return r < t ? r : t;
  }
  __device__ __forceinline__ void skip(int len, const PassSide& s0, const PassSide&) {
    u += len;
    kt += len;
    if (kt == s0.nt) {
      kt = 0;
      ++ob;
    }
  }
  __device__ __forceinline__ void next(const PassSide& s0, const PassSide&) {
    ++u;
    if (++kt == s0.nt) {
      kt = 0;
      ++ob;
    }
  }
};




template <int S>
constexpr int NEPI_OF() { return 4 * (S / 32); }

// Split-K tile (its units span the CTA boundaries bf .. bl): every
// contributor parks its partial in its own slot, the last to arrive sums
// the slots in CTA order and stores -- bit-reproducible, no zeroing of the
// output and no grid-wide wait. A CTA contributes to at most two split tiles
// (its first and its last), so the slots are [2 x grid]: slot 2c for CTA c's
// first tile, 2c + 1 for its last. Out of line: the hot epilogue loop keeps
// its registers. Unit indices fit 32 bits (checked by the launcher).
struct SplitTile {
  int bf, bl, tg;
};

__device__ __forceinline__ int splitk_slot(int c, int tg, int U0, int Ut, int nb0, int nt0, int nt1, int G) {
  const int v = (int)((unsigned)c * (unsigned)Ut / (unsigned)G);  // CTA c's first unit
  const int t = v < U0 ? v / nt0 : nb0 + (v - U0) / nt1;
  return 2 * c + (t == tg ? 0 : 1);
}

// this CTA's slot for the split tile (ob of side p); the partial is stored by
// the caller (inline: the running sums stay in registers)
__device__ __forceinline__ float* splitk_mine(SplitTile& st, int U0, int Ut, int nb0, int nt0, int nt1, int p, int ob,
                                              int nt, int G, int b, float* sk_slots, int tile_floats) {
  const int t_lo = (p ? U0 : 0) + ob * nt, t_hi = t_lo + nt - 1;
  st.bf = (int)(((unsigned)(t_lo + 1) * (unsigned)G - 1u) / (unsigned)Ut);
  st.bl = (int)(((unsigned)(t_hi + 1) * (unsigned)G - 1u) / (unsigned)Ut);
  st.tg = (p ? nb0 : 0) + ob;
  return sk_slots + (size_t)splitk_slot(b, st.tg, U0, Ut, nb0, nt0, nt1, G) * tile_floats;
}

template <int S, int NEPI>
__device__ __noinline__ void splitk_tile(SplitTile st, const PassSide& sd, int U0, int Ut, int nb0, int nt0, int nt1,
                                         int ob, int G, int row_in_sub, int cg, bool leader,
                                         float* __restrict__ sk_slots, unsigned* __restrict__ sk_cnt) {
  const int bf = st.bf, bl = st.bl, tg = st.tg;
  auto slot_of = [&](int c) { return splitk_slot(c, tg, U0, Ut, nb0, nt0, nt1, G); };
  __threadfence();
  asm volatile("bar.sync 2, %0;" ::"n"(NEPI * 32) : "memory");
  __shared__ int s_last;
  if (leader) {
    unsigned* cnt = sk_cnt + slot_of(bf);
    const unsigned old = atomicAdd(cnt, 1u);
    const int last = old == (unsigned)(bl - bf);
    if (last) *cnt = 0u;  // ready for the next launch
    __threadfence();
    s_last = last;
  }
  asm volatile("bar.sync 2, %0;" ::"n"(NEPI * 32) : "memory");
  if (!s_last) return;
#pragma unroll
  for (int j = 0; j < NSUB; ++j) {
    float tot[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) tot[c] = 0.f;
    // contributors in CTA order, two slots' loads in flight at a time
    const size_t off = (size_t)(j * BMT + row_in_sub) * S + cg;
    int k = bf;
    for (; k + 1 <= bl; k += 2) {
      const float* s0p = sk_slots + (size_t)slot_of(k) * (NSUB * BMT * S) + off;
      const float* s1p = sk_slots + (size_t)slot_of(k + 1) * (NSUB * BMT * S) + off;
      float4 va[8], vb[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        va[c] = __ldcg((const float4*)(s0p + 4 * c));
        vb[c] = __ldcg((const float4*)(s1p + 4 * c));
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        tot[4 * c] += va[c].x;
        tot[4 * c + 1] += va[c].y;
        tot[4 * c + 2] += va[c].z;
        tot[4 * c + 3] += va[c].w;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        tot[4 * c] += vb[c].x;
        tot[4 * c + 1] += vb[c].y;
        tot[4 * c + 2] += vb[c].z;
        tot[4 * c + 3] += vb[c].w;
      }
    }
    if (k <= bl) {
      const float* s0p = sk_slots + (size_t)slot_of(k) * (NSUB * BMT * S) + off;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 v = __ldcg((const float4*)(s0p + 4 * c));
        tot[4 * c] += v.x;
        tot[4 * c + 1] += v.y;
        tot[4 * c + 2] += v.z;
        tot[4 * c + 3] += v.w;
      }
    }
    const int64_t row = (int64_t)ob * (NSUB * BMT) + j * BMT + row_in_sub;
    if (row < sd.P) {
      float* dst = sd.out + row * S + cg;
#pragma unroll
      for (int c = 0; c < 32; c += 4) *(float4*)(dst + c) = make_float4(tot[c], tot[c + 1], tot[c + 2], tot[c + 3]);
    }
  }
}

// MODE 0: one forward side, 1: one transpose side, 2: two sides (paired),
// 3: one forward side that also sums A^2 (the residual pass)
template <int S, int MODE>
__global__ void __launch_bounds__(TcCfg2<S>::THREADS, 1)
    stream_pass2(const __grid_constant__ TmaDesc tA0, const __grid_constant__ TmaDesc tB0,
                 const __grid_constant__ TmaDesc tA1, const __grid_constant__ TmaDesc tB1, const PassSide s0,
                 const PassSide s1, int whole, float* __restrict__ sk_slots, unsigned* __restrict__ sk_cnt) {
  using C = TcCfg2<S>;
  constexpr bool SINGLE = MODE != 2;
  using Walk = WalkT<SINGLE>;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sP = smem + C::ST * C::STAGE;          // [AST][BSPL]
  uint64_t* full = (uint64_t*)(sP + C::AST * C::BSPL);  // [ST] stage landed
  uint64_t* empty = full + C::ST;                       // [ST] stage consumed by all splitters
  uint64_t* afull = empty + C::ST;                      // [AST] split A in TMEM + split panel in SMEM
  uint64_t* mdone = afull + C::AST;                     // [AST] MMAs of the slot's K tile retired
  uint64_t* tfull = mdone + C::AST;                     // [NACC] accumulator ready
  uint64_t* tempty = tfull + C::NACC;                   // [NACC] accumulator drained
  uint32_t* tmem_slot = (uint32_t*)(tempty + C::NACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t U0 = s0.nblocks * s0.nt, U1 = s1.nblocks * s1.nt, G = gridDim.x, b = blockIdx.x;
  int64_t u0, u1;
  if (whole) {
    const int64_t T = s0.nblocks + s1.nblocks;
    const int64_t t0 = b * T / G, t1 = (b + 1) * T / G;
    u0 = t0 <= s0.nblocks ? t0 * s0.nt : U0 + (t0 - s0.nblocks) * s1.nt;
    u1 = t1 <= s0.nblocks ? t1 * s0.nt : U0 + (t1 - s0.nblocks) * s1.nt;
  } else {
    u0 = b * (U0 + U1) / G;
    u1 = (b + 1) * (U0 + U1) / G;
  }
  const int64_t lo0 = u0 < U0 ? u0 : U0, hi0 = u1 < U0 ? u1 : U0;
  const int64_t lo1 = u0 > U0 ? u0 - U0 : 0, hi1 = u1 > U0 ? u1 - U0 : 0;
  const int64_t ntiles = (hi0 - lo0) + (hi1 - lo1);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tA0);
    prefetch_tmap(&tB0);
    if (U1 > 0) {
      prefetch_tmap(&tA1);
      prefetch_tmap(&tB1);
    }
    for (int s = 0; s < C::ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NSPL);
    }
    for (int s = 0; s < C::AST; ++s) {
      mbar_init(&afull[s], NSPL);
      mbar_init(&mdone[s], 1);
    }
    for (int i = 0; i < C::NACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], C::NEPI);
    }
    fence_barrier_init();
  }
  if (warp == kWarpMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if constexpr (C::REBAL) {
    if (warp < 4)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::REG_LOW));
    else if (warp >= C::EPI0)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::REG_EPI));
    else if (C::REG_SPL > 96)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::REG_SPL));
  }

  if (warp == kWarpTma) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      Ring<C::ST> r;
      Walk w;
      w.start((int)lo0, (int)hi0, (int)lo1, (int)hi1, s0, s1);
      const uint64_t pol_a = l2_policy_evict_first(), pol_p = l2_policy_evict_last();
      for (int64_t it = 0; it < ntiles; ++it) {
        if (it >= C::ST) mbar_sleep(&empty[r.i], r.ph ^ 1);
        unsigned char* dst = smem + r.i * C::STAGE;
        mbar_arrive_expect_tx(&full[r.i], C::STAGE);
        const PassSide& sd = w.p ? s1 : s0;
        const TmaDesc* ta = w.p ? &tA1 : &tA0;
        const TmaDesc* tb = w.p ? &tB1 : &tB0;
        const int row0 = (int)(w.ob * (NSUB * BMT));
        const bool trans = MODE == 1 || (MODE == 2 && sd.trans);
        if (!trans)  // A rows [row0, +256), cols [kt*32, +32): K-major SW128
          tma_load_2d_hint(dst, ta, &full[r.i], w.kt * BKT, row0, pol_a);
        else  // A rows [kt*32, +32) (K), cols [row0, +256) (M): row-major
          tma_load_2d_hint(dst, ta, &full[r.i], row0, w.kt * BKT, pol_a);
        tma_load_2d_hint(dst + C::ABYTES, tb, &full[r.i], 0, w.kt * BKT, pol_p);
        r.next();
        w.next(s0, s1);
      }
    }
  } else if (warp >= C::EPI0) {
    // ---------------- epilogue (one row per sub-tile x 32 columns per thread) ----------------
    const int q = warp & 3;
    const int cg = 32 * ((warp - C::EPI0) >> 2);
    const int row_in_sub = 32 * q + lane;
    Ring<C::NACC> racc;
    float acc[NSUB][32];
#pragma unroll
    for (int j = 0; j < NSUB; ++j)
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[j][c] = 0.f;
    Walk w;
    w.start((int)lo0, (int)hi0, (int)lo1, (int)hi1, s0, s1);
    for (int64_t it = 0; it < ntiles;) {
      const int nt = w.p ? s1.nt : s0.nt;
      const int64_t left = w.tile_left(nt);
      const int kb_left = C::KB - (w.kt % C::KB);
      const int len = (int)(left < kb_left ? left : kb_left);
      const bool tile_end = (len == left);
      mbar_sleep(&tfull[racc.i], racc.ph);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + racc.i * C::ACC_COLS + cg;
#ifndef CNMF_PASS2_LDW
#define CNMF_PASS2_LDW 8  // columns per TMEM drain load; 16 and 32 measured within +-3 % (tools/gpu_r02_ldw.sh): the drain is not the limiter
#endif
#pragma unroll
      for (int j = 0; j < NSUB; ++j) {
        if constexpr (C::ACC == 2 || CNMF_PASS2_LDW == 8) {
#pragma unroll
          for (int c0 = 0; c0 < 32; c0 += 8) {
            float v[8];
            tmem_ld8(taddr + j * C::AW + c0, v);
            if constexpr (C::ACC == 2) {
              float vl[8];
              tmem_ld8(taddr + j * C::AW + S + c0, vl);
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[j][c0 + e] += v[e] + vl[e];
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[j][c0 + e] += v[e];
            }
          }
        } else if constexpr (CNMF_PASS2_LDW == 16) {
#pragma unroll
          for (int c0 = 0; c0 < 32; c0 += 16) {
            float v[16];
            tmem_ld16(taddr + j * C::AW + c0, v);
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[j][c0 + e] += v[e];
          }
        } else {
          float v[32];
          tmem_ld32(taddr + j * C::AW, v);
#pragma unroll
          for (int e = 0; e < 32; ++e) acc[j][e] += v[e];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[racc.i]);
      racc.next();
      if (tile_end) {
        const PassSide& sd = w.p ? s1 : s0;
        if (w.owned(nt)) {
#pragma unroll
          for (int j = 0; j < NSUB; ++j) {
            const int64_t row = w.ob * (NSUB * BMT) + j * BMT + row_in_sub;
            if (row < sd.P) {
              float* dst = sd.out + row * S + cg;
#pragma unroll
              for (int c = 0; c < 32; c += 4)
                *(float4*)(dst + c) = make_float4(acc[j][c], acc[j][c + 1], acc[j][c + 2], acc[j][c + 3]);
            }
          }
        } else {
          SplitTile stile;
          float* mine = splitk_mine(stile, (int)U0, (int)(U0 + U1), (int)s0.nblocks, s0.nt, s1.nt, w.p, w.ob, nt,
                                    (int)G, (int)b, sk_slots, NSUB * BMT * S);
#pragma unroll
          for (int j = 0; j < NSUB; ++j) {
            float* dst = mine + (j * BMT + row_in_sub) * S + cg;
#pragma unroll
            for (int c = 0; c < 32; c += 4)
              __stcg((float4*)(dst + c), make_float4(acc[j][c], acc[j][c + 1], acc[j][c + 2], acc[j][c + 3]));
          }
          splitk_tile<S, NEPI_OF<S>()>(stile, sd, (int)U0, (int)(U0 + U1), (int)s0.nblocks, s0.nt, s1.nt, w.ob,
                                      (int)G, row_in_sub, cg, warp == C::EPI0 && lane == 0, sk_slots, sk_cnt);
        }
#pragma unroll
        for (int j = 0; j < NSUB; ++j)
#pragma unroll
          for (int c = 0; c < 32; ++c) acc[j][c] = 0.f;
      }
      w.skip(len, s0, s1);
      it += len;
    }
  } else if (warp == kWarpMma) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = idesc_tf32(S);
    constexpr uint32_t idesc_cat = idesc_tf32(2 * S);
    Ring<C::AST> ra;
    Ring<C::NACC> racc;
    Walk w;
    w.start((int)lo0, (int)hi0, (int)lo1, (int)hi1, s0, s1);
    bool block_start = true;
    for (int64_t it = 0; it < ntiles; ++it) {
      const int nt = w.p ? s1.nt : s0.nt;
      const bool tile_end = w.tile_left(nt) == 1;
      const bool block_end = tile_end || ((w.kt + 1) % C::KB == 0);
      if (block_start && racc.wrapped) mbar_sleep(&tempty[racc.i], racc.ph ^ 1);
      mbar_sleep(&afull[ra.i], ra.ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sb = smem_u32(sP + ra.i * C::BSPL);  // K-major SW128 [hi (S rows); lo (S rows)]
        const uint32_t aslot = tmem + C::A_COL0 + ra.i * C::ASLOT;
        const uint32_t d0 = tmem + racc.i * C::ACC_COLS;
#pragma unroll
#ifndef CNMF_VARIANT_NOMMA
        if constexpr (C::ACC == 2) {
#pragma unroll
          for (int k = 0; k < BKT / 8; ++k) {
            const uint64_t bhi = smem_desc(sb + 32 * k, 16, 1024);
            const uint32_t acc0 = (block_start && k == 0) ? 0u : 1u;
#pragma unroll
            for (int j = 0; j < NSUB; ++j) {
              const uint32_t ahi = aslot + j * 2 * BKT + 8 * k, alo = ahi + BKT, d = d0 + j * C::AW;
              tc_mma_ts(d, ahi, bhi, idesc_cat, acc0);  // [A_hi X_hi | A_hi X_lo]   (B rows [hi; lo])
              tc_mma_ts(d + S, alo, bhi, idesc, 1u);    //            + A_lo X_hi
            }
          }
        } else {
          // one S-wide accumulator: the block's small products (A_hi X_lo,
          // A_lo X_hi over all its k steps) accumulate first, from zero, and
          // the large ones (A_hi X_hi) are added on top -- the tensor core's
          // truncating fp32 accumulation then only rounds against the large
          // partial sums as often as the split layout does
#pragma unroll
          for (int k = 0; k < BKT / 8; ++k) {
            const uint64_t bhi = smem_desc(sb + 32 * k, 16, 1024);
            const uint64_t blo = smem_desc(sb + S * 128 + 32 * k, 16, 1024);
            const uint32_t acc0 = (block_start && k == 0) ? 0u : 1u;
#pragma unroll
            for (int j = 0; j < NSUB; ++j) {
              const uint32_t ahi = aslot + j * 2 * BKT + 8 * k, alo = ahi + BKT, d = d0 + j * C::AW;
              tc_mma_ts(d, ahi, blo, idesc, acc0);  // A_hi X_lo
#ifndef CNMF_VARIANT_2PROD  // (timing probe: two of the three products)
              tc_mma_ts(d, alo, bhi, idesc, 1u);    // + A_lo X_hi
#endif
            }
          }
#pragma unroll
          for (int k = 0; k < BKT / 8; ++k) {
            const uint64_t bhi = smem_desc(sb + 32 * k, 16, 1024);
#pragma unroll
            for (int j = 0; j < NSUB; ++j) {
              const uint32_t ahi = aslot + j * 2 * BKT + 8 * k, d = d0 + j * C::AW;
              tc_mma_ts(d, ahi, bhi, idesc, 1u);  // + A_hi X_hi
            }
          }
        }
#endif
        tc_commit(&mdone[ra.i]);  // releases the TMEM A slot and the split panel slot
        if (block_end) tc_commit(&tfull[racc.i]);
      }
      __syncwarp();
      ra.next();
      block_start = block_end;
      if (block_end) racc.next();
      w.next(s0, s1);
    }
  } else if (warp >= C::SPL0) {
    // ---------------- splitters ----------------
    const int q = warp & 3;                      // TMEM lane quarter
    const int half = (warp - C::SPL0) >> 2;  // K half of the A tile
    const int pc = warp - C::SPL0;           // 16-byte K chunk of the panel tile
    const int row_in_sub = 32 * q + lane;
    double sq_acc = 0.0;
    constexpr int PT = S / 32;
    Ring<C::ST> r;
    Ring<C::AST> ra;
    Walk w;
    w.start((int)lo0, (int)hi0, (int)lo1, (int)hi1, s0, s1);
    for (int64_t it = 0; it < ntiles; ++it) {
      mbar_sleep(&full[r.i], r.ph);
      if (ra.wrapped) mbar_sleep(&mdone[ra.i], ra.ph ^ 1);  // the TMEM slot's previous K tile retired
      tc_fence_after();
      const unsigned char* stage = smem + r.i * C::STAGE;
      const bool trans = MODE == 1 || (MODE == 2 && (w.p ? s1.trans : s0.trans));
      constexpr bool sq = MODE == 3;
      // panel K chunk pc: rows k = 4 pc + jj, columns n = lane + 32 t
      {
        float ph[PT][4], pl[PT][4];
        const float* raw = (const float*)(stage + C::ABYTES);
#pragma unroll
        for (int t = 0; t < PT; ++t)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const float v = raw[(4 * pc + jj) * S + lane + 32 * t];
            ph[t][jj] = tf32_rn(v);
            pl[t][jj] = v - ph[t][jj];
          }
        unsigned char* dst = sP + ra.i * C::BSPL;  // the slot is free (mdone above)
#pragma unroll
        for (int t = 0; t < PT; ++t) {
          const int n = lane + 32 * t;
          const uint32_t off = (uint32_t)n * 128 + ((pc ^ (n & 7)) << 4);
          *(float4*)(dst + off) = make_float4(ph[t][0], ph[t][1], ph[t][2], ph[t][3]);
          *(float4*)(dst + S * 128 + off) = make_float4(pl[t][0], pl[t][1], pl[t][2], pl[t][3]);
        }
      }
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + C::A_COL0 + ra.i * C::ASLOT + 16 * half;
      // A: sub-tile by sub-tile (load, split, store to TMEM); every loaded
      // value is consumed before the stage is handed back to the producer
#pragma unroll
      for (int j = 0; j < NSUB; ++j) {
        const int row = j * BMT + row_in_sub;  // row of the 256-row unit
        float hv[16], lv[16];
        if (!trans) {
          const unsigned char* rowp = stage + row * 128;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int c = 4 * half + cc;
            const float4 v = *(const float4*)(rowp + ((c ^ (row & 7)) << 4));
            hv[4 * cc + 0] = v.x;
            hv[4 * cc + 1] = v.y;
            hv[4 * cc + 2] = v.z;
            hv[4 * cc + 3] = v.w;
          }
        } else {
          const float* raw = (const float*)stage + row;
#pragma unroll
          for (int k = 0; k < 16; ++k) hv[k] = raw[(16 * half + k) * (NSUB * BMT)];
        }
        if constexpr (sq) {
          float q2 = 0.f;
#pragma unroll
          for (int k = 0; k < 16; ++k) q2 = fmaf(hv[k], hv[k], q2);
          sq_acc += (double)q2;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float v = hv[k];
          hv[k] = tf32_rn(v);
          lv[k] = v - hv[k];
        }
        tmem_st16(ta + j * 2 * BKT, hv);
        tmem_st16(ta + j * 2 * BKT + BKT, lv);
      }
      // every value loaded from the stage has now been consumed by an
      // instruction that cannot issue before its load returned (the panel
      // STS above, the A tcgen05.st): only then is the stage handed back to
      // the TMA producer. (Releasing it while the panel split could still be
      // scheduled after the arrive let the next TMA overwrite panel rows in
      // flight: ~2 % wrong tiles in 34 of 200 launches, tools/stress_splitk.py.)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[r.i]);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_proxy_async();  // generic-proxy smem stores -> tensor-core (async proxy) reads
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ra.i]);
      r.next();
      ra.next();
      w.next(s0, s1);
    }
    if (MODE == 3) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq_acc += __shfl_xor_sync(0xffffffffu, sq_acc, o);
      if (lane == 0) atomicAdd(s0.sumsq, sq_acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kWarpMma) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

constexpr int kSplitKCtas = 256;  // >= the SM count of the device (148 on B200)

struct SideArgs {
  const float* panel;
  float* out;
  int trans;
  double* sumsq = nullptr;
};

template <int S>
int launch_stream2(const float* A, int64_t m, int64_t n, int64_t lda, const SideArgs* sa, int nsides, cudaStream_t st) {
  using C = TcCfg2<S>;
  TmaDesc tA[2], tB[2];
  PassSide sd[2] = {{nullptr, 0, 0, 1, 0, nullptr}, {nullptr, 0, 0, 1, 0, nullptr}};
  for (int i = 0; i < nsides; ++i) {
    const int64_t K = sa[i].trans ? m : n;
    const int64_t P = sa[i].trans ? n : m;
    if (!sa[i].trans)
      CNMF_TRY(make_tma_2d(&tA[i], A, 4, m, n, lda, BKT, NSUB * BMT, true));
    else
      CNMF_TRY(make_tma_2d(&tA[i], A, 4, m, n, lda, NSUB * BMT, BKT, false));
    CNMF_TRY(make_tma_2d(&tB[i], sa[i].panel, 4, K, S, S, S, BKT, false));
    sd[i] = PassSide{sa[i].out, P, ceil_div(P, NSUB * BMT), (int)ceil_div(K, BKT), sa[i].trans,
                     sa[i].trans ? nullptr : sa[i].sumsq};
  }
  if (nsides == 1) {
    tA[1] = tA[0];
    tB[1] = tB[0];
  }
  const int64_t U = sd[0].nblocks * sd[0].nt + sd[1].nblocks * sd[1].nt;
  const int64_t T = sd[0].nblocks + sd[1].nblocks;
  const int mode = nsides == 2 ? 2 : sa[0].trans ? 1 : sa[0].sumsq ? 3 : 0;
  auto kern = mode == 0 ? stream_pass2<S, 0> : mode == 1 ? stream_pass2<S, 1> : mode == 2 ? stream_pass2<S, 2> : stream_pass2<S, 3>;
  CNMF_TRY(ensure_smem_attr((const void*)kern, (int)C::SMEM));
  static thread_local int occ_cache[64] = {};
  int dev = 0;
  CNMF_CUDA(cudaGetDevice(&dev));
  int& occ = occ_cache[dev & 63];
  if (occ == 0) {
    CNMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM));
    if (occ < 1) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kern);
      return fail(CNMF_ERR_CUDA, "streaming pass kernel does not fit on an SM: regs " + std::to_string(fa.numRegs) +
                                     " max threads " + std::to_string(fa.maxThreadsPerBlock) + " static smem " +
                                     std::to_string(fa.sharedSizeBytes) + " max dyn smem " +
                                     std::to_string(fa.maxDynamicSharedSizeBytes) + " threads " +
                                     std::to_string(C::THREADS) + " smem " + std::to_string(C::SMEM));
    }
  }
  const int64_t slots = (int64_t)device_sms() * occ;
  const int whole = (nsides == 1 && T >= 16 * slots) ? 1 : 0;
  const int64_t grid = std::min<int64_t>(slots, whole ? T : U);
  // split-K slots and arrival counters (fixed size: two slots per CTA; the
  // counters return to zero after every launch). One set per device, shared
  // by the launches of a stream; launches on concurrent streams would need
  // their own set (not done: the library enqueues passes on one stream).
  float* sk_slots = nullptr;
  unsigned* sk_cnt = nullptr;
  if (!whole) {
    const size_t slots = 2 * (size_t)kSplitKCtas;
    if (grid > kSplitKCtas) return fail(CNMF_ERR_CUDA, "split-K slots: grid larger than the device's SM count");
    if ((double)U * (double)grid >= 2147483647.0) return fail(CNMF_ERR_ARGUMENT, "split-K pass: too many units");
    void* p = nullptr;
    CNMF_TRY(device_scratch("pass2-splitk", slots * (NSUB * BMT * 64 * 4) + slots * 4, &p, st));
    sk_slots = (float*)p;
    sk_cnt = (unsigned*)(sk_slots + slots * (NSUB * BMT * 64));
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (pass_profiling()) {
    CNMF_CUDA(cudaEventCreate(&e0));
    CNMF_CUDA(cudaEventCreate(&e1));
    CNMF_CUDA(cudaEventRecord(e0, st));
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)grid);
  lc.blockDim = dim3(C::THREADS);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  CNMF_CUDA(cudaLaunchKernelEx(&lc, kern, tA[0], tB[0], tA[1], tB[1], sd[0], sd[1], whole, sk_slots, sk_cnt));
  CNMF_LAUNCH_CHECK();
  if (e0) {
    CNMF_CUDA(cudaEventRecord(e1, st));
    pass_record(e0, e1, nsides * 4.0 * ((double)m * n + (double)n * S + (double)m * S));
  }
  return CNMF_OK;
}

int launch_any2(const float* A, int64_t m, int64_t n, int64_t lda, const SideArgs* sa, int nsides, int S,
                cudaStream_t st) {
  switch (S) {
    case 32: return launch_stream2<32>(A, m, n, lda, sa, nsides, st);
    case 64: return launch_stream2<64>(A, m, n, lda, sa, nsides, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "tensor-core pass supports panel widths 32 and 64");
}

}  // namespace

int pass_forward_tc2(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y,
                     cudaStream_t st) {
  const SideArgs sa{X, Y, 0};
  return launch_any2(A, m, n, lda, &sa, 1, S, st);
}

int pass_forward_sumsq_tc2(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y,
                           double* sumsq, cudaStream_t st) {
  SideArgs sa{X, Y, 0};
  sa.sumsq = sumsq;
  return launch_any2(A, m, n, lda, &sa, 1, S, st);
}

int pass_transpose_tc2(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, int S, float* Z,
                       cudaStream_t st) {
  const SideArgs sa{W, Z, 1};
  return launch_any2(A, m, n, lda, &sa, 1, S, st);
}

int pass_pair_tc2(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, const float* W,
                  float* Z, int S, cudaStream_t st) {
  const SideArgs sa[2] = {{X, Y, 0}, {W, Z, 1}};
  return launch_any2(A, m, n, lda, sa, 2, S, st);
}

}  // namespace cnmf
