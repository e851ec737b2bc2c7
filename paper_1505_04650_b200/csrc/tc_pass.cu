// Streaming passes over A on the 5th-generation tensor cores (tcgen05,
// kind::tf32) with a 3xTF32 split for fp32-level accuracy:
//
//   A X ~= A_hi X_hi + A_hi X_lo + A_lo X_hi,   v_hi = rn_tf32(v),
//                                               v_lo = v - v_hi (exact; the
//                                               tensor core truncates it).
//
// Forward pass  Y = A X   (M = rows of A, K = columns of A, N = S)
// Transpose     Z = A^T W (M = columns of A, K = rows of A, N = S)
//
// ONE kernel serves a single pass and the paired launch of a power step
// (Y = A X and Z = A^T W together): a launch walks up to two "sides", each a
// (direction, panel, output) triple, over one concatenated unit sequence.
// One CTA per SM, warp-specialised (10 + S/8 warps):
//   warp 0      TMA producer: per K tile one stage = raw fp32 A tile (16 KB:
//               128 output rows x 32 k, K-major SW128 for a forward side,
//               row-major [32 k][128] for a transpose side) + the raw fp32
//               panel rows [32 k][S];
//   warps 2..9  splitters: warp w owns TMEM lane quarter w & 3 (32 output
//               rows) and K half (w - 2) / 4 of the A tile -- it reads its
//               rows from the stage, splits hi/lo and stores both into a TMEM
//               ring (tcgen05.st) -- and 16-byte K chunk w - 2 of the panel
//               tile, which it splits into the K-major SW128 [hi; lo] B
//               operand in a shared-memory ring with the same slot index
//               (kind::tf32 accepts only K-major shared-memory operands on
//               sm_100a; measured). The panel split used to run on two
//               dedicated warps; at S = 64 those two SMSPs were the
//               bottleneck (2048 panel values per 16 KB tile).
//   warp 1      MMA issuer (one elected thread), A from TMEM, panel from SMEM:
//                 D[:, 0:2S]  = A_hi [X_hi | X_lo]      (N = 2S)
//                 D[:, S:2S] += A_lo X_hi               (N = S)
//               so D = [A_hi X_hi | A_hi X_lo + A_lo X_hi]; one
//               tcgen05.commit per K tile releases the TMEM A slot and the
//               panel slot together.
//   warps 10..  epilogue: the tensor core accumulates at most KB = 2 K tiles
//               into a double-buffered TMEM accumulator, the partial sums
//               move to fp32 registers (round-to-nearest adds), so the error
//               does not grow with the tensor-core accumulation chain.
// The stage ring is released as soon as the splitters hold the data in
// registers, so nearly all of it is outstanding DRAM traffic (Little's law:
// the loaded-HBM latency is several microseconds on B200).
//
// Work split: contiguous (side, output tile, K tile) unit ranges over the
// CTAs; a CTA that owns a whole output tile stores it, shared tiles are
// reduced with red.global.add.v4.f32 into an output that the CTAs zero at
// start-up (each a row slice; a CTA polls the arrival count before its first
// reduction). That wait needs every CTA resident at once: the grid is at most
// the SM count times the occupancy the launcher queries (1 CTA per SM).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "pass.cuh"

namespace cnmf {
namespace {

constexpr int BMT = 128;  // output rows per tile (TMEM lanes)
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

template <int S>
struct TcCfg {
  static constexpr int ABYTES = BMT * BKT * 4;  // 16 KB raw A tile
  static constexpr int BRAW = BKT * S * 4;      // raw fp32 panel tile [32 k][S]: 4 or 8 KB
  static constexpr int STAGE = ABYTES + BRAW;   // one TMA stage: A tile + its panel tile
  static constexpr int BSPL = BKT * 2 * S * 4;  // split K-major SW128 panel slot [hi; lo]
  static constexpr int NACC = CNMF_PASS_NACC;   // TMEM accumulator buffers
  static constexpr int AST = S == 64 ? CNMF_PASS_AST64 : 4;  // TMEM A ring = split panel ring = MMA-done ring
  static constexpr int ST = (227 * 1024 - 1024 - AST * BSPL) / STAGE;  // stage ring (DRAM bytes in flight)
  static constexpr int KB = CNMF_PASS_KB;       // K tiles per tensor-core accumulation block
  static constexpr int ACC_COLS = 2 * S;        // per accumulator buffer
  static constexpr int A_COL0 = NACC * ACC_COLS;  // first TMEM column of the A ring
  static constexpr int TMEM_COLS = (A_COL0 + AST * 2 * BKT <= 256) ? 256 : 512;
  static constexpr int NEPI = 4 * (S / 32);     // epilogue warps (lane quarter x 32-column group)
  static constexpr int THREADS = 32 * (2 + NSPL + NEPI);
  static constexpr size_t SMEM = (size_t)ST * STAGE + (size_t)AST * BSPL + 512;
  static_assert(ST >= 4, "stage ring depth");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(A_COL0 + AST * 2 * BKT <= 512, "TMEM budget");
  static_assert(S % 32 == 0, "panel width");
};

constexpr int kWarpTma = 0, kWarpMma = 1, kWarpSplit0 = 2, kWarpEpi0 = 2 + NSPL;

// One side of a launch: Y = A X (trans = 0) or Z = A^T W (trans = 1).
struct PassSide {
  float* out;
  int64_t P;        // output rows
  int64_t nblocks;  // 128-row output tiles
  int nt;           // K tiles per output tile
  int trans;
  double* sumsq;    // forward side only, may be null: += sum of A^2 over the side's tiles
};

// The (side, output tile, K tile) walk of one CTA's units: [lo0, hi0) of
// side 0, then [lo1, hi1) of side 1 (unit indices local to each side; plain
// scalars, no indexed arrays, so nothing lands in local memory).
struct Walk {
  int p;
  int64_t ob, u;
  int kt;
  int64_t lo0, hi0, lo1, hi1;
  __device__ __forceinline__ void start(int64_t a0, int64_t a1, int64_t b0, int64_t b1, const PassSide& s0,
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
    const int64_t t0 = ob * nt;
    return t0 >= (p ? lo1 : lo0) && t0 + nt <= (p ? hi1 : hi0);
  }
  // units left in the current output tile within this CTA's range
  __device__ __forceinline__ int64_t tile_left(int nt) const {
    const int64_t r = (p ? hi1 : hi0) - u, t = nt - kt;
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

// Split-K zeroing handshake (one slot of a per-device ring per launch).
struct ZSync {
  unsigned arrived, finished;
};

// tA0/tB0: A and panel tensor maps of side 0, tA1/tB1 of side 1 (a forward
// side's A map is K-major SW128 boxes of 128 rows x 32 columns, a transpose
// side's row-major boxes of 32 rows x 128 columns). whole = 1: the ranges are
// whole output tiles (no tile is shared, zs unused).
template <int S>
__global__ void __launch_bounds__(TcCfg<S>::THREADS, 1)
    stream_pass(const __grid_constant__ TmaDesc tA0, const __grid_constant__ TmaDesc tB0,
                const __grid_constant__ TmaDesc tA1, const __grid_constant__ TmaDesc tB1, const PassSide s0,
                const PassSide s1, int whole, ZSync* __restrict__ zs) {
  using C = TcCfg<S>;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sP = smem + C::ST * C::STAGE;          // [AST][BSPL]
  uint64_t* full = (uint64_t*)(sP + C::AST * C::BSPL);  // [ST] stage landed
  uint64_t* empty = full + C::ST;                       // [ST] stage consumed by all splitters
  uint64_t* afull = empty + C::ST;                      // [AST] split A in TMEM + split panel in SMEM
  uint64_t* mdone = afull + C::AST;                     // [AST] MMAs of the slot's K tile retired
  uint64_t* tfull = mdone + C::AST;                     // [2] accumulator ready
  uint64_t* tempty = tfull + C::NACC;                   // [NACC] accumulator drained
  uint32_t* tmem_slot = (uint32_t*)(tempty + C::NACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this CTA's share of the concatenated unit sequence (side 0, then side 1)
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
  const int64_t ntiles = (hi0 - lo0) + (hi1 - lo1);  // >= 1: the grid never exceeds the units (tiles)

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
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // programmatic dependent launch: everything above overlapped the tail of
  // the previous kernel in the stream; its outputs are visible from here on
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (zs != nullptr) {
    // split-K outputs start at zero: every CTA zeroes a row slice of each side
    for (int q = 0; q < 2; ++q) {
      const PassSide& sd = q ? s1 : s0;
      if (sd.nblocks == 0) continue;
      const int64_t z0 = b * sd.P / G, z1 = (b + 1) * sd.P / G;
      float4* o4 = reinterpret_cast<float4*>(sd.out + z0 * S);
      for (int64_t i = threadIdx.x; i < (z1 - z0) * S / 4; i += blockDim.x) o4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (zs != nullptr && threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&zs->arrived, 1u);
  }
  const uint32_t tmem = *tmem_slot;

  if (warp == kWarpTma) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      Ring<C::ST> r;
      Walk w;
      w.start(lo0, hi0, lo1, hi1, s0, s1);
      for (int64_t it = 0; it < ntiles; ++it) {
        if (it >= C::ST) mbar_sleep(&empty[r.i], r.ph ^ 1);
        unsigned char* dst = smem + r.i * C::STAGE;
        mbar_arrive_expect_tx(&full[r.i], C::STAGE);
        const PassSide& sd = w.p ? s1 : s0;
        const TmaDesc* ta = w.p ? &tA1 : &tA0;
        const TmaDesc* tb = w.p ? &tB1 : &tB0;
        const int row0 = (int)(w.ob * BMT);
        if (!sd.trans)  // A rows [row0, +128), cols [kt*32, +32): K-major SW128
          tma_load_2d(dst, ta, &full[r.i], w.kt * BKT, row0);
        else  // A rows [kt*32, +32) (K), cols [row0, +128) (M): row-major
          tma_load_2d(dst, ta, &full[r.i], row0, w.kt * BKT);
        // panel rows [kt*32, +32) (K), all S columns: row-major [32][S]
        tma_load_2d(dst + C::ABYTES, tb, &full[r.i], 0, w.kt * BKT);
        r.next();
        w.next(s0, s1);
      }
    }
  } else if (warp >= kWarpEpi0) {
    // ---------------- epilogue (one output row x 32 columns per thread) ----------------
    const int q = warp & 3;                         // TMEM lane quarter this warp may access
    const int cg = 32 * ((warp - kWarpEpi0) >> 2);  // first output column of this warp
    const int row_in_tile = 32 * q + lane;
    Ring<C::NACC> racc;
    acc_t acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    Walk w;
    w.start(lo0, hi0, lo1, hi1, s0, s1);
    // one iteration per accumulation block (<= KB K tiles of one output tile)
    for (int64_t it = 0; it < ntiles;) {
      const int nt = w.p ? s1.nt : s0.nt;
      const int64_t left = w.tile_left(nt);
      const int kb_left = C::KB - (w.kt % C::KB);
      const int len = (int)(left < kb_left ? left : kb_left);
      const bool tile_end = (len == left);
      mbar_sleep(&tfull[racc.i], racc.ph);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + racc.i * C::ACC_COLS + cg;
#pragma unroll
      for (int c0 = 0; c0 < 32; c0 += 8) {  // 8 columns at a time: few live temporaries (96-register cap at S = 64)
        float vh[8], vl[8];
#ifndef CNMF_VARIANT_NOEPI
        tmem_ld8(taddr + c0, vh);
        tmem_ld8(taddr + S + c0, vl);
#else
#pragma unroll
        for (int j = 0; j < 8; ++j) vh[j] = vl[j] = (float)(taddr + j);
#endif
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[c0 + j] += (acc_t)(vh[j] + vl[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[racc.i]);
      racc.next();
      if (tile_end) {
        const PassSide& sd = w.p ? s1 : s0;
        const bool owned = w.owned(nt);
        const int64_t row = w.ob * BMT + row_in_tile;
        if (!owned && zs != nullptr) {  // every CTA's zeroing must have landed
          if (lane == 0) {
            unsigned v;
            do {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&zs->arrived) : "memory");
            } while (v < gridDim.x);
          }
          __syncwarp();
        }
        if (row < sd.P) {
          float* dst = sd.out + row * S + cg;
          if (owned) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *(float4*)(dst + j) = make_float4((float)acc[j], (float)acc[j + 1], (float)acc[j + 2], (float)acc[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              red_add_v4(dst + j, (float)acc[j], (float)acc[j + 1], (float)acc[j + 2], (float)acc[j + 3]);
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.0;
      }
      w.skip(len, s0, s1);
      it += len;
    }
  } else if (warp == kWarpMma) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc_cat = idesc_tf32(2 * S);
    constexpr uint32_t idesc_hi = idesc_tf32(S);
    Ring<C::AST> ra;
    Ring<C::NACC> racc;
    Walk w;
    w.start(lo0, hi0, lo1, hi1, s0, s1);
    bool block_start = true;
    for (int64_t it = 0; it < ntiles; ++it) {
      const int nt = w.p ? s1.nt : s0.nt;
      const bool tile_end = w.tile_left(nt) == 1;
      const bool block_end = tile_end || ((w.kt + 1) % C::KB == 0);
      // reuse of an accumulator buffer waits until the epilogue drained it
      if (block_start && racc.wrapped) mbar_sleep(&tempty[racc.i], racc.ph ^ 1);
      mbar_sleep(&afull[ra.i], ra.ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sb = smem_u32(sP + ra.i * C::BSPL);       // K-major SW128 [hi; lo]
        const uint32_t ahi = tmem + C::A_COL0 + ra.i * 2 * BKT;  // split A in TMEM
        const uint32_t alo = ahi + BKT;
        const uint32_t dcat = tmem + racc.i * C::ACC_COLS;
        const uint32_t dlo = dcat + S;
#pragma unroll
        for (int k = 0; k < BKT / 8; ++k) {
          const uint64_t bcat = smem_desc(sb + 32 * k, 16, 1024);  // 8 tf32 = 32 B per K step
          const uint32_t acc = (block_start && k == 0) ? 0u : 1u;
#ifndef CNMF_VARIANT_NOMMA
          tc_mma_ts(dcat, ahi + 8 * k, bcat, idesc_cat, acc);  // [A_hi X_hi | A_hi X_lo]
          tc_mma_ts(dlo, alo + 8 * k, bcat, idesc_hi, 1u);     //            + A_lo X_hi
#endif
        }
        tc_commit(&mdone[ra.i]);  // releases the TMEM A slot and the split panel slot
        if (block_end) tc_commit(&tfull[racc.i]);
      }
      __syncwarp();
      ra.next();
      block_start = block_end;
      if (block_end) racc.next();
      w.next(s0, s1);
    }
  } else {
    // ---------------- splitters (warps 2..9) ----------------
    const int q = warp & 3;                     // TMEM lane quarter
    const int half = (warp - kWarpSplit0) >> 2; // K half of the A tile
    const int pc = warp - kWarpSplit0;          // 16-byte K chunk of the panel tile (k = 4 pc .. 4 pc + 3)
    const int row_in_tile = 32 * q + lane;
    double sq_acc = 0.0;                        // sum of A^2 (residual pass only)
    constexpr int PT = S / 32;                  // panel columns per lane
    Ring<C::ST> r;
    Ring<C::AST> ra;
    Walk w;
    w.start(lo0, hi0, lo1, hi1, s0, s1);
    for (int64_t it = 0; it < ntiles; ++it) {
      mbar_sleep(&full[r.i], r.ph);
      const unsigned char* stage = smem + r.i * C::STAGE;
      float hi[16], lo[16];
      if (!(w.p ? s1.trans : s0.trans)) {
        // row r of the K-major SW128 tile: 16 B chunk c at chunk c ^ (r & 7)
        const unsigned char* rowp = stage + row_in_tile * 128;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int c = 4 * half + cc;
          const float4 v = *(const float4*)(rowp + ((c ^ (row_in_tile & 7)) << 4));
          hi[4 * cc + 0] = v.x;
          hi[4 * cc + 1] = v.y;
          hi[4 * cc + 2] = v.z;
          hi[4 * cc + 3] = v.w;
        }
        if ((w.p ? s1.sumsq : s0.sumsq) != nullptr) {  // ||A||_F^2 of the residual pass (zero fill adds 0)
          float q2 = 0.f;
#pragma unroll
          for (int k = 0; k < 16; ++k) q2 = fmaf(hi[k], hi[k], q2);
          sq_acc += (double)q2;
        }
      } else {
        // A column = output row: gather 16 K values from the row-major tile
        const float* raw = (const float*)stage + row_in_tile;
#pragma unroll
        for (int k = 0; k < 16; ++k) hi[k] = raw[(16 * half + k) * BMT];
      }
      // panel: rows k = 4 pc + j, columns n = lane + 32 t (consecutive lanes,
      // consecutive columns: conflict-free)
      float ph[PT][4], pl[PT][4];
      {
        const float* raw = (const float*)(stage + C::ABYTES);
#pragma unroll
        for (int t = 0; t < PT; ++t)
#pragma unroll
          for (int j = 0; j < 4; ++j) ph[t][j] = raw[(4 * pc + j) * S + lane + 32 * t];
      }
      // Recycle the stage once every value read from it has landed. The
      // arrive (SYNCS) does not wait for outstanding LDS by itself: without
      // the proxy fence (generic reads -> the next TMA write, an async-proxy
      // write) the producer's next TMA could land before slow loads read the
      // stage -- a whole corrupted output tile in up to 45 % of split-K
      // launches (tools/splitk_diag.py).
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[r.i]);
#ifndef CNMF_VARIANT_NOSPLIT
      // hi = rn_tf32(v); lo = v - hi is exact and signed, so the tensor
      // core's truncation of lo to tf32 is unbiased (<= 2^-22 |v|; measured:
      // same subspace distance to the reference as rounding lo, 6 % faster)
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float v = hi[k];
        hi[k] = tf32_rn(v);
        lo[k] = v - hi[k];
      }
#pragma unroll
      for (int t = 0; t < PT; ++t)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float v = ph[t][j];
          ph[t][j] = tf32_rn(v);
          pl[t][j] = v - ph[t][j];
        }
#else
#pragma unroll
      for (int k = 0; k < 16; ++k) lo[k] = hi[k];
#pragma unroll
      for (int t = 0; t < PT; ++t)
#pragma unroll
        for (int j = 0; j < 4; ++j) pl[t][j] = ph[t][j];
#endif
      if (ra.wrapped) mbar_sleep(&mdone[ra.i], ra.ph ^ 1);  // the slot's previous K tile retired
      tc_fence_after();
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + C::A_COL0 + ra.i * 2 * BKT + 16 * half;
#ifndef CNMF_VARIANT_NOSTTM
      tmem_st16(ta, hi);
      tmem_st16(ta + BKT, lo);
#else
      if (hi[0] == 1.2345f && lo[3] == 2.5f) tmem_st16(ta, hi);
#endif
      unsigned char* dst = sP + ra.i * C::BSPL;
#pragma unroll
      for (int t = 0; t < PT; ++t) {
        const int n = lane + 32 * t;  // output column = B operand row
        const uint32_t off = (uint32_t)n * 128 + ((pc ^ (n & 7)) << 4);
        *(float4*)(dst + off) = make_float4(ph[t][0], ph[t][1], ph[t][2], ph[t][3]);
        *(float4*)(dst + S * 128 + off) = make_float4(pl[t][0], pl[t][1], pl[t][2], pl[t][3]);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_proxy_async();  // generic-proxy smem stores -> tensor-core (async proxy) reads
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ra.i]);
      r.next();
      ra.next();
      w.next(s0, s1);
    }
    if (s0.sumsq != nullptr) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq_acc += __shfl_xor_sync(0xffffffffu, sq_acc, o);
      if (lane == 0) atomicAdd(s0.sumsq, sq_acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (zs != nullptr && threadIdx.x == 0 && atomicAdd(&zs->finished, 1u) == gridDim.x - 1) {
    zs->arrived = 0u;
    zs->finished = 0u;
  }
  if (warp == kWarpMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

struct SideArgs {
  const float* panel;  // X (n x S) for a forward side, W (m x S) for a transpose side
  float* out;
  int trans;
  double* sumsq = nullptr;  // forward side: accumulate ||A||_F^2 (residual pass)
};

// Launch one or two sides over the same A.
template <int S>
int launch_stream(const float* A, int64_t m, int64_t n, int64_t lda, const SideArgs* sa, int nsides, cudaStream_t st) {
  using C = TcCfg<S>;
  TmaDesc tA[2], tB[2];
  PassSide sd[2] = {{nullptr, 0, 0, 1, 0, nullptr}, {nullptr, 0, 0, 1, 0, nullptr}};
  for (int i = 0; i < nsides; ++i) {
    const int64_t K = sa[i].trans ? m : n;  // panel rows
    const int64_t P = sa[i].trans ? n : m;  // output rows
    if (!sa[i].trans)
      CNMF_TRY(make_tma_2d(&tA[i], A, 4, m, n, lda, BKT, BMT, true));
    else
      CNMF_TRY(make_tma_2d(&tA[i], A, 4, m, n, lda, BMT, BKT, false));
    CNMF_TRY(make_tma_2d(&tB[i], sa[i].panel, 4, K, S, S, S, BKT, false));
    sd[i] = PassSide{sa[i].out, P, ceil_div(P, BMT), (int)ceil_div(K, BKT), sa[i].trans, sa[i].trans ? nullptr : sa[i].sumsq};
  }
  if (nsides == 1) {
    tA[1] = tA[0];
    tB[1] = tB[0];
  }
  const int64_t U = sd[0].nblocks * sd[0].nt + sd[1].nblocks * sd[1].nt;
  const int64_t T = sd[0].nblocks + sd[1].nblocks;
  CNMF_TRY(ensure_smem_attr((const void*)stream_pass<S>, (int)C::SMEM));
  static thread_local int occ_cache[64] = {};
  int dev = 0;
  CNMF_CUDA(cudaGetDevice(&dev));
  int& occ = occ_cache[dev & 63];
  if (occ == 0) {
    CNMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stream_pass<S>, C::THREADS, C::SMEM));
    if (occ < 1) return fail(CNMF_ERR_CUDA, "streaming pass kernel does not fit on an SM");
  }
  // every CTA must be resident at once (the split-K zeroing handshake)
  const int64_t slots = (int64_t)device_sms() * occ;
  const int whole = (nsides == 1 && T >= 16 * slots) ? 1 : 0;
  const int64_t grid = std::min<int64_t>(slots, whole ? T : U);
  ZSync* zs = nullptr;
  static const bool memset_zero = [] {
    const char* e = getenv("CNMF_PASS_MEMSET");
    return e && e[0] == '1';
  }();
  if (!whole && memset_zero) {
    for (int i = 0; i < nsides; ++i) CNMF_CUDA(cudaMemsetAsync(sd[i].out, 0, (size_t)sd[i].P * S * 4, st));
  } else if (!whole) {
    void* ring = nullptr;
    CNMF_TRY(device_scratch("pass-zsync", 64 * sizeof(ZSync), &ring, st));
    zs = (ZSync*)ring + (device_ticket("pass-zsync") % 64);
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
  CNMF_CUDA(cudaLaunchKernelEx(&lc, stream_pass<S>, tA[0], tB[0], tA[1], tB[1], sd[0], sd[1], whole, zs));
  CNMF_LAUNCH_CHECK();
  if (e0) {
    CNMF_CUDA(cudaEventRecord(e1, st));
    // algorithmic bytes: A once per side plus the side's panel in and out
    pass_record(e0, e1, nsides * 4.0 * ((double)m * n + (double)n * S + (double)m * S));
  }
  return CNMF_OK;
}

int launch_any(const float* A, int64_t m, int64_t n, int64_t lda, const SideArgs* sa, int nsides, int S,
               cudaStream_t st) {
  switch (S) {
    case 32: return launch_stream<32>(A, m, n, lda, sa, nsides, st);
    case 64: return launch_stream<64>(A, m, n, lda, sa, nsides, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "tensor-core pass supports panel widths 32 and 64");
}

}  // namespace

int pass_forward_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y, cudaStream_t st) {
  const SideArgs sa{X, Y, 0};
  return launch_any(A, m, n, lda, &sa, 1, S, st);
}

// Y = A X and sumsq += ||A||_F^2 in the same read of A (the residual pass)
int pass_forward_sumsq_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y,
                          double* sumsq, cudaStream_t st) {
  SideArgs sa{X, Y, 0};
  sa.sumsq = sumsq;
  return launch_any(A, m, n, lda, &sa, 1, S, st);
}

int pass_transpose_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, int S, float* Z,
                      cudaStream_t st) {
  const SideArgs sa{W, Z, 1};
  return launch_any(A, m, n, lda, &sa, 1, S, st);
}

// Y = A X and Z = A^T W in one launch (the two range finders' passes of a
// power step: one pipeline ramp-up and tail instead of two)
int pass_pair_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, const float* W, float* Z,
                 int S, cudaStream_t st) {
  const SideArgs sa[2] = {{X, Y, 0}, {W, Z, 1}};
  return launch_any(A, m, n, lda, sa, 2, S, st);
}

}  // namespace cnmf
