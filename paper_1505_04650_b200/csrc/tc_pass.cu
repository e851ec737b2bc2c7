// Streaming passes over A on the 5th-generation tensor cores (tcgen05,
// kind::tf32) with a 3xTF32 split for fp32-level accuracy:
//
//   A X ~= A_hi X_hi + A_hi X_lo + A_lo X_hi,   v_hi = rn_tf32(v),
//   v_lo = rn_tf32(v - v_hi).
//
// Forward pass  Y = A X   (M = rows of A, K = columns of A, N = s)
// Transpose     Z = A^T W (M = columns of A, K = rows of A, N = s)
//
// The skinny operand is split once per pass, outside the kernel, into
// [X_hi | X_lo]^T (2S rows, K contiguous): a 32-deep K tile of it is exactly
// the K-major SW128 B operand, so TMA lands it ready for the tensor core.
// One CTA per SM, warp-specialised (11 + S/8 warps):
//   warp 0      A producer: per K tile one raw fp32 A tile (16 KB, K-major
//               SW128 for the forward pass, row-major for the transpose pass)
//               into a deep stage ring (the DRAM bytes in flight per SM);
//   warp 10     panel producer: the split panel tile (2S x 32, 8/16 KB) of
//               the same K tile into a panel ring, released by the MMA commit;
//   warps 2..9  A splitters: warp w owns TMEM lane quarter w & 3 (= 32 output
//               rows) and K half (w - 2) / 4; each thread reads its row from
//               the stage, releases the stage, splits hi/lo and stores both
//               into a TMEM ring (tcgen05.st);
//   warp 1      MMA issuer (one elected thread), A from TMEM, panel from SMEM:
//                 D[:, 0:2S]  = A_hi [X_hi | X_lo]      (N = 2S)
//                 D[:, S:2S] += A_lo X_hi               (N = S)
//               so D = [A_hi X_hi | A_hi X_lo + A_lo X_hi]; one
//               tcgen05.commit per K tile releases the panel slot and the
//               TMEM A slot;
//   warps 11..  epilogue: drain the double-buffered TMEM accumulator every
//               KB K tiles into fp32 registers, store (or reduce) the tile.
// Work is split in contiguous (output tile, K tile) unit ranges over the
// CTAs; split-K tiles are reduced deterministically (see SplitK).
#include <algorithm>

#include "common.cuh"

namespace cnmf {
namespace {

#ifndef CNMF_X
#define CNMF_X 0  // probe-only knockouts (tools/tc_variant.sh); 0 in the library
#endif
constexpr int BMT = 128;              // output rows per tile (TMEM lanes)
constexpr int BKT = 32;               // K per stage (one 128B swizzle atom of fp32)

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

// 32 lanes x 16 consecutive fp32 columns per warp
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
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

// kind::tf32 instruction descriptor: D fp32, A/B tf32, M = 128, N given.
__host__ __device__ constexpr uint32_t idesc_tf32(int n, bool a_mn_major, bool b_mn_major, int m = BMT) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// Round to the nearest tf32 value (10 explicit mantissa bits, ties away from
// zero). The tensor core truncates the low 13 bits of an fp32 operand, so
// both split halves are pre-rounded: hi = rn(v), lo = rn(v - hi) (v - hi is
// exact in fp32), which keeps the split error unbiased and <= 2^-22 |v| --
// truncating would bias every product of nonnegative data toward zero.
__device__ __forceinline__ float tf32_rn(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
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

#ifdef CNMF_TC_TRACE
__device__ long long g_tc_trace[64][16];
__device__ unsigned long long g_tc_span[148][3];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TC_SPAN(slot)                                                          \
  do {                                                                         \
    if (threadIdx.x == 0) g_tc_span[blockIdx.x][slot] = gtimer();              \
  } while (0)
#define TC_TRACE(slot)                                                          \
  do {                                                                          \
    if (blockIdx.x == CNMF_TC_TRACE_CTA && it < 64) g_tc_trace[it][slot] = clock64();           \
  } while (0)
#else
#define TC_TRACE(slot) \
  do {                 \
  } while (0)
#define TC_SPAN(slot) \
  do {                \
  } while (0)
#endif

template <int S>
struct TcCfg {
  static constexpr int ABYTES = BMT * BKT * 4;        // 16 KB raw A tile (one stage)
  static constexpr int PBYTES = 2 * S * BKT * 4;      // split panel tile [X_hi | X_lo]^T: 8 / 16 KB
#ifdef CNMF_TC_RINGS  // (ST32, SSP32, AST32) override for probes
  static constexpr int ST = (S == 32) ? CNMF_TC_ST : 8;
  static constexpr int SSP = (S == 32) ? CNMF_TC_SSP : 4;
  static constexpr int AST = (S == 32) ? CNMF_TC_AST : 4;
#else
  static constexpr int ST = (S == 32) ? 10 : 8;       // A stage ring (DRAM bytes in flight per SM)
  static constexpr int SSP = (S == 32) ? 6 : 4;       // split panel ring
  static constexpr int AST = 4;                       // TMEM ring of split A tiles
#endif
  static constexpr int MD = SSP > AST ? SSP : AST;    // "MMA of K tile j done" ring (>= SSP, AST)
  static constexpr int KB = 2;                        // K tiles per tensor-core accumulation block
  static constexpr int ACC_COLS = 2 * S;              // per accumulator buffer
  static constexpr int A_COL0 = 2 * ACC_COLS;         // first TMEM column of the A ring
  static constexpr int TMEM_COLS = (A_COL0 + AST * 2 * BKT <= 256) ? 256 : 512;
  static constexpr int NSPLIT = 8;                    // A-splitting warps (2 per TMEM lane quarter)
  static constexpr int NEPI = 4 * (S / 32);           // epilogue warps (lane quarter x 32-column group)
  static constexpr int THREADS = 32 * (11 + NEPI);
  static constexpr size_t SMEM = (size_t)ST * ABYTES + (size_t)SSP * PBYTES + 1024 + 512;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(A_COL0 + AST * 2 * BKT <= 512, "TMEM budget");
};

constexpr int kWarpTma = 0, kWarpMma = 1, kWarpSplit0 = 2, kWarpPanel = 10, kWarpEpi0 = 11;

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

// 32 lanes x 16 consecutive 32-bit columns per warp
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}

// Split-K launches reduce shared output tiles deterministically. The CTA
// holding a tile's first K units (slot 0) reaches that tile at the end of its
// unit range, every other contributor at the start of its own, so slot 0
// reduces: contributors store their fp32 partial to their slot of a scratch
// buffer and raise a per-(tile, slot, warp) flag without waiting; slot 0's
// epilogue warps wait for the (long raised) flags, add the slots in slot
// order to their own registers, store the tile and clear the flags. The
// result does not depend on CTA timing (bit-reproducible range finder).
struct SplitK {
  float* part;       // [nblocks][maxsplit][128][S]
  unsigned* flag;    // [nblocks][maxsplit][NEPI], zero between launches
  int maxsplit;
};

// CTA owning unit t of U units spread over G CTAs (CTA b owns [b U / G, (b + 1) U / G))
__device__ __forceinline__ int64_t item_of(int64_t t, int64_t U, int64_t G) { return ((t + 1) * G - 1) / U; }

// TRANS = false: Y = A X; TRANS = true: Z = A^T W. P = output rows of the
// pass (m or n); nt = K tiles per output tile.
template <int S, bool TRANS>
__global__ void __launch_bounds__(TcCfg<S>::THREADS, 1)
    pass_tc(const __grid_constant__ TmaDesc tA, const __grid_constant__ TmaDesc tB, float* __restrict__ out,
            int64_t P, int nt, int64_t nblocks, int whole, const SplitK sk) {
  using C = TcCfg<S>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sP = smem + C::ST * C::ABYTES;                // [SSP][PBYTES]
  uint64_t* full = (uint64_t*)(sP + C::SSP * C::PBYTES);       // [ST] A tile landed
  uint64_t* empty = full + C::ST;                              // [ST] A tile consumed by all splitters
  uint64_t* pfull = empty + C::ST;                             // [SSP] split panel tile landed
  uint64_t* mdone = pfull + C::SSP;                            // [MD] MMAs of K tile j retired
  uint64_t* afull = mdone + C::MD;                             // [AST] split A in TMEM
  uint64_t* tfull = afull + C::AST;                            // [2] accumulator ready
  uint64_t* tempty = tfull + 2;                                // [2] accumulator drained
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t U = nblocks * nt, G = gridDim.x, b = blockIdx.x;
  const int64_t u0 = whole ? (b * nblocks / G) * nt : b * U / G;
  const int64_t u1 = whole ? ((b + 1) * nblocks / G) * nt : (b + 1) * U / G;
  const int64_t ntiles = u1 - u0;
  if (ntiles <= 0) return;
  TC_SPAN(0);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tA);
    prefetch_tmap(&tB);
    for (int s = 0; s < C::ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NSPLIT);
    }
    for (int s = 0; s < C::SSP; ++s) mbar_init(&pfull[s], 1);
    for (int s = 0; s < C::AST; ++s) mbar_init(&afull[s], C::NSPLIT);
    for (int s = 0; s < C::MD; ++s) mbar_init(&mdone[s], 1);
    for (int i = 0; i < 2; ++i) {
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Every role walks the same unit sequence u0..u1-1 with incremental
  // (output tile, K tile) and ring (slot, phase) counters: no 64-bit
  // division and no dynamically indexed arrays in the steady-state loops.
  const int64_t ob0 = u0 / nt;
  const int kt0 = (int)(u0 - ob0 * nt);

  if (warp == kWarpTma) {
    // ---------------- A producer ----------------
    if (elect_one()) {
      Ring<C::ST> r;
      int64_t ob = ob0;
      int kt = kt0;
      for (int64_t it = 0; it < ntiles; ++it) {
        if (it >= C::ST) mbar_wait(&empty[r.i], r.ph ^ 1);
        TC_TRACE(0);
        unsigned char* dst = smem + r.i * C::ABYTES;
        mbar_arrive_expect_tx(&full[r.i], C::ABYTES);
        const int row0 = (int)(ob * BMT);  // this CTA's 128 output rows
        if (!TRANS)  // A rows [row0, +128), cols [kt*32, +32): K-major SW128
          tma_load_2d(dst, &tA, &full[r.i], kt * BKT, row0);
        else         // A rows [kt*32, +32) (K), cols [row0, +128) (M): row-major
          tma_load_2d(dst, &tA, &full[r.i], row0, kt * BKT);
        r.next();
        if (++kt == nt) {
          kt = 0;
          ++ob;
        }
      }
    }
  } else if (warp == kWarpPanel) {
    // ---------------- panel producer: split panel tile [2S][32 k], K-major SW128 ----------------
    if (elect_one()) {
      Ring<C::SSP> rp;
      Ring<C::MD> rd;  // tracks K tile it - SSP (the previous user of slot rp.i)
      int kt = kt0;
      for (int64_t it = 0; it < ntiles; ++it) {
        if (it >= C::SSP) {
          mbar_wait(&mdone[rd.i], rd.ph);
          rd.next();
        }
        TC_TRACE(7);
        mbar_arrive_expect_tx(&pfull[rp.i], C::PBYTES);
        tma_load_2d(sP + rp.i * C::PBYTES, &tB, &pfull[rp.i], kt * BKT, 0);
        rp.next();
        if (++kt == nt) kt = 0;
      }
    }
  } else if (warp >= kWarpEpi0) {
    // ---------------- epilogue (one output row x 32 columns per thread) ----------------
    // The tensor core accumulates at most KB K tiles into a TMEM buffer; the
    // partial sums then move to fp32 registers (round-to-nearest adds), so
    // the error no longer grows with the tensor-core accumulation chain.
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int cg = 32 * ((warp - kWarpEpi0) >> 2);  // first output column of this warp
    const int row_in_tile = 32 * q + lane;
    Ring<2> racc;
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.f;
    int64_t ob = ob0;
    int kt = kt0;
    for (int64_t it = 0; it < ntiles; ++it) {
      const bool tile_end = (it == ntiles - 1) || (kt == nt - 1);
      if (tile_end || ((kt + 1) % C::KB == 0)) {
        mbar_wait(&tfull[racc.i], racc.ph);
        tc_fence_after();
        const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + racc.i * C::ACC_COLS + cg;
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += 16) {
          float vh[16], vl[16];
          tmem_ld16(taddr + c0, vh);
          tmem_ld16(taddr + S + c0, vl);
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[c0 + j] += vh[j] + vl[j];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[racc.i]);
        racc.next();
      }
      if (tile_end) {
        const int64_t t0 = ob * nt;  // first unit of this output tile
        const bool owned = (t0 >= u0) && (t0 + nt <= u1);
        const int64_t row = ob * BMT + row_in_tile;
        if (owned) {
          if (row < P) {
            float* dst = out + row * S + cg;
#pragma unroll
            for (int j = 0; j < 32; j += 4) *(float4*)(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
          }
        } else {
          // shared tile: slot = this CTA's index among the tile's contributors
          const int64_t first = item_of(t0, U, G), last = item_of(t0 + nt - 1, U, G);
          const int slot = (int)(b - first), nsplit = (int)(last - first + 1);
          const int ew = warp - kWarpEpi0;
          float* base = sk.part + (ob * sk.maxsplit) * (int64_t)(BMT * S) + row_in_tile * S + cg;
          unsigned* flags = sk.flag + (ob * sk.maxsplit) * C::NEPI + ew;
          if (slot > 0) {
            float* mine = base + slot * (int64_t)(BMT * S);
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              __stcg((float4*)(mine + j), make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]));
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicExch(flags + slot * C::NEPI, 1u);
          } else {
            for (int q2 = 1; q2 < nsplit; ++q2) {
              if (lane == 0) {
                unsigned v;
                do {
                  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + q2 * C::NEPI) : "memory");
                } while (v == 0u);
                flags[q2 * C::NEPI] = 0u;  // sole reader: reset for the next launch
              }
              __syncwarp();
              const float* src = base + q2 * (int64_t)(BMT * S);
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const float4 v = __ldcg((const float4*)(src + j));
                acc[j] += v.x;
                acc[j + 1] += v.y;
                acc[j + 2] += v.z;
                acc[j + 3] += v.w;
              }
            }
            if (row < P) {
              float* dst = out + row * S + cg;
#pragma unroll
              for (int j = 0; j < 32; j += 4) *(float4*)(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      }
      if (++kt == nt) {
        kt = 0;
        ++ob;
      }
    }
  } else if (warp == kWarpMma) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc_cat = idesc_tf32(2 * S, false, false);
    constexpr uint32_t idesc_hi = idesc_tf32(S, false, false);
    Ring<C::SSP> rp;
    Ring<C::AST> ra;
    Ring<C::MD> rd;
    Ring<2> racc;  // accumulator buffer + its reuse phase
    int kt = kt0;
    bool block_start = true;
    for (int64_t it = 0; it < ntiles; ++it) {
      const bool tile_end = (it == ntiles - 1) || (kt == nt - 1);
      const bool block_end = tile_end || ((kt + 1) % C::KB == 0);
      // reuse of an accumulator buffer waits until the epilogue drained it
      if (block_start && racc.wrapped) mbar_wait(&tempty[racc.i], racc.ph ^ 1);
      mbar_wait(&pfull[rp.i], rp.ph);
      mbar_wait(&afull[ra.i], ra.ph);
      tc_fence_after();
      if (lane == 0) TC_TRACE(4);
      if (elect_one()) {
        const uint32_t sb = smem_u32(sP + rp.i * C::PBYTES);     // K-major SW128 [hi; lo]
        const uint32_t ahi = tmem + C::A_COL0 + ra.i * 2 * BKT;   // split A in TMEM
        const uint32_t alo = ahi + BKT;
        const uint32_t dcat = tmem + racc.i * C::ACC_COLS;
        const uint32_t dlo = dcat + S;
#pragma unroll
        for (int k = 0; k < BKT / 8; ++k) {
          const uint64_t bcat = smem_desc(sb + 32 * k, 16, 1024);  // 8 tf32 = 32 B per K step
          const uint32_t acc = (block_start && k == 0) ? 0u : 1u;
          tc_mma_ts(dcat, ahi + 8 * k, bcat, idesc_cat, acc);  // [A_hi X_hi | A_hi X_lo]
          tc_mma_ts(dlo, alo + 8 * k, bcat, idesc_hi, 1u);     //            + A_lo X_hi
        }
        tc_commit(&mdone[rd.i]);  // one commit releases the panel slot and the TMEM A slot
        if (block_end) tc_commit(&tfull[racc.i]);
        TC_TRACE(5);
      }
      __syncwarp();
      rp.next();
      ra.next();
      rd.next();
      block_start = block_end;
      if (block_end) racc.next();
      if (++kt == nt) kt = 0;
    }
  } else if (warp < kWarpPanel) {
    // ---------------- A splitters (warps 2..9) ----------------
    // warp w serves TMEM lane quarter w & 3 and K half (w - 2) / 4 of every tile
    const int q = warp & 3;
    const int half = (warp - kWarpSplit0) >> 2;
    const int row_in_tile = 32 * q + lane;
    Ring<C::ST> r;
    Ring<C::AST> ra;
    Ring<C::MD> rd;  // tracks K tile it - AST (the previous user of TMEM slot ra.i)
    for (int64_t it = 0; it < ntiles; ++it) {
      mbar_wait(&full[r.i], r.ph);
      if (threadIdx.x == 64) TC_TRACE(1);
      float hi[16], lo[16];
      if (CNMF_X == 2) {
#pragma unroll
        for (int k = 0; k < 16; ++k) hi[k] = (float)(lane + k);
      } else if (!TRANS) {
        // row r of the K-major SW128 tile: 16 B chunk c at chunk c ^ (r & 7)
        const unsigned char* rowp = smem + r.i * C::ABYTES + row_in_tile * 128;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int c = 4 * half + cc;
          const float4 v = *(const float4*)(rowp + ((c ^ (row_in_tile & 7)) << 4));
          hi[4 * cc + 0] = v.x;
          hi[4 * cc + 1] = v.y;
          hi[4 * cc + 2] = v.z;
          hi[4 * cc + 3] = v.w;
        }
      } else {
        // A column = output row: gather 16 K values from the row-major tile
        const float* raw = (const float*)(smem + r.i * C::ABYTES) + row_in_tile;
#pragma unroll
        for (int k = 0; k < 16; ++k) hi[k] = raw[(16 * half + k) * BMT];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[r.i]);  // raw tile is in registers: recycle the stage
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float v = hi[k];
        hi[k] = tf32_rn(v);
        lo[k] = tf32_rn(v - hi[k]);
      }
      if (it >= C::AST) {
        mbar_wait(&mdone[rd.i], rd.ph);
        rd.next();
      }
      tc_fence_after();
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + C::A_COL0 + ra.i * 2 * BKT + 16 * half;
      tmem_st16(ta, hi);
      tmem_st16(ta + BKT, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ra.i]);
      if (threadIdx.x == 64) TC_TRACE(3);
      r.next();
      ra.next();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  TC_SPAN(1);
  if (warp == kWarpMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

// [X_hi | X_lo]^T of a panel X (rows x S, ld S): out[c][r] = rn_tf32(X[r][c]),
// out[S + c][r] = rn_tf32(X[r][c] - hi), row pitch ldk (rows rounded to 4).
// One 32-row x S tile per block through shared memory (coalesced both ways).
template <int S>
__global__ void __launch_bounds__(256) split_panel(const float* __restrict__ X, int64_t rows, int64_t ldk,
                                                   float* __restrict__ out) {
  __shared__ float t[32][S + 1];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.x; i < 32 * S; i += 256) {
    const int r = i / S, c = i % S;
    t[r][c] = (r0 + r < rows) ? X[(r0 + r) * S + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * S; i += 256) {
    const int c = i / 32, r = i % 32;
    if (r0 + r < ldk) {
      const float v = t[r][c];
      const float h = tf32_rn(v);
      out[(int64_t)c * ldk + r0 + r] = h;
      out[(int64_t)(S + c) * ldk + r0 + r] = tf32_rn(v - h);
    }
  }
}

// Library-owned scratch, grown by eager calls (allocation is illegal inside a
// graph capture); kernels on one stream use it in order.
struct Scratch {
  void* p = nullptr;
  size_t cap = 0;
};

static int grow(Scratch& sc, size_t bytes, cudaStream_t st, bool zero) {
  if (sc.cap >= bytes) return CNMF_OK;
  cudaStreamCaptureStatus cs;
  CNMF_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    return fail(CNMF_ERR_CUDA, "pass scratch must be sized by an eager call before graph capture");
  CNMF_CUDA(cudaStreamSynchronize(st));
  if (sc.p) cudaFree(sc.p);
  sc.p = nullptr;
  sc.cap = 0;
  CNMF_CUDA(cudaMalloc(&sc.p, bytes));
  if (zero) CNMF_CUDA(cudaMemset(sc.p, 0, bytes));
  sc.cap = bytes;
  return CNMF_OK;
}

template <int S, bool TRANS>
int launch_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* Bpanel, float* out, cudaStream_t st) {
  using C = TcCfg<S>;
  // skinny operand rows = K extent: n (forward, X) or m (transpose, W)
  const int64_t brows = TRANS ? m : n;
  const int64_t ldk = (brows + 3) / 4 * 4;
  static Scratch split_ws, part_ws, flag_ws;
  CNMF_TRY(grow(split_ws, (size_t)2 * S * ldk * 4, st, false));
  float* Bs = (float*)split_ws.p;
  split_panel<S><<<(unsigned)ceil_div(brows, 32), 256, 0, st>>>(Bpanel, brows, ldk, Bs);
  CNMF_LAUNCH_CHECK();
  TmaDesc tA, tB;
  if (!TRANS)
    CNMF_TRY(make_tma_2d(&tA, A, 4, m, n, lda, BKT, BMT, true));
  else
    CNMF_TRY(make_tma_2d(&tA, A, 4, m, n, lda, BMT, BKT, false));
  CNMF_TRY(make_tma_2d(&tB, Bs, 4, 2 * S, brows, ldk, BKT, 2 * S, true));
  const int64_t P = TRANS ? n : m;   // output rows
  const int nt = (int)ceil_div(brows, BKT);
  const int64_t nblocks = ceil_div(P, BMT);
  const int64_t slots = kNumSMs;
  const int whole = nblocks >= 16 * slots;
  const int64_t grid = std::min<int64_t>(slots, whole ? nblocks : nblocks * nt);
  SplitK sk{nullptr, nullptr, 0};
  if (!whole) {
    const int64_t U = nblocks * nt;
    sk.maxsplit = (int)(ceil_div(nt, U / grid) + 1);
    CNMF_TRY(grow(part_ws, (size_t)nblocks * sk.maxsplit * BMT * S * 4, st, false));
    CNMF_TRY(grow(flag_ws, (size_t)nblocks * sk.maxsplit * C::NEPI * 4, st, true));
    sk.part = (float*)part_ws.p;
    sk.flag = (unsigned*)flag_ws.p;
  }
  static bool attr = false;
  if (!attr) {
    CNMF_CUDA(cudaFuncSetAttribute(pass_tc<S, TRANS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
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
  CNMF_CUDA(cudaLaunchKernelEx(&lc, pass_tc<S, TRANS>, tA, tB, out, P, nt, nblocks, whole, sk));
  CNMF_LAUNCH_CHECK();
  if (e0) {
    CNMF_CUDA(cudaEventRecord(e1, st));
    pass_record(e0, e1, 4.0 * ((double)m * n + (double)n * S + (double)m * S));
  }
  return CNMF_OK;
}

}  // namespace

int pass_forward_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y, cudaStream_t st) {
  switch (S) {
    case 32: return launch_tc<32, false>(A, m, n, lda, X, Y, st);
    case 64: return launch_tc<64, false>(A, m, n, lda, X, Y, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "tensor-core pass supports panel widths 32 and 64");
}

int pass_transpose_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, int S, float* Z,
                      cudaStream_t st) {
  switch (S) {
    case 32: return launch_tc<32, true>(A, m, n, lda, W, Z, st);
    case 64: return launch_tc<64, true>(A, m, n, lda, W, Z, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "tensor-core pass supports panel widths 32 and 64");
}

}  // namespace cnmf
