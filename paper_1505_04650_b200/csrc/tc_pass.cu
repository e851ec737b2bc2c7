// Streaming passes over A on the 5th-generation tensor cores (tcgen05,
// kind::tf32) with a 3xTF32 split for fp32-level accuracy:
//
//   A X ~= A_hi X_hi + A_hi X_lo + A_lo X_hi,   v_hi = v with the low 13
//   mantissa bits cleared (exactly representable in tf32), v_lo = v - v_hi.
//
// Forward pass  Y = A X   (M = rows of A, K = columns of A, N = s)
// Transpose     Z = A^T W (M = columns of A, K = rows of A, N = s)
//
// One CTA per SM, warp-specialised (S/16 + 10 warps):
//   warp 0      TMA producer: per K tile one stage = raw fp32 A tile (16 KB,
//               K-major SW128 for the forward pass, row-major for the
//               transpose pass) + the raw fp32 panel rows [32 k][S];
//   warps 2..9  A splitters: warp w owns TMEM lane quarter w & 3 (= 32 output
//               rows) and K half (w - 2) / 4; each thread reads its row from
//               the stage, releases the stage, splits hi/lo and stores both
//               into a TMEM ring (tcgen05.st); warps 2..5 also drain the
//               accumulator at the end of every output tile;
//   warps 10..  panel splitters: raw [32 k][S] -> K-major SW128 [hi; lo] in a
//               small shared-memory ring (kind::tf32 only accepts K-major
//               shared-memory operands on sm_100a; measured);
//   warp 1      MMA issuer (one elected thread), A from TMEM, panel from SMEM:
//                 D[:, 0:2s]  = A_hi [X_hi | X_lo]      (N = 2s)
//                 D[:, s:2s] += A_lo X_hi               (N = s)
//               so D = [A_hi X_hi | A_hi X_lo + A_lo X_hi] and the epilogue
//               adds the halves; one tcgen05.commit per K tile releases both
//               the panel slot and the TMEM A slot.
// The stage ring is released as soon as the splitters hold the data in
// registers, so nearly all of it is outstanding DRAM traffic (Little's law:
// the loaded-HBM latency is several microseconds on B200).
// Work is distributed exactly like the FFMA passes (contiguous unit ranges,
// flush on tile change, red.global.add when a tile is shared).
#include <algorithm>

#include "common.cuh"
#include "pass.cuh"

namespace cnmf {
namespace {

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

template <int S, bool TRANS, bool PAIR = false>
struct TcCfg {
  static constexpr int ABYTES = BMT * BKT * 4;        // 16 KB raw A tile
  static constexpr int BRAW = BKT * S * 4;            // raw fp32 panel tile [32 k][S]: 4 or 8 KB
  static constexpr int STAGE = ABYTES + BRAW;         // one TMA stage: A tile + its panel tile
  // split K-major SW128 panel slot: [hi; lo] (2S rows), or for a CTA pair this
  // CTA's halves of the two MMAs' B operands: [hi or lo (S rows); hi half (S/2 rows)]
  static constexpr int BSPL = PAIR ? BKT * (S + S / 2) * 4 : BKT * 2 * S * 4;
  // ring depths: a CTA pair's cross-CTA arrivals add ~1 us of latency to the
  // panel and TMEM rings, so those are deeper there
  static constexpr int ST = (S == 32) ? (PAIR ? 9 : 10) : 7;  // stage ring (DRAM bytes in flight per SM)
  static constexpr int SSP = PAIR ? (S == 32 ? 6 : 4) : 3;    // split panel ring
  static constexpr int AST = PAIR && S == 32 ? 6 : 4;         // TMEM ring of split A tiles
  static constexpr int MD = SSP > AST ? SSP : AST;    // "MMA of K tile j done" ring (>= SSP, AST)
  static constexpr int KB = 2;                        // K tiles per tensor-core accumulation block
  static_assert(MD >= SSP && MD >= AST, "one MMA-done ring serves both consumers");
  static constexpr int ACC_COLS = 2 * S;              // per accumulator buffer
  static constexpr int A_COL0 = 2 * ACC_COLS;         // first TMEM column of the A ring
  static constexpr int TMEM_COLS = (A_COL0 + AST * 2 * BKT <= 256) ? 256 : 512;
  static constexpr int NSPLIT = 8;                    // A-splitting warps (2 per TMEM lane quarter)
  static constexpr int NPW = 2;                       // panel-splitting warps
  static constexpr int PU = S / 32;                   // panel units (32 columns x 16 k) per panel warp
  static constexpr int NEPI = 4 * (S / 32);            // epilogue warps (lane quarter x 32-column group)
  static constexpr int THREADS = 32 * (2 + NSPLIT + NPW + NEPI);
  static constexpr size_t SMEM = (size_t)ST * STAGE + (size_t)SSP * BSPL + 512;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(A_COL0 + AST * 2 * BKT <= 512, "TMEM budget");
};

constexpr int kWarpTma = 0, kWarpMma = 1, kWarpSplit0 = 2, kWarpPanel0 = 10, kWarpEpi0 = 12;

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

__device__ __forceinline__ void tc_mma_ts2(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// commit to the same barrier (shared-memory offset) in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((unsigned short)3)
      : "memory");
}

// arrive on the barrier at the same offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}

// wait with cluster-scope acquire (arrivals come from both CTAs of a pair)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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

// 32 lanes x 8 consecutive 32-bit columns per warp
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

// TRANS = false: Y = A X; TRANS = true: Z = A^T W. P = output rows of the
// pass (m or n); nt = K tiles per output tile.
//
// Rings: stage ring in shared memory (one TMA stage = raw fp32 A tile + the
// matching raw panel tile), released once the A-splitting warps hold their
// rows in registers and the panel warp has split the panel tile, so nearly
// the whole ring is outstanding DRAM traffic; split panel ring (K-major SW128
// [hi; lo]) released by the MMA commit; TMEM ring of split A tiles (hi and lo,
// 32 columns each, lane = output row) filled with tcgen05.st and consumed by
// A-from-TMEM MMAs; double-buffered TMEM accumulators.
// Split-K launches reduce shared output tiles with red.global.add, so the
// output must start at zero: every CTA zeroes its slice of rows at start-up
// and counts itself in `arrived`; an epilogue polls the count before its
// first reduction (long satisfied by then). The last CTA to finish resets
// the pair for the next launch that draws this slot.
struct ZSync {
  unsigned arrived, finished;
};

//
// PAIR: a cluster of two CTAs on one TPC shares every MMA (cta_group::2,
// M = 256): each CTA splits its own 128 rows of A into its own TMEM and
// provides half of each B operand ([X_hi | X_lo]: CTA 0 the hi columns, CTA 1
// the lo columns; X_hi for the correction MMA: one half each), CTA 0 issues
// the MMAs and commits to both CTAs' barriers. Half the MMA instructions and
// half the panel splitting per SM.
template <int S, bool TRANS, bool PAIR>
__global__ void __launch_bounds__(TcCfg<S, TRANS, PAIR>::THREADS, 1)
    pass_tc(const __grid_constant__ TmaDesc tA, const __grid_constant__ TmaDesc tB, float* __restrict__ out,
            int64_t P, int nt, int64_t nblocks, int whole, ZSync* __restrict__ zs) {
  using C = TcCfg<S, TRANS, PAIR>;
  constexpr int CW = PAIR ? 2 : 1;          // CTAs per work item
  constexpr int TILE_ROWS = CW * BMT;       // output rows per work item
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sP = smem + C::ST * C::STAGE;                 // [SSP][BSPL]
  uint64_t* full = (uint64_t*)(sP + C::SSP * C::BSPL);         // [ST] stage landed
  uint64_t* empty = full + C::ST;                              // [ST] stage consumed by all splitters
  uint64_t* pfull = empty + C::ST;                             // [SSP] split panel ready
  uint64_t* mdone = pfull + C::SSP;                            // [MD] MMAs of K tile j retired
  uint64_t* afull = mdone + C::MD;                             // [AST] split A in TMEM
  uint64_t* tfull = afull + C::AST;                            // [2] accumulator ready
  uint64_t* tempty = tfull + 2;                                // [2] accumulator drained
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? (blockIdx.x & 1) : 0;  // cluster dims (2, 1, 1)
  const int64_t U = nblocks * nt, G = gridDim.x / CW, b = blockIdx.x / CW;
  const int64_t u0 = whole ? (b * nblocks / G) * nt : b * U / G;
  const int64_t u1 = whole ? ((b + 1) * nblocks / G) * nt : (b + 1) * U / G;
  const int64_t ntiles = u1 - u0;
  if (!PAIR && ntiles <= 0) return;  // (pairs always have work: grid <= units)
  TC_SPAN(0);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tA);
    prefetch_tmap(&tB);
    for (int s = 0; s < C::ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NSPLIT + C::NPW);
    }
    for (int s = 0; s < C::SSP; ++s) {
      mbar_init(&pfull[s], CW * C::NPW);
    }
    for (int s = 0; s < C::AST; ++s) mbar_init(&afull[s], CW * C::NSPLIT);
    for (int s = 0; s < C::MD; ++s) mbar_init(&mdone[s], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], CW * C::NEPI);
    }
    fence_barrier_init();
  }
  if (warp == kWarpMma) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  // programmatic dependent launch: everything above overlapped the tail of
  // the previous kernel in the stream; its outputs are visible from here on
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (zs != nullptr) {
    const int64_t z0 = blockIdx.x * P / gridDim.x, z1 = (blockIdx.x + 1) * P / gridDim.x;
    float4* o4 = reinterpret_cast<float4*>(out + z0 * S);
    for (int64_t i = threadIdx.x; i < (z1 - z0) * S / 4; i += blockDim.x) o4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  tc_fence_before();
  if constexpr (PAIR)
    cluster_sync();  // both CTAs' barriers initialised before any remote arrival
  else
    __syncthreads();
  tc_fence_after();
  if (zs != nullptr && threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&zs->arrived, 1u);
  }
  const uint32_t tmem = *tmem_slot;

  // Every role walks the same unit sequence u0..u1-1 with incremental
  // (output tile, K tile) and ring (slot, phase) counters: no 64-bit
  // division and no dynamically indexed arrays in the steady-state loops.
  const int64_t ob0 = u0 / nt;
  const int kt0 = (int)(u0 - ob0 * nt);

  if (warp == kWarpTma) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      Ring<C::ST> r;
      int64_t ob = ob0;
      int kt = kt0;
      for (int64_t it = 0; it < ntiles; ++it) {
        if (it >= C::ST) mbar_wait(&empty[r.i], r.ph ^ 1);
        TC_TRACE(0);
        unsigned char* dst = smem + r.i * C::STAGE;
        mbar_arrive_expect_tx(&full[r.i], C::STAGE);
        const int row0 = (int)(ob * TILE_ROWS + rank * BMT);  // this CTA's 128 output rows
        if (!TRANS)  // A rows [row0, +128), cols [kt*32, +32): K-major SW128
          tma_load_2d(dst, &tA, &full[r.i], kt * BKT, row0);
        else         // A rows [kt*32, +32) (K), cols [row0, +128) (M): row-major
          tma_load_2d(dst, &tA, &full[r.i], row0, kt * BKT);
        // panel rows [kt*32, +32) (K), all S columns: row-major [32][S]
        tma_load_2d(dst + C::ABYTES, &tB, &full[r.i], 0, kt * BKT);
        r.next();
        if (++kt == nt) {
          kt = 0;
          ++ob;
        }
      }
    }
  } else if (warp >= kWarpEpi0) {
    // ---------------- epilogue (warps 12.., one output row x 32 columns each) ----------------
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
        if (lane == 0) {
          if (PAIR && rank != 0)
            mbar_arrive_remote(&tempty[racc.i], 0);
          else
            mbar_arrive(&tempty[racc.i]);
        }
        racc.next();
      }
      if (tile_end) {
        const int64_t t0 = ob * nt;  // first unit of this output tile
        const bool owned = (t0 >= u0) && (t0 + nt <= u1);
        const int64_t row = ob * TILE_ROWS + rank * BMT + row_in_tile;
        if (!owned && zs != nullptr) {  // every CTA's zeroing must have landed
          if (lane == 0) {
            unsigned v;
            do {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&zs->arrived) : "memory");
            } while (v < gridDim.x);
          }
          __syncwarp();
        }
        if (row < P) {
          float* dst = out + row * S + cg;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            if (owned)
              *(float4*)(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
            else
              red_add_v4(dst + j, acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
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
  } else if (warp >= kWarpPanel0) {
    // ---------------- panel splitters: raw [32 k][S] -> K-major SW128 [hi; lo] ----------------
    // panel warp p covers units p * PU .. p * PU + PU - 1; unit u = columns
    // [32 (u >> 1), +32) x k half u & 1
    const int pw = warp - kWarpPanel0;
    Ring<C::ST> r;
    Ring<C::SSP> rp;
    Ring<C::MD> rd;  // tracks K tile it - SSP (the previous user of slot rp.i)
    for (int64_t it = 0; it < ntiles; ++it) {
      mbar_wait(&full[r.i], r.ph);
      if (threadIdx.x == 32 * kWarpPanel0) TC_TRACE(7);
      const float* raw = (const float*)(smem + r.i * C::STAGE + C::ABYTES);
      float h[C::PU][16], l[C::PU][16];
#pragma unroll
      for (int t = 0; t < C::PU; ++t) {
        const int u = pw * C::PU + t;
        const int n = 32 * (u >> 1) + lane;  // lanes read consecutive columns
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float v = raw[(16 * (u & 1) + k) * S + n];
          h[t][k] = tf32_rn(v);
          l[t][k] = tf32_rn(v - h[t][k]);
        }
      }
      __syncwarp();
      if (threadIdx.x == 32 * kWarpPanel0) TC_TRACE(10);
      if (lane == 0) mbar_arrive(&empty[r.i]);
      if (it >= C::SSP) {
        mbar_wait(&mdone[rd.i], rd.ph);
        rd.next();
      }
      if (threadIdx.x == 32 * kWarpPanel0) TC_TRACE(11);
      unsigned char* dst = sP + rp.i * C::BSPL;
#pragma unroll
      for (int t = 0; t < C::PU; ++t) {
        const int u = pw * C::PU + t;
        const int n = 32 * (u >> 1) + lane;  // output column = operand row
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int c = 4 * (u & 1) + cc;
          const uint32_t off = (uint32_t)n * 128 + ((c ^ (n & 7)) << 4);
          const float4 hv = make_float4(h[t][4 * cc], h[t][4 * cc + 1], h[t][4 * cc + 2], h[t][4 * cc + 3]);
          const float4 lv = make_float4(l[t][4 * cc], l[t][4 * cc + 1], l[t][4 * cc + 2], l[t][4 * cc + 3]);
          if constexpr (PAIR) {
            // B of the [hi | lo] MMA: CTA 0 holds the hi rows, CTA 1 the lo rows;
            // B of the correction MMA (X_hi): rows [rank S/2, +S/2) of X_hi
            *(float4*)(dst + off) = rank == 0 ? hv : lv;
            const int n2 = n - (int)rank * (S / 2);
            if (n2 >= 0 && n2 < S / 2) {
              const uint32_t off2 = (uint32_t)n2 * 128 + ((c ^ (n2 & 7)) << 4);
              *(float4*)(dst + S * 128 + off2) = hv;
            }
          } else {
            *(float4*)(dst + off) = hv;
            *(float4*)(dst + S * 128 + off) = lv;
          }
        }
      }
      if (threadIdx.x == 32 * kWarpPanel0) TC_TRACE(12);
      fence_proxy_async();  // generic-proxy stores -> tensor-core (async proxy) reads
      __syncwarp();
      if (lane == 0) {
        if (PAIR && rank != 0)
          mbar_arrive_remote(&pfull[rp.i], 0);
        else
          mbar_arrive(&pfull[rp.i]);
      }
      if (threadIdx.x == 32 * kWarpPanel0) TC_TRACE(9);
      r.next();
      rp.next();
    }
  } else if (warp == kWarpMma) {
    // ---------------- MMA issuer (CTA 0 of a pair) ----------------
    if (PAIR && rank != 0) goto done;
    constexpr uint32_t idesc_cat = idesc_tf32(2 * S, false, false, CW * BMT);
    constexpr uint32_t idesc_hi = idesc_tf32(S, false, false, CW * BMT);
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
      if constexpr (PAIR) {
        if (block_start && racc.wrapped) mbar_wait_cluster(&tempty[racc.i], racc.ph ^ 1);
        mbar_wait_cluster(&pfull[rp.i], rp.ph);
        mbar_wait_cluster(&afull[ra.i], ra.ph);
      } else {
        if (block_start && racc.wrapped) mbar_wait(&tempty[racc.i], racc.ph ^ 1);
        mbar_wait(&pfull[rp.i], rp.ph);
        mbar_wait(&afull[ra.i], ra.ph);
      }
      tc_fence_after();
      if (lane == 0) TC_TRACE(4);
      if (elect_one()) {
        const uint32_t sb = smem_u32(sP + rp.i * C::BSPL);        // K-major SW128 [hi; lo]
        const uint32_t ahi = tmem + C::A_COL0 + ra.i * 2 * BKT;   // split A in TMEM
        const uint32_t alo = ahi + BKT;
        const uint32_t dcat = tmem + racc.i * C::ACC_COLS;
        const uint32_t dlo = dcat + S;
#pragma unroll
        for (int k = 0; k < BKT / 8; ++k) {
          const uint64_t bcat = smem_desc(sb + 32 * k, 16, 1024);  // 8 tf32 = 32 B per K step
          const uint32_t acc = (block_start && k == 0) ? 0u : 1u;
          if constexpr (PAIR) {
            const uint64_t bhi = smem_desc(sb + S * 128 + 32 * k, 16, 1024);
            tc_mma_ts2(dcat, ahi + 8 * k, bcat, idesc_cat, acc);  // [A_hi X_hi | A_hi X_lo]
            tc_mma_ts2(dlo, alo + 8 * k, bhi, idesc_hi, 1u);      //            + A_lo X_hi
          } else {
            tc_mma_ts(dcat, ahi + 8 * k, bcat, idesc_cat, acc);  // [A_hi X_hi | A_hi X_lo]
            tc_mma_ts(dlo, alo + 8 * k, bcat, idesc_hi, 1u);     //            + A_lo X_hi
          }
        }
        if constexpr (PAIR) {
          tc_commit_pair(&mdone[rd.i]);  // releases the panel slot and the TMEM A slot in both CTAs
          if (block_end) tc_commit_pair(&tfull[racc.i]);
        } else {
          tc_commit(&mdone[rd.i]);  // one commit releases the split panel and the TMEM A slot
          if (block_end) tc_commit(&tfull[racc.i]);
        }
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
  } else {
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
      if (!TRANS) {
        // row r of the K-major SW128 tile: 16 B chunk c at chunk c ^ (r & 7)
        const unsigned char* rowp = smem + r.i * C::STAGE + row_in_tile * 128;
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
        const float* raw = (const float*)(smem + r.i * C::STAGE) + row_in_tile;
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
      if (lane == 0) {
        if (PAIR && rank != 0)
          mbar_arrive_remote(&afull[ra.i], 0);
        else
          mbar_arrive(&afull[ra.i]);
      }
      if (threadIdx.x == 64) TC_TRACE(3);
      r.next();
      ra.next();
    }
  }
done:
  tc_fence_before();
  if constexpr (PAIR)
    cluster_sync();  // the peer's TMEM and barriers stay alive until CTA 0's MMAs retired
  else
    __syncthreads();
  tc_fence_after();
  TC_SPAN(1);
  if (zs != nullptr && threadIdx.x == 0 && atomicAdd(&zs->finished, 1u) == gridDim.x - 1) {
    zs->arrived = 0u;
    zs->finished = 0u;
  }
  if (warp == kWarpMma)
  {
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
}

// CTA-pair (cta_group::2) kernels are opt-in (CNMF_TC_PAIR=1): correct (same
// parity tests), but measured slower on B200 -- every cross-CTA arrival with
// cluster-scope release costs ~1500 cycles on the peer's critical path, and
// the peer's panel splitting does not shrink -- 400 us vs 170 us for a
// 20000 x 10000 forward pass (tools/tc_trace.cu with CNMF_TC_TRACE_CTA=1).
static int g_pair_mode = -1;

template <int S, bool TRANS, bool PAIR>
int launch_tc_t(const float* A, int64_t m, int64_t n, int64_t lda, const float* Bpanel, float* out, cudaStream_t st) {
  using C = TcCfg<S, TRANS, PAIR>;
  constexpr int CW = PAIR ? 2 : 1;
  // skinny operand rows = K extent: n (forward, X) or m (transpose, W)
  const int64_t brows = TRANS ? m : n;
  TmaDesc tA, tB;
  if (!TRANS)
    CNMF_TRY(make_tma_2d(&tA, A, 4, m, n, lda, BKT, BMT, true));
  else
    CNMF_TRY(make_tma_2d(&tA, A, 4, m, n, lda, BMT, BKT, false));
  CNMF_TRY(make_tma_2d(&tB, Bpanel, 4, brows, S, S, S, BKT, false));
  const int64_t P = TRANS ? n : m;   // output rows
  const int nt = (int)ceil_div(brows, BKT);
  const int64_t nblocks = ceil_div(P, CW * BMT);  // work items of CW x 128 output rows
  const int64_t slots = kNumSMs / CW;             // CTAs (pairs) per wave
  const int whole = nblocks >= 16 * slots;
  const int64_t grid = CW * std::min<int64_t>(slots, whole ? nblocks : nblocks * nt);
  ZSync* zs = nullptr;
  if (!whole) {
    static ZSync* ring = nullptr;
    static unsigned next = 0;
    if (ring == nullptr) {
      CNMF_CUDA(cudaMalloc(&ring, 64 * sizeof(ZSync)));
      CNMF_CUDA(cudaMemset(ring, 0, 64 * sizeof(ZSync)));
    }
    zs = ring + (next++ % 64);
  }
  static bool attr = false;
  if (!attr) {
    CNMF_CUDA(cudaFuncSetAttribute(pass_tc<S, TRANS, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)C::SMEM));
    if (PAIR) CNMF_CUDA(cudaFuncSetAttribute(pass_tc<S, TRANS, PAIR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
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
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = CW;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = PAIR ? 2 : 1;
  CNMF_CUDA(cudaLaunchKernelEx(&lc, pass_tc<S, TRANS, PAIR>, tA, tB, out, P, nt, nblocks, whole, zs));
  CNMF_LAUNCH_CHECK();
  if (e0) {
    CNMF_CUDA(cudaEventRecord(e1, st));
    pass_record(e0, e1, 4.0 * ((double)m * n + (double)n * S + (double)m * S));
  }
  return CNMF_OK;
}

template <int S, bool TRANS>
int launch_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* Bpanel, float* out, cudaStream_t st) {
  if (g_pair_mode < 0) {
    const char* e = getenv("CNMF_TC_PAIR");
    g_pair_mode = (e && e[0] == '1') ? 1 : 0;
  }
  if (g_pair_mode) return launch_tc_t<S, TRANS, true>(A, m, n, lda, Bpanel, out, st);
  return launch_tc_t<S, TRANS, false>(A, m, n, lda, Bpanel, out, st);
}

// ---------------------------------------------------------------------------
// Paired pass: Y = A X (unit range 0) and Z = A^T W (unit range 1) in ONE
// launch. The two range finders of the compressed NMF need exactly one
// forward and one transpose pass per power step; a single launch pays the
// pipeline ramp-up and tail once per step instead of twice. Every role walks
// the concatenated unit sequence; the direction (A tile layout, panel,
// output) is a per-tile runtime switch, the pipeline is the same as pass_tc.
// ---------------------------------------------------------------------------
struct PassSide {
  float* out;
  int64_t P;        // output rows
  int64_t nblocks;  // 128-row output tiles
  int nt;           // K tiles per output tile
};

// the (pass, output tile, K tile) walk of one CTA's units: [lo0, hi0) of
// pass 0, then [lo1, hi1) of pass 1 (unit indices local to each pass; plain
// scalars, no indexed arrays, so nothing lands in local memory)
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

// NS A-splitting warps (8: two per TMEM lane quarter, 16 K values each; 16:
// four per quarter, 8 K values each)
template <int NS>
struct PairWarps {
  static constexpr int kSplit0 = 2, kPanel0 = 2 + NS, kEpi0 = 4 + NS, KP = 128 / NS;
};

template <int S, int NS>
__global__ void __launch_bounds__(32 * (4 + NS + 4 * (S / 32)), 1)
    pass_tc_pair(const __grid_constant__ TmaDesc tAf, const __grid_constant__ TmaDesc tX,
                 const __grid_constant__ TmaDesc tAt, const __grid_constant__ TmaDesc tW, const PassSide s0,
                 const PassSide s1, ZSync* __restrict__ zs) {
  using C = TcCfg<S, false, false>;
  using PW = PairWarps<NS>;
  constexpr int kWarpSplit0 = PW::kSplit0, kWarpPanel0 = PW::kPanel0, kWarpEpi0 = PW::kEpi0, KP = PW::KP;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sP = smem + C::ST * C::STAGE;                 // [SSP][BSPL]
  uint64_t* full = (uint64_t*)(sP + C::SSP * C::BSPL);         // [ST] stage landed
  uint64_t* empty = full + C::ST;                              // [ST] stage consumed by all splitters
  uint64_t* pfull = empty + C::ST;                             // [SSP] split panel ready
  uint64_t* mdone = pfull + C::SSP;                            // [MD] MMAs of K tile j retired
  uint64_t* afull = mdone + C::MD;                             // [AST] split A in TMEM
  uint64_t* tfull = afull + C::AST;                            // [2] accumulator ready
  uint64_t* tempty = tfull + 2;                                // [2] accumulator drained
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the concatenated unit sequence (pass 0, then pass 1) is split over the
  // CTAs: the two passes run concurrently on two halves of the GPU and share
  // A through L2 (measured better than every CTA taking a share of each)
  const int64_t U0 = s0.nblocks * s0.nt, U1 = s1.nblocks * s1.nt, G = gridDim.x, b = blockIdx.x;
  const int64_t u0 = b * (U0 + U1) / G, u1 = (b + 1) * (U0 + U1) / G;
  const int64_t lo0 = u0 < U0 ? u0 : U0, hi0 = u1 < U0 ? u1 : U0;
  const int64_t lo1 = u0 > U0 ? u0 - U0 : 0, hi1 = u1 > U0 ? u1 - U0 : 0;
  const int64_t ntiles = (hi0 - lo0) + (hi1 - lo1);  // >= 1: the grid never exceeds the units

  if (threadIdx.x == 0) {
    prefetch_tmap(&tAf);
    prefetch_tmap(&tX);
    prefetch_tmap(&tAt);
    prefetch_tmap(&tW);
    for (int s = 0; s < C::ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NS + C::NPW);
    }
    for (int s = 0; s < C::SSP; ++s) mbar_init(&pfull[s], C::NPW);
    for (int s = 0; s < C::AST; ++s) mbar_init(&afull[s], NS);
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
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // split-K outputs start at zero: every CTA zeroes a row slice of both
  for (int q = 0; q < 2; ++q) {
    const PassSide& sd = q ? s1 : s0;
    const int64_t z0 = blockIdx.x * sd.P / gridDim.x, z1 = (blockIdx.x + 1) * sd.P / gridDim.x;
    float4* o4 = reinterpret_cast<float4*>(sd.out + z0 * S);
    for (int64_t i = threadIdx.x; i < (z1 - z0) * S / 4; i += blockDim.x) o4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
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
        if (it >= C::ST) mbar_wait(&empty[r.i], r.ph ^ 1);
        unsigned char* dst = smem + r.i * C::STAGE;
        mbar_arrive_expect_tx(&full[r.i], C::STAGE);
        const int row0 = (int)(w.ob * BMT);
        if (w.p == 0) {  // A rows [row0, +128), cols [kt*32, +32): K-major SW128; X rows [kt*32, +32)
          tma_load_2d(dst, &tAf, &full[r.i], w.kt * BKT, row0);
          tma_load_2d(dst + C::ABYTES, &tX, &full[r.i], 0, w.kt * BKT);
        } else {  // A rows [kt*32, +32) (K), cols [row0, +128) (M): row-major; W rows [kt*32, +32)
          tma_load_2d(dst, &tAt, &full[r.i], row0, w.kt * BKT);
          tma_load_2d(dst + C::ABYTES, &tW, &full[r.i], 0, w.kt * BKT);
        }
        r.next();
        w.next(s0, s1);
      }
    }
  } else if (warp >= kWarpEpi0) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;
    const int cg = 32 * ((warp - kWarpEpi0) >> 2);
    const int row_in_tile = 32 * q + lane;
    Ring<2> racc;
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.f;
    Walk w;
    w.start(lo0, hi0, lo1, hi1, s0, s1);
    for (int64_t it = 0; it < ntiles; ++it) {
      const int nt = w.p ? s1.nt : s0.nt;
      const bool tile_end = w.last() || (w.kt == nt - 1);
      if (tile_end || ((w.kt + 1) % C::KB == 0)) {
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
        const PassSide& sd = w.p ? s1 : s0;
        const bool owned = w.owned(nt);
        const int64_t row = w.ob * BMT + row_in_tile;
        if (!owned) {  // every CTA's zeroing must have landed
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
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            if (owned)
              *(float4*)(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
            else
              red_add_v4(dst + j, acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      }
      w.next(s0, s1);
    }
  } else if (warp >= kWarpPanel0) {
    // ---------------- panel splitters (direction-independent) ----------------
    const int pw = warp - kWarpPanel0;
    Ring<C::ST> r;
    Ring<C::SSP> rp;
    Ring<C::MD> rd;
    for (int64_t it = 0; it < ntiles; ++it) {
      mbar_wait(&full[r.i], r.ph);
      const float* raw = (const float*)(smem + r.i * C::STAGE + C::ABYTES);
      float h[C::PU][16], l[C::PU][16];
#pragma unroll
      for (int t = 0; t < C::PU; ++t) {
        const int u = pw * C::PU + t;
        const int n = 32 * (u >> 1) + lane;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float v = raw[(16 * (u & 1) + k) * S + n];
          h[t][k] = tf32_rn(v);
          l[t][k] = tf32_rn(v - h[t][k]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[r.i]);
      if (it >= C::SSP) {
        mbar_wait(&mdone[rd.i], rd.ph);
        rd.next();
      }
      unsigned char* dst = sP + rp.i * C::BSPL;
#pragma unroll
      for (int t = 0; t < C::PU; ++t) {
        const int u = pw * C::PU + t;
        const int n = 32 * (u >> 1) + lane;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int c = 4 * (u & 1) + cc;
          const uint32_t off = (uint32_t)n * 128 + ((c ^ (n & 7)) << 4);
          *(float4*)(dst + off) = make_float4(h[t][4 * cc], h[t][4 * cc + 1], h[t][4 * cc + 2], h[t][4 * cc + 3]);
          *(float4*)(dst + S * 128 + off) =
              make_float4(l[t][4 * cc], l[t][4 * cc + 1], l[t][4 * cc + 2], l[t][4 * cc + 3]);
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pfull[rp.i]);
      r.next();
      rp.next();
    }
  } else if (warp == kWarpMma) {
    // ---------------- MMA issuer (direction-independent) ----------------
    constexpr uint32_t idesc_cat = idesc_tf32(2 * S, false, false);
    constexpr uint32_t idesc_hi = idesc_tf32(S, false, false);
    Ring<C::SSP> rp;
    Ring<C::AST> ra;
    Ring<C::MD> rd;
    Ring<2> racc;
    Walk w;
    w.start(lo0, hi0, lo1, hi1, s0, s1);
    bool block_start = true;
    for (int64_t it = 0; it < ntiles; ++it) {
      const int nt = w.p ? s1.nt : s0.nt;
      const bool tile_end = w.last() || (w.kt == nt - 1);
      const bool block_end = tile_end || ((w.kt + 1) % C::KB == 0);
      if (block_start && racc.wrapped) mbar_wait(&tempty[racc.i], racc.ph ^ 1);
      mbar_wait(&pfull[rp.i], rp.ph);
      mbar_wait(&afull[ra.i], ra.ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sb = smem_u32(sP + rp.i * C::BSPL);
        const uint32_t ahi = tmem + C::A_COL0 + ra.i * 2 * BKT;
        const uint32_t alo = ahi + BKT;
        const uint32_t dcat = tmem + racc.i * C::ACC_COLS;
        const uint32_t dlo = dcat + S;
#pragma unroll
        for (int k = 0; k < BKT / 8; ++k) {
          const uint64_t bcat = smem_desc(sb + 32 * k, 16, 1024);
          const uint32_t acc = (block_start && k == 0) ? 0u : 1u;
          tc_mma_ts(dcat, ahi + 8 * k, bcat, idesc_cat, acc);  // [A_hi X_hi | A_hi X_lo]
          tc_mma_ts(dlo, alo + 8 * k, bcat, idesc_hi, 1u);     //            + A_lo X_hi
        }
        tc_commit(&mdone[rd.i]);
        if (block_end) tc_commit(&tfull[racc.i]);
      }
      __syncwarp();
      rp.next();
      ra.next();
      rd.next();
      block_start = block_end;
      if (block_end) racc.next();
      w.next(s0, s1);
    }
  } else {
    // ---------------- A splitters: per-tile direction ----------------
    // warp w serves TMEM lane quarter w & 3 and K part (w - 2) / 4 (KP values)
    const int q = warp & 3;
    const int part = (warp - kWarpSplit0) >> 2;
    const int row_in_tile = 32 * q + lane;
    Ring<C::ST> r;
    Ring<C::AST> ra;
    Ring<C::MD> rd;
    Walk w;
    w.start(lo0, hi0, lo1, hi1, s0, s1);
    for (int64_t it = 0; it < ntiles; ++it) {
      mbar_wait(&full[r.i], r.ph);
      float hi[KP], lo[KP];
      if (w.p == 0) {
        const unsigned char* rowp = smem + r.i * C::STAGE + row_in_tile * 128;
#pragma unroll
        for (int cc = 0; cc < KP / 4; ++cc) {
          const int c = (KP / 4) * part + cc;
          const float4 v = *(const float4*)(rowp + ((c ^ (row_in_tile & 7)) << 4));
          hi[4 * cc + 0] = v.x;
          hi[4 * cc + 1] = v.y;
          hi[4 * cc + 2] = v.z;
          hi[4 * cc + 3] = v.w;
        }
      } else {
        const float* raw = (const float*)(smem + r.i * C::STAGE) + row_in_tile;
#pragma unroll
        for (int k = 0; k < KP; ++k) hi[k] = raw[(KP * part + k) * BMT];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[r.i]);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const float v = hi[k];
        hi[k] = tf32_rn(v);
        lo[k] = tf32_rn(v - hi[k]);
      }
      if (it >= C::AST) {
        mbar_wait(&mdone[rd.i], rd.ph);
        rd.next();
      }
      tc_fence_after();
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + C::A_COL0 + ra.i * 2 * BKT + KP * part;
      if constexpr (KP == 16) {
        tmem_st16(ta, *reinterpret_cast<const float(*)[16]>(hi));
        tmem_st16(ta + BKT, *reinterpret_cast<const float(*)[16]>(lo));
      } else {
        tmem_st8(ta, hi);
        tmem_st8(ta + BKT, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ra.i]);
      r.next();
      ra.next();
      w.next(s0, s1);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0 && atomicAdd(&zs->finished, 1u) == gridDim.x - 1) {
    zs->arrived = 0u;
    zs->finished = 0u;
  }
  if (warp == kWarpMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

#ifndef CNMF_PAIR_NSPLIT
#define CNMF_PAIR_NSPLIT 8
#endif

template <int S>
int launch_pair(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, const float* W, float* Z,
                cudaStream_t st) {
  using C = TcCfg<S, false, false>;
  TmaDesc tAf, tX, tAt, tW;
  CNMF_TRY(make_tma_2d(&tAf, A, 4, m, n, lda, BKT, BMT, true));
  CNMF_TRY(make_tma_2d(&tAt, A, 4, m, n, lda, BMT, BKT, false));
  CNMF_TRY(make_tma_2d(&tX, X, 4, n, S, S, S, BKT, false));
  CNMF_TRY(make_tma_2d(&tW, W, 4, m, S, S, S, BKT, false));
  const PassSide s0{Y, m, ceil_div(m, BMT), (int)ceil_div(n, BKT)};
  const PassSide s1{Z, n, ceil_div(n, BMT), (int)ceil_div(m, BKT)};
  const int64_t U = s0.nblocks * s0.nt + s1.nblocks * s1.nt;
  const int64_t grid = std::min<int64_t>(kNumSMs, U);
  static ZSync* ring = nullptr;
  static unsigned next = 0;
  if (ring == nullptr) {
    CNMF_CUDA(cudaMalloc(&ring, 64 * sizeof(ZSync)));
    CNMF_CUDA(cudaMemset(ring, 0, 64 * sizeof(ZSync)));
  }
  ZSync* zs = ring + (next++ % 64);
  static bool attr = false;
  if (!attr) {
    CNMF_CUDA(cudaFuncSetAttribute(pass_tc_pair<S, CNMF_PAIR_NSPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
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
  lc.blockDim = dim3(32 * (4 + CNMF_PAIR_NSPLIT + 4 * (S / 32)));
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  CNMF_CUDA(cudaLaunchKernelEx(&lc, pass_tc_pair<S, CNMF_PAIR_NSPLIT>, tAf, tX, tAt, tW, s0, s1, zs));
  CNMF_LAUNCH_CHECK();
  if (e0) {
    CNMF_CUDA(cudaEventRecord(e1, st));
    // bytes of two passes: A twice plus the four panels
    pass_record(e0, e1, 2.0 * 4.0 * ((double)m * n + (double)n * S + (double)m * S));
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

// Y = A X and Z = A^T W in one launch (tensor-core path, panel widths 32/64)
int pass_pair_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, const float* W, float* Z,
                 int S, cudaStream_t st) {
  switch (S) {
    case 32: return launch_pair<32>(A, m, n, lda, X, Y, W, Z, st);
    case 64: return launch_pair<64>(A, m, n, lda, X, Y, W, Z, st);
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
