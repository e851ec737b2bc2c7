// Streaming passes over A on the 5th-generation tensor cores (tcgen05,
// kind::tf32) with a 3xTF32 split for fp32-level accuracy:
//
//   A X ~= A_hi X_hi + A_hi X_lo + A_lo X_hi,   v_hi = v with the low 13
//   mantissa bits cleared (exactly representable in tf32), v_lo = v - v_hi.
//
// Forward pass  Y = A X   (M = rows of A, K = columns of A, N = s)
// Transpose     Z = A^T W (M = columns of A, K = rows of A, N = s)
//
// Warp roles (224 threads): warp 0 issues TMA (A tile, 128B swizzle, plus the
// [X_hi | X_lo] panel tile), warp 1 owns TMEM and issues the MMAs (one
// elected thread), warps 2..5 split each landed A tile in shared memory into
// hi (in place) and lo (second buffer) and, at the end of every output tile,
// drain the fp32 accumulator from TMEM (tcgen05.ld) and write the rows.
// The accumulator is [A_hi X_hi | A_hi X_lo + A_lo X_hi] (N = 2s columns,
// double buffered in TMEM); the epilogue adds the two halves.
// kind::tf32 only accepts K-major operands on sm_100a (the transpose bit
// yields zeros; measured), so every operand is presented K-major: the
// forward A tile comes K-major straight from TMA (SW128) and is split in
// place; the transpose-pass A tile (row-major, i.e. MN-major for A^T) is
// transposed by the splitting warps into K-major SW128 hi/lo tiles; the skinny
// panel is pre-split and stored transposed ([hi; lo] rows, K contiguous).
// Work is distributed exactly like the FFMA passes (contiguous unit ranges,
// flush on tile change, red.global.add when a tile is shared).
#include <algorithm>

#include "common.cuh"

namespace cnmf {
namespace {

constexpr int kTcThreads = 192;       // warps 0..5
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

__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32 consecutive fp32 columns per warp (one column per register)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
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
__host__ __device__ constexpr uint32_t idesc_tf32(int n, bool a_mn_major, bool b_mn_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BMT >> 4) << 24);
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <int S, bool TRANS>
struct TcCfg {
  static constexpr int ABYTES = BMT * BKT * 4;        // 16 KB
  static constexpr int BBYTES = BKT * 2 * S * 4;      // [hi; lo] panel tile: 8 or 16 KB
  // forward: A (split to hi in place) + lo + B; transpose: raw A + hi + lo + B
  static constexpr int STAGE = (TRANS ? 3 : 2) * ABYTES + BBYTES;
  static constexpr int ST = (int)((200 * 1024) / STAGE) < 6 ? (int)((200 * 1024) / STAGE) : 6;
  static constexpr int ACC_COLS = 2 * S;              // per accumulator buffer
  static constexpr int TMEM_COLS = (4 * S <= 128) ? 128 : 256;
  static constexpr size_t SMEM = 1024 + (size_t)ST * STAGE + 256;
};

// TRANS = false: Y = A X (A tile K-major); TRANS = true: Z = A^T W (A tile
// MN-major). P = output rows of the pass (m or n); NT = K tiles per output tile.
template <int S, bool TRANS>
__global__ void __launch_bounds__(kTcThreads, 1)
    pass_tc(const __grid_constant__ TmaDesc tA, const __grid_constant__ TmaDesc tB, float* __restrict__ out,
            int64_t P, int nt, int64_t nblocks, int whole) {
  using C = TcCfg<S, TRANS>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + C::ST * C::STAGE);
  uint64_t* conv = full + C::ST;
  uint64_t* empty = conv + C::ST;
  uint64_t* tfull = empty + C::ST;   // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t U = nblocks * nt, G = gridDim.x, b = blockIdx.x;
  const int64_t u0 = whole ? (b * nblocks / G) * nt : b * U / G;
  const int64_t u1 = whole ? ((b + 1) * nblocks / G) * nt : (b + 1) * U / G;
  const int64_t ntiles = u1 - u0;
  if (ntiles <= 0) return;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tA);
    prefetch_tmap(&tB);
    for (int s = 0; s < C::ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      for (int64_t it = 0; it < ntiles; ++it) {
        const int stage = (int)(it % C::ST);
        if (it >= C::ST) mbar_wait(&empty[stage], (uint32_t)(((it / C::ST) - 1) & 1));
        const int64_t u = u0 + it;
        const int64_t ob = u / nt;          // output tile
        const int kt = (int)(u - ob * nt);  // K tile
        unsigned char* sa = smem + stage * C::STAGE;
        unsigned char* sb = sa + (TRANS ? 3 : 2) * C::ABYTES;
        mbar_arrive_expect_tx(&full[stage], C::ABYTES + C::BBYTES);
        if (!TRANS) {
          // A rows [ob*128, +128), cols [kt*32, +32): K-major SW128
          tma_load_2d(sa, &tA, &full[stage], kt * BKT, (int)(ob * BMT));
        } else {
          // A rows [kt*32, +32) (K), cols [ob*128, +128) (M): row-major, no swizzle
          tma_load_2d(sa, &tA, &full[stage], (int)(ob * BMT), kt * BKT);
        }
        // transposed panel: rows [0, 2S) = [hi; lo] output columns, K cols [kt*32, +32)
        tma_load_2d(sb, &tB, &full[stage], kt * BKT, 0);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc_cat = idesc_tf32(2 * S, false, false);
    constexpr uint32_t idesc_hi = idesc_tf32(S, false, false);
    int buf = 0;
    uint32_t tphase[2] = {0, 0};
    bool first = true;
    for (int64_t it = 0; it < ntiles; ++it) {
      const int stage = (int)(it % C::ST);
      const int64_t u = u0 + it;
      const bool tile_start = first || (u % nt == 0);
      const bool tile_end = (it == ntiles - 1) || ((u + 1) % nt == 0);
      // reuse of an accumulator buffer waits until the epilogue drained it
      if (tile_start && tphase[buf] > 0) mbar_wait(&tempty[buf], (tphase[buf] - 1) & 1);
      mbar_wait(&full[stage], (uint32_t)((it / C::ST) & 1));
      mbar_wait(&conv[stage], (uint32_t)((it / C::ST) & 1));
      tc_fence_after();
      if (elect_one()) {
        const uint32_t base = smem_u32(smem + stage * C::STAGE);
        const uint32_t shi = TRANS ? base + C::ABYTES : base;        // K-major SW128 hi tile
        const uint32_t slo = shi + C::ABYTES;                          // K-major SW128 lo tile
        const uint32_t sb = base + (TRANS ? 3 : 2) * C::ABYTES;       // K-major SW128 [hi; lo]
        const uint32_t dcat = tmem + buf * C::ACC_COLS;
        const uint32_t dlo = dcat + S;
#pragma unroll
        for (int k = 0; k < BKT / 8; ++k) {
          // K-major: advance 8 tf32 (32 B) within the 128 B swizzled rows
          const uint64_t ahi = smem_desc(shi + 32 * k, 16, 1024);
          const uint64_t alo = smem_desc(slo + 32 * k, 16, 1024);
          const uint64_t bcat = smem_desc(sb + 32 * k, 16, 1024);
          const uint32_t acc = (tile_start && k == 0) ? 0u : 1u;
          tc_mma(dcat, ahi, bcat, idesc_cat, acc);  // [A_hi X_hi | A_hi X_lo]
          tc_mma(dlo, alo, bcat, idesc_hi, 1u);     //            + A_lo X_hi
        }
        tc_commit(&empty[stage]);
        if (tile_end) tc_commit(&tfull[buf]);
      }
      __syncwarp();
      first = false;
      if (tile_end) {
        tphase[buf] += 1;
        buf ^= 1;
      }
    }
  } else if (warp >= 2 && warp < 6) {
    // ---------------- converter + epilogue (128 threads) ----------------
    const int ct = threadIdx.x - 64;  // 0..127
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    int buf = 0;
    uint32_t tph[2] = {0, 0};
    for (int64_t it = 0; it < ntiles; ++it) {
      const int stage = (int)(it % C::ST);
      const int64_t u = u0 + it;
      mbar_wait(&full[stage], (uint32_t)((it / C::ST) & 1));
      if (!TRANS) {
        // split the landed K-major A tile: hi in place, lo into the second buffer
        float4* a4 = (float4*)(smem + stage * C::STAGE);
        float4* l4 = (float4*)(smem + stage * C::STAGE + C::ABYTES);
#pragma unroll
        for (int j = 0; j < C::ABYTES / 16 / 128; ++j) {
          const int idx = ct + 128 * j;
          const float4 v = a4[idx];
          const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
          a4[idx] = h;
          l4[idx] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        }
      } else {
        // thread ct owns output row (A column) ct: gather its 32 K values from
        // the row-major tile, split, and store them as row ct of K-major SW128
        // hi / lo tiles (16 B chunk c of row r lives at chunk c ^ (r & 7))
        const float* raw = (const float*)(smem + stage * C::STAGE);
        unsigned char* hi = smem + stage * C::STAGE + C::ABYTES;
        unsigned char* lo = hi + C::ABYTES;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e] = raw[(4 * c + e) * BMT + ct];
          const float4 h = make_float4(tf32_hi(v[0]), tf32_hi(v[1]), tf32_hi(v[2]), tf32_hi(v[3]));
          const int off = ct * 128 + ((c ^ (ct & 7)) << 4);
          *(float4*)(hi + off) = h;
          *(float4*)(lo + off) = make_float4(v[0] - h.x, v[1] - h.y, v[2] - h.z, v[3] - h.w);
        }
      }
      fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[stage]);
      const bool tile_end = (it == ntiles - 1) || ((u + 1) % nt == 0);
      if (tile_end) {
        const int64_t ob = u / nt;
        const bool owned = (ob * nt >= u0) && ((ob + 1) * nt <= u1);
        mbar_wait(&tfull[buf], tph[buf] & 1);
        tph[buf] += 1;
        tc_fence_after();
        const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + buf * C::ACC_COLS;
        const int64_t row = ob * BMT + 32 * q + lane;
#pragma unroll
        for (int c0 = 0; c0 < S; c0 += 32) {
          float vh[32], vl[32];
          tmem_ld32(taddr + c0, vh);
          tmem_ld32(taddr + S + c0, vl);
          if (row < P) {
            float* dst = out + row * S + c0;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float x0 = vh[j] + vl[j], x1 = vh[j + 1] + vl[j + 1];
              const float x2 = vh[j + 2] + vl[j + 2], x3 = vh[j + 3] + vl[j + 3];
              if (owned)
                *(float4*)(dst + j) = make_float4(x0, x1, x2, x3);
              else
                red_add_v4(dst + j, x0, x1, x2, x3);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        buf ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
}

// Split an fp32 panel P (rows x S) into the transposed [hi; lo] operand
// PT (2S x ldt): PT[c][r] = hi(P[r][c]), PT[S + c][r] = lo(P[r][c]).
// 32 x 32 tiles through shared memory keep both sides coalesced.
__global__ void split_panel_t(const float* __restrict__ src, int64_t rows, int S, float* __restrict__ dst,
                              int64_t ldt) {
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i;
    tile[i][tx] = (r < rows && c0 + tx < S) ? src[r * S + c0 + tx] : 0.f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int c = c0 + i;
    const int64_t r = r0 + tx;
    if (c < S && r < rows) {
      const float x = tile[tx][i];
      const float h = tf32_hi(x);
      dst[(int64_t)c * ldt + r] = h;
      dst[(int64_t)(S + c) * ldt + r] = x - h;
    }
  }
}

template <int S, bool TRANS>
int launch_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* Bpanel, float* out, float* split_buf,
              cudaStream_t st) {
  using C = TcCfg<S, TRANS>;
  // skinny operand rows = K extent: n (forward, X) or m (transpose, W)
  const int64_t brows = TRANS ? m : n;
  const int64_t ldt = (brows + 31) / 32 * 32;
  split_panel_t<<<dim3((unsigned)ceil_div(brows, 32), (unsigned)(S / 32)), 256, 0, st>>>(Bpanel, brows, S, split_buf,
                                                                                       ldt);
  CNMF_LAUNCH_CHECK();
  TmaDesc tA, tB;
  if (!TRANS)
    CNMF_TRY(make_tma_2d(&tA, A, 4, m, n, lda, BKT, BMT, true));
  else
    CNMF_TRY(make_tma_2d(&tA, A, 4, m, n, lda, BMT, BKT, false));
  CNMF_TRY(make_tma_2d(&tB, split_buf, 4, 2 * S, brows, ldt, BKT, 2 * S, true));
  const int64_t P = TRANS ? n : m;   // output rows
  const int nt = (int)ceil_div(brows, BKT);
  const int64_t nblocks = ceil_div(P, BMT);
  const int whole = nblocks >= 16 * kNumSMs;
  const int64_t grid = std::min<int64_t>(kNumSMs, whole ? nblocks : nblocks * nt);
  if (!whole) CNMF_CUDA(cudaMemsetAsync(out, 0, (size_t)P * S * 4, st));
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
  pass_tc<S, TRANS><<<(unsigned)grid, kTcThreads, C::SMEM, st>>>(tA, tB, out, P, nt, nblocks, whole);
  CNMF_LAUNCH_CHECK();
  if (e0) {
    CNMF_CUDA(cudaEventRecord(e1, st));
    pass_record(e0, e1, 4.0 * ((double)m * n + (double)n * S + (double)m * S));
  }
  return CNMF_OK;
}

}  // namespace

size_t tc_split_bytes(int64_t rows, int S) { return (size_t)((rows + 31) / 32 * 32) * 2 * S * 4 + 256; }

int pass_forward_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y, float* split,
                    cudaStream_t st) {
  switch (S) {
    case 32: return launch_tc<32, false>(A, m, n, lda, X, Y, split, st);
    case 64: return launch_tc<64, false>(A, m, n, lda, X, Y, split, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "tensor-core pass supports panel widths 32 and 64");
}

int pass_transpose_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, int S, float* Z,
                      float* split, cudaStream_t st) {
  switch (S) {
    case 32: return launch_tc<32, true>(A, m, n, lda, W, Z, split, st);
    case 64: return launch_tc<64, true>(A, m, n, lda, W, Z, split, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "tensor-core pass supports panel widths 32 and 64");
}

}  // namespace cnmf
