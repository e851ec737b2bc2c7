// Streaming skinny-GEMM passes over A (the bytes that dominate the method).
//
// Reference: store.py:578-597 matmul_blocked (A @ B over row blocks) and
// store.py:600-627 matmul_transposed_blocked (A^T @ B), as used by
// compress.py:186-198 (sketch + power passes), snmf.py:154-167 (Q^T A) and
// nmf.py:138-149 / nmf.py:329-332 (projections).
//
// Design (B200): A is fp32 row-major and read exactly once per pass. Tiles of
// A are staged by TMA into a multi-stage shared-memory ring (mbarrier
// complete_tx), the skinny operand tile rides along in the same stage, and
// each thread keeps a 2 x 32 (forward) or 4 x 32 (transpose) register block of
// FP32 accumulators fed by one 128-bit A load plus warp-broadcast operand
// loads. Forward uses the 128B TMA swizzle so that eight consecutive rows hit
// eight distinct bank groups. The long reduction stays on chip; only the
// (rare) split-K partials go to L2 through vectorised red.global.add.v4.f32.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "pass.cuh"

namespace cnmf {
namespace {

constexpr int kThreads = 256;

template <int S>
struct FwdCfg;
template <>
struct FwdCfg<32> {
  static constexpr int WC = 1, TS = 32, TM = 2, BM = 512, ST = 3;
};
template <>
struct FwdCfg<64> {
  static constexpr int WC = 2, TS = 32, TM = 2, BM = 256, ST = 4;
};
template <>
struct FwdCfg<128> {
  static constexpr int WC = 4, TS = 32, TM = 2, BM = 128, ST = 4;
};

template <int S>
constexpr size_t fwd_smem() {
  using C = FwdCfg<S>;
  return 1024 + (size_t)C::ST * (C::BM * 32 * 4 + 32 * S * 4) + 64;
}

__device__ __forceinline__ unsigned char* align1024(unsigned char* p) {
  return (unsigned char*)(((uintptr_t)p + 1023) & ~(uintptr_t)1023);
}

__device__ __forceinline__ float f4c(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Y[m x S] = A[m x n] X[n x S]. Work unit = one BM x 32 tile of A (row block
// rb, k-tile kt), flattened rb-major. Each CTA (one per SM) streams a
// contiguous range of units — whole row blocks when there are many, else an
// even split of all units — and flushes its register accumulator whenever
// the row block changes: a plain store when it owned the whole row block,
// a red.global.add.v4 into the zeroed output otherwise. Balanced to within
// one 64 KB tile per SM.
template <int S>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_ffma(const __grid_constant__ TmaDesc tA, const __grid_constant__ TmaDesc tX, float* __restrict__ Y,
             int64_t m, int nkt, int64_t mb, int whole_blocks) {
  using C = FwdCfg<S>;
  constexpr int BM = C::BM, BK = 32, ST = C::ST;
  constexpr int ABYTES = BM * BK * 4, XBYTES = BK * S * 4;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = align1024(smem_raw);
  unsigned char* sA = smem;
  float* sX = (float*)(smem + ST * ABYTES);
  uint64_t* bars = (uint64_t*)(smem + ST * (ABYTES + XBYTES));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp / C::WC, wc = warp % C::WC;
  const int64_t U = mb * nkt, G = gridDim.x, b = blockIdx.x;
  const int64_t u0 = whole_blocks ? (b * mb / G) * nkt : b * U / G;
  const int64_t u1 = whole_blocks ? ((b + 1) * mb / G) * nkt : (b + 1) * U / G;
  const int64_t ntiles = u1 - u0;
  if (ntiles <= 0) return;

  if (tid == 0) {
    prefetch_tmap(&tA);
    prefetch_tmap(&tX);
    for (int s = 0; s < ST; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int stage, int64_t u) {
    const int64_t rb = u / nkt;
    const int kt = (int)(u - rb * nkt);
    mbar_arrive_expect_tx(&bars[stage], ABYTES + XBYTES);
#pragma unroll
    for (int h = 0; h < (BM + 255) / 256; ++h)
      tma_load_2d(sA + stage * ABYTES + h * 256 * 128, &tA, &bars[stage], kt * BK, (int)(rb * BM + h * 256));
    tma_load_2d(sX + stage * (BK * S), &tX, &bars[stage], 0, kt * BK);
  };
  if (tid == 0)
    for (int s = 0; s < ST && s < ntiles; ++s) issue(s, u0 + s);

  float acc[C::TM][C::TS];
#pragma unroll
  for (int i = 0; i < C::TM; ++i)
#pragma unroll
    for (int j = 0; j < C::TS; ++j) acc[i][j] = 0.f;

  for (int64_t it = 0; it < ntiles; ++it) {
    const int stage = (int)(it % ST);
    const int64_t u = u0 + it;
    mbar_wait(&bars[stage], (uint32_t)((it / ST) & 1));
    const unsigned char* As = sA + stage * ABYTES;
    const float* Xs = sX + stage * (BK * S) + wc * C::TS;
#pragma unroll 2
    for (int k4 = 0; k4 < 8; ++k4) {
      float4 a[C::TM];
#pragma unroll
      for (int i = 0; i < C::TM; ++i) {
        const int row = wr * 32 * C::TM + lane + 32 * i;
        a[i] = *(const float4*)(As + row * 128 + ((k4 ^ (row & 7)) << 4));
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float* xr = Xs + (4 * k4 + kk) * S;
#pragma unroll
        for (int j4 = 0; j4 < C::TS / 4; ++j4) {
          const float4 x = *(const float4*)(xr + 4 * j4);
#pragma unroll
          for (int i = 0; i < C::TM; ++i) {
            const float av = f4c(a[i], kk);
            acc[i][4 * j4 + 0] = fmaf(av, x.x, acc[i][4 * j4 + 0]);
            acc[i][4 * j4 + 1] = fmaf(av, x.y, acc[i][4 * j4 + 1]);
            acc[i][4 * j4 + 2] = fmaf(av, x.z, acc[i][4 * j4 + 2]);
            acc[i][4 * j4 + 3] = fmaf(av, x.w, acc[i][4 * j4 + 3]);
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0 && it + ST < ntiles) issue(stage, u + ST);
    const int64_t rb = u / nkt;
    if (it == ntiles - 1 || (u + 1) / nkt != rb) {
      // flush this row block
      const bool owned = (rb * nkt >= u0) && ((rb + 1) * nkt <= u1);
#pragma unroll
      for (int i = 0; i < C::TM; ++i) {
        const int64_t row = rb * BM + wr * 32 * C::TM + lane + 32 * i;
        if (row < m) {
          float* yr = Y + row * S + wc * C::TS;
#pragma unroll
          for (int j4 = 0; j4 < C::TS / 4; ++j4) {
            if (owned)
              *(float4*)(yr + 4 * j4) =
                  make_float4(acc[i][4 * j4], acc[i][4 * j4 + 1], acc[i][4 * j4 + 2], acc[i][4 * j4 + 3]);
            else
              red_add_v4(yr + 4 * j4, acc[i][4 * j4], acc[i][4 * j4 + 1], acc[i][4 * j4 + 2],
                         acc[i][4 * j4 + 3]);
          }
        }
#pragma unroll
        for (int j = 0; j < C::TS; ++j) acc[i][j] = 0.f;
      }
    }
  }
}

template <int S>
struct TrnCfg;
template <>
struct TrnCfg<32> {
  static constexpr int WC = 1, TS = 32, BN = 1024, BR = 16, ST = 3;
};
template <>
struct TrnCfg<64> {
  static constexpr int WC = 2, TS = 32, BN = 512, BR = 16, ST = 4;
};
template <>
struct TrnCfg<128> {
  static constexpr int WC = 4, TS = 32, BN = 256, BR = 32, ST = 4;
};

template <int S>
constexpr size_t trn_smem() {
  using C = TrnCfg<S>;
  return 1024 + (size_t)C::ST * (C::BN * C::BR * 4 + C::BR * S * 4) + 64;
}

// Z[n x S] = A[m x n]^T W[m x S]. Work unit = one BR x BN tile (column block
// cb, row tile rt), flattened cb-major; CTAs stream contiguous unit ranges
// and flush per column block exactly like the forward pass.
template <int S>
__global__ void __launch_bounds__(kThreads, 1)
    trn_ffma(const __grid_constant__ TmaDesc tA, const __grid_constant__ TmaDesc tW, float* __restrict__ Z,
             int64_t n, int nrt, int64_t nb, int whole_blocks) {
  using C = TrnCfg<S>;
  constexpr int BN = C::BN, BR = C::BR, ST = C::ST;
  constexpr int ABYTES = BN * BR * 4, WBYTES = BR * S * 4;
  constexpr int NSUB = BN / 256;  // TMA boxes of 256 columns
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = align1024(smem_raw);
  float* sA = (float*)smem;
  float* sW = (float*)(smem + ST * ABYTES);
  uint64_t* bars = (uint64_t*)(smem + ST * (ABYTES + WBYTES));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wn = warp / C::WC, wc = warp % C::WC;
  const int64_t U = nb * nrt, G = gridDim.x, b = blockIdx.x;
  const int64_t u0 = whole_blocks ? (b * nb / G) * nrt : b * U / G;
  const int64_t u1 = whole_blocks ? ((b + 1) * nb / G) * nrt : (b + 1) * U / G;
  const int64_t ntiles = u1 - u0;
  if (ntiles <= 0) return;

  if (tid == 0) {
    prefetch_tmap(&tA);
    prefetch_tmap(&tW);
    for (int s = 0; s < ST; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int stage, int64_t u) {
    const int64_t cb = u / nrt;
    const int rt = (int)(u - cb * nrt);
    mbar_arrive_expect_tx(&bars[stage], ABYTES + WBYTES);
#pragma unroll
    for (int h = 0; h < NSUB; ++h)
      tma_load_2d(sA + stage * (BN * BR) + h * (256 * BR), &tA, &bars[stage], (int)(cb * BN + h * 256), rt * BR);
    tma_load_2d(sW + stage * (BR * S), &tW, &bars[stage], 0, rt * BR);
  };
  if (tid == 0)
    for (int s = 0; s < ST && s < ntiles; ++s) issue(s, u0 + s);

  const int cl = wn * 128 + 4 * lane;  // first of this thread's 4 columns in the tile
  const int sub = cl / 256, cin = cl % 256;
  float acc[4][C::TS];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < C::TS; ++j) acc[i][j] = 0.f;

  for (int64_t it = 0; it < ntiles; ++it) {
    const int stage = (int)(it % ST);
    const int64_t u = u0 + it;
    mbar_wait(&bars[stage], (uint32_t)((it / ST) & 1));
    const float* As = sA + stage * (BN * BR) + sub * (256 * BR) + cin;
    const float* Ws = sW + stage * (BR * S) + wc * C::TS;
#pragma unroll 4
    for (int r = 0; r < BR; ++r) {
      const float4 a = *(const float4*)(As + r * 256);
#pragma unroll
      for (int j4 = 0; j4 < C::TS / 4; ++j4) {
        const float4 w = *(const float4*)(Ws + r * S + 4 * j4);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float av = f4c(a, i);
          acc[i][4 * j4 + 0] = fmaf(av, w.x, acc[i][4 * j4 + 0]);
          acc[i][4 * j4 + 1] = fmaf(av, w.y, acc[i][4 * j4 + 1]);
          acc[i][4 * j4 + 2] = fmaf(av, w.z, acc[i][4 * j4 + 2]);
          acc[i][4 * j4 + 3] = fmaf(av, w.w, acc[i][4 * j4 + 3]);
        }
      }
    }
    __syncthreads();
    if (tid == 0 && it + ST < ntiles) issue(stage, u + ST);
    const int64_t cb = u / nrt;
    if (it == ntiles - 1 || (u + 1) / nrt != cb) {
      const bool owned = (cb * nrt >= u0) && ((cb + 1) * nrt <= u1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t col = cb * BN + cl + i;
        if (col < n) {
          float* zr = Z + col * S + wc * C::TS;
#pragma unroll
          for (int j4 = 0; j4 < C::TS / 4; ++j4) {
            if (owned)
              *(float4*)(zr + 4 * j4) =
                  make_float4(acc[i][4 * j4], acc[i][4 * j4 + 1], acc[i][4 * j4 + 2], acc[i][4 * j4 + 3]);
            else
              red_add_v4(zr + 4 * j4, acc[i][4 * j4], acc[i][4 * j4 + 1], acc[i][4 * j4 + 2],
                         acc[i][4 * j4 + 3]);
          }
        }
#pragma unroll
        for (int j = 0; j < C::TS; ++j) acc[i][j] = 0.f;
      }
    }
  }
}

// P <- P T (T upper-triangular S x S, fp64 given, applied in fp32), grid-
// strided over 64-row tiles (cnmf_panel_apply; the CholeskyQR sweeps of the
// range finders apply their transform inside csrc/sweep.cu).
template <int S>
__global__ void __launch_bounds__(kThreads) apply_panel(float* __restrict__ P, int64_t rows, const double* T) {
  constexpr int TR = 64;
  extern __shared__ float fsm[];
  float* sT = fsm;              // S x S
  float* sIn = sT + S * S;      // TR x S
  float* sOut = sIn + TR * S;   // TR x S
  const int tid = threadIdx.x;
  for (int i = tid; i < S * S; i += kThreads) sT[i] = (float)T[i];
  for (int64_t t0 = (int64_t)blockIdx.x * TR; t0 < rows; t0 += (int64_t)gridDim.x * TR) {
    __syncthreads();
    const int nr = (int)min64(TR, rows - t0);
    for (int i = tid; i < TR * S / 4; i += kThreads) {
      const int r = (i * 4) / S;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nr) v = *(const float4*)(P + t0 * S + 4 * (int64_t)i);
      *(float4*)(sIn + 4 * i) = v;
    }
    __syncthreads();
    for (int i = tid; i < TR * S; i += kThreads) {
      const int r = i / S, c = i % S;
      float acc = 0.f;
      for (int j = 0; j <= c; ++j) acc = fmaf(sIn[r * S + j], sT[j * S + c], acc);
      sOut[i] = acc;
    }
    __syncthreads();
    for (int i = tid; i < TR * S / 4; i += kThreads) {
      const int r = (i * 4) / S;
      if (r < nr) *(float4*)(P + t0 * S + 4 * (int64_t)i) = *(const float4*)(sOut + 4 * i);
    }
  }
}

template <int S>
int launch_forward(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, cudaStream_t st) {
  using C = FwdCfg<S>;
  TmaDesc tA, tX;
  CNMF_TRY(make_tma_2d(&tA, A, 4, m, n, lda, 32, std::min(C::BM, 256), true));
  CNMF_TRY(make_tma_2d(&tX, X, 4, n, S, S, S, 32, false));
  const int nkt = (int)ceil_div(n, 32);
  const int64_t mb = ceil_div(m, C::BM);
  // whole row blocks per CTA when there are many (no atomics, no memset)
  const int whole = mb >= 16 * kNumSMs;
  const int64_t grid = std::min<int64_t>(kNumSMs, whole ? mb : mb * nkt);
  if (!whole) CNMF_CUDA(cudaMemsetAsync(Y, 0, (size_t)m * S * 4, st));
  constexpr size_t smem = fwd_smem<S>();
  CNMF_TRY(ensure_smem_attr((const void*)fwd_ffma<S>, (int)smem));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (pass_profiling()) {
    CNMF_CUDA(cudaEventCreate(&e0));
    CNMF_CUDA(cudaEventCreate(&e1));
    CNMF_CUDA(cudaEventRecord(e0, st));
  }
  fwd_ffma<S><<<(unsigned)grid, kThreads, smem, st>>>(tA, tX, Y, m, nkt, mb, whole);
  CNMF_LAUNCH_CHECK();
  if (e0) {
    CNMF_CUDA(cudaEventRecord(e1, st));
    pass_record(e0, e1, 4.0 * ((double)m * n + (double)n * S + (double)m * S));
  }
  return CNMF_OK;
}

template <int S>
int launch_transpose(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, float* Z, cudaStream_t st) {
  using C = TrnCfg<S>;
  TmaDesc tA, tW;
  CNMF_TRY(make_tma_2d(&tA, A, 4, m, n, lda, 256, C::BR, false));
  CNMF_TRY(make_tma_2d(&tW, W, 4, m, S, S, S, C::BR, false));
  const int nrt = (int)ceil_div(m, C::BR);
  const int64_t nb = ceil_div(n, C::BN);
  const int whole = nb >= 16 * kNumSMs;
  const int64_t grid = std::min<int64_t>(kNumSMs, whole ? nb : nb * nrt);
  if (!whole) CNMF_CUDA(cudaMemsetAsync(Z, 0, (size_t)n * S * 4, st));
  constexpr size_t smem = trn_smem<S>();
  CNMF_TRY(ensure_smem_attr((const void*)trn_ffma<S>, (int)smem));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (pass_profiling()) {
    CNMF_CUDA(cudaEventCreate(&e0));
    CNMF_CUDA(cudaEventCreate(&e1));
    CNMF_CUDA(cudaEventRecord(e0, st));
  }
  trn_ffma<S><<<(unsigned)grid, kThreads, smem, st>>>(tA, tW, Z, n, nrt, nb, whole);
  CNMF_LAUNCH_CHECK();
  if (e0) {
    CNMF_CUDA(cudaEventRecord(e1, st));
    pass_record(e0, e1, 4.0 * ((double)m * n + (double)n * S + (double)m * S));
  }
  return CNMF_OK;
}

template <int S>
int launch_apply(float* P, int64_t rows, const double* T, cudaStream_t st) {
  constexpr size_t smem = (size_t)(S * S + 2 * 64 * S) * 4;
  CNMF_TRY(ensure_smem_attr((const void*)apply_panel<S>, (int)smem));
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 64), 2 * kNumSMs));
  apply_panel<S><<<grid, kThreads, smem, st>>>(P, rows, T);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

}  // namespace

int panel_ld(int s) {
  if (s <= 32) return 32;
  if (s <= 64) return 64;
  if (s <= 128) return 128;
  return -1;
}



// Pass implementation: tcgen05 3xTF32 (default for panel widths 32/64) or the
// FFMA kernels (CNMF_PASS=ffma, and widths 128).
static int g_pass_mode = -1;  // 0 = FFMA, 1 = tcgen05
void set_pass_impl(int mode) { g_pass_mode = mode; }
static bool use_tc(int S) {
  if (g_pass_mode < 0) {
    const char* e = getenv("CNMF_PASS");
    g_pass_mode = (e && std::string(e) == "ffma") ? 0 : 1;
  }
  return g_pass_mode == 1 && (S == 32 || S == 64);
}

bool pass_uses_tc(int S) { return use_tc(S); }

// streaming-pass kernel version on the tensor-core path: 2 = 256-row units
// (csrc/tc_pass2.cu, default), 1 = 128-row units (csrc/tc_pass.cu); CNMF_PASS_V
static int pass_version() {
  const char* e = getenv("CNMF_PASS_V");
  return (e && e[0] == '1') ? 1 : 2;
}

int pass_forward_sumsq(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y,
                       double* sumsq, cudaStream_t st) {
  if (!use_tc(S)) return fail(CNMF_ERR_ARGUMENT, "the residual pass needs the tensor-core pass");
  return pass_version() == 2 ? pass_forward_sumsq_tc2(A, m, n, lda, X, S, Y, sumsq, st)
                             : pass_forward_sumsq_tc(A, m, n, lda, X, S, Y, sumsq, st);
}

int pass_forward(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y,
                 cudaStream_t st) {
  if (use_tc(S))
    return pass_version() == 2 ? pass_forward_tc2(A, m, n, lda, X, S, Y, st) : pass_forward_tc(A, m, n, lda, X, S, Y, st);
  switch (S) {
    case 32: return launch_forward<32>(A, m, n, lda, X, Y, st);
    case 64: return launch_forward<64>(A, m, n, lda, X, Y, st);
    case 128: return launch_forward<128>(A, m, n, lda, X, Y, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "panel width must be 32, 64 or 128");
}

// the paired launch on the tensor-core path for matrices up to 4 GB (it
// saves a pipeline ramp-up and tail per power step and lets the two
// directions share A through L2: 1.31 -> 1.27 ms for configs[1]'s range
// finders); for 80 GB matrices the two concurrent access patterns cost ~5 %
// (configs[4]: 514 -> 540 ms), so those run two launches, as does
// CNMF_PAIR_PASS=0
int pass_pair(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, const float* W, float* Z,
              int S, cudaStream_t st) {
  static int paired = -1;
  static double max_bytes = 4e9;
  if (paired < 0) {
    const char* e = getenv("CNMF_PAIR_PASS");
    paired = (e && e[0] == '0') ? 0 : 1;
    const char* g = getenv("CNMF_PAIR_MAX_GB");  // A/B: the size limit of the paired launch
    if (g) max_bytes = atof(g) * 1e9;
  }
  if (paired && use_tc(S) && 4.0 * (double)m * (double)n <= max_bytes)
    return pass_version() == 2 ? pass_pair_tc2(A, m, n, lda, X, Y, W, Z, S, st)
                               : pass_pair_tc(A, m, n, lda, X, Y, W, Z, S, st);
  CNMF_TRY(pass_forward(A, m, n, lda, X, S, Y, st));
  return pass_transpose(A, m, n, lda, W, S, Z, st);
}

int pass_transpose(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, int S, float* Z,
                   cudaStream_t st) {
  if (use_tc(S))
    return pass_version() == 2 ? pass_transpose_tc2(A, m, n, lda, W, S, Z, st)
                               : pass_transpose_tc(A, m, n, lda, W, S, Z, st);
  switch (S) {
    case 32: return launch_transpose<32>(A, m, n, lda, W, Z, st);
    case 64: return launch_transpose<64>(A, m, n, lda, W, Z, st);
    case 128: return launch_transpose<128>(A, m, n, lda, W, Z, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "panel width must be 32, 64 or 128");
}

int panel_finalize(float* P, int64_t rows, int S, const double* T, double* G, cudaStream_t st) {
  if (G != nullptr) return fail(CNMF_ERR_ARGUMENT, "panel_finalize: Gram accumulation moved to panel_sweep");
  switch (S) {
    case 32: return launch_apply<32>(P, rows, T, st);
    case 64: return launch_apply<64>(P, rows, T, st);
    case 128: return launch_apply<128>(P, rows, T, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "panel width must be 32, 64 or 128");
}

}  // namespace cnmf

namespace cnmf {
namespace {

// out (S x S, fp64) = P1^T P2 for two row-aligned S-wide panels.
template <int S>
__global__ void __launch_bounds__(256)
    panel_cross_kernel(const float* __restrict__ P1, const float* __restrict__ P2, int64_t rows,
                       double* __restrict__ out) {  // out: [gridDim.x][S * S] block partials
  constexpr int TR = S > 64 ? 32 : 64, NB = S / 4, NBLK = NB * NB, BPT = (NBLK + 255) / 256;
  __shared__ __align__(16) float s1[TR * S];
  __shared__ __align__(16) float s2[TR * S];
  const int tid = threadIdx.x;
  double g[BPT][16];
#pragma unroll
  for (int q = 0; q < BPT; ++q)
#pragma unroll
    for (int e = 0; e < 16; ++e) g[q][e] = 0.0;
  for (int64_t t0 = (int64_t)blockIdx.x * TR; t0 < rows; t0 += (int64_t)gridDim.x * TR) {
    const int nr = (int)min64(TR, rows - t0);
    __syncthreads();
    for (int i = tid; i < TR * S / 4; i += 256) {
      const int r = (i * 4) / S;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      if (r < nr) {
        a = *(const float4*)(P1 + t0 * S + 4 * (int64_t)i);
        b = *(const float4*)(P2 + t0 * S + 4 * (int64_t)i);
      }
      *(float4*)(s1 + 4 * i) = a;
      *(float4*)(s2 + 4 * i) = b;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      const int blk = tid + 256 * q;
      if (blk >= NBLK) continue;
      const int bi = blk / NB, bj = blk % NB;
      for (int r = 0; r < nr; ++r) {
        const float4 x = *(const float4*)(s1 + r * S + 4 * bi);
        const float4 y = *(const float4*)(s2 + r * S + 4 * bj);
        const double xs[4] = {x.x, x.y, x.z, x.w};
        const double ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) g[q][a * 4 + b] = fma(xs[a], ys[b], g[q][a * 4 + b]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    const int blk = tid + 256 * q;
    if (blk >= NBLK) continue;
    const int bi = blk / NB, bj = blk % NB;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) out[(size_t)blockIdx.x * S * S + (4 * bi + a) * S + 4 * bj + b] = g[q][a * 4 + b];
  }
}

// out[e] = sum over blocks of part[block][e], four block segments summed in
// block order and combined in segment order (bit-reproducible)
__global__ void __launch_bounds__(256) cross_reduce(const double* __restrict__ part, int nb, int len,
                                                    double* __restrict__ out) {
  __shared__ double seg[4][64];
  const int el = threadIdx.x & 63, sg = threadIdx.x >> 6, e = blockIdx.x * 64 + el;
  double acc = 0.0;
  if (e < len) {
    const int per = (nb + 3) / 4, j1 = min(nb, (sg + 1) * per);
    for (int j0 = sg * per; j0 < j1; j0 += 8) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (j0 + j < j1) ? part[(size_t)(j0 + j) * len + e] : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += v[j];
    }
  }
  seg[sg][el] = acc;
  __syncthreads();
  if (sg == 0 && e < len) out[e] = ((seg[0][el] + seg[1][el]) + seg[2][el]) + seg[3][el];
}

template <int S>
int launch_cross(const float* P1, const float* P2, int64_t rows, double* out, cudaStream_t st) {
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 64), 2 * device_sms()));
  void* part = nullptr;  // per-block partials (every block writes all S x S entries)
  CNMF_TRY(device_scratch("panel-cross", (size_t)2 * device_sms() * 128 * 128 * 8, &part, st));
  panel_cross_kernel<S><<<grid, 256, 0, st>>>(P1, P2, rows, (double*)part);
  CNMF_LAUNCH_CHECK();
  cross_reduce<<<S * S / 64, 256, 0, st>>>((const double*)part, (int)grid, S * S, out);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

}  // namespace

int panel_cross(const float* P1, const float* P2, int64_t rows, int S, double* out, cudaStream_t st) {
  switch (S) {
    case 32: return launch_cross<32>(P1, P2, rows, out, st);
    case 64: return launch_cross<64>(P1, P2, rows, out, st);
    case 128: return launch_cross<128>(P1, P2, rows, out, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "panel_cross supports widths 32, 64 and 128");
}

}  // namespace cnmf
