// Fused residual norms over A: ||A - X Y||_F^2 and ||A||_F^2 in one pass.
//
// Reference: nmf.py:53-75 relative_error (blocked over A's rows) and
// snmf.py:223-230 (full-space error of A[:, K] Y). The product X Y is never
// materialised: each 128 x 128 tile of A is read once (coalesced float4),
// the matching rank-r product is formed in registers from shared-memory
// slices of X and Y, and squared differences are accumulated in fp64.
#include <algorithm>

#include "common.cuh"
#include "pass.cuh"

namespace cnmf {
int gram_tn_f64(const double* X, int64_t p, int a, const double* Y, int b, double* out, cudaStream_t st);
namespace {

constexpr int kRM = 128, kRN = 128, kRT = 256, kRMax = 128;  // ranks up to 64 and up to 128 are separate instantiations

// Work units: (column strip of 128 columns, chunk of kChunk row tiles),
// spread round-robin over the CTAs so that every SM gets the same share. X
// and Y arrive pre-converted to fp32 (xf: m x r, yf: n x r). A CTA keeps its
// strip's Y slice in shared memory across the chunk's row tiles (k-major:
// Ys[k][column]) and stages each tile's X rows k-major too (Xs[k][row]), so
// that a thread's 8 x 8 block of X Y costs four 128-bit shared loads per 64
// FMAs (the round-1/2 kernel's 4 x 8 blocks took six loads per 32 and were
// bound by shared-memory bandwidth: 26 TFLOP/s). A is read once, straight
// into registers, after the products (two CTAs per SM overlap one's loads
// with the other's FMAs). Squared differences are summed in fp32 per thread
// and tile, then in fp64.
constexpr int kChunk = 16;
constexpr int kRLD = 132;
static_assert(kRM == kRN && kRLD >= kRM && kRLD % 4 == 0, "slice layout");

template <int RMAX>
__global__ void __launch_bounds__(kRT, 1)
    resid_kernel(const float* __restrict__ A, int64_t m, int64_t n, int64_t lda, const float* __restrict__ xf,
                 const float* __restrict__ yf, int r, double* __restrict__ out, const int* __restrict__ skip) {
  if (skip != nullptr && *skip) return;  // the pass path's result stands
  extern __shared__ __align__(16) float rsm[];
  // k-major slices with a row stride of 132 floats: the staging stores (a warp
  // writes 32 consecutive k of one row / column) then hit 8 banks instead of 1
  float(*Xs)[kRLD] = (float(*)[kRLD])rsm;                  // r x kRM
  float(*Ys)[kRLD] = (float(*)[kRLD])(rsm + RMAX * kRLD);  // r x kRN
  __shared__ double red[2][kRT / 32];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t mt = ceil_div(m, kRM), nt = ceil_div(n, kRN), chunks = ceil_div(mt, kChunk);
  const int64_t units = nt * chunks;
  double res = 0.0, ref = 0.0;
  const bool vec = (lda & 3) == 0;
  // a tile's rows of X are one contiguous run of kRM * r floats of xf; thread
  // t takes elements t, t + 256, ...: (row, k) of element e advance by
  // (256 / r, 256 % r) per step -- no division in the loops
  constexpr int NX = kRM * RMAX / kRT;
  const int q256 = kRT / r, m256 = kRT - q256 * r;
  const int rr0 = tid / r, k0 = tid - rr0 * r;
  const int nx = kRM * r;
  float xn[NX];
  auto x_fetch = [&](int64_t r0) {  // the tile at row r0 -> registers
    const int64_t lim = min64((int64_t)nx, (m - r0) * r);
    const float* src = xf + r0 * r;
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      const int i = tid + j * kRT;
      xn[j] = (i < lim) ? src[i] : 0.f;
    }
  };
  auto x_store = [&]() {  // registers -> Xs (k-major)
    int rr = rr0, k = k0;
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      if (tid + j * kRT < nx) Xs[k][rr] = xn[j];
      rr += q256;
      k += m256;
      if (k >= r) {
        k -= r;
        ++rr;
      }
    }
  };
  int64_t cur_strip = -1;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t strip = u / chunks, ch = u - strip * chunks;
    const int64_t c0 = strip * kRN;
    const int64_t rt0 = ch * kChunk, rt1 = min64(mt, (ch + 1) * kChunk);
    x_fetch(rt0 * kRM);
    if (strip != cur_strip) {
      __syncthreads();
      for (int i = tid; i < kRN * r; i += kRT) {
        const int cc = i / r, k = i - cc * r;
        const int64_t col = c0 + cc;
        Ys[k][cc] = (col < n) ? yf[col * r + k] : 0.f;
      }
      cur_strip = strip;
    }
    for (int64_t rt = rt0; rt < rt1; ++rt) {
      const int64_t r0 = rt * kRM;
      const int nrow = (int)min64(kRM, m - r0);
      __syncthreads();  // the previous tile's products are done with Xs
      x_store();
      __syncthreads();
      if (rt + 1 < rt1) x_fetch(r0 + kRM);  // the next tile's X rows, in flight during the products
      // this thread's block of A: rows 8 ty .. + 7, columns 4 tx .. + 3 and
      // 64 + 4 tx .. + 3, loaded first (in flight during the products too)
      float a[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t row = r0 + 8 * ty + i;
        const bool rok = 8 * ty + i < nrow;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t col = c0 + 64 * h + 4 * tx;
          if (rok && col + 3 < n && vec) {
            const float4 v = __ldcs((const float4*)(A + row * lda + col));
            a[i][4 * h] = v.x;
            a[i][4 * h + 1] = v.y;
            a[i][4 * h + 2] = v.z;
            a[i][4 * h + 3] = v.w;
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) a[i][4 * h + q] = (rok && col + q < n) ? A[row * lda + col + q] : 0.f;
          }
        }
      }
      float acc[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll 2
      for (int k = 0; k < r; ++k) {
        const float4 x0 = *(const float4*)&Xs[k][8 * ty];
        const float4 x1 = *(const float4*)&Xs[k][8 * ty + 4];
        const float4 y0 = *(const float4*)&Ys[k][4 * tx];
        const float4 y1 = *(const float4*)&Ys[k][64 + 4 * tx];
        const float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        const float ys[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(xs[i], ys[j], acc[i][j]);
      }
      // rows >= nrow and columns >= n hold a = 0 and X Y = 0 (zero-filled slices)
      float tr = 0.f, tf = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = a[i][j] - acc[i][j];
          tr = fmaf(d, d, tr);
          tf = fmaf(a[i][j], a[i][j], tf);
        }
      res += (double)tr;
      ref += (double)tf;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    res += __shfl_xor_sync(0xffffffffu, res, o);
    ref += __shfl_xor_sync(0xffffffffu, ref, o);
  }
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = res;
    red[1][tid >> 5] = ref;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kRT / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    atomicAdd(&out[0], a);
    atomicAdd(&out[1], b);
  }
}

// fp32 copies of the factors: xf (m x r) = X, or the picked columns of A
// (cols != null); yf (n x r) = Yt
__global__ void factors_f32(const float* __restrict__ A, int64_t m, int64_t lda, const double* __restrict__ X,
                            const int64_t* __restrict__ cols, int64_t n, const double* __restrict__ Yt, int r,
                            float* __restrict__ xf, float* __restrict__ yf, const int* __restrict__ skip) {
  if (skip != nullptr && *skip) return;
  const int64_t tot = (m + n) * r;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < m * r) {
      const int64_t row = i / r, k = i - row * r;
      xf[i] = cols ? A[row * lda + cols[k]] : (float)X[i];
    } else {
      yf[i - m * r] = (float)Yt[i - m * r];
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// Pass path: ||A - X Y||^2 = ||A||^2 - 2 <A Y^T, X> + <X^T X, Y Y^T>, with
// A Y^T and ||A||^2 from ONE tensor-core forward pass over A (the streaming
// pass kernel, 3xTF32, the squares summed by its splitters) -- the direct
// kernel is FP32-FFMA bound (2 m n r flops; 72 ms at configs[4]), the pass is
// HBM bound. The expansion cancels: it is used only when the residual is
// large enough that the pass's rounding (<= 1e-6 of <A Y^T, X>, estimated
// conservatively; fp32-level products of nonnegative data) stays below 1e-4
// of the residual; otherwise the combine kernel leaves the flag clear and the
// direct kernel runs (graph-capturable: the decision stays on the device).
// ---------------------------------------------------------------------------
__global__ void yt_panel(const double* __restrict__ Yt, int64_t n, int r, int S, float* __restrict__ P) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * S; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / S;
    const int k = (int)(i - row * S);
    P[i] = k < r ? (float)Yt[row * r + k] : 0.f;
  }
}

__global__ void gather_cols_f64(const float* __restrict__ A, int64_t m, int64_t lda, const int64_t* __restrict__ cols,
                                int r, double* __restrict__ X) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m * r; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / r;
    X[i] = (double)A[row * lda + cols[i - row * r]];
  }
}

// acc[1] += sum_{i < m, k < r} T[i][k] X[i][k]
__global__ void __launch_bounds__(256) dot_tx(const float* __restrict__ T, int64_t m, int S, const double* __restrict__ X,
                                              int r, double* __restrict__ acc) {
  __shared__ double red[8];
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m * r; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / r;
    v = fma((double)T[row * S + (i - row * r)], X[i], v);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    atomicAdd(&acc[1], t);
  }
}

// acc = {||A||^2, <A Y^T, X>}, G1 = X^T X, G2 = Y Y^T (r x r): out and the
// skip flag when the expansion is accurate enough, else zeroed out / flag 0
__global__ void resid_combine(const double* __restrict__ acc, const double* __restrict__ G1,
                              const double* __restrict__ G2, int r, double* __restrict__ out, int* __restrict__ skip) {
  __shared__ double red[8];
  double g = 0.0;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) g = fma(G1[i], G2[i], g);
#pragma unroll
  for (int o = 16; o; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = g;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    const double a2 = acc[0], d = acc[1];
    const double res = a2 - 2.0 * d + t;
    const bool ok = res > 0.0 && 1e-6 * fabs(d) <= 1e-4 * res;
    out[0] = ok ? res : 0.0;
    out[1] = ok ? a2 : 0.0;
    *skip = ok ? 1 : 0;
  }
}

bool resid_pass_enabled(int64_t m, int64_t n, int r) {
  const char* e = getenv("CNMF_RESID_PASS");  // "0": direct kernel only (A/B and tests)
  const int mode = (e && e[0] == '0') ? 0 : 1;
  // the pass path pays off where the direct kernel's 2 m n r flops exceed the
  // pass's read of A (r >= 8) on matrices large enough to amortise its launches
  return mode == 1 && r >= 8 && r <= 64 && (double)m * (double)n >= (double)(1 << 26) && pass_uses_tc(r <= 32 ? 32 : 64);
}

int residual_norms(const float* A, int64_t m, int64_t n, int64_t lda, const double* X, const int64_t* cols,
                   const double* Yt, int r, double* out, cudaStream_t st) {
  if (r < 1 || r > kRMax) return fail(CNMF_ERR_ARGUMENT, "residual_norms: 1 <= r <= 128");
  if ((X == nullptr) == (cols == nullptr)) return fail(CNMF_ERR_ARGUMENT, "give exactly one of X and cols");
  const int* skip = nullptr;
  bool try_pass = resid_pass_enabled(m, n, r);
  bool factors_done = false;
  void* fscr = nullptr;
  CNMF_TRY(device_scratch("resid-factors", (size_t)(m + n) * r * 4 + 256, &fscr, st));
  float* xf = (float*)fscr;
  float* yf = xf + (size_t)m * r;
  const unsigned fgrid = (unsigned)std::min<int64_t>(ceil_div((m + n) * r, 256), 8 * device_sms());
  auto direct = [&](int64_t rows, double* dst, const int* flag) -> int {
    const int64_t units = ceil_div(n, kRN) * ceil_div(ceil_div(rows, kRM), kChunk);
    auto launch = [&](auto kernel, size_t smem) -> int {
      CNMF_TRY(ensure_smem_attr((const void*)kernel, (int)smem));
      int occ = 0;
      CNMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kRT, smem));
      const unsigned grid =
          (unsigned)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)std::max(occ, 1) * device_sms()));
      kernel<<<grid, kRT, smem, st>>>(A, rows, n, lda, xf, yf, r, dst, flag);
      CNMF_LAUNCH_CHECK();
      return CNMF_OK;
    };
    if (r <= 64) return launch(resid_kernel<64>, (size_t)(2 * 64 * kRLD) * 4);
    return launch(resid_kernel<128>, (size_t)(2 * 128 * kRLD) * 4);
  };
  if (try_pass) {
    // The expansion below is only accepted for relative residuals above ~0.1
    // (resid_combine); a well-fitted factorisation (configs[3]: 0.013) would
    // pay for a pass whose result is then thrown away. The residual of the
    // top rows (1/256 of the matrix, the direct kernel) decides which path
    // to try; a wrong guess costs time, never accuracy (the guard still runs).
    // Needs one host round trip, so it is skipped under graph capture.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CNMF_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusNone) {
      void* sscr = nullptr;
      CNMF_TRY(device_scratch("resid-sample", 64, &sscr, st));
      double* sm2 = (double*)sscr;
      CNMF_CUDA(cudaMemsetAsync(sm2, 0, 16, st));
      factors_f32<<<fgrid, 256, 0, st>>>(A, m, lda, X, cols, n, Yt, r, xf, yf, nullptr);
      CNMF_LAUNCH_CHECK();
      factors_done = true;
      const int64_t rows = std::min<int64_t>(m, std::max<int64_t>(256, (m / 256 + 63) / 64 * 64));
      CNMF_TRY(direct(rows, sm2, nullptr));
      double h[2] = {0.0, 0.0};
      CNMF_CUDA(cudaMemcpyAsync(h, sm2, 16, cudaMemcpyDeviceToHost, st));
      CNMF_CUDA(cudaStreamSynchronize(st));
      if (h[1] > 0.0 && h[0] < 5e-3 * h[1]) try_pass = false;
    }
  }
  if (try_pass) {
    const int S = r <= 32 ? 32 : 64;
    const size_t small = 64 + 2 * (size_t)r * r * 8;
    const size_t need = small + (size_t)n * S * 4 + (size_t)m * S * 4 + (cols ? (size_t)m * r * 8 : 0) + 512;
    void* scr = nullptr;
    CNMF_TRY(device_scratch("resid-pass", need, &scr, st));
    unsigned char* p = (unsigned char*)scr;
    double* acc = (double*)p;          // [0] ||A||^2, [1] <A Y^T, X>
    int* flag = (int*)(p + 32);
    double* G1 = (double*)(p + 64);
    double* G2 = G1 + (size_t)r * r;
    float* P = (float*)(p + ((small + 255) & ~(size_t)255));
    float* T = P + (size_t)n * S;
    double* Xg = (double*)(T + (size_t)m * S);
    CNMF_CUDA(cudaMemsetAsync(acc, 0, 16, st));
    const unsigned g8 = (unsigned)(8 * device_sms());
    yt_panel<<<g8, 256, 0, st>>>(Yt, n, r, S, P);
    CNMF_LAUNCH_CHECK();
    if (cols) {
      gather_cols_f64<<<g8, 256, 0, st>>>(A, m, lda, cols, r, Xg);
      CNMF_LAUNCH_CHECK();
      X = Xg;
    }
    CNMF_TRY(pass_forward_sumsq(A, m, n, lda, P, S, T, acc, st));
    dot_tx<<<g8, 256, 0, st>>>(T, m, S, X, r, acc);
    CNMF_LAUNCH_CHECK();
    CNMF_TRY(gram_tn_f64(X, m, r, X, r, G1, st));
    CNMF_TRY(gram_tn_f64(Yt, n, r, Yt, r, G2, st));
    resid_combine<<<1, 256, 0, st>>>(acc, G1, G2, r, out, flag);
    CNMF_LAUNCH_CHECK();
    skip = flag;
    if (cols) X = nullptr;
  } else {
    CNMF_CUDA(cudaMemsetAsync(out, 0, 16, st));
  }
  if (!factors_done) {
    factors_f32<<<fgrid, 256, 0, st>>>(A, m, lda, X, cols, n, Yt, r, xf, yf, skip);
    CNMF_LAUNCH_CHECK();
  }
  CNMF_TRY(direct(m, out, skip));
  return CNMF_OK;
}

}  // namespace cnmf
