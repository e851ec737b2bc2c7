// Fused residual norms over A: ||A - X Y||_F^2 and ||A||_F^2 in one pass.
//
// Reference: nmf.py:53-75 relative_error (blocked over A's rows) and
// snmf.py:223-230 (full-space error of A[:, K] Y). The product X Y is never
// materialised: each 64 x 128 tile of A is read once (coalesced float4),
// the matching rank-r product is formed in registers from shared-memory
// slices of X and Y, and squared differences are accumulated in fp64.
#include <algorithm>

#include "common.cuh"

namespace cnmf {
namespace {

constexpr int kRM = 64, kRN = 128, kRT = 256, kRMax = 64;

// Grid: column strips of 128 columns x row groups; a CTA keeps its strip's
// Y slice in shared memory for all its row tiles and issues the loads of the
// next A tile before forming X Y for the current one, so the DRAM latency of
// A overlaps the rank-r products.
__global__ void __launch_bounds__(kRT)
    resid_kernel(const float* __restrict__ A, int64_t m, int64_t n, int64_t lda, const double* __restrict__ X,
                 const int64_t* __restrict__ cols, const double* __restrict__ Yt, int r, int row_groups,
                 double* __restrict__ out) {
  extern __shared__ __align__(16) float rsm[];
  float(*Xs)[kRMax] = (float(*)[kRMax])rsm;                // kRM x kRMax
  float(*Ys)[kRN] = (float(*)[kRN])(rsm + kRM * kRMax);     // kRMax x kRN
  __shared__ double red[2][kRT / 32];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t mt = ceil_div(m, kRM), nt = ceil_div(n, kRN);
  const int64_t strip = blockIdx.x / row_groups, grp = blockIdx.x % row_groups;
  double res = 0.0, ref = 0.0;
  const bool vec = (lda & 3) == 0;
  for (int64_t cs = strip; cs < nt; cs += gridDim.x / row_groups) {
    const int64_t c0 = cs * kRN;
    __syncthreads();
    for (int i = tid; i < kRN * r; i += kRT) {
      const int cc = i / r, k = i % r;
      const int64_t col = c0 + cc;
      Ys[k][cc] = (col < n) ? (float)Yt[col * r + k] : 0.f;
    }
    for (int64_t rt = grp; rt < mt; rt += row_groups) {
      const int64_t r0 = rt * kRM;
      // this thread's 4 rows x 8 columns of the A tile, loaded first
      float a[4][8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t row = r0 + 4 * ty + i;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t col = c0 + 64 * h + 4 * tx;
          if (row < m && col + 3 < n && vec) {
            const float4 v = __ldcs((const float4*)(A + row * lda + col));
            a[i][4 * h] = v.x;
            a[i][4 * h + 1] = v.y;
            a[i][4 * h + 2] = v.z;
            a[i][4 * h + 3] = v.w;
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) a[i][4 * h + q] = (row < m && col + q < n) ? A[row * lda + col + q] : 0.f;
          }
        }
      }
      __syncthreads();
      for (int i = tid; i < kRM * r; i += kRT) {
        const int rr = i / r, k = i % r;
        const int64_t row = r0 + rr;
        float v = 0.f;
        if (row < m) v = cols ? A[row * lda + cols[k]] : (float)X[row * r + k];
        Xs[rr][k] = v;
      }
      __syncthreads();
      float acc[4][8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
      for (int k = 0; k < r; ++k) {
        const float4 y0 = *(const float4*)&Ys[k][4 * tx];
        const float4 y1 = *(const float4*)&Ys[k][64 + 4 * tx];
        const float ys[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float xv = Xs[4 * ty + i][k];
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(xv, ys[j], acc[i][j]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t row = r0 + 4 * ty + i;
        if (row >= m) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int64_t col = c0 + 64 * (j >> 2) + 4 * tx + (j & 3);
          if (col < n) {
            const double d = (double)a[i][j] - (double)acc[i][j];
            res = fma(d, d, res);
            ref = fma((double)a[i][j], (double)a[i][j], ref);
          }
        }
      }
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

}  // namespace

int residual_norms(const float* A, int64_t m, int64_t n, int64_t lda, const double* X, const int64_t* cols,
                   const double* Yt, int r, double* out, cudaStream_t st) {
  if (r < 1 || r > kRMax) return fail(CNMF_ERR_ARGUMENT, "residual_norms: 1 <= r <= 64");
  if ((X == nullptr) == (cols == nullptr)) return fail(CNMF_ERR_ARGUMENT, "give exactly one of X and cols");
  CNMF_CUDA(cudaMemsetAsync(out, 0, 16, st));
  // strips x row groups, about four CTAs per SM
  const int64_t strips = ceil_div(n, kRN), mt = ceil_div(m, kRM);
  const int64_t want = 4 * kNumSMs;
  const int row_groups = (int)std::max<int64_t>(1, std::min<int64_t>(mt, want / std::max<int64_t>(strips, 1)));
  const unsigned grid = (unsigned)(std::min<int64_t>(strips, std::max<int64_t>(1, want / row_groups)) * row_groups);
  constexpr size_t smem = (size_t)(kRM * kRMax + kRMax * kRN) * 4;
  static bool attr = false;
  if (!attr) {
    CNMF_CUDA(cudaFuncSetAttribute(resid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  resid_kernel<<<grid, kRT, smem, st>>>(A, m, n, lda, X, cols, Yt, r, row_groups, out);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

}  // namespace cnmf
