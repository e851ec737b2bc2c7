// fp64 range finder for float64 inputs (BASELINE.json configs[0] is an fp64
// workload): the same algorithm as the fp32 path (csrc/linalg.cu) -- the
// seeded Gaussian test matrix, 2w + 1 passes over A, every pass output
// re-orthonormalised -- with A, the panels and every product in fp64 (DFMA),
// and CholeskyQR2 (fp64 Gram, chol.cuh's factor + inverse, fp64 apply) after
// each pass. Meant for the CPU-sized configurations: the passes are plain
// shared-memory tiled DFMA kernels, not the tensor-core streaming kernels.
//
// Reference: compress.py:156-227 (structured_compress[_rows] with
// reorthogonalize), compress.py:136-145 (canonical QR, diag(R) > 0).
#include <algorithm>

#include "common.cuh"

namespace cnmf {

int gram_tn_f64(const double* X, int64_t p, int a, const double* Y, int b, double* out, cudaStream_t st);
int chol_inv(const double* G, int s, int S, double* T, double* R, int* info, int pass_id, cudaStream_t st);
int gaussian_fill(uint64_t seed, int64_t rows, int64_t cols, int64_t chunk_rows, int dtype, void* out, int64_t ld,
                  cudaStream_t stream);
int panel_ld(int s);

namespace {

constexpr int kFT = 64;  // rows (forward) / columns (transpose) per tile
constexpr int kFK = 16;  // K per shared-memory step

// Y (m x S) = A X, A fp64 m x n (lda), X n x S. Block: 64 rows x S columns;
// thread (row, column group of S / 4).
template <int S>
__global__ void __launch_bounds__(256) f64_forward(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                                   const double* __restrict__ X, double* __restrict__ Y) {
  __shared__ double As[kFT][kFK + 1];
  __shared__ double Xs[kFK][S];
  constexpr int CPT = S / 4;  // columns per thread
  const int tid = threadIdx.x, tr = tid >> 2, tc = tid & 3;  // 64 rows x 4 column groups
  const int64_t r0 = (int64_t)blockIdx.x * kFT;
  double acc[CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) acc[j] = 0.0;
  for (int64_t k0 = 0; k0 < n; k0 += kFK) {
    __syncthreads();
    for (int i = tid; i < kFT * kFK; i += 256) {
      const int rr = i / kFK, kk = i % kFK;
      As[rr][kk] = (r0 + rr < m && k0 + kk < n) ? A[(r0 + rr) * lda + k0 + kk] : 0.0;
    }
    for (int i = tid; i < kFK * S; i += 256) {
      const int kk = i / S, c = i % S;
      Xs[kk][c] = (k0 + kk < n) ? X[(k0 + kk) * S + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kFK; ++kk) {
      const double a = As[tr][kk];
#pragma unroll
      for (int j = 0; j < CPT; ++j) acc[j] = fma(a, Xs[kk][tc + 4 * j], acc[j]);
    }
  }
  if (r0 + tr < m)
#pragma unroll
    for (int j = 0; j < CPT; ++j) Y[(r0 + tr) * S + tc + 4 * j] = acc[j];
}

// Z (n x S) += A^T W over this block's row range: block (column tile, row
// slice); the partial sums of the row slices meet in fp64 atomics (Z zeroed
// by the caller).
template <int S>
__global__ void __launch_bounds__(256) f64_transpose(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                                     const double* __restrict__ W, double* __restrict__ Z,
                                                     int64_t rows_per_slice) {
  __shared__ double As[kFK][kFT + 1];
  __shared__ double Ws[kFK][S];
  constexpr int CPT = S / 4;
  const int tid = threadIdx.x, tr = tid >> 2, tc = tid & 3;  // 64 A columns x 4 column groups
  const int64_t c0 = (int64_t)blockIdx.x * kFT;
  const int64_t k_begin = (int64_t)blockIdx.y * rows_per_slice, k_end = min64(m, k_begin + rows_per_slice);
  double acc[CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) acc[j] = 0.0;
  for (int64_t k0 = k_begin; k0 < k_end; k0 += kFK) {
    __syncthreads();
    for (int i = tid; i < kFK * kFT; i += 256) {
      const int kk = i / kFT, cc = i % kFT;
      As[kk][cc] = (k0 + kk < k_end && c0 + cc < n) ? A[(k0 + kk) * lda + c0 + cc] : 0.0;
    }
    for (int i = tid; i < kFK * S; i += 256) {
      const int kk = i / S, c = i % S;
      Ws[kk][c] = (k0 + kk < k_end) ? W[(k0 + kk) * S + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kFK; ++kk) {
      const double a = As[kk][tr];
#pragma unroll
      for (int j = 0; j < CPT; ++j) acc[j] = fma(a, Ws[kk][tc + 4 * j], acc[j]);
    }
  }
  if (c0 + tr < n)
#pragma unroll
    for (int j = 0; j < CPT; ++j) atomicAdd(&Z[(c0 + tr) * S + tc + 4 * j], acc[j]);
}

// P <- P T in place (T upper triangular S x S, fp64): one thread per row
template <int S>
__global__ void f64_apply(double* __restrict__ P, int64_t rows, const double* __restrict__ T) {
  __shared__ double Ts[S * S];
  for (int i = threadIdx.x; i < S * S; i += blockDim.x) Ts[i] = T[i];
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    double in[S], o[S];
#pragma unroll
    for (int c = 0; c < S; ++c) in[c] = P[r * S + c];
#pragma unroll
    for (int c = 0; c < S; ++c) {
      double acc = 0.0;
      for (int j = 0; j <= c; ++j) acc = fma(in[j], Ts[j * S + c], acc);
      o[c] = acc;
    }
#pragma unroll
    for (int c = 0; c < S; ++c) P[r * S + c] = o[c];
  }
}

__global__ void f64_init_info(int* info) {
  info[0] = 0;
  info[1] = 1 << 30;
}

template <int S>
int run_f64(const double* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed, int side, double* Q,
            void* ws, size_t ws_bytes, cudaStream_t st) {
  const int64_t big = std::max(m, n);
  const size_t need = ((size_t)big * S * 2 + 2 * (size_t)S * S) * 8 + 64;
  if (ws_bytes < need) return fail(CNMF_ERR_ARGUMENT, "fp64 range finder: workspace too small");
  double* Pm = side == 0 ? Q : (double*)ws;                     // m x S panel
  double* Pn = side == 0 ? (double*)ws : Q;                     // n x S panel
  double* G = (double*)ws + (size_t)big * S * 2;
  double* T = G + (size_t)S * S;
  int* info = (int*)(T + (size_t)S * S);
  f64_init_info<<<1, 1, 0, st>>>(info);
  CNMF_LAUNCH_CHECK();
  const int dev_sms = device_sms();
  auto forward = [&](const double* X, double* Y) -> int {  // Y = A X
    f64_forward<S><<<(unsigned)ceil_div(m, kFT), 256, 0, st>>>(A, m, n, lda, X, Y);
    CNMF_LAUNCH_CHECK();
    return CNMF_OK;
  };
  auto transpose = [&](const double* W, double* Z) -> int {  // Z = A^T W
    CNMF_CUDA(cudaMemsetAsync(Z, 0, (size_t)n * S * 8, st));
    const int64_t ctiles = ceil_div(n, kFT);
    const int64_t slices = std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 4 * dev_sms / std::max<int64_t>(ctiles, 1)));
    const int64_t rps = ceil_div(ceil_div(m, slices), kFK) * kFK;
    f64_transpose<S><<<dim3((unsigned)ctiles, (unsigned)ceil_div(m, rps)), 256, 0, st>>>(A, m, n, lda, W, Z, rps);
    CNMF_LAUNCH_CHECK();
    return CNMF_OK;
  };
  int pass_id = 0;
  auto orth = [&](double* P, int64_t rows) -> int {  // CholeskyQR2
    for (int sweep = 0; sweep < 2; ++sweep) {
      CNMF_CUDA(cudaMemsetAsync(G, 0, (size_t)S * S * 8, st));
      CNMF_TRY(gram_tn_f64(P, rows, S, P, S, G, st));
      CNMF_TRY(chol_inv(G, s, S, T, nullptr, info, pass_id, st));
      f64_apply<S><<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 128), 4 * dev_sms)), 128,
                     0, st>>>(P, rows, T);
      CNMF_LAUNCH_CHECK();
    }
    ++pass_id;
    return CNMF_OK;
  };
  // the seeded test matrix (compress.py:125-127), rows = A.cols (column
  // basis) or A.rows (row basis), padding columns zero
  double* omega = side == 0 ? Pn : Pm;
  const int64_t orows = side == 0 ? n : m;
  CNMF_CUDA(cudaMemsetAsync(omega, 0, (size_t)orows * S * 8, st));
  CNMF_TRY(gaussian_fill(child_seed(seed, "omega"), orows, s, 4096, CNMF_F64, omega, S, st));
  if (side == 0) {
    CNMF_TRY(forward(Pn, Pm));
    CNMF_TRY(orth(Pm, m));
    for (int t = 0; t < w; ++t) {
      CNMF_TRY(transpose(Pm, Pn));
      CNMF_TRY(orth(Pn, n));
      CNMF_TRY(forward(Pn, Pm));
      CNMF_TRY(orth(Pm, m));
    }
  } else {
    CNMF_TRY(transpose(Pm, Pn));
    CNMF_TRY(orth(Pn, n));
    for (int t = 0; t < w; ++t) {
      CNMF_TRY(forward(Pn, Pm));
      CNMF_TRY(orth(Pm, m));
      CNMF_TRY(transpose(Pm, Pn));
      CNMF_TRY(orth(Pn, n));
    }
  }
  int h[2];
  CNMF_CUDA(cudaMemcpyAsync(h, info, sizeof(h), cudaMemcpyDeviceToHost, st));
  CNMF_CUDA(cudaStreamSynchronize(st));
  if (h[1] != (1 << 30)) return fail(CNMF_ERR_NUMERIC, "fp64 range finder: Gram matrix not factorable");
  return CNMF_OK;
}

// ||A - X Y||_F^2 and ||A||_F^2 of an fp64 A (X: m x r, Yt: n x r, fp64), or
// of A - A[:, cols] Y (cols != null)
__global__ void f64_resid(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                          const double* __restrict__ X, const int64_t* __restrict__ cols,
                          const double* __restrict__ Yt, int r, double* __restrict__ out) {
  double res = 0.0, ref = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m * n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / n, col = i - row * n;
    double p = 0.0;
    for (int k = 0; k < r; ++k) {
      const double x = cols ? A[row * lda + cols[k]] : X[row * r + k];
      p = fma(x, Yt[col * r + k], p);
    }
    const double a = A[row * lda + col], d = a - p;
    res = fma(d, d, res);
    ref = fma(a, a, ref);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    res += __shfl_xor_sync(0xffffffffu, res, o);
    ref += __shfl_xor_sync(0xffffffffu, ref, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], res);
    atomicAdd(&out[1], ref);
  }
}

}  // namespace

size_t compress_f64_workspace(int64_t m, int64_t n, int s) {
  const int S = panel_ld(s);
  if (S < 0) return 0;
  return ((size_t)std::max(m, n) * S * 2 + 2 * (size_t)S * S) * 8 + 64;
}

int structured_compress_f64(const double* A, int64_t m, int64_t n, int64_t lda, int s, int w, uint64_t seed, int side,
                            double* Q, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (A == nullptr || m < 1 || n < 1 || lda < n) return fail(CNMF_ERR_ARGUMENT, "A must be a non-empty fp64 matrix");
  if (s < 1 || w < 0) return fail(CNMF_ERR_ARGUMENT, "bad width or power exponent");
  if (s > std::min(m, n))
    return fail(CNMF_ERR_INFEASIBLE_RANK, "basis width " + std::to_string(s) + " exceeds min(m, n) = " +
                                              std::to_string(std::min(m, n)) + "; adjust_config first");
  switch (panel_ld(s)) {
    case 32: return run_f64<32>(A, m, n, lda, s, w, seed, side, Q, ws, ws_bytes, st);
    case 64: return run_f64<64>(A, m, n, lda, s, w, seed, side, Q, ws, ws_bytes, st);
  }
  return fail(CNMF_ERR_ARGUMENT, "fp64 range finder supports widths <= 64");
}

int pass_transpose_f64(const double* A, int64_t m, int64_t n, int64_t lda, const double* W, int s, double* Z,
                       cudaStream_t st) {
  const int S = panel_ld(s);
  CNMF_CUDA(cudaMemsetAsync(Z, 0, (size_t)n * S * 8, st));
  const int64_t ctiles = ceil_div(n, kFT);
  const int64_t slices =
      std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 4 * device_sms() / std::max<int64_t>(ctiles, 1)));
  const int64_t rps = ceil_div(ceil_div(m, slices), kFK) * kFK;
  const dim3 grid((unsigned)ctiles, (unsigned)ceil_div(m, rps));
  if (S == 32)
    f64_transpose<32><<<grid, 256, 0, st>>>(A, m, n, lda, W, Z, rps);
  else if (S == 64)
    f64_transpose<64><<<grid, 256, 0, st>>>(A, m, n, lda, W, Z, rps);
  else
    return fail(CNMF_ERR_ARGUMENT, "fp64 pass supports widths <= 64");
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

int residual_norms_f64(const double* A, int64_t m, int64_t n, int64_t lda, const double* X, const int64_t* cols,
                       const double* Yt, int r, double* out, cudaStream_t st) {
  if ((X == nullptr) == (cols == nullptr)) return fail(CNMF_ERR_ARGUMENT, "give exactly one of X and cols");
  CNMF_CUDA(cudaMemsetAsync(out, 0, 16, st));
  f64_resid<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m * n, 256), 8 * device_sms())), 256, 0,
              st>>>(A, m, n, lda, X, cols, Yt, r, out);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

}  // namespace cnmf
