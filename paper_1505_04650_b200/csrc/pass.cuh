// Streaming passes over A (csrc/pass.cu dispatch, csrc/tc_pass.cu tensor-core kernels).
#pragma once

#include "common.cuh"

namespace cnmf {

int panel_ld(int s);
// Y = A X (forward) / Z = A^T W (transpose)
int pass_forward(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y, cudaStream_t st);
int pass_transpose(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, int S, float* Z,
                   cudaStream_t st);
int pass_forward_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y,
                    cudaStream_t st);
int pass_forward_sumsq_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y,
                          double* sumsq, cudaStream_t st);
bool pass_uses_tc(int S);
int pass_forward_sumsq(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y,
                       double* sumsq, cudaStream_t st);
int pass_forward_tc2(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y,
                     cudaStream_t st);
int pass_forward_sumsq_tc2(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, int S, float* Y,
                           double* sumsq, cudaStream_t st);
int pass_transpose_tc2(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, int S, float* Z,
                       cudaStream_t st);
int pass_pair_tc2(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, const float* W,
                  float* Z, int S, cudaStream_t st);
int pass_transpose_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* W, int S, float* Z,
                      cudaStream_t st);
// Y = A X and Z = A^T W in one launch (one A-read pipeline ramp per pair)
int pass_pair(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, const float* W, float* Z,
              int S, cudaStream_t st);
int pass_pair_tc(const float* A, int64_t m, int64_t n, int64_t lda, const float* X, float* Y, const float* W, float* Z,
                 int S, cudaStream_t st);

}  // namespace cnmf
