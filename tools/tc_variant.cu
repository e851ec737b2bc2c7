// Time pass_tc (no tracing) for one ring configuration; build several with
// -DCNMF_TC_RINGS -DCNMF_TC_ST=.. -DCNMF_TC_SSP=.. -DCNMF_TC_AST=.. (tools/tc_variant.sh)
#include "../paper_1505_04650_b200/csrc/tc_pass.cu"

#include <cstdio>
#include <cstdlib>

int main(int argc, char** argv) {
  const int64_t M = argc > 1 ? atoll(argv[1]) : 10000, N = argc > 2 ? atoll(argv[2]) : 5000;
  const int S = 32, reps = 30;
  float *A, *X, *W, *Y, *Z;
  cudaMalloc(&A, M * N * 4);
  cudaMemset(A, 0x3c, M * N * 4);
  cudaMalloc(&X, N * S * 4);
  cudaMemset(X, 0x3c, N * S * 4);
  cudaMalloc(&W, M * S * 4);
  cudaMemset(W, 0x3c, M * S * 4);
  cudaMalloc(&Y, M * S * 4);
  cudaMalloc(&Z, N * S * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int t = 0; t < 2; ++t) {
    auto run = [&]() {
      return t ? cnmf::pass_transpose_tc(A, M, N, N, W, S, Z, 0) : cnmf::pass_forward_tc(A, M, N, N, X, S, Y, 0);
    };
    for (int r = 0; r < 3; ++r) run();
    cudaDeviceSynchronize();
    float best = 1e9, tot = 0;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0);
      run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
      tot += ms;
    }
    const double bytes = 4.0 * (M * N + (M + N) * S);
    printf("%s %s: avg %.1f us (%.0f GB/s) best %.1f us\n", argv[0], t ? "trn" : "fwd", tot / reps * 1e3,
           bytes / (tot / reps * 1e-3) / 1e9, best * 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
