// Run-to-run bitwise check of the tensor-core passes (includes the kernel
// source given by -DTC_SRC) on random data: tools/tc_check.sh
#include TC_SRC

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

int main(int argc, char** argv) {
  const int64_t M = argc > 1 ? atoll(argv[1]) : 4000, N = argc > 2 ? atoll(argv[2]) : 3000;
  const int S = 32, reps = 8;
  std::vector<float> h(M * N), hw(M * S);
  srand(1);
  for (auto& x : h) x = rand() / (float)RAND_MAX;
  for (auto& x : hw) x = rand() / (float)RAND_MAX - 0.5f;
  float *A, *W, *Z;
  cudaMalloc(&A, M * N * 4);
  cudaMalloc(&W, M * S * 4);
  cudaMalloc(&Z, N * S * 4);
  cudaMemcpy(A, h.data(), M * N * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(W, hw.data(), M * S * 4, cudaMemcpyHostToDevice);
  std::vector<float> z0(N * S), z(N * S);
  int diffs = 0;
  for (int r = 0; r < reps; ++r) {
    cudaMemset(Z, 0, N * S * 4);
    int st = TC_CALL;
    if (st) printf("status %d\n", st);
    cudaMemcpy(r ? z.data() : z0.data(), Z, N * S * 4, cudaMemcpyDeviceToHost);
    if (r) {
      int bad = 0;
      for (int64_t i = 0; i < N * S; ++i) bad += z[i] != z0[i];
      if (bad) ++diffs;
      if (bad) printf("rep %d: %d entries differ\n", r, bad);
    }
  }
  printf("%s %lldx%lld: %d of %d repeats differ (%s)\n", argv[0], (long long)M, (long long)N, diffs, reps - 1,
         cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
