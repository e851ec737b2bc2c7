// Composition of one CholeskyQR sweep on a configs[1]-sized panel:
// Gram only / Gram + last-block factor / full cooperative sweep (Gram,
// factor, apply), CUDA-event timed back to back.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/sweep_probe.cu
//        paper_1505_04650_b200/csrc/build/{pass,tc_pass,common}.o -o tools/sweep_probe.bin -lcuda
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

namespace cnmf {
int panel_finalize_chol(float*, int64_t, int, const double*, double*, int, double*, double*, int*, int, unsigned*,
                        cudaStream_t, int apply_after);
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 10000;
  const int s = 30, S = 32, reps = 50;
  float* P;
  double *G, *T;
  int* info;
  unsigned* counter;
  cudaMalloc(&P, rows * S * 4);
  cudaMalloc(&G, S * S * 8);
  cudaMalloc(&T, S * S * 8);
  cudaMalloc(&info, 64);
  cudaMalloc(&counter, 64);
  cudaMemset(G, 0, S * S * 8);
  cudaMemset(info, 0, 64);
  cudaMemset(counter, 0, 64);
  float* h = (float*)malloc(rows * S * 4);
  srand(3);
  for (int64_t i = 0; i < rows * S; ++i) h[i] = (i % S) < s ? rand() / (float)RAND_MAX - 0.5f : 0.f;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"gram only", "gram+factor", "gram+factor+apply (coop)"};
  for (int mode = 0; mode < 3; ++mode) {
    float tot = 0;
    for (int r = 0; r < reps; ++r) {
      cudaMemcpy(P, h, rows * S * 4, cudaMemcpyHostToDevice);
      cudaMemset(G, 0, S * S * 8);
      cudaEventRecord(e0);
      cnmf::panel_finalize_chol(P, rows, S, nullptr, G, s, T, nullptr, info, 0, mode ? counter : nullptr, 0,
                                mode == 2 ? 1 : 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 5) tot += ms;
    }
    printf("rows %lld %-28s %7.1f us (%s)\n", (long long)rows, names[mode], tot / (reps - 5) * 1e3,
           cudaGetErrorString(cudaGetLastError()));
  }
  // back-to-back sweeps (what the range finder does between passes)
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r)
    cnmf::panel_finalize_chol(P, rows, S, nullptr, G, s, T, nullptr, info, 0, counter, 0, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("rows %lld back-to-back full sweeps: %7.1f us each\n", (long long)rows, ms / reps * 1e3);
  return 0;
}
