// Time the small Cholesky-inverse device routines on a random SPD Gram matrix.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/chol_bench.cu
//        paper_1505_04650_b200/csrc/common.cu -o tools/chol_bench.bin
#define CHOL_TIMING 1
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1505_04650_b200/csrc/chol.cuh"

using namespace cnmf;

__global__ void k_block(double* G, int s, int S, double* T, int* info) {
  extern __shared__ double a[];
  chol_block(G, s, S, T, nullptr, info, 0, a);
}
__global__ void k_tile(double* G, int s, int S, double* T, int* info) {
  __shared__ double buf[32 * 33 + 128];
  chol_tile32(G, s, S, T, nullptr, info, 0, buf);
}

__global__ void k_empty(double* G, int s, int S, double* T, int* info) {}

int main() {
  const int s = 30, S = 32;
  std::vector<double> h(S * S, 0.0), M(S * S);
  srand(1);
  for (auto& x : M) x = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j) {
      double v = (i == j) ? 4.0 : 0.0;
      for (int k = 0; k < S; ++k) v += M[i * S + k] * M[j * S + k];
      h[i * S + j] = v;
    }
  double *G, *G0, *T;
  int* info;
  cudaMalloc(&G, S * S * 8);
  cudaMalloc(&G0, S * S * 8);
  cudaMalloc(&T, S * S * 8);
  cudaMalloc(&info, 64);
  cudaMemcpy(G0, h.data(), S * S * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 2; v >= 0; --v) {
    float tot = 0;
    for (int r = 0; r < 20; ++r) {
      cudaMemcpy(G, G0, S * S * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      if (v == 2)
        k_empty<<<1, 256>>>(G, s, S, T, info);
      else if (v == 0)
        k_block<<<1, 256, (s * s + 2 * s) * 8>>>(G, s, S, T, info);
      else
        k_tile<<<1, 256>>>(G, s, S, T, info);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 5) tot += ms;
    }
    std::vector<double> t(S * S);
    cudaMemcpy(t.data(), T, S * S * 8, cudaMemcpyDeviceToHost);
    // check T^T G T = I
    double err = 0;
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) {
        double v = 0;
        for (int a = 0; a < s; ++a)
          for (int b = 0; b < s; ++b) v += t[a * S + i] * h[a * S + b] * t[b * S + j];
        err = fmax(err, fabs(v - (i == j)));
      }
    printf("%s: %.1f us  |T^T G T - I| = %.2e  (%s)\n", v == 2 ? "empty" : v ? "tile" : "block", tot / 15 * 1e3, err,
           cudaGetErrorString(cudaGetLastError()));
  }
  long long ht[8];
  cudaMemcpyFromSymbol(ht, g_chol_t, sizeof ht);
  printf("tile phases: load %lld, elim %lld, out %lld cycles\n", ht[1] - ht[0], ht[2] - ht[1], ht[3] - ht[2]);
  return 0;
}
