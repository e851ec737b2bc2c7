// DFMA and FFMA issue throughput per SM (independent chains), to size the
// fp64 pieces (Gram, Cholesky, ADMM state).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void k(T* out, int iters) {
  T a[8];
  for (int j = 0; j < 8; ++j) a[j] = (T)(threadIdx.x + j);
  const T b = (T)1.0000001, c = (T)0.5;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = a[j] * b + c;
  T s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == (T)12345) out[0] = s;
}
int main() {
  double* d;
  float* f;
  cudaMalloc(&d, 8);
  cudaMalloc(&f, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, blocks = 148 * 4, threads = 256;
  for (int t = 0; t < 2; ++t) {
    for (int r = 0; r < 2; ++r) t ? k<float><<<blocks, threads>>>(f, iters) : k<double><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e0);
    t ? k<float><<<blocks, threads>>>(f, iters) : k<double><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fma = (double)blocks * threads * iters * 8;
    printf("%s: %.2f TFMA/s = %.1f TFLOP/s (%.1f per SM per clock at 1.965 GHz)\n", t ? "FFMA" : "DFMA",
           fma / (ms * 1e-3) / 1e12, 2 * fma / (ms * 1e-3) / 1e12, fma / (ms * 1e-3) / 148 / 1.965e9);
  }
}
