// Throughput of fp64 mma.sync (DMMA m8n8k4) vs DFMA on this GPU: register
// operands only, 8 independent accumulator tiles per warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) c[t] = fma(a, b, c[t]);
  }
  double s = 0;
  for (int t = 0; t < 16; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    int it = 4000; float ms;
    dmma_loop<<<148 * 4, 32 * warps>>>(out, 10);
    cudaEventRecord(e0); dmma_loop<<<148 * 4, 32 * warps>>>(out, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * it * (148.0 * 4 * warps);
    printf("DMMA warps/block %d: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    dfma_loop<<<148 * 4, 32 * warps>>>(out, 10);
    cudaEventRecord(e0); dfma_loop<<<148 * 4, 32 * warps>>>(out, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * it * (148.0 * 4 * warps * 32);
    printf("DFMA warps/block %d: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
