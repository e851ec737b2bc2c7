// Cost of block barriers in a loop (512 threads): named bar.sync, __syncthreads,
// and a publish (one thread stores, barrier, all load) round trip.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double sh[2][64];
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, %0;" :: "r"(blockDim.x) : "memory");
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) {
    if (threadIdx.x == (i & 511)) sh[i & 1][0] = acc + i;
    asm volatile("bar.sync 1, %0;" :: "r"(blockDim.x) : "memory");
    acc += sh[i & 1][0];
  }
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) {
    if (threadIdx.x == (i & 511)) sh[i & 1][0] = 1.0 / (acc + i);
    asm volatile("bar.sync 1, %0;" :: "r"(blockDim.x) : "memory");
    acc = fma(acc, 0.5, sh[i & 1][0]);
  }
  long long t4 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  long long h[4];
  for (int nt : {128, 512}) {
  k<<<1, nt>>>(o, c, 100); cudaDeviceSynchronize();
  k<<<1, nt>>>(o, c, 1000); cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("threads %d: bar.sync %.1f  __syncthreads %.1f  publish %.1f  publish+div chain %.1f cycles per iteration (%s)\n", nt, h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, cudaGetErrorString(cudaGetLastError()));
  }
}
