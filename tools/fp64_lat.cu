// Latency of dependent DFMA / DMUL / DADD chains and of shared-memory
// round trips with one warp (B200).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, int n) {
  double x = threadIdx.x * 1e-9 + 1.0, y = 1.0000001;
  __shared__ double sh[64];
  sh[threadIdx.x & 63] = x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  long long t2 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) { sh[threadIdx.x & 31] = z; __syncwarp(); z = sh[(threadIdx.x + 1) & 31] + 1e-9; __syncwarp(); }
  long long t3 = clock64();
  float f = x;
  for (int i = 0; i < n; ++i) f = fmaf(f, 1.0000001f, 1e-7f);
  long long t4 = clock64();
  out[threadIdx.x] = x + z + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  long long h[4];
  for (int w : {32, 128}) {
    lat<<<1, w>>>(o, c, 1000); cudaDeviceSynchronize();
    lat<<<1, w>>>(o, c, 1000); cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("threads %d: DFMA %.1f  DMUL %.1f  STS+LDS(fp64) %.1f  FFMA %.1f cycles per dependent op\n", w, h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0);
  }
}
