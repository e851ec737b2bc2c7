// Latency of a dependent fp64 reciprocal chain: IEEE division, __drcp_rn,
// and MUFU.RCP64H + two Newton steps.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_nr(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}
__global__ void lat(double* out, long long* cyc, int n) {
  double x = 1.5 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = rcp_nr(x + 1.0);
  long long t3 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  long long h[3];
  lat<<<1, 32>>>(o, c, 100); cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, 1000); cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("1.0/x %.1f  __drcp_rn %.1f  rcp.approx+2NR %.1f cycles per dependent op\n", h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0);
}
