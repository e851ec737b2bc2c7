// cycles per elimination step of the 256-thread register-tile Cholesky (chol.cuh) and variants
#include <cstdio>
#include "../paper_1505_04650_b200/csrc/chol.cuh"
using namespace cnmf;

template <int V>
__global__ void k(double* out, long long* cyc, int s) {
  __shared__ double buf[256];
  const int t = threadIdx.x, j = t & 31, i0 = t >> 5;
  double a[4];
  for (int q = 0; q < 4; ++q) a[q] = (i0 + 8 * q == j) ? 40.0 : 0.01 * ((i0 + 8 * q + j) % 7);
  __syncthreads();
  long long t0 = clock64();
  bool ok = true;
  for (int kk = 0; kk < s; ++kk) {
    double* colk = buf + (kk & 1) * 64;
    double* rowk = colk + 32;
    if (j == kk)
#pragma unroll
      for (int q = 0; q < 4; ++q) colk[i0 + 8 * q] = a[q];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i0 + 8 * q == kk) rowk[j] = a[q];
    __syncthreads();
    const double d = rowk[kk];
    ok = ok && (d > 1e-30);
    double inv;
    if (V == 0) inv = rcp64(d);
    else if (V == 1) inv = 1.0 / d;
    else inv = 0.025;
    const double rkj = rowk[j];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + 8 * q;
      if (i > kk) {
        const double f = colk[i] * inv;
        a[q] = (j == kk) ? -f : fma(-f, rkj, a[q]);
      }
    }
  }
  long long t1 = clock64();
  out[t] = a[0] + a[1] + a[2] + a[3] + ok;
  if (t == 0) cyc[V] = (t1 - t0) / s;
}
__global__ void syncloop(long long* cyc, int s) {
  __shared__ double buf[64];
  long long t0 = clock64();
  double x = 0;
  for (int kk = 0; kk < s; ++kk) { if (threadIdx.x == kk) buf[kk & 63] = x + kk; __syncthreads(); x += buf[kk & 63]; }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / s + (x > 1e30);
}
int main() {
  double* o; long long* c; long long h[4];
  cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 256>>>(o, c, 30); k<1><<<1, 256>>>(o, c, 30); k<2><<<1, 256>>>(o, c, 30); syncloop<<<1, 256>>>(c, 30);
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("cycles/step: rcp64 %lld, div %lld, no-div %lld, bare sync+lds %lld\n", h[0], h[1], h[2], h[3]);
  }
  return 0;
}
