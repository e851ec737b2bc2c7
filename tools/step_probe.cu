// cycles per barrier-separated step of small fp64 shared-memory work (256 threads)
#include <cstdio>
template <int V>
__global__ void k(long long* cyc, double* out, int steps) {
  __shared__ double buf[2][32 * 33];
  const int tid = threadIdx.x;
  for (int i = tid; i < 2 * 32 * 33; i += 256) (&buf[0][0])[i] = 1.0 + 0.001 * (i % 7);
  __syncthreads();
  double acc = 0.0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const int src = s & 1, dst = src ^ 1;
    if (V == 0) {  // barrier only
    } else if (V == 1) {  // + 1 broadcast load + 1 fma
      acc = fma(buf[src][(s & 31) * 33], 1.0001, acc);
    } else if (V == 2) {  // + one element: 3 loads, fma, store
      const int i = tid >> 5, j = tid & 31;
      buf[dst][i * 33 + j] = buf[src][i * 33 + j] - buf[src][i * 33 + (s & 31)] * buf[src][(s & 31) * 33 + j];
    } else if (V == 3) {  // four elements per thread (the Gauss-Jordan pattern)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int idx = tid + 256 * t, i = idx >> 5, j = idx & 31;
        buf[dst][i * 33 + j] = buf[src][i * 33 + j] - buf[src][i * 33 + (s & 31)] * buf[src][(s & 31) * 33 + j];
      }
    } else if (V == 4) {  // four elements, pivot-row element loaded once
      const int j = tid & 31;
      const double pr = buf[src][(s & 31) * 33 + j];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int i = (tid >> 5) + 8 * t;
        buf[dst][i * 33 + j] = buf[src][i * 33 + j] - buf[src][i * 33 + (s & 31)] * pr;
      }
    } else if (V == 5) {  // four elements in registers, column via shuffle, row via smem
      // (register state carried in acc-like variables)
    }
    __syncthreads();
  }
  long long t1 = clock64();
  out[tid] = acc + buf[0][tid % 64];
  if (tid == 0) cyc[V] = (t1 - t0) / steps;
}
int main() {
  long long* c; double* o; long long h[6];
  cudaMalloc(&c, 64); cudaMalloc(&o, 4096);
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 256>>>(c, o, 200); k<1><<<1, 256>>>(c, o, 200); k<2><<<1, 256>>>(c, o, 200);
    k<3><<<1, 256>>>(c, o, 200); k<4><<<1, 256>>>(c, o, 200);
    cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("cycles/step: barrier %lld | +bcast fma %lld | 1 elem %lld | 4 elem %lld | 4 elem hoisted %lld\n", h[0], h[1], h[2], h[3], h[4]);
  }
  return 0;
}
