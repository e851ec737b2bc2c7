// cycles per pivot of small block Gauss-Jordan variants (the ADMM core solves)
#include <cstdio>
__device__ __forceinline__ double rcp64(double d) {
  double x = (double)__frcp_rn((float)d);
  x = x * fma(-d, x, 2.0);
  x = x * fma(-d, x, 2.0);
  return fma(x, fma(-d, x, 1.0), x);
}
// Gauss-Jordan inverse of the leading r x r block of the RP x RP SPD matrix M
// (RP <= 32) with the matrix in registers: warp w owns rows w + 8 t, lane j
// column j. Per pivot k the owner warp publishes row k to shared memory (one
// store), column k reaches every row owner by a shuffle from lane k, and one
// barrier separates the pivots; shared-memory traffic per pivot is ~1/6 of the
// shared-memory formulation, which is what bounds these tiny fp64 kernels.
// Padded entries: diagonal pen is inverted, off-diagonal stay zero. In place.
template <int RP, int DV = 0>
__device__ void gj_inverse_reg(double* M, double* strip, int r) {
  static_assert(RP <= 32 && RP % 8 == 0, "one column per lane, RP/8 rows per warp");
  constexpr int LR = RP + 1, RT = RP / 8;
  const int w = threadIdx.x >> 5, j = threadIdx.x & 31;
  double a[RT];
#pragma unroll
  for (int t = 0; t < RT; ++t) a[t] = (j < RP) ? M[(w + 8 * t) * LR + j] : 0.0;
#pragma unroll
  for (int k = 0; k < RP; ++k) {
    if (k >= r) break;  // uniform; k is a compile-time constant inside the unrolled body
    double* prow = strip + (k & 1) * 32;
    if (w == (k & 7) && j < RP) {
      // select chain (a dynamically indexed read would demote a[] to local memory)
      double v = a[0];
#pragma unroll
      for (int t = 1; t < RT; ++t) v = (t == (k >> 3)) ? a[t] : v;
      prow[j] = v;
    }
    double colk[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) colk[t] = __shfl_sync(0xffffffffu, a[t], k);
    __syncthreads();
    const double inv = DV == 0 ? 1.0 / prow[k] : (DV == 1 ? rcp64(prow[k]) : 0.025);
    const double pk = (j == k) ? 1.0 : prow[j];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int i = w + 8 * t;
      if (i < r && j < r) {
        const double nk = pk * inv;
        a[t] = (i == k) ? nk : ((j == k) ? 0.0 : a[t]) - colk[t] * nk;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < RT; ++t) {
    const int i = w + 8 * t;
    if (j < RP) M[i * LR + j] = (i >= r && i == j) ? 1.0 / a[t] : a[t];
  }
  __syncthreads();
}

template <int V>
__global__ void probe3(long long* cyc, double* out, int r) {
  __shared__ double M[32 * 33], strip[64];
  for (int i = threadIdx.x; i < 32 * 33; i += blockDim.x) M[i] = (i % 34 == 0) ? 40.0 : 0.01 * (i % 5);
  __syncthreads();
  long long t0 = clock64();
  gj_inverse_reg<32, V>(M, strip, r);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[6 + V] = t1 - t0;
  out[threadIdx.x] = M[threadIdx.x];
}

template <int V>
__device__ void gj(double* M, double* T, int r) {
  constexpr int RP = 32, LR = 33;
  const int tid = threadIdx.x;
  double* src = M;
  double* dst = T;
  for (int k = 0; k < r; ++k) {
    const double inv = (V == 1) ? 0.025 : (V == 3 ? 1.0 / src[k * LR + k] : rcp64(src[k * LR + k]));
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int idx = tid + t * 256;
      const int i = idx / RP, j = idx % RP;
      if (i < r && j < r) {
        if (V == 2) {
          dst[i * LR + j] = src[i * LR + j] * inv;
        } else {
          const double nk = ((j == k) ? 1.0 : src[k * LR + j]) * inv;
          dst[i * LR + j] = (i == k) ? nk : ((j == k) ? 0.0 : src[i * LR + j]) - src[i * LR + k] * nk;
        }
      }
    }
    __syncthreads();
    double* tmp = src;
    src = dst;
    dst = tmp;
  }
}
// V = 4: shared buffers indexed by pivot parity (no pointer swap: the compiler
// keeps shared-memory addressing); V = 5: same plus scale-only
template <int V>
__device__ void gj_par(int r) {
  constexpr int RP = 32, LR = 33;
  __shared__ double buf[2][32 * 33];
  const int tid = threadIdx.x;
  for (int k = 0; k < r; ++k) {
    const int s = k & 1, d = s ^ 1;
    const double inv = rcp64(buf[s][k * LR + k]);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int idx = tid + t * 256;
      const int i = idx / RP, j = idx % RP;
      if (i < r && j < r) {
        if (V == 5) {
          buf[d][i * LR + j] = buf[s][i * LR + j] * inv;
        } else {
          const double nk = ((j == k) ? 1.0 : buf[s][k * LR + j]) * inv;
          buf[d][i * LR + j] = (i == k) ? nk : ((j == k) ? 0.0 : buf[s][i * LR + j]) - buf[s][i * LR + k] * nk;
        }
      }
    }
    __syncthreads();
  }
}
template <int V>
__global__ void probe2(long long* cyc, double* out, int r) {
  long long t0 = clock64();
  gj_par<V>(r);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[V] = t1 - t0;
}
template <int V>
__global__ void probe(long long* cyc, double* out, int r) {
  __shared__ double M[32 * 33], T[32 * 33];
  for (int i = threadIdx.x; i < 32 * 33; i += blockDim.x) M[i] = (i % 34 == 0) ? 40.0 : 0.01 * (i % 5);
  __syncthreads();
  long long t0 = clock64();
  gj<V>(M, T, r);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[V] = t1 - t0;
  out[threadIdx.x] = M[threadIdx.x] + T[threadIdx.x];
}
int main() {
  long long* c; double* o; long long h[10];
  cudaMalloc(&c, 128); cudaMalloc(&o, 8192);
  for (int rep = 0; rep < 2; ++rep) {
    probe<0><<<1, 256>>>(c, o, 20); probe<1><<<1, 256>>>(c, o, 20); probe<2><<<1, 256>>>(c, o, 20); probe<3><<<1, 256>>>(c, o, 20);
    probe2<4><<<1, 256>>>(c, o, 20); probe2<5><<<1, 256>>>(c, o, 20); probe3<0><<<1, 256>>>(c, o, 20);
    probe3<1><<<1, 256>>>(c, o, 20); probe3<2><<<1, 256>>>(c, o, 20);
    cudaMemcpy(h, c, 72, cudaMemcpyDeviceToHost);
    printf("register GJ cycles/pivot: ddiv %lld, rcp64 %lld, no division %lld\n", h[6] / 20, h[7] / 20, h[8] / 20);
    printf("cycles/pivot: rcp64 %lld, const-inv %lld, scale-only %lld, ddiv %lld | shared-indexed %lld, scale-only %lld\n",
           h[0] / 20, h[1] / 20, h[2] / 20, h[3] / 20, h[4] / 20, h[5] / 20);
  }
  return 0;
}
