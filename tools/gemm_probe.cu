
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kCT = 512;
#ifndef GEMMFN
#define GEMMFN small_gemm
#endif
// D (8 x 8) += A (8 x 4, row g, column t) B (4 x 8, row t, column g); the
// accumulator holds row g, columns 2 t, 2 t + 1 (g = lane / 4, t = lane % 4)
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// C(m, n) = sum_k A[m * am + k * ak] * B[k * bk + n * bn] for m < M, n < N <= 64,
// M <= 64; out(m, n, value) consumes every result exactly once. On the fp64
// tensor cores: the (ceil(M/8) x ceil(N/8)) 8 x 8 output tiles are dealt to
// the 16 warps (up to 4 each, accumulated together so the k loop has 4
// independent DMMA chains); per k step of 4 a lane loads one A and one B
// element per tile (zero outside the bounds).
template <class F>
__device__ __forceinline__ void small_gemm(int M, int N, int K, const double* A, int am, int ak, const double* B,
                                           int bk, int bn, F out) {
  static_assert(kCT == 512, "16 warps x 4 tiles cover 64 x 64");
  constexpr int NW = kCT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int tn = (N + 7) >> 3, nt = ((M + 7) >> 3) * tn;
  if (warp >= nt) return;
  int ma[4], nb[4];
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int t = warp + NW * j;
    const int tm_ = t < nt ? t / tn : 0, tn_ = t < nt ? t - tm_ * tn : 0;
    ma[j] = 8 * tm_ + g;  // this lane's A row
    nb[j] = 8 * tn_ + g;  // this lane's B column
    acc[j][0] = acc[j][1] = 0.0;
  }
  const int ntw = (nt - warp + NW - 1) / NW;  // tiles of this warp (1..4), warp-uniform
  for (int k0 = 0; k0 < K; k0 += 4) {
    const int k = k0 + tq;
    const bool kon = k < K;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < ntw) {
        const double a = (kon && ma[j] < M) ? A[ma[j] * am + k * ak] : 0.0;
        const double b = (kon && nb[j] < N) ? B[k * bk + nb[j] * bn] : 0.0;
        dmma(acc[j], a, b);
      }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (j < ntw) {
      const int m = ma[j], n0 = nb[j] - g + 2 * tq;
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (m < M && n0 + e < N) out(m, n0 + e, acc[j][e]);
    }
}



// 2 x 2 tile blocks per warp, clamped indices (rows >= M / columns >= N are
// computed on clamped data and dropped at the output), k tail masked
template <class F>
__device__ __forceinline__ void small_gemm2(int M, int N, int K, const double* A, int am, int ak, const double* B,
                                            int bk, int bn, F out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int bm_ = warp >> 2, bn_ = warp & 3;
  if (16 * bm_ >= M || 16 * bn_ >= N) return;
  const int m0 = min(16 * bm_ + g, M - 1), m1 = min(16 * bm_ + 8 + g, M - 1);
  const int n0 = min(16 * bn_ + g, N - 1), n1 = min(16 * bn_ + 8 + g, N - 1);
  const double* a0p = A + m0 * am + tq * ak;
  const double* a1p = A + m1 * am + tq * ak;
  const double* b0p = B + tq * bk + n0 * bn;
  const double* b1p = B + tq * bk + n1 * bn;
  double c[2][2][2] = {};
  const int K4 = K & ~3;
  int k0 = 0;
  if (K4 > 0) {
    double x0 = a0p[0], x1 = a1p[0], y0 = b0p[0], y1 = b1p[0];
    for (k0 = 4; k0 < K4; k0 += 4) {
      const double nx0 = a0p[k0 * ak], nx1 = a1p[k0 * ak], ny0 = b0p[k0 * bk], ny1 = b1p[k0 * bk];
      dmma(c[0][0], x0, y0);
      dmma(c[0][1], x0, y1);
      dmma(c[1][0], x1, y0);
      dmma(c[1][1], x1, y1);
      x0 = nx0; x1 = nx1; y0 = ny0; y1 = ny1;
    }
    dmma(c[0][0], x0, y0);
    dmma(c[0][1], x0, y1);
    dmma(c[1][0], x1, y0);
    dmma(c[1][1], x1, y1);
  }
  if (K4 < K) {  // tail: k = K4 + tq may pass K
    const bool kon = K4 + tq < K;
    const double x0 = kon ? a0p[K4 * ak] : 0.0, x1 = kon ? a1p[K4 * ak] : 0.0;
    const double y0 = kon ? b0p[K4 * bk] : 0.0, y1 = kon ? b1p[K4 * bk] : 0.0;
    dmma(c[0][0], x0, y0);
    dmma(c[0][1], x0, y1);
    dmma(c[1][0], x1, y0);
    dmma(c[1][1], x1, y1);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = 16 * bm_ + 8 * i + g, n = 16 * bn_ + 8 * j + 2 * tq + e;
        if (m < M && n < N) out(m, n, c[i][j][e]);
      }
}

__global__ void k_gemm(double* out, int M, int N, int K, long long* cyc) {
  extern __shared__ double sm[];
  double* A = sm; double* B = sm + 64 * 64; double* C = B + 64 * 64;
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) { A[i] = i * 1e-3; B[i] = 1.0 - i * 1e-4; }
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 10; ++rep) {
    GEMMFN(M, N, K, A, K, 1, B, N, 1, [&](int m, int n, double v) { C[m * N + n] = v; });
    __syncthreads();
  }
  long long t1 = clock64();
  for (int i = threadIdx.x; i < M * N; i += blockDim.x) out[i] = C[i];
  if (threadIdx.x == 0) *cyc = (t1 - t0) / 10;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 64 * 8); cudaMalloc(&c, 8);
  cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 64 * 64 * 8);
  int shapes[4][3] = {{60, 50, 60}, {50, 50, 60}, {60, 50, 50}, {64, 64, 64}};
  for (auto& sh : shapes) {
    k_gemm<<<1, 512, 3 * 64 * 64 * 8>>>(o, sh[0], sh[1], sh[2], c);
    long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("%dx%dx%d: %lld cycles per gemm (%s)\n", sh[0], sh[1], sh[2], cyc, cudaGetErrorString(cudaGetLastError()));
  }
}
