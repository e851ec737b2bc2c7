// Gauss-Jordan SPD inverse variants for the streaming ADMM core step, timed
// on one block (512 threads) with clock64 and checked on the host.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
constexpr int kPivLD = 72;

// smem-resident, 8 threads per row (8 columns each), one named barrier per
// step; the owners of row k + 1 publish the next pivot row right after their
// own update of step k.
__device__ void gj_smem(double* M, double* piv, int r) {
  // thread (a, q): row a, columns c(j, e) = 2 q + 16 j + e (j < 4, e < 2): a
  // quarter warp reads one contiguous 128-byte run per double2 (ld 66)
  constexpr int LD = 66;
  __syncthreads();
  const int t = threadIdx.x, a = t >> 3, q = t & 7, lane = t & 31;
  const bool on = a < r;
  double* row = M + a * LD;
  if (a == 0) {
    const double p = __shfl_sync(0xffu, row[0], 0);
    const double inv = 1.0 / p;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = 2 * q + 16 * j;
      *(double2*)(piv + c) = make_double2(row[c] * inv, row[c + 1] * inv);
    }
    if (q == 0) piv[64] = inv;
  }
  for (int k = 0; k < r; ++k) {
    asm volatile("bar.sync 1, 512;" ::: "memory");
    const double* pv = piv + (k & 1) * kPivLD;
    const double inv = pv[64];
    const double f = row[k];
    double v[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = 2 * q + 16 * j;
      const double2 x = *(const double2*)(row + c), p = *(const double2*)(pv + c);
      if (a == k) {
        v[2 * j] = p.x;
        v[2 * j + 1] = p.y;
      } else {
        v[2 * j] = fma(-f, p.x, x.x);
        v[2 * j + 1] = fma(-f, p.y, x.y);
      }
    }
    const double ck = (a == k) ? inv : -f * inv;
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (2 * q + 16 * (j >> 1) + (j & 1) == k) ? ck : v[j];
    if (on) {
#pragma unroll
      for (int j = 0; j < 4; ++j) *(double2*)(row + 2 * q + 16 * j) = make_double2(v[2 * j], v[2 * j + 1]);
    }
    if (a == k + 1 && k + 1 < r) {  // the next pivot row, from registers
      const int kn = k + 1;
      double pe = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) pe = (2 * q + 16 * (j >> 1) + (j & 1) == kn) ? v[j] : pe;
      const double p2 = __shfl_sync(0xffu << (lane & 24), pe, (lane & ~7) | ((kn & 15) >> 1));
      const double inv2 = 1.0 / p2;
      double* pn = piv + (kn & 1) * kPivLD;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *(double2*)(pn + 2 * q + 16 * j) = make_double2(v[2 * j] * inv2, v[2 * j + 1] * inv2);
      if (q == 0) pn[64] = inv2;
    }
  }
  __syncthreads();
}

__global__ void k_inv(double* Mg, int r, long long* cyc) {
  extern __shared__ double sm[];
  double* M = sm; double* piv = sm + 64 * 66;
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) { int a = i / 64, c = i % 64; M[a * 66 + c] = (a < r && c < r) ? Mg[a * r + c] : 0.0; }
  __syncthreads();
  long long t0 = clock64();
  gj_smem(M, piv, r);
  long long t1 = clock64();
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) Mg[i] = M[(i / r) * 66 + i % r];
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  for (int r : {5, 33, 50, 64}) {
    double* A = (double*)malloc(r * r * 8); double* X = (double*)malloc(r * r * 8); double* B = (double*)malloc(r * r * 8);
    srand(1);
    for (int i = 0; i < r * r; ++i) B[i] = rand() / (double)RAND_MAX;
    for (int i = 0; i < r; ++i) for (int j = 0; j < r; ++j) { double s = 0; for (int k = 0; k < r; ++k) s += B[i*r+k]*B[j*r+k]; A[i*r+j] = s + (i==j ? 1.0 : 0.0); }
    double* d; long long* c; cudaMalloc(&d, r*r*8); cudaMalloc(&c, 8);
    cudaMemcpy(d, A, r*r*8, cudaMemcpyHostToDevice);
    k_inv<<<1, 512, (64 * 66 + 2 * kPivLD) * 8>>>(d, r, c);
    long long cyc; cudaMemcpy(X, d, r*r*8, cudaMemcpyDeviceToHost); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    double err = 0; for (int i = 0; i < r; ++i) for (int j = 0; j < r; ++j) { double s = 0; for (int k = 0; k < r; ++k) s += A[i*r+k]*X[k*r+j]; err = fmax(err, fabs(s - (i==j))); }
    printf("r=%d err=%.3e cycles=%lld (%.0f per step) %s\n", r, err, cyc, (double)cyc / r, cudaGetErrorString(cudaGetLastError()));
  }
}
