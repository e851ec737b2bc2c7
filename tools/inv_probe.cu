#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_1505_04650_b200/csrc/common.cuh"
namespace cnmf {
constexpr int kCT = 512;
// In-place inverse of an SPD r x r matrix (ld r, r <= 64) by Gauss-Jordan
// without pivoting (the ridge term keeps the pivots >= the penalty). Thread t
// of the first 64 * TPR owns row t / TPR, columns EPT (t % TPR) .. + EPT - 1
// (EPT = 64 / TPR) in registers. Per elimination step the owners of the
// pivot row publish it (scaled) and the reciprocal pivot in a double-buffered
// shared row, one named barrier, and every thread updates its entries
// branch-free (a divergent branch per entry serialised every DFMA behind its
// predecessor); the pivot-column entry of a row comes from the lane holding
// it by shuffle, picked out of the registers by a select tree.
constexpr int kPivLD = 72;  // per buffer: 64 pivot-row entries + the reciprocal pivot at [64]
constexpr int kPivDoubles = 2 * kPivLD;  // two pivot-row buffers
// (a version passing the pivot rows through an mbarrier-guarded ring, so that
// only the next pivot row's owners sit on the critical path, measured the
// same ~1.2k cycles per step and deadlocked when called twice per launch)
#ifndef CNMF_GJ_TPR
#define CNMF_GJ_TPR 2
#endif

__device__ void spd_inverse(double* M, double* piv, int r) {
  constexpr int TPR = CNMF_GJ_TPR, EPT = 64 / TPR, NT = 64 * TPR;
  static_assert(kCT >= NT && (TPR & (TPR - 1)) == 0 && TPR <= 32, "threads per row");
  __syncthreads();  // M complete
  const int t = threadIdx.x;
  if (t < NT) {
    const int a = t / TPR, q = t % TPR, cb = EPT * q, lane = t & 31;
    double m[EPT];
#pragma unroll
    for (int j = 0; j < EPT; ++j) m[j] = (a < r && cb + j < r) ? M[a * r + cb + j] : 0.0;
    double fk = m[0];  // this thread's entry in the next pivot column (column 0 first)
    for (int k = 0; k < r; ++k) {
      double* pv = piv + (k & 1) * kPivLD;
      const double f = __shfl_sync(0xffffffffu, fk, (lane & ~(TPR - 1)) | (k / EPT));  // row a, column k
      if (a == k) {
        const double inv = 1.0 / f;
#pragma unroll
        for (int j = 0; j < EPT; j += 2) *(double2*)(pv + cb + j) = make_double2(m[j] * inv, m[j + 1] * inv);
        if (q == 0) pv[64] = inv;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
      const double inv = pv[64];
      //   row k:      m = piv (column k: inv)
      //   other rows: m = m - f piv (column k: -f inv)
      const bool own = (a == k);
      const double coef = own ? 0.0 : -f, ck = own ? inv : -f * inv;
      const int kc = k - cb;  // the pivot column, relative to this thread's entries
      double2 p2[EPT / 2];
#pragma unroll
      for (int j = 0; j < EPT / 2; ++j) p2[j] = *(const double2*)(pv + cb + 2 * j);
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const double pj = (j & 1) ? p2[j >> 1].y : p2[j >> 1].x;
        const double v = fma(coef, pj, own ? pj : m[j]);
        m[j] = (j == kc) ? ck : v;
      }
      // this thread's entry in the next pivot column: a select tree
      const int kn = k + 1 - cb;
      double tr[EPT];
#pragma unroll
      for (int j = 0; j < EPT; ++j) tr[j] = m[j];
#pragma unroll
      for (int w = EPT / 2; w >= 1; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) tr[j] = (kn & w) ? tr[j + w] : tr[j];
      fk = tr[0];
    }
#pragma unroll
    for (int j = 0; j < EPT; ++j)
      if (a < r && cb + j < r) M[a * r + cb + j] = m[j];
  }
  __syncthreads();
}


}  // namespace cnmf
using namespace cnmf;
__global__ void k_inv(double* Mg, int r, long long* cyc) {
  extern __shared__ double sm[];
  double* M = sm; double* piv = sm + ((r * r + 1) & ~1);
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) M[i] = Mg[i];
  __syncthreads();
  long long t0 = clock64();
  spd_inverse(M, piv, r);
  long long t1 = clock64();
#ifdef TWICE
  spd_inverse(M, piv, r);  // inverse of the inverse
  spd_inverse(M, piv, r);
#endif
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) Mg[i] = M[i];
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
    k_inv<<<1, 512, (r*r + 2 + kPivDoubles)*8>>>(d, r, c);
    long long cyc; cudaMemcpy(X, d, r*r*8, cudaMemcpyDeviceToHost); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    double err = 0; for (int i = 0; i < r; ++i) for (int j = 0; j < r; ++j) { double s = 0; for (int k = 0; k < r; ++k) s += A[i*r+k]*X[k*r+j]; err = fmax(err, fabs(s - (i==j))); }
    printf("r=%d err=%.3e cycles=%lld (%.0f per step) %s\n", r, err, cyc, (double)cyc / r, cudaGetErrorString(cudaGetLastError()));
  }
}
