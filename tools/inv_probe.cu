#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_1505_04650_b200/csrc/common.cuh"
namespace cnmf {
constexpr int kCT = 512;
// In-place inverse of an SPD r x r matrix (ld r, r <= 64) by Gauss-Jordan
// without pivoting (the ridge term keeps the pivots >= the penalty),
// pipelined: thread t of the first four warps owns row t / 2, columns
// 32 (t % 2) .. + 31 in registers. The scaled pivot rows travel through a
// ring of kPivNB shared rows guarded by mbarriers: the two owners of row
// k + 1 update their row from pivot row k, pick its pivot, and publish
// pivot row k + 1 at once, while every other thread updates its own row --
// only the owners' chain (wait, 32 DFMA, select, shuffle, reciprocal,
// publish) is on the critical path, no block barrier per step. The earlier
// versions synchronised all 512 (then 128) threads twice (then once) per
// step: 47 us, then ~33 us per 50 x 50 inverse.
constexpr int kPivLD = 72;   // per ring row: 64 pivot-row entries + the reciprocal pivot at [64]
constexpr int kPivNB = 4;    // pivot rows in flight
constexpr int kPivDoubles = kPivNB * kPivLD + 2 * kPivNB;  // ring + its full / empty mbarriers

__device__ __forceinline__ void gj_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#ifndef CNMF_GJ_TPR
#define CNMF_GJ_TPR 8
#endif

__device__ void spd_inverse(double* M, double* piv, int r) {
  constexpr int TPR = CNMF_GJ_TPR, EPT = 64 / TPR, NT = 64 * TPR;  // threads per row, entries per thread
  static_assert(kCT >= NT && (TPR & (TPR - 1)) == 0 && TPR <= 32 && EPT % 2 == 0, "row mapping");
  uint64_t* full = (uint64_t*)(piv + kPivNB * kPivLD);
  uint64_t* empty = full + kPivNB;
  const int t = threadIdx.x;
  if (t == 0) {
    for (int i = 0; i < kPivNB; ++i) {
      mbar_init(&full[i], TPR);  // the owners of the pivot row
      mbar_init(&empty[i], NT);  // every row thread has read it
    }
    fence_barrier_init();
  }
  __syncthreads();  // M complete, barriers initialised
  if (t < NT) {
    const int a = t / TPR, q = t % TPR, cb = EPT * q, lane = t & 31;
    const unsigned grp = (TPR == 32 ? 0xffffffffu : ((1u << TPR) - 1u)) << (lane & ~(TPR - 1));
    double m[EPT];
#pragma unroll
    for (int j = 0; j < EPT; ++j) m[j] = (a < r && cb + j < r) ? M[a * r + cb + j] : 0.0;
    auto select = [&](int kk) {  // m[kk - cb] (0 when outside this thread's columns): a select tree
      const int kn = kk - cb;
      double tr[EPT];
#pragma unroll
      for (int j = 0; j < EPT; ++j) tr[j] = m[j];
#pragma unroll
      for (int wdt = EPT / 2; wdt >= 1; wdt >>= 1)
#pragma unroll
        for (int j = 0; j < wdt; ++j) tr[j] = (kn & wdt) ? tr[j + wdt] : tr[j];
      return (kn >= 0 && kn < EPT) ? tr[0] : 0.0;
    };
    auto publish = [&](int kk, double fkk) {  // the owners of row kk: pivot row kk into ring slot kk % NB
      const double p = __shfl_sync(grp, fkk, (lane & ~(TPR - 1)) | (kk / EPT));
      const double inv = 1.0 / p;
      double* pv = piv + (kk % kPivNB) * kPivLD;
      if (kk >= kPivNB) mbar_wait(&empty[kk % kPivNB], ((kk / kPivNB) - 1) & 1);
#pragma unroll
      for (int j = 0; j < EPT; j += 2) *(double2*)(pv + cb + j) = make_double2(m[j] * inv, m[j + 1] * inv);
      if (q == 0) pv[64] = inv;
      gj_arrive(&full[kk % kPivNB]);  // release: the row is visible to the waiters
    };
    double fk = select(0);  // this row's entry in the next pivot column
    if (a == 0) publish(0, fk);
    for (int k = 0; k < r; ++k) {
      const double f = __shfl_sync(0xffffffffu, fk, (lane & ~(TPR - 1)) | (k / EPT));  // row a, column k
      const double* pv = piv + (k % kPivNB) * kPivLD;
      mbar_wait(&full[k % kPivNB], (k / kPivNB) & 1);
      const double inv = pv[64];
      double2 p2[EPT / 2];
#pragma unroll
      for (int j = 0; j < EPT / 2; ++j) p2[j] = *(const double2*)(pv + cb + 2 * j);
      gj_arrive(&empty[k % kPivNB]);
      //   row k:      m = piv (column k: inv)
      //   other rows: m = m - f piv (column k: -f inv)
      const bool own = (a == k);
      const double coef = own ? 0.0 : -f, ck = own ? inv : -f * inv;
      const int kc = k - cb;
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const double pj = (j & 1) ? p2[j >> 1].y : p2[j >> 1].x;
        const double v = fma(coef, pj, own ? pj : m[j]);
        m[j] = (j == kc) ? ck : v;
      }
      fk = select(k + 1);
      if (a == k + 1 && k + 1 < r) publish(k + 1, fk);
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
