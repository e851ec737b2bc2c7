"""Writes tools/inv_probe.cu: the core step's spd_inverse (extracted from
csrc/admm_stream.cu) timed on one block with clock64 and checked on host.
Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/inv_probe.cu -o tools/inv_a.bin"""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = open(os.path.join(ROOT, "paper_1505_04650_b200/csrc/admm_stream.cu")).read()
a = src.index("// In-place inverse of an SPD r x r matrix")
b = src.index("#ifdef CNMF_CORE_TRACE\n// phase timestamps")
HEAD = """#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_1505_04650_b200/csrc/common.cuh"
namespace cnmf {
constexpr int kCT = 512;
"""
TAIL = """
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
    printf("r=%d err=%.3e cycles=%lld (%.0f per step) %s\\n", r, err, cyc, (double)cyc / r, cudaGetErrorString(cudaGetLastError()));
  }
}
"""
open(os.path.join(ROOT, "tools/inv_probe.cu"), "w").write(HEAD + src[a:b] + TAIL)
