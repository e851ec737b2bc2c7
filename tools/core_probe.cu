// cycles of the ADMM core-step pieces on one CTA, outside the persistent kernel
#include "../paper_1505_04650_b200/csrc/admm.cu"
#include <cstdio>
namespace cnmf { namespace {
__global__ void probe(long long* cyc, Acc* acc) {
  extern __shared__ double smraw[];
  const Smem<32, 32> sm(smraw, 8);
  constexpr int LS = 33, LR = 33;
  for (int i = threadIdx.x; i < 32 * 33; i += blockDim.x) {
    const int a = i / 33, b = i % 33;
    sm.C[i] = (a == b ? 3.0 : 0.01 * ((a * 7 + b) % 11));
    sm.xc[i] = 0.1 * ((a + 2 * b) % 5);
    sm.yc[i] = 0.1 * ((3 * a + b) % 7);
    sm.M[i] = sm.Q[i] = sm.T[i] = sm.W[i] = 0.0;
  }
  if (threadIdx.x < 2) sm.misc[threadIdx.x] = 0.0;
  __syncthreads();
  long long t[8];
  t[0] = clock64();
  dgemm_tc<32, 32, 32>([&](int i, int k) { return sm.yc[i * LS + k]; }, [&](int k, int j) { return sm.yc[j * LS + k]; },
                       [&](int i, int j, double v) { sm.M[i * LR + j] = v + (i == j ? 1.0 : 0.0); });
  __syncthreads();
  t[1] = clock64();
  bgemm<32, 32, 32>([&](int i, int k) { return sm.yc[i * LS + k]; }, [&](int k, int j) { return sm.yc[j * LS + k]; },
                    [&](int i, int j, double v) { sm.W[i * LR + j] = v + (i == j ? 1.0 : 0.0); });
  __syncthreads();
  t[2] = clock64();
  gj_inverse<32>(sm.W, sm.T, 20);
  t[3] = clock64();
  core_step<32, 32>(sm, acc, 30, 20, 1.0, 1.0);  // cold: Gauss-Jordan inverses
  t[4] = clock64();
  core_step<32, 32>(sm, acc, 30, 20, 1.0, 1.0);  // warm: Newton-Schulz
  t[5] = clock64();
  if (threadIdx.x == 0)
    for (int i = 0; i < 5; ++i) cyc[i] = t[i + 1] - t[i];
}
}}
int main() {
  long long* c; cnmf::Acc* acc; long long h[5];
  cudaMalloc(&c, 64); cudaMalloc(&acc, sizeof(cnmf::Acc)); cudaMemset(acc, 0, sizeof(cnmf::Acc));
  const size_t sm = cnmf::Smem<32, 32>::bytes(8);
  cudaFuncSetAttribute(cnmf::probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int rep = 0; rep < 3; ++rep) {
    cnmf::probe<<<1, 256, sm>>>(c, acc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("dgemm_tc32 %lld | bgemm32 %lld | gj_inverse r=20 %lld | core_step cold %lld | warm %lld cycles (%s)\n", h[0], h[1], h[2], h[3], h[4], cudaGetErrorString(e));
  }
  return 0;
}
