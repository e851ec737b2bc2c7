// cooperative launch overhead baseline: an empty kernel with the sweep's grid
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_k(int* p) { if (p && threadIdx.x == 1234) *p = 0; }
int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int coop = 0; coop < 2; ++coop) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(236);
    lc.blockDim = dim3(256);
    lc.dynamicSmemBytes = 52 * 1024;
    cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = coop;
    int* p = nullptr;
    for (int r = 0; r < 5; ++r) cudaLaunchKernelEx(&lc, empty_k, p);
    cudaEventRecord(e0);
    for (int r = 0; r < 40; ++r) cudaLaunchKernelEx(&lc, empty_k, p);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("empty kernel, 236 blocks, cooperative=%d: %.2f us per launch\n", coop, ms / 40 * 1e3);
  }
}
