// Streaming-read ceiling probe: how fast can one CTA per SM pull A through a
// TMA ring into shared memory, as a function of box shape and ring depth?
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/tma_probe.cu -o /tmp/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));     \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

struct alignas(64) Desc {
  unsigned char b[128];
};

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su(bar)),
      "r"(ph)
      : "memory");
}

// mode 0: 2D TMA boxes {bc, br} (one box per stage); mode 1: 1D bulk copies of stage bytes (contiguous)
__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ Desc tA, const float* A, int mode, int bc, int br,
                                               int ST, int64_t units, int tiles_c, float* sink) {
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  const int SB = bc * br * 4;
  uint64_t* full = (uint64_t*)(sm + ST * SB);
  uint64_t* empty = full + ST;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t u0 = b * units / G, u1 = (b + 1) * units / G;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t it = 0; it < u1 - u0; ++it) {
      const int s = (int)(it % ST);
      if (it >= ST) wait(&empty[s], (uint32_t)(((it / ST) - 1) & 1));
      const int64_t u = u0 + it;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(SB) : "memory");
      if (mode == 0) {
        const int c = (int)(u % tiles_c) * bc, r = (int)(u / tiles_c) * br;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                su(sm + s * SB)),
            "l"(&tA), "r"(su(&full[s])), "r"(c), "r"(r)
            : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su(sm + s * SB)),
            "l"(A + u * (SB / 4)), "r"(SB), "r"(su(&full[s]))
            : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    float acc = 0.f;
    for (int64_t it = 0; it < u1 - u0; ++it) {
      const int s = (int)(it % ST);
      wait(&full[s], (uint32_t)((it / ST) & 1));
      acc += *(volatile float*)(sm + s * SB);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
    if (acc == 12345.f) sink[0] = acc;
  }
}

__global__ void ldg_read(const float4* __restrict__ a, int64_t n4, float* sink) {
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(a + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t M = 20000, N = 10000;
  float* A;
  float* sink;
  CK(cudaMalloc(&A, M * N * 4));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(A, 0, M * N * 4));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  int nsm = 148;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  auto timeit = [&](auto&& launch, const char* name) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("%-44s %8.1f us %8.1f GB/s\n", name, ms * 1e3, M * N * 4 / ms / 1e6);
  };
  char name[128];
  for (int gmul = 1; gmul <= 2; ++gmul) {
    snprintf(name, sizeof name, "ldg float4 grid=%d x 1024", nsm * gmul * 2);
    timeit([&] { ldg_read<<<nsm * gmul * 2, 1024>>>((const float4*)A, M * N / 4, sink); }, name);
  }
  const int shapes[][3] = {{32, 128, 1}, {64, 64, 0}, {128, 32, 0}, {256, 16, 0}, {128, 64, 0}, {32, 256, 1}, {256, 32, 0}};
  for (auto& sh : shapes) {
    const int bc = sh[0], br = sh[1];
    Desc d;
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t str[1] = {(cuuint64_t)(N * 4)};
    cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
    cuuint32_t es[2] = {1, 1};
    if (enc((CUtensorMap*)&d, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            sh[2] ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed %d %d\n", bc, br);
      continue;
    }
    const int SB = bc * br * 4;
    const int tiles_c = (int)((N + bc - 1) / bc);
    const int64_t units = (int64_t)((M + br - 1) / br) * tiles_c;
    for (int ST : {4, 6, 8, 10, 12}) {
      const size_t smem = 1024 + (size_t)ST * SB + 256;
      if (smem > 227 * 1024) continue;
      for (int cps : {1, 2}) {
        if (cps == 2 && 2 * smem > 227 * 1024) continue;
        snprintf(name, sizeof name, "tma box{%d,%d}%s ST=%d ctas/sm=%d", bc, br, sh[2] ? " sw128" : "", ST, cps);
        timeit([&] { probe<<<nsm * cps, 64, smem>>>(d, A, 0, bc, br, ST, units, tiles_c, sink); }, name);
      }
    }
  }
  for (int kb : {16, 32}) {
    const int SB = kb * 1024;
    const int64_t units = M * N * 4 / SB;
    for (int ST : {4, 8, 12}) {
      const size_t smem = 1024 + (size_t)ST * SB + 256;
      if (smem > 227 * 1024) continue;
      snprintf(name, sizeof name, "bulk1d %d KB ST=%d", kb, ST);
      Desc d{};
      timeit([&] { probe<<<nsm, 64, smem>>>(d, A, 1, SB / 4 / 16, 16, ST, units, 1, sink); }, name);
    }
  }
  return 0;
}
