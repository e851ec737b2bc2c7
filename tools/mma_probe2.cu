// Tensor-pipe throughput of the pass kernel's per-K-tile MMA pattern with a
// tight (branch-free, compile-time) issue loop:
//   4 x { D[:,0:64] (+)= A_hi(TMEM) [X_hi|X_lo] (N=64); D[:,32:64] += A_lo(TMEM) X_hi (N=32) }
//   + COMMITS tcgen05.commit per K tile,
// optionally with other warps streaming tcgen05.st (BG=1) / tcgen05.ld (BG=2)
// into/from TMEM like the splitters / epilogue do.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/mma_probe2.cu -o tools/mma_probe2.bin
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc(int n, int m = 128) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}

// VAR 0: 3xTF32 pattern (N=64 + N=32, A from TMEM); VAR 1: only the N=64 MMA
// (4 per tile); VAR 2: both N=64 (A_lo [X_hi|X_lo]); VAR 3: A from SMEM (SS), N=64 + N=32
template <int VAR, int COMMITS, int BG>
__global__ void __launch_bounds__(128, 1) pat(int iters, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ int stop_flag;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    stop_flag = 0;
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) ((float*)sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  constexpr uint32_t icat = idesc(64), ihi = idesc(VAR == 2 ? 64 : 32);
  if (threadIdx.x == 0) {
    const uint32_t b_s = su(sm);
    const uint64_t b0 = sdesc(b_s);
    const uint64_t a0 = sdesc(b_s + 16384);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t a = tmem + 256 + (i & 3) * 64;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t bd = b0 + 2 * k;  // +32 B
        if (VAR == 3) {
          mma_ss(tmem, a0 + 2 * k, bd, icat, 1);
          mma_ss(tmem + 32, a0 + 512 + 2 * k, bd, ihi, 1);
        } else {
          mma(tmem, a + 8 * k, bd, icat, k | (i & 1));
          if (VAR != 1) mma(tmem + 32, a + 32 + 8 * k, bd, ihi, 1);
        }
      }
#pragma unroll
      for (int c = 0; c < COMMITS; ++c)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         su(&bar[c]))
                     : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar[3]))
                 : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
            su(&bar[3]))
        : "memory");
    cycles[blockIdx.x] = clock64() - t0;
    *(volatile int*)&stop_flag = 1;
  } else if (warp > 0 && BG) {
    const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + 256 + 16 * warp;
    uint32_t r[16] = {};
    while (*(volatile int*)&stop_flag == 0) {
#pragma unroll 1
      for (int rep = 0; rep < 16; ++rep) {
        if (BG & 1)
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
              "%13, %14, %15, %16};\ntcgen05.wait::st.sync.aligned;" ::"r"(ta + 64 * (rep & 3)),
              "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
              "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
              : "memory");
        if (BG & 2)
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
              "%14, %15}, [%16];\ntcgen05.wait::ld.sync.aligned;"
              : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
              : "r"(tmem + ((uint32_t)(32 * warp) << 16) + 16 * (rep & 3))
              : "memory");
      }
    }
    if (r[3] == 12345) cycles[0] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int VAR, int COMMITS, int BG>
void run(long long* d) {
  const int iters = 4096;
  cudaFuncSetAttribute(pat<VAR, COMMITS, BG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 49 * 1024);
  pat<VAR, COMMITS, BG><<<148, 128, 49 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("var=%d commits=%d bg=%d: %7.1f cycles/K-tile (%s)\n", VAR, COMMITS, BG, avg / iters, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<0, 0, 0>(d);
  run<0, 1, 0>(d);
  run<0, 2, 0>(d);
  run<1, 0, 0>(d);
  run<1, 1, 0>(d);
  run<2, 0, 0>(d);
  run<3, 0, 0>(d);
  run<3, 1, 0>(d);
  run<0, 1, 1>(d);
  run<0, 1, 2>(d);
  run<0, 1, 3>(d);
  run<3, 1, 3>(d);
  return 0;
}
