// tcgen05.mma kind::tf32 issue-throughput probe (M = 128, cta_group::1):
// cycles per MMA for N in {32, 64, 128, 256}, A from shared memory (SS) or
// from TMEM (TS). Operand contents are irrelevant (zeros).
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/mma_probe.cu -o tools/mma_probe.bin
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

template <int N, bool TS, int MM = 128>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float*)sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a_s = su(sm), b_s = su(sm + 32768);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t bd = sdesc(b_s + 32 * k);
        if (TS) {
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
              "r"(tmem + 256 + 8 * k), "l"(bd), "r"(idesc(N, MM))
              : "memory");
        } else {
          const uint64_t ad = sdesc(a_s + 32 * k);
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc(N, MM))
              : "memory");
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar))
                 : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su(&bar))
        : "memory");
    const long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// The pass kernel's per-K-tile pattern: 4 x (N = 2S from TMEM A_hi, N = S from
// TMEM A_lo) + `commits` tcgen05.commit per iteration.
template <int S>
__global__ void __launch_bounds__(128, 1) pattern(int iters, int commits, int mode, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ __align__(8) uint64_t ready;
  __shared__ int stop_flag;
  if (threadIdx.x == 0) stop_flag = 0;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&ready)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&ready)) : "memory");
  }
  for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) ((float*)sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t b_s = su(sm);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (mode & 2)
        asm volatile(
            "{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n" ::"r"(
                su(&ready))
            : "memory");
      if (mode & 1) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a = tmem + 256 + ((mode & 512) ? 0 : (i & 3) * 64);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t bd = sdesc(b_s + 32 * k);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
            "r"(a + 8 * k), "l"(bd), "r"(idesc(2 * S)), "r"((mode & 256) ? 1 : k)
            : "memory");
        if (!(mode & 1024)) asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + ((mode & 64) ? 0 : (mode & 16) ? 2 * S : S)),
            "r"(a + ((mode & 128) ? 0 : 32) + 8 * k), "l"((mode & 2048) ? sdesc(b_s + 8192 + 32 * k) : bd), "r"(idesc((mode & 32) ? 2 * S : S))
            : "memory");
      }
      for (int c = 0; c < commits; ++c)
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
    stop_flag = 1;
  } else if (warp > 0 && (mode & 12)) {
    const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + 448;
    uint32_t r[16] = {};
    while (*(volatile int*)&stop_flag == 0) {
      for (int rep = 0; rep < 16; ++rep) {
        if (mode & 4)
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
              "%13, %14, %15, %16};\ntcgen05.wait::st.sync.aligned;" ::"r"(ta),
              "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
              "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
              : "memory");
        if (mode & 8)
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
              "%14, %15}, [%16];\ntcgen05.wait::ld.sync.aligned;"
              : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
              : "r"(ta)
              : "memory");
      }
    }
    if (r[3] == 12345) cycles[0] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int S>
void run_pattern(long long* d, int commits, int mode = 0) {
  const int iters = 2048;
  cudaFuncSetAttribute(pattern<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  pattern<S><<<148, 128, 33 * 1024>>>(iters, commits, mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("pattern S=%d commits=%d mode=%d: %7.1f cycles/K-tile (%s)\n", S, commits, mode, avg / iters,
         cudaGetErrorString(e));
}

template <int N, bool TS, int MM = 128>
void run(long long* d) {
  const int iters = 4096;
  cudaFuncSetAttribute(probe<N, TS, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  probe<N, TS, MM><<<148, 128, 65 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("M=%3d N=%3d %s: %7.1f cycles/MMA  (%s)\n", MM, N, TS ? "TS" : "SS", avg / (iters * 4.0), cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<64, false, 64>(d);
  run<128, false, 64>(d);
  run<256, false, 64>(d);
  run<32, false>(d);
  run<64, false>(d);
  run<128, false>(d);
  run<256, false>(d);
  run<32, true>(d);
  run<64, true>(d);
  run<128, true>(d);
  run<256, true>(d);
  for (int c = 0; c <= 2; ++c) run_pattern<32>(d, c);
  for (int c = 0; c <= 2; ++c) run_pattern<64>(d, c);
  for (int m = 1; m <= 3; ++m) run_pattern<32>(d, 1, m);
  for (int m = 1; m <= 3; ++m) run_pattern<64>(d, 1, m);
  for (int c = 0; c <= 2; ++c) run_pattern<32>(d, c, 16);
  run_pattern<32>(d, 0, 48 + 64);
  run_pattern<32>(d, 0, 48 + 128);
  run_pattern<32>(d, 0, 48 + 64 + 128);
  run_pattern<32>(d, 0, 1024);
  run_pattern<32>(d, 0, 1024 + 768);
  run_pattern<32>(d, 0, 2048);
  run_pattern<32>(d, 0, 2048 + 768 + 32 + 64);
  run_pattern<32>(d, 0, 256);
  run_pattern<32>(d, 0, 512);
  run_pattern<32>(d, 0, 768);
  run_pattern<32>(d, 1, 256);
  run_pattern<32>(d, 1, 768);
  run_pattern<32>(d, 2, 768);
  run_pattern<32>(d, 1, 4);
  run_pattern<32>(d, 1, 8);
  run_pattern<32>(d, 1, 12);
  return 0;
}
