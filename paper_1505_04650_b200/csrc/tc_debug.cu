// Self-test kernels for the tcgen05 building blocks (not part of the C ABI
// header; used by tools/tc_debug.py when bringing up tc_pass.cu).
#include "common.cuh"

namespace cnmf {
namespace {

__device__ __forceinline__ void tcf_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tcf_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// test 0: TMEM st/ld round trip. test 1: one MMA 128x32x8 with ones.
__global__ void tc_selftest(int test, float* out) {
  __shared__ __align__(1024) float sa[128 * 32];
  __shared__ __align__(1024) float sb[32 * 32];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const float one = (test == 3 || test == 7) ? __uint_as_float(0x3F803F80u) : 1.0f;
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) sa[i] = one;
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) sb[i] = one;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tcf_before();
  __syncthreads();
  tcf_after();
  const uint32_t tmem = slot;
  const uint32_t taddr = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
  if (test == 0) {
    uint32_t v = __float_as_uint(100.0f * (32 * warp + lane) + 1.0f);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  } else if (warp == 0) {
    // A: 128 x 8 K-major SW128 (rows 128 B apart), B: 8 x 32 MN-major SW128
    const uint32_t a = smem_u32(sa), b = smem_u32(sb);
    auto desc = [](uint32_t addr, uint32_t lbo, uint32_t sbo) {
      uint64_t d = 0;
      d |= (uint64_t)((addr >> 4) & 0x3FFF);
      d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
      d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
      d |= (uint64_t)1 << 46;
      d |= (uint64_t)2 << 61;
      return d;
    };
    uint64_t ad = desc(a, 16, 1024), bd = desc(b, 4096, 1024);
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) | ((32u >> 3) << 17) |
                     ((128u >> 4) << 24);
    if (test == 2 || test == 6) idesc &= ~(1u << 16);            // B K-major
    if (test == 6) idesc |= (1u << 15);                          // A MN-major
    if (test == 4) {                                             // no swizzle
      ad &= ~((uint64_t)7 << 61);
      bd &= ~((uint64_t)7 << 61);
    }
    if (test == 5) idesc = (idesc & ~(0x1Fu << 24)) | ((64u >> 4) << 24);  // M = 64
    if (lane == 0) {
      if (test == 3 || test == 7) {
        // bf16: A, B all 1.0 (0x3F80), K = 16 per instruction (test 7: B MN-major)
        const uint32_t id16 = (1u << 4) | (1u << 7) | (1u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24) |
                              (test == 7 ? (1u << 16) : 0u);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(id16), "r"(0)
            : "memory");
      } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(0)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar))
                   : "memory");
    }
    __syncwarp();
  }
  if (test >= 1) mbar_wait(&bar, 0);
  tcf_before();
  __syncthreads();
  tcf_after();
  uint32_t r0, r1;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r0), "=r"(r1)
      : "r"(taddr)
      : "memory");
  out[(32 * warp + lane) * 2 + 0] = __uint_as_float(r0);
  out[(32 * warp + lane) * 2 + 1] = __uint_as_float(r1);
  tcf_before();
  __syncthreads();
  tcf_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

}  // namespace
}  // namespace cnmf

extern "C" int cnmf_debug_tc(int test, float* out) {
  cnmf::tc_selftest<<<1, 128>>>(test, out);
  cudaError_t e = cudaDeviceSynchronize();
  return e == cudaSuccess ? 0 : (int)e;
}
