// Shared device/host helpers for the cnmf B200 library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/cnmf_b200.h"

namespace cnmf {

// ---------------------------------------------------------------------------
// error plumbing: every C-ABI call returns a cnmf_status and leaves a message
// ---------------------------------------------------------------------------
void set_error(int code, const std::string& msg);
int fail(int code, const std::string& msg);

#define CNMF_CUDA(expr)                                                          \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess)                                                       \
      return ::cnmf::fail(CNMF_ERR_CUDA, std::string(#expr) + ": " +             \
                                             cudaGetErrorString(_e));            \
  } while (0)

#define CNMF_TRY(expr)                   \
  do {                                   \
    int _s = (expr);                     \
    if (_s != CNMF_OK) return _s;        \
  } while (0)

// every kernel launch site calls CNMF_LAUNCH_CHECK() once: it also counts
// the launch (cnmf_launch_count) so benchmarks can report their kernel count
void count_launches(int64_t n);
#define CNMF_LAUNCH_CHECK()                 \
  do {                                      \
    ::cnmf::count_launches(1);              \
    CNMF_CUDA(cudaGetLastError());          \
  } while (0)

// optional CUDA-event timing of the streaming passes (the dominant kernels)
bool pass_profiling();
void pass_record(cudaEvent_t start, cudaEvent_t stop, double bytes);

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

constexpr int kNumSMs = 148;  // B200; launch sites size grids with device_sms()

// ---------------------------------------------------------------------------
// per-device library state (thread-safe; every entry is keyed by the current
// device, so a process driving several GPUs gets one of each per GPU)
// ---------------------------------------------------------------------------
// SM count of the current device (cudaDevAttrMultiProcessorCount, cached)
int device_sms();
// cudaFuncAttributeMaxDynamicSharedMemorySize = bytes, once per (device, fn)
int ensure_smem_attr(const void* fn, int bytes);
// a library-owned device buffer, one per (device, tag), zero-filled when it
// is (re)allocated; grows on demand, which is refused during graph capture
int device_scratch(const char* tag, size_t bytes, void** out, cudaStream_t st);
// next value of a per-(device, tag) counter (lock-free)
unsigned device_ticket(const char* tag);



// ---------------------------------------------------------------------------
// Philox4x64-10 (the reference's bit generator, rng.py:49-51), counter-based.
// Raw draw i of a stream keyed by `key` is word (i & 3) of the block with
// counter (i / 4) + 1 (numpy pre-increments the counter).
// ---------------------------------------------------------------------------
struct U64x4 {
  uint64_t v[4];
};

__device__ __forceinline__ U64x4 philox4x64(uint64_t c0, uint64_t c1, uint64_t k0, uint64_t k1) {
  uint64_t c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    const uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0;
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    const uint64_t lo1 = 0xCA5A826395121157ULL * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0;
    const uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  U64x4 out;
  out.v[0] = c0;
  out.v[1] = c1;
  out.v[2] = c2;
  out.v[3] = c3;
  return out;
}

__device__ __forceinline__ uint64_t philox_raw(uint64_t key, uint64_t pos) {
  U64x4 b = philox4x64((pos >> 2) + 1, 0, key, 0);
  return b.v[pos & 3];
}

// numpy's next_double: 53 random bits -> [0, 1)
__device__ __forceinline__ double raw_to_unit(uint64_t r) {
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

void keep_pool();

// host-side seed derivation (rng.py:23-35, 56-58, 73-75)
uint64_t fnv1a64(const char* s);
uint64_t splitmix64(uint64_t x);
inline uint64_t child_seed(uint64_t seed, const char* tag) { return splitmix64(seed ^ fnv1a64(tag)); }

// ---------------------------------------------------------------------------
// small PTX helpers: mbarrier + TMA (cp.async.bulk.tensor)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// vectorised fp32 reduction into global memory (sm_90+)
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// ---------------------------------------------------------------------------
// TMA descriptor creation (driver entry point fetched at runtime; no -lcuda)
// ---------------------------------------------------------------------------
struct alignas(64) TmaDesc {
  unsigned char bytes[128];
};

// 2-D row-major tensor [rows][cols] with leading dimension `ld` (elements).
// box = {box_cols, box_rows}; swizzle128 selects CU_TENSOR_MAP_SWIZZLE_128B.
int make_tma_2d(TmaDesc* out, const void* base, int elem_bytes, int64_t rows, int64_t cols, int64_t ld,
                int box_cols, int box_rows, bool swizzle128);

}  // namespace cnmf
