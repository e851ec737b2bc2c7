// Library runtime: error state, seed derivation, TMA descriptor encoding.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace cnmf {

static thread_local std::string g_last_error;

void set_error(int code, const std::string& msg) {
  g_last_error = "[cnmf " + std::to_string(code) + "] " + msg;
}

int fail(int code, const std::string& msg) {
  set_error(code, msg);
  return code;
}

const char* last_error() { return g_last_error.c_str(); }

static std::atomic<int64_t> g_launches{0};
void count_launches(int64_t n) { g_launches += n; }
int64_t launch_count() { return g_launches.load(); }

static bool g_prof = false;
struct PassEvent {
  cudaEvent_t a, b;
  double bytes;
};
static std::vector<PassEvent> g_events;
static std::mutex g_prof_mu;

bool pass_profiling() { return g_prof; }
void pass_record(cudaEvent_t start, cudaEvent_t stop, double bytes) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_events.push_back({start, stop, bytes});
}
void set_pass_profiling(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& e : g_events) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  g_events.clear();
  g_prof = on != 0;
}
int pass_stats(double* total_ms, int64_t* launches, double* bytes) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double ms = 0.0, by = 0.0;
  for (auto& e : g_events) {
    CNMF_CUDA(cudaEventSynchronize(e.b));
    float t = 0.f;
    CNMF_CUDA(cudaEventElapsedTime(&t, e.a, e.b));
    ms += t;
    by += e.bytes;
  }
  *total_ms = ms;
  *launches = (int64_t)g_events.size();
  *bytes = by;
  return CNMF_OK;
}

// Keep freed stream-ordered allocations in the default pool instead of
// returning them to the driver at every synchronisation (the default release
// threshold of 0 makes every cudaMallocAsync remap physical memory).
void keep_pool() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

namespace {
std::mutex g_dev_mu;
int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  return dev;
}
}  // namespace

int device_sms() {
  static std::mutex mu;
  static std::map<int, int> cache;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) sms = kNumSMs;
  cache[dev] = sms;
  return sms;
}

int ensure_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, fn);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return CNMF_OK;
  CNMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done[key] = bytes;
  return CNMF_OK;
}

int device_scratch(const char* tag, size_t bytes, void** out, cudaStream_t st) {
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  static std::map<std::pair<int, std::string>, Buf> bufs;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  Buf& b = bufs[std::make_pair(dev, std::string(tag))];
  if (b.cap < bytes) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CNMF_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return fail(CNMF_ERR_CUDA, std::string("library scratch '") + tag +
                                     "' must be allocated by an eager call before graph capture");
    CNMF_CUDA(cudaDeviceSynchronize());  // the old buffer may still be in use
    if (b.p) CNMF_CUDA(cudaFree(b.p));
    b.p = nullptr;
    b.cap = 0;
    CNMF_CUDA(cudaMalloc(&b.p, bytes));
    CNMF_CUDA(cudaMemset(b.p, 0, bytes));
    b.cap = bytes;
  }
  *out = b.p;
  return CNMF_OK;
}

unsigned device_ticket(const char* tag) {
  static std::map<std::pair<int, std::string>, std::atomic<unsigned>> counters;
  const int dev = current_device();
  std::atomic<unsigned>* c;
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    c = &counters[std::make_pair(dev, std::string(tag))];
  }
  return c->fetch_add(1u);
}

uint64_t fnv1a64(const char* s) {
  uint64_t h = 0xCBF29CE484222325ULL;
  for (const unsigned char* p = (const unsigned char*)s; *p; ++p) h = (h ^ *p) * 0x100000001B3ULL;
  return h;
}

uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

int make_tma_2d(TmaDesc* out, const void* base, int elem_bytes, int64_t rows, int64_t cols, int64_t ld,
                int box_cols, int box_rows, bool swizzle128) {
  static_assert(sizeof(CUtensorMap) == sizeof(TmaDesc), "descriptor size");
  auto enc = get_encode();
  if (!enc) return fail(CNMF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (((uintptr_t)base & 15) || ((ld * elem_bytes) & 15))
    return fail(CNMF_ERR_ARGUMENT, "TMA needs a 16-byte aligned base and leading dimension");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * elem_bytes)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(out),
                   elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CNMF_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return CNMF_OK;
}

}  // namespace cnmf
