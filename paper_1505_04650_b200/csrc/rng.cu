// Device RNG: numpy-compatible Philox4x64 uniform and ziggurat normal streams.
//
// Reference: rng.py:38-98 (Rng over numpy Generator(Philox)), compress.py:115-127
// (_drawn_in_chunks: fixed 4096-row chunks, child stream per chunk).
//
// The normal sampler consumes a variable number of raw 64-bit draws per
// variate (≈0.75% of draws hit the wedge/tail path), so a stream is decoded in
// parallel by splitting its raw sequence into fixed segments:
//   k1  one warp per segment walks the variate chain speculatively from the
//       segment start (128 raws per warp step, one Philox block per lane) and
//       records the exit position, the variate count and which of the first
//       128 positions start a variate;
//   k2  one CTA per stream re-anchors every segment at the previous segment's
//       exit (chains merge at the first shared start position, almost always
//       the entry itself) and prefix-sums the corrected counts;
//   k3  one warp per segment decodes again from its true entry and writes its
//       variates at the scanned offset.
// Any segment whose chain does not merge inside its first window, or a stream
// whose segments end before its last variate, flags the stream, which is then
// decoded by one warp sequentially. The segments cover the stream's variate
// count plus a 5 % margin of raw positions: with 2 % one 4096 x 60 chunk of
// configs[4]'s right test matrix (child_seed(5, "right-basis")) ran short and
// its serial decode took 10 ms (tools/zig_probe.py); the streams are the same
// either way.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "glibc_log1p.cuh"
#include "ziggurat_tables.h"

namespace cnmf {
namespace {

constexpr int kWin = 128;  // raw positions per warp step (32 lanes x 4 words)

struct StreamDesc {
  uint64_t key;
  int64_t base;     // raw position of the stream's first variate
  int64_t count;    // variates in this stream
  int64_t row0;     // first output row
  int64_t seg0;     // first segment index (global)
  int32_t nseg;     // segments of this stream
  int32_t seglen;   // raw positions per segment (multiple of kWin)
};

struct SegState {
  int64_t exit;          // first chain start >= segment end (absolute position)
  int64_t count;         // variates started in [entry, exit)
  int64_t entry;         // true entry (after k2)
  int64_t offset;        // output offset (after k2)
  uint32_t chain[4];     // chain-start bits for [seg_start, seg_start + 128)
};

// The streams of one fill: a single stream (gaussian_matrix) or fixed-size row
// chunks, chunk c drawn from child_seed(seed, f"chunk{c}") (compress.py:115).
// Every segment derives its stream from this by arithmetic — no host-built
// descriptor tables are copied to the device.
struct Layout {
  uint64_t key;         // single-stream key, or the parent seed of the chunks
  int64_t rows, cols;
  int64_t chunk_rows;   // rows per chunk (== rows for a single stream)
  int64_t nchunks;
  int32_t chunked;
  int32_t nseg_full, nseg_last;
  int32_t seglen_full, seglen_last;
  int64_t total_segs;
  int64_t start;        // single stream: raw position of its first variate (stream continuation)
};

__device__ uint64_t dev_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

// child_seed(seed, "chunk" + str(c)) (rng.py:23-35, 56-58)
__device__ uint64_t dev_chunk_key(uint64_t seed, int64_t c) {
  uint64_t h = 0xCBF29CE484222325ULL;
  const char pre[5] = {'c', 'h', 'u', 'n', 'k'};
  for (int i = 0; i < 5; ++i) h = (h ^ (uint64_t)(unsigned char)pre[i]) * 0x100000001B3ULL;
  char dig[20];
  int nd = 0;
  do {
    dig[nd++] = (char)('0' + (int)(c % 10));
    c /= 10;
  } while (c > 0);
  while (nd > 0) h = (h ^ (uint64_t)(unsigned char)dig[--nd]) * 0x100000001B3ULL;
  return dev_splitmix64(seed ^ h);
}

__device__ StreamDesc stream_of(const Layout& L, int64_t c) {
  StreamDesc sd;
  const bool last = c == L.nchunks - 1;
  sd.key = L.chunked ? dev_chunk_key(L.key, c) : L.key;
  sd.base = L.chunked ? 0 : L.start;
  sd.row0 = c * L.chunk_rows;
  sd.count = (last ? L.rows - sd.row0 : L.chunk_rows) * L.cols;
  sd.seg0 = c * L.nseg_full;
  sd.nseg = last ? L.nseg_last : L.nseg_full;
  sd.seglen = last ? L.seglen_last : L.seglen_full;
  return sd;
}

__device__ __forceinline__ int64_t chunk_of_seg(const Layout& L, int64_t g) {
  const int64_t c = g / L.nseg_full;
  return c < L.nchunks - 1 ? c : L.nchunks - 1;
}

// A tail variate (|x| > r): numpy draws xx = -log1p(-u1) / r and
// yy = -log1p(-u2) with the C library's log1p (random_standard_normal), which
// is not correctly rounded; glibc_log1p.cuh restates that exact function, so
// the acceptance test and the variate are bit-identical on the device.
// Slow path of numpy's random_standard_normal starting at raw position `pos`
// whose first draw `r0` failed the fast acceptance. Returns the variate and
// sets *next to the position after the last consumed draw.
__device__ double slow_normal(uint64_t key, int64_t pos, uint64_t r0, int64_t* next) {
  uint64_t r = r0;
  int64_t p = pos + 1;
  for (;;) {
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = __dmul_rn((double)rabs, cnmf_zig::kWi[idx]);
    if (sign) x = -x;
    if (rabs < cnmf_zig::kKi[idx]) {
      *next = p;
      return x;
    }
    if (idx == 0) {
      for (;;) {
        const double u1 = raw_to_unit(philox_raw(key, (uint64_t)p));
        const double u2 = raw_to_unit(philox_raw(key, (uint64_t)(p + 1)));
        p += 2;
        const double xx = __dmul_rn(-cnmf_zig::kTailInvR, glibc_log1p(-u1));
        const double yy = -glibc_log1p(-u2);
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          *next = p;
          const double v = __dadd_rn(cnmf_zig::kTailR, xx);
          return ((rabs >> 8) & 1) ? -v : v;
        }
      }
    }
    const double u = raw_to_unit(philox_raw(key, (uint64_t)p));
    p += 1;
    const double lhs = __dadd_rn(__dmul_rn(__dadd_rn(cnmf_zig::kFi[idx - 1], -cnmf_zig::kFi[idx]), u),
                                 cnmf_zig::kFi[idx]);
    if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
      *next = p;
      return x;
    }
    r = philox_raw(key, (uint64_t)p);
    p += 1;
  }
}

// Per-block shared-memory copies of the ziggurat tables used on the fast
// path: every lane indexes them with its own random layer, which __constant__
// memory serialises (one access per distinct address per warp).
__shared__ uint64_t s_zki[256];
__shared__ double s_zwi[256];

__device__ __forceinline__ void load_zig_tables() {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    s_zki[i] = cnmf_zig::kKi[i];
    s_zwi[i] = cnmf_zig::kWi[i];
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ void store_variate(T* out, int64_t ld, int64_t cols, int64_t row0, int64_t k,
                                              int64_t count, double x) {
  if (k < count) {
    const int64_t row = row0 + k / cols;
    const int64_t col = k - (k / cols) * cols;
    out[row * ld + col] = (T)x;
  }
}

// Walk the chain of one segment from `head` until the head reaches `stop`.
// When WRITE, variates are stored from output index `k0`. Returns the number
// of variates started; *exit_pos receives the final head. When chain != null
// the start bits of the first window [seg_start, seg_start+128) are recorded.
// When end != null, the raw position after the stream's last variate (output
// index count - 1) is stored there (Rng stream continuation).
template <bool WRITE, typename T>
__device__ int64_t walk(uint64_t key, int64_t head, int64_t stop, int64_t seg_start, uint32_t* chain, T* out,
                        int64_t ld, int64_t cols, int64_t row0, int64_t k0, int64_t count, int64_t* exit_pos,
                        int64_t* end = nullptr) {
  const int lane = threadIdx.x & 31;
  int64_t k = 0;
  int64_t base = (head / kWin) * kWin;
  while (head < stop) {
    // one Philox block per lane: positions base + 4*lane + {0..3}
    const U64x4 blk = philox4x64((uint64_t)(base / 4 + lane) + 1, 0, key, 0);
    uint32_t slow = 0;
    double xs[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint64_t r = blk.v[j];
      const int idx = (int)(r & 0xff);
      r >>= 8;
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      double x = __dmul_rn((double)rabs, s_zwi[idx]);
      xs[j] = (r & 1) ? -x : x;
      if (!(rabs < s_zki[idx])) slow |= 1u << j;
    }
    uint32_t m[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      m[q] = __reduce_or_sync(0xffffffffu, (lane >> 3) == q ? (slow << (4 * (lane & 7))) : 0u);

    int p = (int)(head - base);
    while (p < kWin && base + p < stop) {
      // first slow position >= p (static indices only: a dynamically
      // indexed m[] would live in local memory)
      int f = kWin;
      const int pq = p >> 5;
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        const uint32_t w = q < pq ? 0u : m[q] & (q == pq ? (0xffffffffu << (p & 31)) : 0xffffffffu);
        if (w) f = q * 32 + __ffs(w) - 1;
      }
      // fast run [p, f) — but never start a variate at or beyond `stop`
      int fe = f;
      if (base + fe > stop) fe = (int)(stop - base);
      if (chain != nullptr && base == seg_start) {
        // record chain starts p..fe-1 in the first window
        for (int q = 0; q < 4; ++q) {
          const int lo = q * 32, hi = lo + 32;
          const int a = max(p, lo), b = min(fe, hi);
          if (a < b) {
            const uint32_t bits = (b - a == 32) ? 0xffffffffu : (((1u << (b - a)) - 1u) << (a - lo));
            chain[q] |= bits;
          }
        }
      }
      if (WRITE) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int pos = 4 * lane + j;
          if (pos >= p && pos < fe) {
            store_variate(out, ld, cols, row0, k0 + k + (pos - p), count, xs[j]);
            if (end != nullptr && k0 + k + (pos - p) == count - 1) *end = base + pos + 1;
          }
        }
      }
      k += fe - p;
      p = fe;
      if (fe < f || f == kWin) break;  // reached stop or window end
      // slow variate starting at base + f (warp-uniform, all lanes compute)
      const uint64_t r0 = __shfl_sync(0xffffffffu, blk.v[0], f >> 2);
      const uint64_t r1 = __shfl_sync(0xffffffffu, blk.v[1], f >> 2);
      const uint64_t r2 = __shfl_sync(0xffffffffu, blk.v[2], f >> 2);
      const uint64_t r3 = __shfl_sync(0xffffffffu, blk.v[3], f >> 2);
      const int jj = f & 3;
      const uint64_t rf = jj == 0 ? r0 : jj == 1 ? r1 : jj == 2 ? r2 : r3;
      int64_t nxt;
      const double x = slow_normal(key, base + f, rf, &nxt);
      if (chain != nullptr && base == seg_start) {
#pragma unroll
        for (int q = 0; q < 4; ++q) chain[q] |= ((f >> 5) == q) ? (1u << (f & 31)) : 0u;
      }
      if (WRITE && lane == 0) {
        store_variate(out, ld, cols, row0, k0 + k, count, x);
        if (end != nullptr && k0 + k == count - 1) *end = nxt;
      }
      k += 1;
      p = (int)(nxt - base);
    }
    head = base + p;
    base = (head / kWin) * kWin;
  }
  *exit_pos = head;
  return k;
}

#ifdef CNMF_RNG_PROBE
__device__ unsigned long long g_rng_probe[4096][2];
__device__ __forceinline__ unsigned long long probe_time() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

__global__ void k1_speculate(const Layout L, SegState* segs) {
#ifdef CNMF_RNG_PROBE
  const unsigned long long pt0 = probe_time();
#endif
  load_zig_tables();
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (g >= L.total_segs) return;
  const StreamDesc sd = stream_of(L, chunk_of_seg(L, g));
  const int64_t w = g - sd.seg0;
  const int64_t s0 = sd.base + w * sd.seglen, s1 = s0 + sd.seglen;
  uint32_t chain[4] = {0, 0, 0, 0};
  int64_t ex;
  const int64_t n = walk<false, float>(sd.key, s0, s1, s0, chain, nullptr, 0, 1, 0, 0, 0, &ex);
#ifdef CNMF_RNG_PROBE
  if ((threadIdx.x & 31) == 0 && g < 4096) {
    g_rng_probe[g][0] = pt0;
    g_rng_probe[g][1] = probe_time();
  }
#endif
  if ((threadIdx.x & 31) == 0) {
    segs[g].exit = ex;
    segs[g].count = n;
#pragma unroll
    for (int q = 0; q < 4; ++q) segs[g].chain[q] = chain[q];
  }
}

// One CTA per stream: re-anchor each segment at its true entry, scan counts.
__global__ void k2_anchor_scan(const Layout L, SegState* segs, int* flags) {
  load_zig_tables();
  const StreamDesc sd = stream_of(L, blockIdx.x);
  __shared__ int64_t s_cnt[1024];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (int w = threadIdx.x; w < sd.nseg; w += blockDim.x) {
    SegState& st = segs[sd.seg0 + w];
    const int64_t s0 = sd.base + (int64_t)w * sd.seglen;
    const int64_t entry = (w == 0) ? sd.base : segs[sd.seg0 + w - 1].exit;
    int64_t d = 0;
    int64_t p = entry;
    bool merged = false;
    // serial single-thread walk from the entry until hitting a recorded start
    for (int guard = 0; guard < 64; ++guard) {
      const int64_t rel = p - s0;
      if (rel >= 0 && rel < kWin && ((st.chain[rel >> 5] >> (rel & 31)) & 1u)) {
        merged = true;
        break;
      }
      if (rel >= kWin || rel < 0) break;
      const uint64_t r = philox_raw(sd.key, (uint64_t)p);
      uint64_t rr = r >> 8;
      const int idx = (int)(r & 0xff);
      const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
      int64_t nxt = p + 1;
      if (!(rabs < s_zki[idx])) (void)slow_normal(sd.key, p, r, &nxt);
      d += 1;
      p = nxt;
    }
    int64_t cnt = 0;
    if (merged) {
      const int64_t rel = p - s0;
      int64_t below = 0;
      for (int q = 0; q < 4; ++q) {
        const int lo = q * 32;
        if (rel >= lo + 32)
          below += __popc(st.chain[q]);
        else if (rel > lo)
          below += __popc(st.chain[q] & ((1u << (rel - lo)) - 1u));
      }
      cnt = d + st.count - below;
    } else {
      s_bad = 1;
    }
    st.entry = entry;
    s_cnt[w] = cnt;
  }
  __syncthreads();
  // block-wide exclusive scan of the corrected counts (blockDim = 256, 4 each)
  __shared__ int64_t s_part[256];
  const int t = threadIdx.x;
  int64_t loc = 0;
  for (int q = 0; q < 4; ++q) {
    const int w = 4 * t + q;
    if (w < sd.nseg) loc += s_cnt[w];
  }
  s_part[t] = loc;
  __syncthreads();
  for (int off = 1; off < 256; off <<= 1) {
    const int64_t v = (t >= off) ? s_part[t - off] : 0;
    __syncthreads();
    s_part[t] += v;
    __syncthreads();
  }
  int64_t acc = s_part[t] - loc;
  for (int q = 0; q < 4; ++q) {
    const int w = 4 * t + q;
    if (w < sd.nseg) {
      segs[sd.seg0 + w].offset = acc;
      acc += s_cnt[w];
    }
  }
  if (t == 255) {
    if (s_part[255] < sd.count) s_bad = 1;
  }
  __syncthreads();
  if (t == 0) flags[blockIdx.x] = s_bad;
}

template <typename T>
__global__ void k3_emit(const Layout L, const SegState* segs, const int* flags, T* out, int64_t ld, int64_t* end) {
  load_zig_tables();
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (g >= L.total_segs) return;
  const int64_t c = chunk_of_seg(L, g);
  if (flags[c]) return;
  const StreamDesc sd = stream_of(L, c);
  const int64_t w = g - sd.seg0;
  const SegState st = segs[g];
  if (st.offset >= sd.count) return;
  const int64_t s1 = sd.base + (w + 1) * sd.seglen;
  int64_t ex;
  walk<true, T>(sd.key, st.entry, s1, -1, nullptr, out, ld, L.cols, sd.row0, st.offset, sd.count, &ex,
                end);
}

// Fallback: one warp decodes a whole stream sequentially.
template <typename T>
__global__ void k_serial(const Layout L, const int* flags, T* out, int64_t ld, int64_t* end) {
  load_zig_tables();
  if (!flags[blockIdx.x]) return;
  const StreamDesc sd = stream_of(L, blockIdx.x);
  int64_t head = sd.base, k = 0;
  while (k < sd.count) {
    int64_t ex;
    k += walk<true, T>(sd.key, head, head + 64 * kWin, -1, nullptr, out, ld, L.cols, sd.row0, k, sd.count, &ex,
                       end);
    head = ex;
  }
}

template <typename T>
__global__ void uniform_kernel(uint64_t key, int64_t start, int64_t rows, int64_t cols, double low, double high,
                               int transpose, T* out) {
  // raw draw start + i feeds variate i; thread b covers Philox block
  // start / 4 + b (words before `start` in the first block are skipped)
  const int64_t total = rows * cols;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t b0 = start / 4;
  if ((b0 + b) * 4 >= start + total) return;
  const U64x4 blk = philox4x64((uint64_t)(b0 + b) + 1, 0, key, 0);
  const double span = __dadd_rn(high, -low);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t i = (b0 + b) * 4 + j - start;
    if (i >= 0 && i < total) {
      const double v = __dadd_rn(low, __dmul_rn(span, raw_to_unit(blk.v[j])));
      if (transpose) {
        const int64_t r = i / cols, c = i - (i / cols) * cols;
        out[c * rows + r] = (T)v;
      } else {
        out[i] = (T)v;
      }
    }
  }
}

}  // namespace

static Layout make_layout(uint64_t seed, int64_t rows, int64_t cols, int64_t chunk_rows, int64_t start = 0) {
  Layout L{};
  L.start = chunk_rows > 0 ? 0 : start;
  L.rows = rows;
  L.cols = cols;
  L.chunked = chunk_rows > 0;
  L.chunk_rows = L.chunked ? std::min(chunk_rows, rows) : rows;
  L.nchunks = ceil_div(rows, L.chunk_rows);
  L.key = seed;
  auto seg = [](int64_t count, int32_t* seglen, int32_t* nseg) {
#ifndef CNMF_ZIG_MARGIN
#define CNMF_ZIG_MARGIN 1.05
#endif
    const int64_t need = (int64_t)(count * CNMF_ZIG_MARGIN) + 4 * kWin;
    int64_t len = kWin;  // one window per segment: 4x the warps of 4-window segments (latency-bound walk)
    while (ceil_div(need, len) > 1024) len *= 2;
    *seglen = (int32_t)len;
    *nseg = (int32_t)ceil_div(need, len);
  };
  seg(L.chunk_rows * cols, &L.seglen_full, &L.nseg_full);
  seg((rows - (L.nchunks - 1) * L.chunk_rows) * cols, &L.seglen_last, &L.nseg_last);
  L.total_segs = (L.nchunks - 1) * (int64_t)L.nseg_full + L.nseg_last;
  return L;
}

size_t gaussian_workspace(int64_t rows, int64_t cols, int64_t chunk_rows) {
  const Layout L = make_layout(0, rows, cols, chunk_rows);
  return (size_t)L.total_segs * sizeof(SegState) + (size_t)L.nchunks * 4 + 64 + 512;
}

template <typename T>
static int gaussian_streams(const Layout& L, T* out, int64_t ld, void* ws, size_t ws_bytes, cudaStream_t stream,
                            int64_t* end = nullptr) {
  if (ws_bytes < gaussian_workspace(L.rows, L.cols, L.chunked ? L.chunk_rows : 0))
    return fail(CNMF_ERR_ARGUMENT, "gaussian_fill: workspace too small");
  char* p = (char*)(((uintptr_t)ws + 15) & ~(uintptr_t)15);
  SegState* d_seg = (SegState*)p;
  p += (size_t)L.total_segs * sizeof(SegState);
  int* d_flags = (int*)p;
  const int wpb = 4;  // warps per block
  const unsigned grid = (unsigned)ceil_div(L.total_segs, wpb);
  k1_speculate<<<grid, 32 * wpb, 0, stream>>>(L, d_seg);
  CNMF_LAUNCH_CHECK();
  k2_anchor_scan<<<(unsigned)L.nchunks, 256, 0, stream>>>(L, d_seg, d_flags);
  CNMF_LAUNCH_CHECK();
  k3_emit<T><<<grid, 32 * wpb, 0, stream>>>(L, d_seg, d_flags, out, ld, end);
  CNMF_LAUNCH_CHECK();
  k_serial<T><<<(unsigned)L.nchunks, 32, 0, stream>>>(L, d_flags, out, ld, end);
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

int gaussian_fill_ws(uint64_t seed, int64_t rows, int64_t cols, int64_t chunk_rows, int dtype, void* out, int64_t ld,
                     void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (rows < 1 || cols < 1) return fail(CNMF_ERR_ARGUMENT, "gaussian_fill needs positive dims");
  if (ld < cols) return fail(CNMF_ERR_ARGUMENT, "gaussian_fill: ld < cols");
  const Layout L = make_layout(seed, rows, cols, chunk_rows);
  if (dtype == CNMF_F64) return gaussian_streams(L, (double*)out, ld, ws, ws_bytes, stream);
  if (dtype == CNMF_F32) return gaussian_streams(L, (float*)out, ld, ws, ws_bytes, stream);
  return fail(CNMF_ERR_ARGUMENT, "unknown dtype");
}

int gaussian_fill(uint64_t seed, int64_t rows, int64_t cols, int64_t chunk_rows, int dtype, void* out, int64_t ld,
                  cudaStream_t stream) {
  if (rows < 1 || cols < 1) return fail(CNMF_ERR_ARGUMENT, "gaussian_fill needs positive dims");
  const size_t bytes = gaussian_workspace(rows, cols, chunk_rows);
  keep_pool();
  void* ws = nullptr;
  CNMF_CUDA(cudaMallocAsync(&ws, bytes, stream));
  const int rc = gaussian_fill_ws(seed, rows, cols, chunk_rows, dtype, out, ld, ws, bytes, stream);
  cudaFreeAsync(ws, stream);
  return rc;
}

int uniform_fill_at(uint64_t seed, int64_t start, int64_t rows, int64_t cols, double low, double high, int dtype,
                    int transpose, void* out, cudaStream_t stream) {
  if (rows < 1 || cols < 1) return fail(CNMF_ERR_ARGUMENT, "uniform_fill needs positive dims");
  if (start < 0) return fail(CNMF_ERR_ARGUMENT, "uniform_fill: negative stream position");
  const int64_t blocks = ceil_div(start % 4 + rows * cols, 4);
  const unsigned grid = (unsigned)ceil_div(blocks, 256);
  if (dtype == CNMF_F64)
    uniform_kernel<double><<<grid, 256, 0, stream>>>(seed, start, rows, cols, low, high, transpose, (double*)out);
  else if (dtype == CNMF_F32)
    uniform_kernel<float><<<grid, 256, 0, stream>>>(seed, start, rows, cols, low, high, transpose, (float*)out);
  else
    return fail(CNMF_ERR_ARGUMENT, "unknown dtype");
  CNMF_LAUNCH_CHECK();
  return CNMF_OK;
}

int uniform_fill(uint64_t seed, int64_t rows, int64_t cols, double low, double high, int dtype, int transpose,
                 void* out, cudaStream_t stream) {
  return uniform_fill_at(seed, 0, rows, cols, low, high, dtype, transpose, out, stream);
}

// One stream of `count` standard normals starting at raw position `start`;
// *d_end (device int64) receives the raw position after the last variate.
int normal_fill_at(uint64_t seed, int64_t start, int64_t count, int dtype, void* out, int64_t* d_end,
                   cudaStream_t stream) {
  if (count < 1) return fail(CNMF_ERR_ARGUMENT, "normal_fill needs a positive count");
  if (start < 0) return fail(CNMF_ERR_ARGUMENT, "normal_fill: negative stream position");
  const Layout L = make_layout(seed, 1, count, 0, start);
  const size_t bytes = gaussian_workspace(1, count, 0);
  keep_pool();
  void* ws = nullptr;
  CNMF_CUDA(cudaMallocAsync(&ws, bytes, stream));
  int rc;
  if (dtype == CNMF_F64)
    rc = gaussian_streams(L, (double*)out, count, ws, bytes, stream, d_end);
  else if (dtype == CNMF_F32)
    rc = gaussian_streams(L, (float*)out, count, ws, bytes, stream, d_end);
  else
    rc = fail(CNMF_ERR_ARGUMENT, "unknown dtype");
  cudaFreeAsync(ws, stream);
  return rc;
}

}  // namespace cnmf
