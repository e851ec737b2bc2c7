// Per-warp timeline of the test-matrix kernels (k1 speculate): start/end of
// each warp's walk, to tell a long per-warp walk from late-starting warps.
#define CNMF_RNG_PROBE 1
#include "../paper_1505_04650_b200/csrc/rng.cu"
#include <algorithm>
#include <cstdio>
#include <vector>
int main() {
  const int64_t rows = 10000, cols = 30;
  float* out;
  cudaMalloc(&out, rows * 32 * 4);
  for (int rep = 0; rep < 3; ++rep) cnmf::gaussian_fill(12345, rows, cols, 4096, CNMF_F32, out, 32, 0);
  cudaDeviceSynchronize();
  unsigned long long h[4096][2];
  cudaMemcpyFromSymbol(h, cnmf::g_rng_probe, sizeof h);
  unsigned long long t0 = ~0ull, t1 = 0;
  std::vector<double> dur;
  for (int i = 0; i < 4096; ++i)
    if (h[i][0]) {
      t0 = std::min(t0, h[i][0]);
      t1 = std::max(t1, h[i][1]);
      dur.push_back((h[i][1] - h[i][0]) * 1e-3);
    }
  std::sort(dur.begin(), dur.end());
  unsigned long long smax = 0;
  for (int i = 0; i < 4096; ++i)
    if (h[i][0]) smax = std::max(smax, h[i][0] - t0);
  printf("warps %zu: span %.1f us, start spread %.1f us, walk min %.1f median %.1f max %.1f us\n", dur.size(),
         (t1 - t0) * 1e-3, smax * 1e-3, dur.front(), dur[dur.size() / 2], dur.back());
  return 0;
}
