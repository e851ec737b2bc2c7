// Time one dual CholeskyQR sweep (configs[1] panels: 10000 and 5000 rows,
// s = 30) back to back; build variants with -DSWEEP_X=1 (no factorisation:
// the last block publishes T = I) to see the factorisation's share.
// Build: tools/sweep_probe.sh
#include "../paper_1505_04650_b200/csrc/sweep.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

int main() {
  // SW_S / SW_ROWS0 / SW_ROWS1: basis width and panel heights (default configs[1]; configs[4]: 60 200000 100000)
  const int s = getenv("SW_S") ? atoi(getenv("SW_S")) : 30, S = s <= 32 ? 32 : 64, reps = 40;
  const int64_t rows[2] = {getenv("SW_ROWS0") ? atoll(getenv("SW_ROWS0")) : 10000,
                           getenv("SW_ROWS1") ? atoll(getenv("SW_ROWS1")) : 5000};
  cnmf::SweepPanel p[2];
  std::vector<float> h((size_t)rows[0] * S);
  srand(3);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (i % S) < (size_t)s ? rand() / (float)RAND_MAX - 0.5f : 0.f;
  for (int k = 0; k < 2; ++k) {
    float* P;
    double *G, *T;
    int* info;
    unsigned* counter;
    cudaMalloc(&P, rows[k] * S * 4);
    cudaMalloc(&G, S * S * 8);
    cudaMalloc(&T, S * S * 8);
    cudaMalloc(&info, 64);
    cudaMalloc(&counter, 64);
    cudaMemset(G, 0, S * S * 8);
    cudaMemset(info, 0, 64);
    cudaMemset(counter, 0, 64);
    cudaMemcpy(P, h.data(), rows[k] * S * 4, cudaMemcpyHostToDevice);
    p[k] = cnmf::SweepPanel{P, rows[k], G, T, nullptr, info, counter, s, 0, 0};
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int np = 1; np <= 2; ++np) {
    for (int r = 0; r < 3; ++r) cnmf::panel_sweep(p, np, S, 0);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) cnmf::panel_sweep(p, np, S, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%d panel(s): %.1f us per sweep (%s)\n", np, ms / reps * 1e3, cudaGetErrorString(cudaGetLastError()));
#ifdef SWEEP_TRACE
    unsigned long long t[512][12];
    cudaMemcpyFromSymbol(t, cnmf::g_sw_t, sizeof t);
    unsigned long long t0 = ~0ull;
    const int nbk = 296;
    for (int b = 0; b < nbk; ++b) t0 = t[b][0] < t0 ? t[b][0] : t0;
    auto mx = [&](int k) { unsigned long long m = 0; for (int b = 0; b < nbk; ++b) if (t[b][k] > m && t[b][k] < t0 + 100000000) m = t[b][k]; return (m - t0) * 1e-3; };
    auto mn = [&](int k) { unsigned long long m = ~0ull; for (int b = 0; b < nbk; ++b) if (t[b][k] >= t0 && t[b][k] < m) m = t[b][k]; return (m - t0) * 1e-3; };
    printf("  tile loaded max %.2f | gram computed max %.2f\n", mx(8), mx(9));
    printf("  start spread %.2f | gram done max %.2f | partial stored max %.2f | reducers done max %.2f | final reduce %.2f..%.2f | factor done %.2f | T seen min %.2f max %.2f | apply done max %.2f us\n",
           mx(0), mx(1), mx(2), mx(3), mn(4), mx(4), mx(5), mn(6), mx(6), mx(7));
#endif
  }
  return 0;
}
