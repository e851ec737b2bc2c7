// Per-iteration timeline of pass_tc (block 0): which role gates the pipeline?
// Build: see tools/tc_trace.sh
#define CNMF_TC_TRACE 1
#ifndef CNMF_TC_TRACE_CTA
#define CNMF_TC_TRACE_CTA 0
#endif
#include "../paper_1505_04650_b200/csrc/tc_pass.cu"

#include <algorithm>
#include <cstdlib>

int main(int argc, char** argv) {
  const int S = argc > 1 ? atoi(argv[1]) : 32;
  const bool trn = argc > 2 && atoi(argv[2]);
  const int64_t M = argc > 3 ? atoll(argv[3]) : 20000, N = argc > 4 ? atoll(argv[4]) : 10000;
  float *A, *X, *Y;
  cudaMalloc(&A, M * N * 4);
  cudaMemset(A, 0, M * N * 4);
  cudaMalloc(&X, M * S * 4);
  cudaMemset(X, 0, M * S * 4);
  cudaMalloc(&Y, M * S * 4);

  for (int r = 0; r < 3; ++r) {
    int st = trn ? cnmf::pass_transpose_tc(A, M, N, N, X, S, Y, 0) : cnmf::pass_forward_tc(A, M, N, N, X, S, Y, 0);
    if (st) printf("status %d\n", st);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  long long h[64][16];
  cudaMemcpyFromSymbol(h, cnmf::g_tc_trace, sizeof h);
  long long t0 = h[0][0];
  printf(" it   prodA  prodB  splA  splAE  splAF  bRaw  bSlot  bDone   mmaW   mmaI\n");
  for (int i = 0; i < 64; ++i)
    printf("%3d %7lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld\n", i, h[i][0] - t0,
           h[i][6] - t0, h[i][1] - t0, h[i][2] - t0, h[i][3] - t0, h[i][7] - t0, h[i][8] - t0, h[i][9] - t0,
           h[i][4] - t0, h[i][5] - t0, h[i][10] - t0, h[i][11] - t0, h[i][12] - t0);
  unsigned long long sp[148][3];
  cudaMemcpyFromSymbol(sp, cnmf::g_tc_span, sizeof sp);
  unsigned long long t_lo = ~0ull, t_hi = 0, s_lo = ~0ull, s_hi = 0, e_lo = ~0ull;
  double avg = 0;
  for (int b = 0; b < 148; ++b) {
    t_lo = std::min(t_lo, sp[b][0]);
    s_hi = std::max(s_hi, sp[b][0]);
    t_hi = std::max(t_hi, sp[b][1]);
    e_lo = std::min(e_lo, sp[b][1]);
    avg += (double)(sp[b][1] - sp[b][0]) / 148;
  }
  printf("kernel span %.1f us: starts spread %.1f us, ends spread %.1f us, avg CTA %.1f us\n",
         (t_hi - t_lo) * 1e-3, (s_hi - t_lo) * 1e-3, (t_hi - e_lo) * 1e-3, avg * 1e-3);
  for (int b = 0; b < 148; b += 8) printf("cta %3d: start %7.1f end %7.1f\n", b, (sp[b][0] - t_lo) * 1e-3, (sp[b][1] - t_lo) * 1e-3);
  return 0;
}
