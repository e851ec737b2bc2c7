// One CholeskyQR sweep over one or two tall-skinny panels in one cooperative
// launch (csrc/sweep.cu).
#pragma once

#include "common.cuh"

namespace cnmf {

// A panel to orthonormalise in place: P (rows x S fp32, s logical columns),
// its Gram accumulator G (S x S fp64, zero on entry, handed back zeroed),
// the transform T = R^{-1} and optionally R (S x S fp64), the failure word
// `info` (info[1] = min pass id whose Gram matrix was not factorable) and
// three zeroed counters (left zeroed).
struct SweepPanel {
  float* P;
  int64_t rows;
  double* G;
  double* T;
  double* R;
  int* info;
  unsigned* counter;
  int s;
  int pass_id;
  int blocks;  // set by panel_sweep
};

// P <- P R^{-1} with G = P^T P = R^T R for np (1 or 2) panels of the same
// width S. Two panels share the launch: their Gram passes, factorisations
// (one block each, concurrently) and applies overlap.
int panel_sweep(SweepPanel* panels, int np, int S, cudaStream_t st);

}  // namespace cnmf
