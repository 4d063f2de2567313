// Tensor-core logistic-regression energy engine (k_lr_energy.cu, lr_engine.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "nss_internal.cuh"

namespace nss {

struct LrEngine {
  long long N = 0, n_pad = 0;
  int d = 0, n_tiles = 0, p_stride = 0, max_probe = 0, n_splits = 1;
  int bn = 128;                 // data-tile width of the tensor-core pass (UMMA N): 128 or 256
  __nv_bfloat16 *Xb = nullptr;  // [n_pad][128] bf16 data rows (K padded with zeros)
  // linear part of the energy: sum_r (1/2 - y_r) a_r = theta . g, g = X^T (1/2 - y)
  // (fp64 on the host, 128 floats, zero past d); per-row values live in the
  // extra slot n_splits of partial[parity]
  float *g = nullptr;
  __nv_bfloat16 *A[2] = {nullptr, nullptr};   // per round parity: [3][p_stride][128] splits hi / mid / lo
  float *partial[2] = {nullptr, nullptr};     // per round parity: [n_splits + 1][p_stride]
  int *slices = nullptr;                      // [2] data slices used by the last pass of each parity
  CUtensorMap tmA[2]{}, tmB{};
};

bool lr_data_bf16_exact(const double *X, long long count);
cudaError_t lr_setup(LrEngine &L, const double *X, const double *y, long long N, int d, int max_probe);
void lr_free(LrEngine &L);
// Splits the fp32 probe rows P (row stride ldp) into A[parity] and reduces the
// split partial sums into E (kernel-check path of nss_lr_energy_batch).
void lr_energies(const LrEngine &L, const float *P, int ldp, const int *n_probe, float *E, const LaunchCtx &lc);
// Energy pass of the batch engine: A[parity] was written by the advance kernel;
// partial[parity] receives the split sums; *reset_counter is cleared.
void lr_energy_pass(const LrEngine &L, int parity, const int *n_probe, int *reset_counter, const LaunchCtx &lc);

}  // namespace nss
