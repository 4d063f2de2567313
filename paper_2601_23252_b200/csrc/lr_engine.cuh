// Tensor-core logistic-regression energy engine (k_lr_energy.cu, lr_engine.cu).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include "nss_internal.cuh"

namespace nss {

struct LrEngine {
  long long N = 0, n_pad = 0;
  int d = 0, n_tiles = 0, p_stride = 0, max_probe = 0;
  int bn = 256;                 // data-tile width of the tensor-core pass (UMMA N): 128 or 256
  int xs = 1;                   // X terms: 1 (fp16-exact data) or 2 (X = Xhi + Xlo, R-28)
  __half *Xb = nullptr;         // [n_pad][128] fp16 data rows Xhi (K padded with zeros)
  __half *Xl = nullptr;         // [n_pad][128] fp16 Xlo = fp16(X - Xhi) (xs = 2), else null
  // linear part of the energy: sum_r (1/2 - y_r) a_r = theta . g, g = X^T (1/2 - y)
  // (fp64 on the host, 128 floats, zero past d); per-row values in lin[parity]
  float *g = nullptr;
  __half *A[2] = {nullptr, nullptr};          // per round parity: [2][p_stride][128] splits hi / lo
  double *eacc[2] = {nullptr, nullptr};       // per round parity: [p_stride] exact fp64 softplus sums
  float *lin[2] = {nullptr, nullptr};         // per round parity: [p_stride] theta~ . g
  CUtensorMap tmA[2]{}, tmB{}, tmB2{};
};

// Data the tensor-core path takes: d <= 128 and every |X| within the fp16
// range; *exact: every value fp16-exact (one X term), else split (two).
bool lr_data_ok(const double *X, long long count, int d, bool *exact);
cudaError_t lr_setup(LrEngine &L, const double *X, const double *y, long long N, int d, int max_probe);
void lr_free(LrEngine &L);
// Splits the fp32 probe rows P (row stride ldp) into A[0] and reduces the
// split partial sums into E (kernel-check path of nss_lr_energy_batch).
void lr_energies(const LrEngine &L, const float *P, int ldp, const int *n_probe, float *E, const LaunchCtx &lc);
// Energy pass of the batch engine: A[parity], lin[parity] and the zeroed
// eacc[parity] rows were written by the advance kernel; eacc[parity] receives
// the softplus sums; *reset_counter is cleared.
void lr_energy_pass(const LrEngine &L, int parity, const int *n_probe, int *reset_counter, const LaunchCtx &lc);

}  // namespace nss
