// Round-synchronous batched HRSS engine (k_batch.cu) for energies that are too
// expensive for one warp: every round, each chain advances its HRSS state
// machine until it needs an energy, writes that probe point into a shared
// probe buffer, and one batched energy kernel evaluates all probes at once
// (tensor cores for logistic regression, batched Cholesky for GP).
#pragma once
#include <cuda_fp16.h>

#include "nss_internal.cuh"

namespace nss {

enum BatchPhase : int { kPhDir = 0, kPhStepOut = 1, kPhShrink = 2, kPhDone = 3 };

constexpr int kChainWords = 8;  // int4 words per chain record (128 bytes)

struct BatchDev {
  int k, dp, max_rows, n_splits, p_stride;
  // per-chain state: one 128-byte record per chain (batch_chain.cuh, ChainRegs
  // packed: 9 ints, 11 floats, 5 counters {probes, evals, expansions, shrinks,
  // nulls}), read and written as seven 16-byte words of one cache line
  int4 *cs;                   // [k][8]
  float *x, *v;               // [k][dp]
  // probe buffers, double-buffered by round parity
  float *P[2];                // [max_rows][dp] probe points (fp32)
  int *n_probe;               // [2] rows issued in the round of that parity
  float *partial[2];          // [slices][p_stride] energy partial sums per row
  int *slices;                // [2] slices written by the energy pass of each parity
  __half *A[2];               // logistic regression: [2][p_stride][128] fp16 splits hi / lo, else null
  float *lin[2];              // logistic regression: per-row linear part theta~ . g, else null
  double *eacc[2];            // logistic regression: per-row exact fp64 softplus sums (energy pass), else null
  const float *g;             // logistic regression: g = X^T (1/2 - y) (128 floats), else null
};

// k_batch.cu
void batch_begin(const RunDev &r, const PriorDev &pr, const BatchDev &b, const LaunchCtx &lc);
void batch_advance(const RunDev &r, const PriorDev &pr, const BatchDev &b, int parity, const LaunchCtx &lc);
void batch_energy_generic(const RunDev &r, const EnergyDev &en, const BatchDev &b, int parity, const LaunchCtx &lc);
void batch_finish(const RunDev &r, const BatchDev &b, const LaunchCtx &lc);
// one pass of the device-side round loop decides whether the WHILE node repeats
void launch_round_cond(cudaGraphConditionalHandle h, const BatchDev &b, const RunDev &r, int per_body,
                       int max_rounds, const LaunchCtx &lc);
bool batch_generic_ok(const EnergyDev &en);
void batch_init_draw(const RunDev &r, const PriorDev &pr, const BatchDev &b, const int *pending, int *map,
                     uint32_t attempt, const LaunchCtx &lc);
void batch_init_accept(const RunDev &r, const BatchDev &b, const int *map, int *pending, int *n_pending,
                       const LaunchCtx &lc);

// k_gp.cu: fp64 batched GP marginal likelihood (one CTA per probe matrix)
bool gp_setup(void **handle, const double *X, const double *y, int N, int D, double jitter);
void gp_free(void *handle);
void gp_set_out64(void *handle, double *e64);  // also write fp64 energies (kernel checks)
void gp_energy_pass(void *handle, const BatchDev &b, int parity, const LaunchCtx &lc);
// the fused engine: every chain of [r.c0, r.c1) run to completion by one CTA
// (HRSS state machine + GP energies of its probes), no per-round barrier
bool gp_chains_pass(void *handle, const RunDev &r, const PriorDev &pr, const BatchDev &b, const LaunchCtx &lc);

}  // namespace nss
