// Internal declarations of the B200 NSS library (not part of the ABI).
// "P:n" cites /root/reference/PAPER.md; "R-n" a DESIGN.md section 2 reading.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "nss.h"

namespace nss {

constexpr int kMaxDim = NSS_MAX_DIM;
constexpr int kMaxComp = 16;
constexpr uint32_t kPhaseInit = 1, kPhaseResample = 2, kPhaseHrss = 3, kPhaseVolume = 4, kPhasePosterior = 5,
                   kPhaseRw = 6, kPhaseSmc = 7;

// ----------------------------------------------------------------------------
// Device-resident run state (one small struct, read by every kernel).
// ----------------------------------------------------------------------------
struct DevState {
  long long n_dead;        // records in the dead store
  long long dead_base;     // first dead record of the current iteration
  int iter;                // completed iterations (next one is iter + 1)
  int terminated;          // R-19 criterion met after the last iteration
  int error;               // nss_status raised on the device (NaN, capacity, support)
  int has_pend;            // trapezoid point waiting for X_{i+1}
  float e_star;            // E* of the last iteration
  float width;             // slice width for the next iteration (R-7)
  float emin;              // min live energy after the last iteration
  int finalised;
  double pend_e;           // energy of the pending trapezoid point
  double log_z_live;
  unsigned long long probes, evals, expansions, shrinks, nulls;
  unsigned long long init_evals, init_attempts;
  unsigned long long stamp[16];  // %globaltimer stamps (ns) for latency profiling
  double smc_beta, smc_logz;     // F3 tempered SMC: current temperature, accumulated log Z
  unsigned long long dev_launches;  // kernels launched by device-side loops (graph WHILE nodes)
  int loop_rounds;                  // rounds of the current iteration's device-side loop
};

// Energy parameters laid out for the kernels (device pointers, fp32).
struct EnergyDev {
  int kind;
  int d;
  int n_comp;
  int d_in;
  long long n_data;
  float c;
  float sigma_y;
  float jitter;
  const float *mu;      // GAUSS/CORR: d; MOG: K*d
  const float *isig;    // GAUSS: d; MOG: K*d  (1/sigma)
  const float *logc;    // MOG: K  (log w_j - sum log sigma_j - d/2 log 2pi)
  const float *prec;    // CORR: d*d
  const float *ufac;    // CORR: U (d*d row-major, upper) with P = U^T U, or null
  const float *data_x;  // LOGREG: N*d; GP: N*d_in
  const float *data_y;  // LOGREG / GP: N
  // one-probe-per-lane engine tables, padded to 32 coordinates with neutral
  // values: [K][2][32] = {1/sigma, -mu/sigma} per component (GAUSS: K = 1)
  const float *lane_ab;
};

struct PriorDev {
  int kind;
  const float *lo, *hi;       // BOX
  const float *mean, *isd, *sd;  // GAUSS_DIAG (isd = 1/sd)
  float log_norm;             // BOX: -sum log(hi-lo); GAUSS: -sum log sd - d/2 log 2pi
  // [2][32] padded: BOX {lo (-inf), hi (+inf)}; GAUSS {mean (0), 1/sd (0)}
  const float *lane_pab;
};

// Everything a kernel needs about the live set and the run.
struct RunDev {
  int n, k, d, dp, p;         // dp = row stride of X (floats)
  int max_stepout, max_shrink;
  int dir_norm, quadrature;
  int R;
  int engine;                 // nss_hrss_engine (host-side choice)
  int c0, c1;                 // HRSS chains [c0, c1) run here (all on one GPU);
                              // with `crange` the grid bound only (c1 - c0 = the most chains this GPU runs)
  // sharded live set: rank `rank` of `world` owns the gids
  // [rank_lo[rank], rank_lo[rank + 1]) -- whole segments of kSegs fixed gid
  // segments -- and runs the chains whose destination it owns, the ordinal
  // range crange[0..1) of the ascending destination list (written by the
  // merge kernel).  Start rows of chains whose parent another rank owns are
  // read from that rank's live set over NVLink through peerX / peerE.
  int world, rank;
  int rank_lo[9];
  const int *crange;          // device [2], or null (host range c0, c1)
  float *const *peerX;        // device [world] row bases of every rank's X (own included), or null
  float *const *peerE;
  double *mshift;             // d: shift of the metric's moment sums (the previous metric's mean, R-8)
  // HRSS chains of the iteration: nch = k (destinations = deleted slots) or n
  // (F4 update-all: every slot); chain c writes slot cdest[c] starting from
  // row cpar[c] of the start arrays Xs/Es (X/E themselves, or a snapshot of
  // the pre-mutation live set when survivors move too)
  int nch;
  int *cdest, *cpar;
  int mutation;               // NSS_MUT_HRSS or NSS_MUT_RW (F1)
  int tempered;               // F3: HRSS on Pi exp(-beta E) (beta = st->smc_beta), no threshold
  float *Vpre;                // warp engine, large d: directions of every (chain, step) of the
                              // iteration, computed up front by k_dirs ((c1-c0) p rows of dp), or null
  float rw_sigma;             // RW proposal scale c 2.38 / sqrt(d)
  const float *Xs, *Es;
  long long max_dead;
  uint32_t seed_lo, seed_hi;
  float term_log_ratio;
  float *X, *E, *birth;       // live set
  float *L;                   // lower Cholesky of Sigma, fp32, row stride dp
  float *LT;                  // its transpose (column j of L contiguous), row stride dp
  double *L64;                // fp64 copy, d*d
  // dead store
  float *dE, *dbirth, *dX;
  int *dnlive, *dgid, *dord, *diter;
  // per-iteration scratch
  int *dead_gid, *dest_gid, *parent_gid, *surv;
  uint32_t *counts;           // k*p packed {nL, nR, nS, acc}
  unsigned long long *sort_scratch;  // n + pow2(max(n, k)) keys
  unsigned long long *sel_scratch;   // 2k keys: selected (gid order), sorted
  // evidence replicas
  double *lx_prev, *lx_cur, *lz;
  DevState *st;
};

constexpr int kSegs = 8;  // fixed gid segments: the metric's summation tree and the shard unit

// Segment s of the n gids: [seg_lo(n, s), seg_lo(n, s + 1)).
__host__ __device__ __forceinline__ int seg_lo(int n, int s) {
  return static_cast<int>((static_cast<long long>(s) * n) / kSegs);
}

// Chains [x, y) this GPU runs.
__device__ __forceinline__ int2 chain_range(const RunDev &r) {
  return r.crange ? make_int2(r.crange[0], r.crange[1]) : make_int2(r.c0, r.c1);
}

// Rank owning gid g (sharded live set).
__device__ __forceinline__ int owner_of(const RunDev &r, int g) {
  int o = 0;
  while (o + 1 < r.world && g >= r.rank_lo[o + 1]) ++o;
  return o;
}

// Start row / energy of a chain whose parent (start point) is gid g: the
// start arrays Xs/Es, or the owner's live set (possibly a peer GPU's memory).
__device__ __forceinline__ const float *start_row(const RunDev &r, int g) {
  const float *base = r.peerX ? r.peerX[owner_of(r, g)] : r.Xs;
  return base + static_cast<long long>(g) * r.dp;
}
__device__ __forceinline__ float start_e(const RunDev &r, int g) {
  return r.peerE ? r.peerE[owner_of(r, g)][g] : r.Es[g];
}

// ----------------------------------------------------------------------------
// Philox4x32-10 and the draw contract
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ uint4 philox_block(const RunDev &r, uint32_t iter, uint32_t gid,
                                              uint32_t phase, uint32_t sub, uint32_t block) {
  return philox(make_uint4(block, (phase << 24) | (sub & 0xFFFFFFu), gid, iter), r.seed_lo,
                r.seed_hi);
}

__device__ __forceinline__ uint32_t word(uint4 b, uint32_t w) {
  return w == 0 ? b.x : (w == 1 ? b.y : (w == 2 ? b.z : b.w));
}

// u = ((r >> 9) + 1/2) * 2^-23, exact in fp32 (R-25)
__device__ __forceinline__ float u01(uint32_t r) {
  return (static_cast<float>(r >> 9) + 0.5f) * 1.1920928955078125e-07f;
}

// D(8x8) += A(8x4) B(4x8) on the fp64 tensor cores (DMMA): a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], d = D[lane/4][2 (lane%4) + {0, 1}]
__device__ __forceinline__ void dmma_f64(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Orderable u32 of an fp32 (ascending), -0 canonicalised to +0 (R-1).
__device__ __forceinline__ uint32_t ord_f32(float e) {
  uint32_t b = __float_as_uint(e);
  if (b == 0x80000000u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ unsigned long long key_of(float e, int gid) {
  return (static_cast<unsigned long long>(ord_f32(e)) << 32) | static_cast<uint32_t>(gid);
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void raise_error(DevState *st, int code) { atomicCAS(&st->error, 0, code); }

// A9 / R-19: the run stops when the live bound log Z_live = -min E_live +
// log X (replica 0) is below e^{term} of log Z_0 + Z_live.  Evaluated before
// each iteration by the select kernel (one thread) and by k_term_probe when
// the host asks; records E_min and log Z_live; returns the decision.
__device__ inline bool term_check_v(const RunDev &r, DevState *st, float emin, double lx0, double lz0) {
  const double lz_live = -static_cast<double>(emin) + lx0;
  const double mm = fmax(lz0, lz_live);
  const double tot = (mm == -INFINITY) ? -INFINITY : mm + log(exp(lz0 - mm) + exp(lz_live - mm));
  const bool stop = st->n_dead > 0 && (lz_live - tot) < static_cast<double>(r.term_log_ratio);
  st->emin = emin;
  st->log_z_live = lz_live;
  if (stop) st->terminated = 1;
  return stop;
}
__device__ inline bool term_check(const RunDev &r, DevState *st, float emin) {
  return term_check_v(r, st, emin, r.lx_cur[0], r.lz[0]);
}

// ----------------------------------------------------------------------------
// Launchers (host side, one per kernel file)
// ----------------------------------------------------------------------------
// Every kernel of the library runs with the same (maximum) shared-memory
// carveout: a different carveout per kernel forces the SM to reconfigure its
// L1/shared split between consecutive launches.
// Function attributes apply per device, so the "already set" caches below are
// kept per (call site, device): a second context on another GPU of the same
// process sets them again for its device.
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d & 63;
}
template <class Kern>
inline void pin_carveout(Kern *kernel) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}
#define NSS_PIN_CARVEOUT(kern)                 \
  do {                                         \
    static bool pinned_[64] = {};              \
    const int dv_ = ::nss::current_device();   \
    if (!pinned_[dv_]) {                       \
      ::nss::pin_carveout(kern);               \
      pinned_[dv_] = true;                     \
    }                                          \
  } while (0)
// Raise a kernel's dynamic shared-memory limit to at least `bytes` on the
// current device (once per size increase).
#define NSS_MAX_SMEM(kern, bytes)                                                              \
  do {                                                                                         \
    static size_t set_[64] = {};                                                               \
    const int dv_ = ::nss::current_device();                                                   \
    const size_t b_ = static_cast<size_t>(bytes);                                              \
    if (set_[dv_] < b_) {                                                                      \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(b_)); \
      set_[dv_] = b_;                                                                          \
    }                                                                                          \
  } while (0)

struct LaunchCtx {
  cudaStream_t stream;
  long long *launch_counter;
};

// Programmatic dependent launch (the batch engine's round kernels): the
// kernel may start while its predecessor drains (setup overlaps the tail and
// the launch latency) and waits in pdl_wait() for the predecessor's results;
// pdl_trigger() lets the successor start.  NSS_NO_PDL=1 launches normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool on = getenv("NSS_NO_PDL") == nullptr;
  return on;
}
template <typename... KArgs, typename... Args>
inline void launch_maybe_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// k_select.cu: A2 delete + A3 dead records + A4 resample (one iteration)
void launch_select(const RunDev &r, const LaunchCtx &lc);
// k_select.cu: finalisation (R-18): all n live points become dead records
void launch_finalise_sort(const RunDev &r, const LaunchCtx &lc);
// k_evidence.cu: A8 volume replicas + quadrature for `count` new deaths
void launch_evidence(const RunDev &r, int finalise, const LaunchCtx &lc);
// k_hrss.cu: A6/A7 (+A1) HRSS chains; init draws
void launch_hrss(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc);
void launch_init(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc);
size_t energy_smem_bytes(const EnergyDev &en);
bool energy_supported(const EnergyDev &en);
int hrss_engine(const RunDev &r, const EnergyDev &en);  // 0 warp-cooperative, 1 one probe per lane
// k_hrss_multi.cu: several chains per warp sharing the factor's loads (correlated Gaussian, large d)
bool multi_engine_ok(const RunDev &r, const EnergyDev &en);
void launch_hrss_multi(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc);
// k_hrss_group.cu: four speculative probes per warp in groups of 8 lanes (cheap energies, large d)
bool group_engine_ok(const RunDev &r, const EnergyDev &en);
void launch_hrss_group(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc);
// k_hrss_lane.cu
bool lane_engine_ok(const RunDev &r, const EnergyDev &en);
void launch_hrss_lane(const RunDev &r, const PriorDev &pr, const EnergyDev &en, const LaunchCtx &lc);
// k_metric.cu: A5 metric (+ A9 termination when iterating)
void launch_term_probe(const RunDev &r, const LaunchCtx &lc, int probe = 1, DevState *mirror = nullptr,
                       double *lz0_mirror = nullptr);
void launch_dirs(const RunDev &r, const LaunchCtx &lc);  // k_dirs when r.Vpre (k_hrss.cu)
void launch_smc_stage(const RunDev &r, double rho, double *cum, int *parents, float *Xsnap, float *Esnap,
                      const LaunchCtx &lc);
void launch_chains_all(const RunDev &r, int *cdest, int *cpar, float *Xs, float *Es, const LaunchCtx &lc);
void launch_metric(const RunDev &r, double metric_reg, int width_rule, double width_param,
                   int end_of_iteration, double *partials, unsigned *ticket, int n_blocks, const LaunchCtx &lc);
int metric_blocks(int n, int d);

}  // namespace nss
