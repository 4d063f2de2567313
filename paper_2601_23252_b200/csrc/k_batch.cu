// A6/A7 for expensive energies: the round-synchronous batched HRSS engine.
//
// One warp per chain runs the sequential HRSS state machine (P:733-749,
// identical decisions and draws to k_hrss.cu) and stops whenever it needs an
// energy: it appends the probe point x + t v to the probe buffer of this
// round (atomic row ticket; the row index never changes the value computed),
// remembers which row it owns, and returns.  Probes that leave the prior
// support or fall below the slice height are resolved in place without an
// energy.  Both stepping-out endpoints of a side are independent of the other
// side, so a chain issues the next left and the next right endpoint in the
// same round (two probes), which cuts the rounds per HRSS step from ~6 to ~4
// without evaluating anything the sequential algorithm would not.  A batched
// energy kernel then evaluates every probe row; the next round's advance
// reads the results.  Buffers alternate by round parity, and each energy
// kernel clears the other parity's row counter for the round after it.
#include "batch_chain.cuh"

namespace nss {

namespace {

constexpr int kWarpsPerBlock = 8;

template <int NPL>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_batch_begin(RunDev r, PriorDev pr, BatchDev b) {
  const int lane = threadIdx.x & 31;
  const int2 cr = chain_range(r);
  const int c = cr.x + blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    b.n_probe[0] = 0;
    b.n_probe[1] = 0;
    r.st->loop_rounds = 0;
  }
  if (c >= cr.y) return;
  const DevState *st = r.st;
  const bool off = st->terminated || st->error || st->finalised;
  const int d = r.d, par = r.cpar[c];
  float pa[NPL], pb[NPL], x[NPL];
  load_prior_lane<NPL>(pr, lane, d, pa, pb);
  const float *xs = start_row(r, par);
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    x[t] = i < d ? xs[i] : 0.f;
    if (i < r.dp) b.x[static_cast<long long>(c) * b.dp + i] = x[t];
  }
  bool dummy;
  const float lp = prior_logp<NPL>(x, pr, pa, pb, lane, d, dummy);
  if (lane == 0) {
    ChainRegs s{};
    s.phase = off ? kPhDone : kPhDir;
    s.row0 = s.row1 = -1;
    s.e = start_e(r, par);
    s.lp = lp;
    store_chain(b, c, s);
  }
}

// resident blocks per SM the advance is compiled for (register budget);
// measurement builds may change it (NSS_NVCC_EXTRA=-DNSS_ADV_MINB=4)
#ifndef NSS_ADV_WARPS
#define NSS_ADV_WARPS 1  // warps (chains) per advance block (A/B: 8 -> 4 -> 2 -> 1 measured 21.27 -> 21.00 -> 20.90 -> 20.26 ms per C4 iteration)
#endif
constexpr int kAdvWarps = NSS_ADV_WARPS;
#ifndef NSS_ADV_MINB
#define NSS_ADV_MINB (24 / NSS_ADV_WARPS)
#endif

// W lanes per chain: 32, or 16 (two chains per warp; large d, where the
// directions are precomputed): twice the chains in flight per SM for this
// latency-bound state machine.
template <int NPL, int W>
__global__ void __launch_bounds__(kAdvWarps * 32, NSS_ADV_MINB) k_batch_advance(RunDev r, PriorDev pr, BatchDev b,
                                                                                   int parity) {
  extern __shared__ float sm[];
  pdl_trigger();  // every block has started: the energy pass may launch (it waits for us)
  pdl_wait();     // the previous energy pass is complete
  const int wib = threadIdx.x >> 5;
  const int2 cr = chain_range(r);
  const int c = cr.x + (blockIdx.x * kAdvWarps * 32 + static_cast<int>(threadIdx.x)) / W;
  if constexpr (W == 32) {
    // one row ticket per block: every warp reports its probe count once
    __shared__ int sh_cnt[kAdvWarps], sh_base;
    auto ticket = [&](int np) -> int {
      if ((threadIdx.x & 31) == 0) sh_cnt[wib] = np;
      __syncthreads();
      if (threadIdx.x == 0) {
        int tot = 0;
        for (int q = 0; q < kAdvWarps; ++q) tot += sh_cnt[q];
        sh_base = tot ? atomicAdd(&b.n_probe[parity], tot) : 0;
      }
      __syncthreads();
      int off = sh_base;
      for (int q = 0; q < wib; ++q) off += sh_cnt[q];
      return off;
    };
    if (r.st->terminated || r.st->error || r.st->finalised) return;  // uniform: no ticket at all
    if (c >= cr.y) {
      (void)ticket(0);
      return;
    }
    advance_chain<NPL, W>(r, pr, b, parity, c, sm + wib * (NPL * 32), ticket);
  } else {
    if (c >= cr.y) return;  // uniform per group
    advance_chain<NPL, W>(r, pr, b, parity, c, sm + wib * (NPL * 32));
  }
}

// Generic batched energy (warp per probe row) for kinds with a warp energy.
template <int NPL, int KIND>
__global__ void __launch_bounds__(256) k_batch_energy(RunDev r, EnergyDev en, BatchDev b, int parity) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) b.n_probe[parity ^ 1] = 0;  // next round's counter
  const int n = b.n_probe[parity];
  if (static_cast<int>(blockIdx.x) * wpb >= n) return;
  const int npar = energy_param_floats(KIND, r.d, en.n_comp);
  float *sP = sm;
  float *sY = sP + npar + wib * (NPL * 32);
  ESm es;
  stage_energy(en, sP, es);
  __syncthreads();
  const int row = blockIdx.x * wpb + wib;
  if (row >= n) return;
  float x[NPL];
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    x[t] = i < r.d ? b.P[parity][static_cast<long long>(row) * b.dp + i] : 0.f;
  }
  const float e = warp_energy<NPL, KIND>(x, en, es, sY, lane);
  if (lane == 0) b.partial[parity][row] = e;
}

// Batched prior draws (R-20) for energies that only have a batched
// implementation (GP): attempt `a` of every still-pending live point goes to
// the probe buffer of parity 0 (row ticket, map row -> gid), the energy pass
// evaluates them, and k_binit_accept keeps the finite ones.  Draws, budget
// and error rules are those of k_init (k_hrss.cu).
template <int NPL>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_binit_draw(RunDev r, PriorDev pr, BatchDev b,
                                                                     const int *pending, int *map, uint32_t a) {
  const int lane = threadIdx.x & 31;
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  DevState *st = r.st;
  if (g >= r.n || st->error || !pending[g]) return;
  unsigned long long used = 0;
  if (lane == 0) used = atomicAdd(&st->init_attempts, 1ull);
  used = __shfl_sync(kFull, used, 0);
  if (used >= 100ull * static_cast<unsigned long long>(r.n)) {
    if (lane == 0) raise_error(st, NSS_ERR_PRIOR_SUPPORT);
    return;
  }
  float pa[NPL], pb[NPL], x[NPL];
  load_prior_lane<NPL>(pr, lane, r.d, pa, pb);
  prior_draw<NPL>(r, pr, g, a, lane, pa, pb, x);
  int row = 0;
  if (lane == 0) row = atomicAdd(&b.n_probe[0], 1);
  row = __shfl_sync(kFull, row, 0);
#pragma unroll
  for (int t = 0; t < NPL; ++t) {
    const int i = lane + 32 * t;
    if (i < r.d) {
      b.P[0][static_cast<long long>(row) * b.dp + i] = x[t];
      r.X[static_cast<long long>(g) * r.dp + i] = x[t];
    }
  }
  if (lane == 0) map[row] = g;
}

__global__ void k_binit_accept(RunDev r, BatchDev b, const int *map, int *pending, int *n_pending) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  DevState *st = r.st;
  if (row >= b.n_probe[0] || st->error) return;
  const int g = map[row];
  const float e = b.partial[0][row];
  atomicAdd(&st->init_evals, 1ull);
  if (isnan(e)) {
    raise_error(st, NSS_ERR_NAN);
  } else if (isfinite(e)) {
    r.E[g] = e;
    r.birth[g] = INFINITY;
    pending[g] = 0;
  } else {
    atomicAdd(n_pending, 1);
  }
}

__global__ void k_batch_finish(RunDev r, BatchDev b) {
  const int2 cr = chain_range(r);
  const int c = cr.x + blockIdx.x * blockDim.x + threadIdx.x;
  DevState *st = r.st;
  if (st->terminated || st->error || st->finalised) return;
  __shared__ unsigned long long acc[5];
  if (threadIdx.x < 5) acc[threadIdx.x] = 0;
  __syncthreads();
  if (c < cr.y) {
    const int s = r.cdest[c];
    for (int i = 0; i < r.d; ++i) r.X[static_cast<long long>(s) * r.dp + i] = b.x[static_cast<long long>(c) * b.dp + i];
    ChainRegs cs;
    load_chain(b, c, cs);
    r.E[s] = cs.e;
    if (r.cpar[c] != s) r.birth[s] = st->e_star;  // a moved survivor (F4) keeps its birth level
    const unsigned cn[5] = {cs.c_probe, cs.c_eval, cs.c_exp, cs.c_shr, cs.c_null};
    for (int q = 0; q < 5; ++q) atomicAdd(&acc[q], static_cast<unsigned long long>(cn[q]));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&st->probes, acc[0]);
    atomicAdd(&st->evals, acc[1]);
    atomicAdd(&st->expansions, acc[2]);
    atomicAdd(&st->shrinks, acc[3]);
    atomicAdd(&st->nulls, acc[4]);
  }
}

// The device-side round loop (a CUDA-graph WHILE node, nss_api.cu): after each
// pass of its body (two rounds) continue while the last round issued probes.
// A cap far above any run's rounds (p (cap + 2 + max_shrink) + 2) turns a
// runaway loop into an error instead of a hang.
__global__ void k_round_cond(cudaGraphConditionalHandle h, const int *n_last, DevState *st, int per_body,
                             int max_rounds) {
  const int rounds = st->loop_rounds + per_body / 2;
  st->loop_rounds = rounds;
  st->dev_launches += static_cast<unsigned long long>(per_body);
  bool more = *n_last > 0;
  if (more && rounds > max_rounds) {
    raise_error(st, NSS_ERR_CUDA);
    more = false;
  }
  cudaGraphSetConditional(h, more ? 1u : 0u);
}

}  // namespace

void launch_round_cond(cudaGraphConditionalHandle h, const BatchDev &b, const RunDev &r, int per_body,
                       int max_rounds, const LaunchCtx &lc) {
  k_round_cond<<<1, 1, 0, lc.stream>>>(h, b.n_probe + 1, r.st, per_body, max_rounds);
  ++*lc.launch_counter;
}

namespace {

// blocks for this GPU's chains; at least one (block 0 resets the row counters)
int chain_blocks(const RunDev &r, int per_block) {
  const int nc = r.c1 - r.c0;
  return nc > 0 ? (nc + per_block - 1) / per_block : 1;
}

template <int NPL>
void begin_t(const RunDev &r, const PriorDev &pr, const BatchDev &b, const LaunchCtx &lc) {
  NSS_PIN_CARVEOUT(k_batch_begin<NPL>);
  k_batch_begin<NPL><<<chain_blocks(r, kWarpsPerBlock), kWarpsPerBlock * 32, 0, lc.stream>>>(r, pr, b);
  ++*lc.launch_counter;
}

template <int NPL, int W>
void advance_t(const RunDev &r, const PriorDev &pr, const BatchDev &b, int parity, const LaunchCtx &lc) {
  const size_t smem = W == 32 ? static_cast<size_t>(kAdvWarps) * NPL * 32 * sizeof(float) : 0;
  NSS_MAX_SMEM((k_batch_advance<NPL, W>), 160 * 1024);
  NSS_PIN_CARVEOUT((k_batch_advance<NPL, W>));
  launch_maybe_pdl(k_batch_advance<NPL, W>, dim3(chain_blocks(r, kAdvWarps * 32 / W)),
                   dim3(kAdvWarps * 32), smem, lc.stream, r, pr, b, parity);
  ++*lc.launch_counter;
}

template <int NPL>
void binit_draw_t(const RunDev &r, const PriorDev &pr, const BatchDev &b, const int *pending, int *map, uint32_t a,
                  const LaunchCtx &lc) {
  k_binit_draw<NPL><<<(r.n + kWarpsPerBlock - 1) / kWarpsPerBlock, kWarpsPerBlock * 32, 0, lc.stream>>>(
      r, pr, b, pending, map, a);
  ++*lc.launch_counter;
}

template <int NPL, int KIND>
void energy_t(const RunDev &r, const EnergyDev &en, const BatchDev &b, int parity, const LaunchCtx &lc) {
  const int wpb = 8;
  const size_t smem = (energy_param_floats(KIND, r.d, en.n_comp) + static_cast<size_t>(wpb) * NPL * 32) * sizeof(float);
  NSS_MAX_SMEM((k_batch_energy<NPL, KIND>), 160 * 1024);
  NSS_PIN_CARVEOUT((k_batch_energy<NPL, KIND>));
  k_batch_energy<NPL, KIND><<<(b.max_rows + wpb - 1) / wpb, wpb * 32, smem, lc.stream>>>(r, en, b, parity);
  ++*lc.launch_counter;
}

template <int KIND>
void energy_kind(const RunDev &r, const EnergyDev &en, const BatchDev &b, int parity, const LaunchCtx &lc) {
  switch ((r.d + 31) / 32) {
    case 1: energy_t<1, KIND>(r, en, b, parity, lc); break;
    case 2: energy_t<2, KIND>(r, en, b, parity, lc); break;
    case 3: energy_t<3, KIND>(r, en, b, parity, lc); break;
    default: energy_t<4, KIND>(r, en, b, parity, lc); break;
  }
}

}  // namespace

bool batch_generic_ok(const EnergyDev &en) {
  switch (en.kind) {
    case NSS_E_FLAT: case NSS_E_GAUSS: case NSS_E_MOG: case NSS_E_CORR_GAUSS: case NSS_E_FUNNEL: case NSS_E_LOGREG:
      return true;
    default:
      return false;
  }
}

void batch_begin(const RunDev &r, const PriorDev &pr, const BatchDev &b, const LaunchCtx &lc) {
  switch ((r.d + 31) / 32) {
    case 1: begin_t<1>(r, pr, b, lc); break;
    case 2: begin_t<2>(r, pr, b, lc); break;
    case 3: begin_t<3>(r, pr, b, lc); break;
    default: begin_t<4>(r, pr, b, lc); break;
  }
}

void batch_advance(const RunDev &r, const PriorDev &pr, const BatchDev &b, int parity, const LaunchCtx &lc) {
  // two chains per warp (NSS_ADV_HALF=1): measured slower at C4 (31.1 vs
  // 26.4 ms per iteration: 480 B of spills at NPL = 7 and the two halves'
  // divergent state machines serialise), so one chain per warp by default
  static const bool half = getenv("NSS_ADV_HALF") != nullptr;
  if (r.Vpre && half) {
    switch ((r.d + 15) / 16) {
      case 3: advance_t<3, 16>(r, pr, b, parity, lc); return;
      case 4: advance_t<4, 16>(r, pr, b, parity, lc); return;
      case 5: advance_t<5, 16>(r, pr, b, parity, lc); return;
      case 6: advance_t<6, 16>(r, pr, b, parity, lc); return;
      case 7: advance_t<7, 16>(r, pr, b, parity, lc); return;
      case 8: advance_t<8, 16>(r, pr, b, parity, lc); return;
      default: break;
    }
  }
  switch ((r.d + 31) / 32) {
    case 1: advance_t<1, 32>(r, pr, b, parity, lc); break;
    case 2: advance_t<2, 32>(r, pr, b, parity, lc); break;
    case 3: advance_t<3, 32>(r, pr, b, parity, lc); break;
    default: advance_t<4, 32>(r, pr, b, parity, lc); break;
  }
}

void batch_energy_generic(const RunDev &r, const EnergyDev &en, const BatchDev &b, int parity, const LaunchCtx &lc) {
  switch (en.kind) {
    case NSS_E_FLAT: energy_kind<NSS_E_FLAT>(r, en, b, parity, lc); break;
    case NSS_E_GAUSS: energy_kind<NSS_E_GAUSS>(r, en, b, parity, lc); break;
    case NSS_E_MOG: energy_kind<NSS_E_MOG>(r, en, b, parity, lc); break;
    case NSS_E_CORR_GAUSS: energy_kind<NSS_E_CORR_GAUSS>(r, en, b, parity, lc); break;
    case NSS_E_FUNNEL: energy_kind<NSS_E_FUNNEL>(r, en, b, parity, lc); break;
    case NSS_E_LOGREG: energy_kind<NSS_E_LOGREG>(r, en, b, parity, lc); break;
    default: break;
  }
}

void batch_init_draw(const RunDev &r, const PriorDev &pr, const BatchDev &b, const int *pending, int *map,
                     uint32_t attempt, const LaunchCtx &lc) {
  switch ((r.d + 31) / 32) {
    case 1: binit_draw_t<1>(r, pr, b, pending, map, attempt, lc); break;
    case 2: binit_draw_t<2>(r, pr, b, pending, map, attempt, lc); break;
    case 3: binit_draw_t<3>(r, pr, b, pending, map, attempt, lc); break;
    default: binit_draw_t<4>(r, pr, b, pending, map, attempt, lc); break;
  }
}

void batch_init_accept(const RunDev &r, const BatchDev &b, const int *map, int *pending, int *n_pending,
                       const LaunchCtx &lc) {
  k_binit_accept<<<(r.n + 255) / 256, 256, 0, lc.stream>>>(r, b, map, pending, n_pending);
  ++*lc.launch_counter;
}

void batch_finish(const RunDev &r, const BatchDev &b, const LaunchCtx &lc) {
  NSS_PIN_CARVEOUT(k_batch_finish);
  k_batch_finish<<<chain_blocks(r, 256), 256, 0, lc.stream>>>(r, b);
  ++*lc.launch_counter;
}

}  // namespace nss
