#include <chrono>
// C ABI (include/nss.h) and host orchestration of one NSS run on one GPU.
//
// The host only validates, allocates, uploads the problem once, enqueues the
// per-iteration kernels on one stream and copies results back; every step of
// the method runs on the device.  Iterations after the
// termination criterion is met are no-ops on the device, so nss_run can enqueue
// ahead and poll a small state struct instead of synchronising every iteration.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "batch.cuh"
#include "lr_engine.cuh"
#include "nss_internal.cuh"

// NVTX ranges around the host calls and per-iteration enqueues (SURVEY
// section 5 tracing); header-only, inert unless a profiler attaches.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

#define NSS_API extern "C" __attribute__((visibility("default")))

using namespace nss;

namespace nss {
bool nccl_unique_id(uint8_t out[128]);
bool nccl_comm_init(void **comm, int world, const uint8_t uid[128], int rank, std::string *err);
void nccl_comm_free(void *comm);
bool exchange_chains(const RunDev &r, void *comm, float *buf, float *all, int kc, const LaunchCtx &lc,
                     std::string *err);
void launch_evidence_summary(const RunDev &r, double *out, const LaunchCtx &lc);
void launch_samples(const RunDev &r, long long N, double *logw, double *scratch, int chunk, const LaunchCtx &lc,
                    double beta, double *zacc);
void launch_resample(const RunDev &r, long long N, const double *logw, double *cum, long long m, uint64_t seed,
                     long long *idx, double *x, const LaunchCtx &lc);
// sharded live set (k_shard.cu, k_metric.cu, dist.cu)
bool nccl_allgather_inplace(void *comm, void *buf, size_t bytes, int rank, cudaStream_t stream, std::string *err);
bool ipc_exchange(void *comm, int world, int rank, void *const *mine, int nptr, void **peers,
                  std::vector<void *> *opened, cudaStream_t stream, std::string *err);
size_t shard_block_bytes(int k, int own_max, int world, int d);
size_t shard_metric_offset(int k, int own_max);
void launch_shard_cand(const RunDev &r, char *block, int kc_cap, const LaunchCtx &lc);
void launch_shard_merge(const RunDev &r, const char *gather, size_t block_bytes, int m_max, int *crange,
                        const LaunchCtx &lc);
void launch_shard_dead_rows(const RunDev &r, const LaunchCtx &lc);
void launch_shard_pack_live(const RunDev &r, float *block, const LaunchCtx &lc);
void launch_shard_unpack_live(const RunDev &r, const float *buf, long long rows_cap, const LaunchCtx &lc);
void launch_shard_mask_rows(const RunDev &r, const LaunchCtx &lc);
void launch_metric_shard_partials(const RunDev &r, double *partials, int bps, int seg0, int nseg, double *seg_out,
                                  const LaunchCtx &lc);
void launch_metric_shard_final(const RunDev &r, double metric_reg, int width_rule, double width_param,
                               const double *seg_rows, long long rank_stride, double *sums, unsigned *ticket,
                               const LaunchCtx &lc);
}  // namespace nss

// Ranks of one sharded run emulated in one process on one GPU (nss_group_*):
// the members share one stream and one gather buffer, so an "all-gather" is
// every member writing its block in place, and a member's peer table points
// at the other members' arrays.  Freed with the last member.
struct nss_group {
  int world = 0, alive = 0;
  char *gather = nullptr;
  float *live = nullptr;
  cudaStream_t stream = nullptr;
};

static const int kPhases = 5;

struct nss_ctx {
  nss_config cfg{};
  int d = 0, dp = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  RunDev r{};
  PriorDev pr{};
  EnergyDev en{};
  std::vector<void *> allocs;
  char *arena = nullptr;  // current small-allocation arena (dalloc)
  size_t arena_used = 0;
  double *partials = nullptr;
  unsigned *ticket = nullptr;   // last-block-done counter of k_metric
  cudaStream_t side = nullptr;  // evidence runs here, concurrently with HRSS
  cudaStream_t side2 = nullptr;  // the previous iteration's metric, concurrently with the select
  cudaEvent_t ev_sel = nullptr, ev_evid = nullptr, ev_fork = nullptr, ev_met = nullptr;
  // A5 of iteration i only feeds HRSS of iteration i+1, so it is deferred into
  // the next iteration (overlapping its select) and computed on demand when the
  // host asks for the metric; A9 is evaluated by the select kernel, and on
  // demand (k_term_probe) when the host reads the state.
  bool metric_pending = false;
  bool term_stale = false;
  int bps = 1;  // metric blocks per gid segment (k_metric.cu)
  double *summary = nullptr;  // device: [mean, std, closed lz_0..R]
  void *h_block = nullptr;    // one pinned (host-mapped) allocation for all host mirrors below
  DevState *d_h_st = nullptr;  // device aliases of h_st / h_lz0 (mapped)
  double *d_h_lz0 = nullptr;
  DevState *h_st = nullptr;   // pinned mirror of the device state
  int *h_one = nullptr;       // pinned constant 1 (finalised flag)
  double *h_lz0 = nullptr;    // pinned mirror of replica 0's log Z (step info)
  bool poisoned = false;
  std::string err;
  long long launches = 0;
  bool timing = false;
  bool serial_evidence = false;  // run A8 on the main stream (no overlap)
  struct Timed {
    int phase;  // 0 hrss, 1 select, 2 evidence, 3 metric, 4 batched energy passes (inside 0)
    cudaEvent_t a, b;
  };
  std::vector<cudaEvent_t> ev_free;
  std::vector<Timed> ev_pending;
  double time_ms[kPhases] = {0, 0, 0, 0, 0};
  long long timed[kPhases] = {0, 0, 0, 0, 0};
  int host_finalised = 0;
  // one iteration captured as a CUDA graph (about 1 us per kernel node
  // instead of about 3.4 us per stream launch on B200)
  bool use_graph = true;
  cudaGraphExec_t graph = nullptr, graph0 = nullptr;  // with / without the deferred metric
  long long graph_launches = 0, graph0_launches = 0;
  // `graph` + the termination probe writing the state to the mapped host
  // mirror, for nss_step with info: the host then only synchronises
  cudaGraphExec_t graph_info = nullptr;
  long long graph_info_launches = 0;
  bool probe_in_graph = false;  // the last iteration's graph already ran the probe
  // round-synchronous batch engine (k_batch.cu) and its energy backends
  BatchDev bd{};
  bool batch_alloc = false;
  int batch_backend = 0;  // 1 generic warp-per-probe energy, 2 tensor-core logistic regression, 3 GP
  bool gp_rounds = getenv("NSS_GP_ROUNDS") != nullptr;  // GP: round-synchronous engine instead of the fused chains
  LrEngine lr{};
  bool lr_ok = false;     // logistic-regression data fit the tensor-core path (d <= 128, fp16 range)
  std::vector<double> lr_x, lr_y;
  cudaGraphExec_t round_graph = nullptr;
  long long round_graph_launches = 0;
  // the rounds as a device-side loop: one graph with a WHILE node whose body
  // is two rounds + k_round_cond (no host polling); NSS_HOST_ROUNDS=1 keeps
  // the host-polled chunks
  cudaGraphExec_t loop_graph = nullptr;
  bool host_rounds = getenv("NSS_HOST_ROUNDS") != nullptr;
  int loop_body = getenv("NSS_LOOP_ROUNDS") ? std::max(2, atoi(getenv("NSS_LOOP_ROUNDS")) & ~1) : 16;
  int *h_nprobe = nullptr;  // pinned (inside h_block)
  void *gp = nullptr;       // fp64 batched GP marginal likelihood (k_gp.cu)
  // multi-GPU (dist.cu): chain block [r.c0, r.c1) of kc chains, NCCL all-gather of new rows
  void *comm = nullptr;
  int rank = 0, world = 1, kc = 0;
  float *xbuf = nullptr, *xall = nullptr;
  float *vpre = nullptr;  // k_dirs output (warp engine, d > 32)
  size_t vpre_floats = 0;
  // sharded live set (k_shard.cu): this rank owns segments
  // [seg0, seg0 + nseg) = gids [r.rank_lo[rank], r.rank_lo[rank + 1])
  bool sharded = false;
  nss_group *group = nullptr;  // in-process emulation of the ranks (nss_group_*), else NCCL
  int seg0 = 0, nseg = 0, own_max = 0, kc_cap = 0;
  size_t blk_bytes = 0, met_off = 0;
  char *gather = nullptr;       // world * blk_bytes
  float *live_buf = nullptr;    // world * own_max * (dp + 2): live-set gather
  double *shard_sums = nullptr;
  int *crange = nullptr;
  bool stage_wm = false;        // with-metric flag between the group stages of an iteration
  bool live_gathered = true;    // every rank's rows present locally (init, after a gather)
  std::vector<void *> ipc_open, raw_allocs;
  // F3 tempered SMC-SS (k_smc.cu): particles are the live set
  bool smc = false;
  double smc_rho = 0.9;
  double *smc_cum = nullptr;
  int *smc_par = nullptr;
  float *smc_xs = nullptr, *smc_es = nullptr;
};

static const int kRoundsPerChunk = 32;

namespace {

nss_status fail(nss_ctx *c, nss_status s, const std::string &msg) {
  if (c) c->err = msg;
  return s;
}

nss_status exchange(nss_ctx *c);

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      c->poisoned = true;                                                          \
      return fail(c, NSS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                              \
  } while (0)

// Zeroed device memory owned by the context.  Small requests are carved from
// 16 MB arenas (one cudaMalloc + memset each: nss_init makes dozens of
// allocations), large ones get their own; 256-byte alignment throughout.
// Device memory comes from the device's stream-ordered pool (cudaMallocAsync
// on the context's stream), which keeps freed blocks for the next context
// (release threshold), so nss_init / nss_destroy cycles cost microseconds
// instead of cudaMalloc + synchronous memset per buffer.
void ensure_pool() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> g(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = uint64_t(8) << 30;  // freed blocks kept for reuse, up to 8 GB
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}

// The mapped page-locked 4 KB host mirror of a context: page locking costs
// milliseconds, so destroyed contexts return their block to a process-wide
// free list.
std::mutex g_pinned_mu;
std::vector<void *> g_pinned_free;
void *pinned_block() {
  {
    std::lock_guard<std::mutex> g(g_pinned_mu);
    if (!g_pinned_free.empty()) {
      void *p = g_pinned_free.back();
      g_pinned_free.pop_back();
      memset(p, 0, 4096);
      return p;
    }
  }
  void *p = nullptr;
  if (cudaHostAlloc(&p, 4096, cudaHostAllocMapped) != cudaSuccess) return nullptr;
  memset(p, 0, 4096);
  return p;
}
void pinned_release(void *p) {
  std::lock_guard<std::mutex> g(g_pinned_mu);
  g_pinned_free.push_back(p);
}

template <typename T>
nss_status dalloc(nss_ctx *c, T **p, size_t count) {
  const size_t bytes = (count * sizeof(T) + 16 + 255) & ~size_t(255);
  constexpr size_t kArena = size_t(16) << 20;
  auto get = [&](size_t nb, void **q) -> nss_status {
    cudaError_t e = cudaMallocAsync(q, nb, c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(*q, 0, nb, c->stream);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      return fail(c, NSS_ERR_OOM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    }
    c->allocs.push_back(*q);
    return NSS_OK;
  };
  if (bytes <= kArena / 8) {
    if (!c->arena || c->arena_used + bytes > kArena) {
      void *q = nullptr;
      nss_status s = get(kArena, &q);
      if (s) return s;
      c->arena = static_cast<char *>(q);
      c->arena_used = 0;
    }
    *p = reinterpret_cast<T *>(c->arena + c->arena_used);
    c->arena_used += bytes;
    return NSS_OK;
  }
  void *q = nullptr;
  nss_status s = get(bytes, &q);
  if (s) return s;
  *p = static_cast<T *>(q);
  return NSS_OK;
}

nss_status upload_f32(nss_ctx *c, float **dst, const double *src, size_t count) {
  nss_status s = dalloc(c, dst, count ? count : 1);
  if (s != NSS_OK) return s;
  if (!count || !src) return NSS_OK;
  std::vector<float> tmp(count);
  for (size_t i = 0; i < count; ++i) tmp[i] = static_cast<float>(src[i]);
  // stream-ordered after the allocation; a pageable source is staged before the call returns
  CK(cudaMemcpyAsync(*dst, tmp.data(), count * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  return NSS_OK;
}

bool validate(const nss_prior *p, const nss_energy *e, const nss_config *cfg) {
  if (!p || !e || !cfg) return false;
  const int d = p->d;
  if (d < 1 || d > NSS_MAX_DIM || e->d != d) return false;
  if (cfg->n_live < 2 || cfg->n_live > (1 << 30) || cfg->k < 1 || cfg->k > cfg->n_live - 1) return false;
  if (cfg->steps < 0 || cfg->max_stepout < 1 || cfg->max_shrink < 1 || cfg->max_stepout > 255 ||
      cfg->max_shrink > 255)
    return false;
  if (cfg->n_volume_sims < 2 || !(cfg->width > 0.0) || cfg->max_dead < cfg->n_live) return false;
  if (cfg->update_all != 0 && cfg->update_all != 1) return false;
  if (cfg->mutation != NSS_MUT_HRSS && cfg->mutation != NSS_MUT_RW) return false;
  if (cfg->width_rule != NSS_W_OPTIMAL && cfg->width_rule != NSS_W_FIXED) return false;
  if (cfg->dir_norm != NSS_DIR_MAHALANOBIS && cfg->dir_norm != NSS_DIR_EUCLIDEAN) return false;
  if (cfg->quadrature != NSS_Q_TRAPEZOID && cfg->quadrature != NSS_Q_RECTANGLE) return false;
  if (p->kind == NSS_PRIOR_BOX) {
    if (!p->lo || !p->hi) return false;
    for (int i = 0; i < d; ++i)
      if (!(p->lo[i] < p->hi[i])) return false;
  } else if (p->kind == NSS_PRIOR_GAUSS_DIAG) {
    if (!p->mean || !p->sd) return false;
    for (int i = 0; i < d; ++i)
      if (!(p->sd[i] > 0.0)) return false;
  } else {
    return false;
  }
  switch (e->kind) {
    case NSS_E_FLAT: case NSS_E_FUNNEL: return true;
    case NSS_E_GAUSS: return e->mu && e->sigma;
    case NSS_E_MOG: return e->n_comp >= 1 && e->w && e->mu && e->sigma;
    case NSS_E_CORR_GAUSS: return e->mu && e->prec;
    case NSS_E_LOGREG: return e->n_data >= 1 && e->data_x && e->data_y;
    case NSS_E_GP_ARD: return e->n_data >= 1 && e->d_in >= 1 && d == e->d_in + 2 && e->data_x && e->data_y;
    default: return false;
  }
}

LaunchCtx lctx(nss_ctx *c) { return LaunchCtx{c->stream, &c->launches}; }

nss_status device_error(nss_ctx *c) {
  if (c->h_st->error) {
    int code = c->h_st->error;
    const char *what = code == NSS_ERR_NAN ? "energy returned NaN"
                       : code == NSS_ERR_CAPACITY ? "dead store full"
                       : code == NSS_ERR_PRIOR_SUPPORT ? "no finite energy within 100 n prior draws"
                                                       : "device error";
    return fail(c, static_cast<nss_status>(code), what);
  }
  return NSS_OK;
}

// The device state into the host mirror: one kernel (A9 at the end of the
// last enqueued iteration when stale, R-19) that also writes the state into
// host-mapped pinned memory, then a synchronisation.
nss_status pull_state(nss_ctx *c) {
  LaunchCtx lc{c->stream, &c->launches};
  if (c->probe_in_graph) {  // the iteration's graph ended with the probe
    c->probe_in_graph = false;
    c->term_stale = false;
  } else if (c->d_h_st && c->r.lz) {
    // sharded: the termination test runs in the next merge (global minimum);
    // this rank's E holds only its own rows
    launch_term_probe(c->r, lc, (c->term_stale && !c->sharded) ? 1 : 0, c->d_h_st, c->d_h_lz0);
    c->term_stale = false;
    CK(cudaGetLastError());
  } else {
    if (c->term_stale) {
      launch_term_probe(c->r, lc);
      c->term_stale = false;
    }
    CK(cudaMemcpyAsync(c->h_st, c->r.st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
    if (c->r.lz) CK(cudaMemcpyAsync(c->h_lz0, c->r.lz, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  return NSS_OK;
}

void fill_info(nss_ctx *c, nss_step_info *info) {
  const DevState &s = *c->h_st;
  info->iteration = s.iter;
  info->e_star = s.e_star;
  info->probes = static_cast<int64_t>(s.probes);
  info->energy_evals = static_cast<int64_t>(s.evals);
  info->expansions = static_cast<int64_t>(s.expansions);
  info->shrinks = static_cast<int64_t>(s.shrinks);
  info->null_moves = static_cast<int64_t>(s.nulls);
  info->init_evals = static_cast<int64_t>(s.init_evals);
  info->log_z_live = s.log_z_live;
  info->terminated = s.terminated;
  info->finalised = s.finalised;
  info->log_z_det = *c->h_lz0;  // copied with the state by pull_state
}

nss_status collect_timing(nss_ctx *c) {
  for (const auto &t : c->ev_pending) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, t.a, t.b));
    c->time_ms[t.phase] += ms;
    c->timed[t.phase] += 1;
    c->ev_free.push_back(t.a);
    c->ev_free.push_back(t.b);
  }
  c->ev_pending.clear();
  return NSS_OK;
}

cudaEvent_t take_event(nss_ctx *c) {
  if (c->ev_free.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = c->ev_free.back();
  c->ev_free.pop_back();
  return e;
}

// Runs `launch` on `stream`, bracketed by timing events in timing mode.
template <class F>
nss_status timed_launch(nss_ctx *c, int phase, cudaStream_t stream, F &&launch) {
  if (!c->timing) {
    launch();
    return NSS_OK;
  }
  cudaEvent_t a = take_event(c), b = take_event(c);
  CK(cudaEventRecord(a, stream));
  launch();
  CK(cudaEventRecord(b, stream));
  c->ev_pending.push_back({phase, a, b});
  return NSS_OK;
}

nss_status launch_metric_on(nss_ctx *c, cudaStream_t stream, int end_of_iter) {
  LaunchCtx l{stream, &c->launches};
  return timed_launch(c, 3, stream, [&] {
    launch_metric(c->r, c->cfg.metric_reg, c->cfg.width_rule, c->cfg.width, end_of_iter, c->partials, c->ticket,
                  c->bps, l);
  });
}

// Stages of a sharded iteration: kPre (rank-local
// candidates and moment sums into this rank's block), the all-gather, kPost
// (replicated metric + merge, then this rank's chains).  A one-process context
// runs kAll; the in-process group drives kPre on every member, then kPost.
enum Stage { kAll = 0, kPre = 1, kPost = 2 };

nss_status shard_pre(nss_ctx *c, bool with_metric) {
  LaunchCtx lc = lctx(c);
  char *mine = c->gather + static_cast<size_t>(c->r.rank) * c->blk_bytes;
  if (with_metric)
    launch_metric_shard_partials(c->r, c->partials, c->bps, c->seg0, c->nseg,
                                 reinterpret_cast<double *>(mine + c->met_off), lc);
  launch_shard_cand(c->r, mine, c->kc_cap, lc);
  CK(cudaGetLastError());
  return NSS_OK;
}

nss_status shard_exchange(nss_ctx *c) {
  if (c->group) return NSS_OK;  // members wrote their blocks into the shared buffer
  std::string err;
  if (!nccl_allgather_inplace(c->comm, c->gather, c->blk_bytes, c->r.rank, c->stream, &err)) {
    c->poisoned = true;
    return fail(c, NSS_ERR_COMM, err);
  }
  return NSS_OK;
}

// Replicated part of a sharded iteration's select phase: metric (fork) and
// merge, then this rank's dead rows; returns with the metric joined.
nss_status shard_post_select(nss_ctx *c, bool with_metric) {
  LaunchCtx lc = lctx(c);
  nss_status s;
  if (with_metric) {
    CK(cudaEventRecord(c->ev_fork, c->stream));
    CK(cudaStreamWaitEvent(c->side2, c->ev_fork, 0));
    LaunchCtx l2{c->side2, &c->launches};
    if ((s = timed_launch(c, 3, c->side2, [&] {
           launch_metric_shard_final(c->r, c->cfg.metric_reg, c->cfg.width_rule, c->cfg.width,
                                     reinterpret_cast<const double *>(c->gather + c->met_off),
                                     static_cast<long long>(c->blk_bytes / 8), c->shard_sums, c->ticket, l2);
         })))
      return s;
    CK(cudaEventRecord(c->ev_met, c->side2));
  }
  if ((s = timed_launch(c, 1, c->stream, [&] {
         launch_shard_merge(c->r, c->gather, c->blk_bytes, c->r.world * c->kc_cap, c->crange, lc);
         launch_shard_dead_rows(c->r, lc);
       })))
    return s;
  if (with_metric) CK(cudaStreamWaitEvent(c->stream, c->ev_met, 0));
  return NSS_OK;
}

// One iteration: [deferred A5 of the previous iteration || A2-A4 select] ->
// [A8 evidence on the side stream || A6 HRSS] (-> multi-GPU exchange).
nss_status enqueue_iteration_eager(nss_ctx *c, bool with_metric, Stage stage = kAll) {
  LaunchCtx lc = lctx(c);
  nss_status s;
  if (c->sharded) {
    if (stage != kPost && (s = shard_pre(c, with_metric))) return s;
    if (stage == kPre) return NSS_OK;
    if (stage == kAll && (s = shard_exchange(c))) return s;
    if ((s = shard_post_select(c, with_metric))) return s;
    with_metric = false;  // joined above
  } else if (with_metric) {
    if (c->serial_evidence) {
      if ((s = launch_metric_on(c, c->stream, 1))) return s;
    } else {
      CK(cudaEventRecord(c->ev_fork, c->stream));
      CK(cudaStreamWaitEvent(c->side2, c->ev_fork, 0));
      if ((s = launch_metric_on(c, c->side2, 1))) return s;
      CK(cudaEventRecord(c->ev_met, c->side2));
    }
  }
  if (!c->sharded && (s = timed_launch(c, 1, c->stream, [&] {
                        launch_select(c->r, lc);
                        if (c->cfg.update_all)
                          launch_chains_all(c->r, c->r.cdest, c->r.cpar, const_cast<float *>(c->r.Xs),
                                            const_cast<float *>(c->r.Es), lc);
                      })))
    return s;
  if (c->serial_evidence) {
    if ((s = timed_launch(c, 2, c->stream, [&] { launch_evidence(c->r, 0, lc); }))) return s;
  } else {
    // A8 only needs this iteration's dead records: fork it onto the side
    // stream so it overlaps HRSS; joined at the end of the iteration.
    CK(cudaEventRecord(c->ev_sel, c->stream));
    CK(cudaStreamWaitEvent(c->side, c->ev_sel, 0));
    LaunchCtx ls{c->side, &c->launches};
    if ((s = timed_launch(c, 2, c->side, [&] { launch_evidence(c->r, 0, ls); }))) return s;
    CK(cudaEventRecord(c->ev_evid, c->side));
  }
  if (with_metric && !c->serial_evidence) CK(cudaStreamWaitEvent(c->stream, c->ev_met, 0));
  if ((s = timed_launch(c, 0, c->stream, [&] { launch_hrss(c->r, c->pr, c->en, lc); }))) return s;
  if ((s = exchange(c))) return s;
  if (!c->serial_evidence) CK(cudaStreamWaitEvent(c->stream, c->ev_evid, 0));
  CK(cudaGetLastError());
  return NSS_OK;
}

// Multi-GPU: every rank's new chain rows to every rank.
nss_status exchange(nss_ctx *c) {
  if (!c->comm || c->sharded) return NSS_OK;
  std::string err;
  if (!exchange_chains(c->r, c->comm, c->xbuf, c->xall, c->kc, lctx(c), &err)) {
    c->poisoned = true;
    return fail(c, NSS_ERR_CUDA, err);
  }
  return NSS_OK;
}

// 0 warp, 1 lane, 2 batch
int resolve_engine(const nss_ctx *c) {
  const int want = c->r.engine;
  if (c->smc) return 0;  // F3: tempered HRSS on the warp engine
  if (c->r.mutation == NSS_MUT_RW) return 0;  // F1: warp-per-chain random walk (launch_hrss)
  if (c->en.kind == NSS_E_GP_ARD) return 2;  // no per-warp GP energy
  const bool expensive = c->en.kind == NSS_E_LOGREG && c->lr_ok;
  if (want == NSS_ENGINE_BATCH) return 2;
  if (want == NSS_ENGINE_AUTO && expensive) return 2;
  return hrss_engine(c->r, c->en);
}

nss_status ensure_batch(nss_ctx *c) {
  const int backend = c->en.kind == NSS_E_GP_ARD ? 3 : (c->en.kind == NSS_E_LOGREG && c->lr_ok) ? 2 : 1;
  if (c->batch_alloc && c->batch_backend == backend) return NSS_OK;
  if (backend == 1 && !batch_generic_ok(c->en)) return fail(c, NSS_ERR_UNSUPPORTED, "no batched energy for this kind");
  BatchDev &b = c->bd;
  const int k = c->r.nch;  // chains per iteration
  if (!c->batch_alloc) {
    b.k = k;
    b.dp = c->dp;
    b.max_rows = backend >= 2 ? std::max(2 * k, c->r.n) : 2 * k;  // GP / LR also draw the n initial points
    nss_status s;
    if ((s = dalloc(c, &b.cs, static_cast<size_t>(k) * kChainWords))) return s;  // one 128-B record per chain
    if ((s = dalloc(c, &b.x, static_cast<size_t>(k) * c->dp))) return s;
    if ((s = dalloc(c, &b.v, static_cast<size_t>(k) * c->dp))) return s;
    for (int q = 0; q < 2; ++q)
      if ((s = dalloc(c, &b.P[q], static_cast<size_t>(b.max_rows) * c->dp))) return s;
    if ((s = dalloc(c, &b.n_probe, 2))) return s;
    // c->h_nprobe lives in the pinned block allocated by nss_init
    c->batch_alloc = true;
  }
  if (backend == 2) {
    if (!c->lr.Xb) {
      if (lr_setup(c->lr, c->lr_x.data(), c->lr_y.data(), c->en.n_data, c->d, b.max_rows) != cudaSuccess)
        return fail(c, NSS_ERR_CUDA, "tensor-core logistic-regression setup failed");
    }
    b.n_splits = 1;
    b.p_stride = c->lr.p_stride;
    b.slices = nullptr;
    for (int q = 0; q < 2; ++q) {
      nss_status s;  // float energies of the batched init draws (k_binit_accept)
      if (!b.partial[q] && (s = dalloc(c, &b.partial[q], static_cast<size_t>(b.max_rows)))) return s;
      b.A[q] = c->lr.A[q];
      b.lin[q] = c->lr.lin[q];
      b.eacc[q] = c->lr.eacc[q];
    }
    b.g = c->lr.g;
  } else {
    b.n_splits = 1;
    b.p_stride = b.max_rows;
    {
      nss_status s;
      if ((s = dalloc(c, &b.slices, 2))) return s;
      const int ones[2] = {1, 1};
      CK(cudaMemcpyAsync(b.slices, ones, sizeof(ones), cudaMemcpyHostToDevice, c->stream));
    }
    for (int q = 0; q < 2; ++q) {
      nss_status s;
      if ((s = dalloc(c, &b.partial[q], static_cast<size_t>(b.max_rows)))) return s;
      b.A[q] = nullptr;
      b.lin[q] = nullptr;
      b.eacc[q] = nullptr;
    }
    b.g = nullptr;
  }
  c->batch_backend = backend;
  return NSS_OK;
}

void enqueue_rounds(nss_ctx *c, int count) {
  LaunchCtx lc = lctx(c);
  for (int i = 0; i < count; ++i) {
    const int par = i & 1;
    batch_advance(c->r, c->pr, c->bd, par, lc);
    auto energy = [&] {
      if (c->batch_backend == 2)
        lr_energy_pass(c->lr, par, c->bd.n_probe + par, c->bd.n_probe + (par ^ 1), lc);
      else if (c->batch_backend == 3)
        gp_energy_pass(c->gp, c->bd, par, lc);
      else
        batch_energy_generic(c->r, c->en, c->bd, par, lc);
    };
    if (c->timing)
      (void)timed_launch(c, 4, c->stream, energy);  // per-launch energy timing (nss_phase_times)
    else
      energy();
  }
}

void drop_graph(nss_ctx *c) {
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  if (c->graph0) {
    cudaGraphExecDestroy(c->graph0);
    c->graph0 = nullptr;
  }
  if (c->round_graph) {
    cudaGraphExecDestroy(c->round_graph);
    c->round_graph = nullptr;
  }
  if (c->graph_info) {
    cudaGraphExecDestroy(c->graph_info);
    c->graph_info = nullptr;
  }
  if (c->loop_graph) {
    cudaGraphExecDestroy(c->loop_graph);
    c->loop_graph = nullptr;
  }
}

// One iteration with the batch engine: the HRSS part is a data-dependent
// number of rounds, replayed in chunks from a captured graph; the host polls
// the last round's probe count after each chunk (zero: every chain is done).
nss_status enqueue_iteration_batch(nss_ctx *c, Stage stage = kAll) {
  nss_status s;
  if ((s = ensure_batch(c))) return s;
  LaunchCtx lc = lctx(c);
  if (c->sharded) {
    if (stage != kPost && (s = shard_pre(c, c->metric_pending))) return s;
    if (stage == kPre) return NSS_OK;
    if (stage == kAll && (s = shard_exchange(c))) return s;
    if ((s = shard_post_select(c, c->metric_pending))) return s;
  }
  // the metric of the live set beside the select (as in the per-probe
  // engines): neither reads what the other writes; joined before the rounds
  const bool fork_met = !c->sharded && c->metric_pending && !c->serial_evidence;
  if (!c->sharded) {
    if (fork_met) {
      CK(cudaEventRecord(c->ev_fork, c->stream));
      CK(cudaStreamWaitEvent(c->side2, c->ev_fork, 0));
      if ((s = launch_metric_on(c, c->side2, 1))) return s;
      CK(cudaEventRecord(c->ev_met, c->side2));
    } else if (c->metric_pending && (s = launch_metric_on(c, c->stream, 1))) {
      return s;
    }
    if ((s = timed_launch(c, 1, c->stream, [&] {
           launch_select(c->r, lc);
           if (c->cfg.update_all) launch_chains_all(c->r, c->r.cdest, c->r.cpar, const_cast<float *>(c->r.Xs),
                                                    const_cast<float *>(c->r.Es), lc);
         })))
      return s;
  }
  CK(cudaEventRecord(c->ev_sel, c->stream));
  CK(cudaStreamWaitEvent(c->side, c->ev_sel, 0));
  LaunchCtx ls{c->side, &c->launches};
  if ((s = timed_launch(c, 2, c->side, [&] { launch_evidence(c->r, 0, ls); }))) return s;
  CK(cudaEventRecord(c->ev_evid, c->side));
  if (fork_met) CK(cudaStreamWaitEvent(c->stream, c->ev_met, 0));
  auto rounds = [&]() -> nss_status {
    launch_dirs(c->r, lc);  // large d: every direction of the iteration up front
    batch_begin(c->r, c->pr, c->bd, lc);
    if (c->batch_backend == 3 && !c->gp_rounds) {  // fused chains: one launch, no host polling
      bool ok = true;
      const nss_status st = timed_launch(c, 4, c->stream, [&] { ok = gp_chains_pass(c->gp, c->r, c->pr, c->bd, lc); });
      if (st) return st;
      if (!ok) return fail(c, NSS_ERR_OOM, "GP chain buffers");
      batch_finish(c->r, c->bd, lc);
      return NSS_OK;
    }
    const long long max_rounds =
        static_cast<long long>(c->r.p) * (c->r.max_stepout + 2 + c->r.max_shrink) + kRoundsPerChunk;
    if (c->use_graph && !c->timing && !c->host_rounds) {
      // device-side loop: a WHILE node repeating {2 rounds, k_round_cond}
      if (!c->loop_graph) {
        const long long before = c->launches;
        cudaGraph_t g = nullptr;
        CK(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams np{};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, g, nullptr, 0, &np));
        cudaGraph_t body = np.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        enqueue_rounds(c, c->loop_body);  // rounds past the last probe are no-ops
        const int per_body = static_cast<int>(c->launches - before) + 1;
        launch_round_cond(h, c->bd, c->r, per_body, static_cast<int>(max_rounds), lc);
        const cudaError_t e = cudaStreamEndCapture(c->stream, &body);
        if (e != cudaSuccess) {
          cudaGraphDestroy(g);
          c->poisoned = true;
          return fail(c, NSS_ERR_CUDA, std::string("round loop capture: ") + cudaGetErrorString(e));
        }
        const cudaError_t e2 = cudaGraphInstantiate(&c->loop_graph, g, 0);
        cudaGraphDestroy(g);
        if (e2 != cudaSuccess) {
          c->poisoned = true;
          return fail(c, NSS_ERR_CUDA, std::string("round loop graph: ") + cudaGetErrorString(e2));
        }
        c->launches = before;  // counted on the device (DevState::dev_launches)
      }
      CK(cudaGraphLaunch(c->loop_graph, c->stream));
      batch_finish(c->r, c->bd, lc);
      return NSS_OK;
    }
    for (long long done = 0; done < max_rounds; done += kRoundsPerChunk) {
      if (c->use_graph && !c->timing) {
        if (!c->round_graph) {
          const long long before = c->launches;
          cudaGraph_t g = nullptr;
          CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
          enqueue_rounds(c, kRoundsPerChunk);
          const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
          if (e != cudaSuccess) {
            c->poisoned = true;
            return fail(c, NSS_ERR_CUDA, std::string("round graph capture: ") + cudaGetErrorString(e));
          }
          const cudaError_t e2 = cudaGraphInstantiate(&c->round_graph, g, 0);
          cudaGraphDestroy(g);
          if (e2 != cudaSuccess) {
            c->poisoned = true;
            return fail(c, NSS_ERR_CUDA, std::string("round graph: ") + cudaGetErrorString(e2));
          }
          c->round_graph_launches = c->launches - before;
          c->launches = before;
        }
        CK(cudaGraphLaunch(c->round_graph, c->stream));
        c->launches += c->round_graph_launches;
      } else {
        enqueue_rounds(c, kRoundsPerChunk);
      }
      CK(cudaMemcpyAsync(c->h_nprobe, c->bd.n_probe + ((kRoundsPerChunk - 1) & 1), sizeof(int),
                         cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (*c->h_nprobe == 0) break;
    }
    batch_finish(c->r, c->bd, lc);
    return NSS_OK;
  };
  if (c->timing) {
    cudaEvent_t a = take_event(c), b = take_event(c);
    CK(cudaEventRecord(a, c->stream));
    if ((s = rounds())) return s;
    CK(cudaEventRecord(b, c->stream));
    c->ev_pending.push_back({0, a, b});
  } else if ((s = rounds())) {
    return s;
  }
  if ((s = exchange(c))) return s;
  CK(cudaStreamWaitEvent(c->stream, c->ev_evid, 0));
  CK(cudaGetLastError());
  return NSS_OK;
}

// One outer iteration: replayed from a captured graph, or launched eagerly in
// timing mode (events bracket each kernel) or when graphs are disabled.
// Warp engine at large d: room for every (chain, step) direction of an
// iteration, precomputed by k_dirs (allocated once, before any graph capture).
nss_status ensure_vpre(nss_ctx *c) {
  RunDev &r = c->r;
  const int eng = resolve_engine(c);
  const bool want = r.d > 32 && r.mutation == NSS_MUT_HRSS &&
                    ((eng == 0 && hrss_engine(r, c->en) == 0) || eng == 2);
  const size_t need = static_cast<size_t>(r.c1 - r.c0) * (r.p > 0 ? r.p : 1) * c->dp;
  if (!want || need == 0 || need * sizeof(float) > (1ull << 30)) {
    r.Vpre = nullptr;
    return NSS_OK;
  }
  if (!c->vpre || c->vpre_floats < need) {
    nss_status s;
    if ((s = dalloc(c, &c->vpre, need))) return s;
    c->vpre_floats = need;
  }
  r.Vpre = c->vpre;
  return NSS_OK;
}

nss_status enqueue_iteration(nss_ctx *c, bool with_probe = false, Stage stage = kAll) {
  NvtxRange nvtx_(stage == kPre ? "iteration (pre)" : stage == kPost ? "iteration (post)" : "iteration");
  nss_status vs = ensure_vpre(c);
  if (vs) return vs;
  // group stages: kPre records the with-metric flag, kPost reuses it
  const bool wm = stage == kPost ? c->stage_wm : c->metric_pending;
  c->stage_wm = wm;
  if (stage == kPre) {
    c->metric_pending = wm;
  } else {
    c->term_stale = true;
    c->metric_pending = true;
    c->live_gathered = !c->sharded;
  }
  c->probe_in_graph = false;
  if (resolve_engine(c) == 2) {
    c->metric_pending = wm;  // the batch path launches the deferred metric itself
    const nss_status s = enqueue_iteration_batch(c, stage);
    c->metric_pending = stage == kPre ? wm : true;
    return s;
  }
  if (c->timing || !c->use_graph || stage != kAll) return enqueue_iteration_eager(c, wm, stage);
  const bool probe = with_probe && wm && c->d_h_st && c->r.lz;
  cudaGraphExec_t &g = probe ? c->graph_info : wm ? c->graph : c->graph0;
  long long &gl = probe ? c->graph_info_launches : wm ? c->graph_launches : c->graph0_launches;
  if (!g) {
    const long long before = c->launches;
    cudaGraph_t cg = nullptr;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    nss_status s = enqueue_iteration_eager(c, wm);
    if (s == NSS_OK && probe) launch_term_probe(c->r, lctx(c), 1, c->d_h_st, c->d_h_lz0);
    const cudaError_t e = cudaStreamEndCapture(c->stream, &cg);
    if (s != NSS_OK) return s;
    if (e != cudaSuccess) {
      c->poisoned = true;
      return fail(c, NSS_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    }
    const cudaError_t e2 = cudaGraphInstantiate(&g, cg, 0);
    cudaGraphDestroy(cg);
    if (e2 != cudaSuccess) {
      c->poisoned = true;
      return fail(c, NSS_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e2));
    }
    gl = c->launches - before;
    c->launches = before;
  }
  CK(cudaGraphLaunch(g, c->stream));
  c->launches += gl;
  c->probe_in_graph = probe;
  return NSS_OK;
}

// R-20 for energies with a batched implementation (GP, tensor-core LR): every attempt draws
// the still-pending live points into the probe buffer, one energy pass
// evaluates them, and the accept pass keeps the finite ones.
nss_status init_batched(nss_ctx *c) {
  nss_status s;
  if ((s = ensure_batch(c))) return s;
  int *pending = nullptr, *map = nullptr, *npend = nullptr;
  if ((s = dalloc(c, &pending, c->r.n))) return s;
  if ((s = dalloc(c, &map, c->r.n))) return s;
  if ((s = dalloc(c, &npend, 1))) return s;
  std::vector<int> ones(c->r.n, 1);
  CK(cudaMemcpyAsync(pending, ones.data(), ones.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  LaunchCtx lc = lctx(c);
  for (uint32_t a = 0;; ++a) {
    CK(cudaMemsetAsync(c->bd.n_probe, 0, 2 * sizeof(int), c->stream));
    CK(cudaMemsetAsync(npend, 0, sizeof(int), c->stream));
    batch_init_draw(c->r, c->pr, c->bd, pending, map, a, lc);
    if (c->batch_backend == 3)
      gp_energy_pass(c->gp, c->bd, 0, lc);
    else  // tensor-core logistic regression: energies written in place over slice 0 of the partials
      lr_energies(c->lr, c->bd.P[0], c->dp, c->bd.n_probe, c->bd.partial[0], lc);
    batch_init_accept(c->r, c->bd, map, pending, npend, lc);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(c->h_nprobe, npend, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if ((s = pull_state(c))) return s;  // synchronises the stream
    if (c->h_st->error || *c->h_nprobe == 0) break;
  }
  CK(cudaMemsetAsync(c->bd.n_probe, 0, 2 * sizeof(int), c->stream));
  return NSS_OK;
}

nss_status check_usable(nss_ctx *c) {
  if (!c) return NSS_ERR_INVALID_ARG;
  if (c->poisoned) return fail(c, NSS_ERR_CUDA, "context poisoned by an earlier CUDA failure");
  return NSS_OK;
}

}  // namespace

NSS_API nss_status nss_get_unique_id(uint8_t out[128]) {
  if (!out) return NSS_ERR_INVALID_ARG;
  std::memset(out, 0, 128);
  return nccl_unique_id(out) ? NSS_OK : NSS_ERR_UNSUPPORTED;
}

// nss_init and its variants: smc_mode keeps the replicated multi-GPU layout
// (F3); `group` != null builds rank `dist->rank` of an in-process group.
static nss_status init_impl(const nss_prior *prior, const nss_energy *energy, const nss_config *cfg,
                            const nss_dist *dist, bool smc_mode, nss_group *group, nss_ctx **out) {
  if (!out) return NSS_ERR_INVALID_ARG;
  *out = nullptr;
  if (!validate(prior, energy, cfg)) return NSS_ERR_INVALID_ARG;
  if (dist && (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world ||
               (dist->world > 1 && !dist->nccl_uid && !group)))
    return NSS_ERR_INVALID_ARG;
  // sharded live set: NS over several ranks (or an in-process group)
  const bool sharded = !smc_mode && dist && (dist->world > 1 || dist->nccl_uid || group);
  if (sharded) {
    if (kSegs % dist->world != 0) return NSS_ERR_INVALID_ARG;  // world in {1, 2, 4, 8}
    if (cfg->update_all) return NSS_ERR_UNSUPPORTED;
  }
  nss_ctx *c = new nss_ctx();
  c->sharded = sharded;
  c->group = group;
  // measurement hook (NSS_INIT_PROF): host wall time of the phases of nss_init
  const bool iprof = getenv("NSS_INIT_PROF") != nullptr;
  auto it0 = std::chrono::steady_clock::now();
  auto ip = [&](const char *what) {
    if (!iprof) return;
    cudaDeviceSynchronize();
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "nss_init %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - it0).count());
    it0 = t;
  };
  c->cfg = *cfg;
  const int d = prior->d;
  c->d = d;
  c->dp = (d + 3) & ~3;
  const long long n = cfg->n_live, k = cfg->k;
  const int R = cfg->n_volume_sims;
  auto bail = [&](nss_status s) {
    nss_destroy(c);
    return s;
  };
  if (dist && dist->cuda_stream) {
    c->stream = static_cast<cudaStream_t>(dist->cuda_stream);
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(NSS_ERR_CUDA);
    c->own_stream = true;
  }
  // one page-locked block for the host mirrors (page locking is slow: one call)
  ensure_pool();
  if (!(c->h_block = pinned_block())) return bail(NSS_ERR_CUDA);
  {
    char *hb = static_cast<char *>(c->h_block);
    c->h_st = reinterpret_cast<DevState *>(hb);
    c->h_lz0 = reinterpret_cast<double *>(hb + ((sizeof(DevState) + 63) & ~size_t(63)));
    c->h_one = reinterpret_cast<int *>(reinterpret_cast<char *>(c->h_lz0) + 64);
    c->h_nprobe = c->h_one + 16;
    void *dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, c->h_block, 0) == cudaSuccess) {
      c->d_h_st = static_cast<DevState *>(dp);
      c->d_h_lz0 = reinterpret_cast<double *>(static_cast<char *>(dp) + (reinterpret_cast<char *>(c->h_lz0) -
                                                                         static_cast<char *>(c->h_block)));
    }
  }
  *c->h_lz0 = -INFINITY;
  ip("pinned");
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess) return bail(NSS_ERR_CUDA);
  if (cudaEventCreateWithFlags(&c->ev_sel, cudaEventDisableTiming) != cudaSuccess) return bail(NSS_ERR_CUDA);
  if (cudaEventCreateWithFlags(&c->ev_evid, cudaEventDisableTiming) != cudaSuccess) return bail(NSS_ERR_CUDA);
  if (cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess) return bail(NSS_ERR_CUDA);
  if (cudaEventCreateWithFlags(&c->ev_met, cudaEventDisableTiming) != cudaSuccess) return bail(NSS_ERR_CUDA);
  if (cudaStreamCreateWithFlags(&c->side2, cudaStreamNonBlocking) != cudaSuccess) return bail(NSS_ERR_CUDA);
  *c->h_one = 1;

  // ---- energy parameters (fp64 host -> fp32 device) ----
  EnergyDev &en = c->en;
  en.kind = energy->kind;
  en.d = d;
  en.n_comp = energy->n_comp;
  en.d_in = energy->d_in;
  en.n_data = energy->n_data;
  en.c = static_cast<float>(energy->c);
  en.sigma_y = static_cast<float>(energy->sigma_y);
  en.jitter = static_cast<float>(energy->jitter);
  if ((en.kind == NSS_E_GP_ARD && cfg->mutation == NSS_MUT_RW) ||
      (en.kind != NSS_E_GP_ARD && !energy_supported(en))) {
    nss_destroy(c);
    return NSS_ERR_UNSUPPORTED;
  }
  nss_status s = NSS_OK;
  float *tmp = nullptr;
  if (en.kind == NSS_E_GAUSS) {
    std::vector<double> is(d);
    for (int i = 0; i < d; ++i) is[i] = 1.0 / energy->sigma[i];
    if ((s = upload_f32(c, &tmp, energy->mu, d))) return bail(s);
    en.mu = tmp;
    if ((s = upload_f32(c, &tmp, is.data(), d))) return bail(s);
    en.isig = tmp;
  } else if (en.kind == NSS_E_MOG) {
    const int K = en.n_comp;
    std::vector<double> is(static_cast<size_t>(K) * d), lc(K);
    for (int j = 0; j < K; ++j) {
      double acc = std::log(energy->w[j]) - 0.5 * d * std::log(2.0 * M_PI);
      for (int i = 0; i < d; ++i) {
        is[j * d + i] = 1.0 / energy->sigma[j * d + i];
        acc -= std::log(energy->sigma[j * d + i]);
      }
      lc[j] = acc;
    }
    if ((s = upload_f32(c, &tmp, energy->mu, static_cast<size_t>(K) * d))) return bail(s);
    en.mu = tmp;
    if ((s = upload_f32(c, &tmp, is.data(), is.size()))) return bail(s);
    en.isig = tmp;
    if ((s = upload_f32(c, &tmp, lc.data(), K))) return bail(s);
    en.logc = tmp;
  } else if (en.kind == NSS_E_CORR_GAUSS) {
    if ((s = upload_f32(c, &tmp, energy->mu, d))) return bail(s);
    en.mu = tmp;
    if ((s = upload_f32(c, &tmp, energy->prec, static_cast<size_t>(d) * d))) return bail(s);
    en.prec = tmp;
    // P = L L^T in fp64 (host); U = L^T lets the warp energy form |U r|^2
    // with half the multiply-adds of r^T P r (same value up to rounding)
    std::vector<double> Lc(static_cast<size_t>(d) * d, 0.0);
    bool pd = true;
    for (int j = 0; j < d && pd; ++j) {
      double s2 = energy->prec[j * d + j];
      for (int q = 0; q < j; ++q) s2 -= Lc[j * d + q] * Lc[j * d + q];
      if (!(s2 > 0.0)) { pd = false; break; }
      Lc[j * d + j] = std::sqrt(s2);
      for (int i = j + 1; i < d; ++i) {
        double t = energy->prec[i * d + j];
        for (int q = 0; q < j; ++q) t -= Lc[i * d + q] * Lc[j * d + q];
        Lc[i * d + j] = t / Lc[j * d + j];
      }
    }
    if (pd) {
      std::vector<double> U(static_cast<size_t>(d) * d, 0.0);
      for (int i = 0; i < d; ++i)
        for (int m = i; m < d; ++m) U[i * d + m] = Lc[m * d + i];
      if ((s = upload_f32(c, &tmp, U.data(), U.size()))) return bail(s);
      en.ufac = tmp;
    }
  } else if (en.kind == NSS_E_LOGREG) {
    const size_t nx = static_cast<size_t>(energy->n_data) * d;
    bool exact = true;
    c->lr_ok = lr_data_ok(energy->data_x, static_cast<long long>(nx), d, &exact);
    if (c->lr_ok) {
      c->lr_x.assign(energy->data_x, energy->data_x + nx);
      c->lr_y.assign(energy->data_y, energy->data_y + energy->n_data);
    }
    if ((s = upload_f32(c, &tmp, energy->data_x, nx))) return bail(s);
    en.data_x = tmp;
    if ((s = upload_f32(c, &tmp, energy->data_y, energy->n_data))) return bail(s);
    en.data_y = tmp;
  } else if (en.kind == NSS_E_GP_ARD) {
    if (!gp_setup(&c->gp, energy->data_x, energy->data_y, static_cast<int>(energy->n_data), energy->d_in,
                  energy->jitter))
      return bail(c->gp ? NSS_ERR_UNSUPPORTED : NSS_ERR_OOM);
  }

  // ---- prior ----
  PriorDev &pr = c->pr;
  pr.kind = prior->kind;
  if (pr.kind == NSS_PRIOR_BOX) {
    double ln = 0.0;
    for (int i = 0; i < d; ++i) ln -= std::log(prior->hi[i] - prior->lo[i]);
    pr.log_norm = static_cast<float>(ln);
    if ((s = upload_f32(c, &tmp, prior->lo, d))) return bail(s);
    pr.lo = tmp;
    if ((s = upload_f32(c, &tmp, prior->hi, d))) return bail(s);
    pr.hi = tmp;
  } else {
    std::vector<double> is(d);
    double ln = -0.5 * d * std::log(2.0 * M_PI);
    for (int i = 0; i < d; ++i) {
      is[i] = 1.0 / prior->sd[i];
      ln -= std::log(prior->sd[i]);
    }
    pr.log_norm = static_cast<float>(ln);
    if ((s = upload_f32(c, &tmp, prior->mean, d))) return bail(s);
    pr.mean = tmp;
    if ((s = upload_f32(c, &tmp, is.data(), d))) return bail(s);
    pr.isd = tmp;
    if ((s = upload_f32(c, &tmp, prior->sd, d))) return bail(s);
    pr.sd = tmp;
  }

  // ---- padded tables of the one-probe-per-lane engine (k_hrss_lane.cu) ----
  {
    const int K = (en.kind == NSS_E_MOG) ? en.n_comp : 1;
    std::vector<double> ab(static_cast<size_t>(K) * 64, 0.0), pab(64, 0.0);
    if (en.kind == NSS_E_MOG || en.kind == NSS_E_GAUSS) {
      for (int j = 0; j < K; ++j)
        for (int i = 0; i < d && i < 32; ++i) {
          const double is = 1.0 / energy->sigma[j * d + i];
          ab[j * 64 + i] = is;
          ab[j * 64 + 32 + i] = -energy->mu[j * d + i] * is;
        }
    }
    for (int i = 0; i < 32; ++i) {
      if (pr.kind == NSS_PRIOR_BOX) {
        pab[i] = i < d ? prior->lo[i] : -INFINITY;
        pab[32 + i] = i < d ? prior->hi[i] : INFINITY;
      } else {
        pab[i] = i < d ? prior->mean[i] : 0.0;
        pab[32 + i] = i < d ? 1.0 / prior->sd[i] : 0.0;
      }
    }
    if ((s = upload_f32(c, &tmp, ab.data(), ab.size()))) return bail(s);
    en.lane_ab = tmp;
    if ((s = upload_f32(c, &tmp, pab.data(), pab.size()))) return bail(s);
    pr.lane_pab = tmp;
  }

  // ---- live set, dead store, scratch ----
  RunDev &r = c->r;
  r.n = static_cast<int>(n);
  r.k = static_cast<int>(k);
  r.d = d;
  r.dp = c->dp;
  r.p = cfg->steps;
  r.max_stepout = cfg->max_stepout;
  r.max_shrink = cfg->max_shrink;
  r.dir_norm = cfg->dir_norm;
  r.quadrature = cfg->quadrature;
  r.R = R;
  r.max_dead = cfg->max_dead;
  const long long nch = cfg->update_all ? n : k;
  r.nch = static_cast<int>(nch);
  r.mutation = cfg->mutation;
  r.rw_sigma = static_cast<float>(cfg->width * 2.38 / std::sqrt(static_cast<double>(d)));
  r.c0 = 0;
  r.c1 = static_cast<int>(nch);
  r.seed_lo = static_cast<uint32_t>(cfg->seed);
  r.seed_hi = static_cast<uint32_t>(cfg->seed >> 32);
  r.term_log_ratio = static_cast<float>(cfg->term_log_ratio);
  const size_t cap = static_cast<size_t>(cfg->max_dead);
  ip("setup");
  if (sharded && !group) {
    // other ranks map X and E with CUDA IPC: plain cudaMalloc allocations
    for (int q = 0; q < 2; ++q) {
      const size_t bytes = (q == 0 ? static_cast<size_t>(n) * c->dp : static_cast<size_t>(n)) * sizeof(float);
      void *p = nullptr;
      if (cudaMalloc(&p, bytes) != cudaSuccess || cudaMemset(p, 0, bytes) != cudaSuccess) return bail(NSS_ERR_OOM);
      c->raw_allocs.push_back(p);
      (q == 0 ? r.X : r.E) = static_cast<float *>(p);
    }
  } else {
    if ((s = dalloc(c, &r.X, static_cast<size_t>(n) * c->dp))) return bail(s);
    if ((s = dalloc(c, &r.E, n))) return bail(s);
  }
  if ((s = dalloc(c, &r.birth, n))) return bail(s);
  if ((s = dalloc(c, &r.L, static_cast<size_t>(d) * c->dp))) return bail(s);
  if ((s = dalloc(c, &r.LT, static_cast<size_t>(d) * c->dp))) return bail(s);
  if ((s = dalloc(c, &r.L64, static_cast<size_t>(d) * d))) return bail(s);
  if ((s = dalloc(c, &r.dE, cap))) return bail(s);
  if ((s = dalloc(c, &r.dbirth, cap))) return bail(s);
  if ((s = dalloc(c, &r.dX, cap * c->dp))) return bail(s);
  if ((s = dalloc(c, &r.dnlive, cap))) return bail(s);
  if ((s = dalloc(c, &r.dgid, cap))) return bail(s);
  if ((s = dalloc(c, &r.dord, cap))) return bail(s);
  if ((s = dalloc(c, &r.diter, cap))) return bail(s);
  if ((s = dalloc(c, &r.dead_gid, k))) return bail(s);
  if ((s = dalloc(c, &r.dest_gid, k))) return bail(s);
  if ((s = dalloc(c, &r.parent_gid, k))) return bail(s);
  if ((s = dalloc(c, &r.surv, n))) return bail(s);
  if ((s = dalloc(c, &r.counts, static_cast<size_t>(nch) * (cfg->steps > 0 ? cfg->steps : 1)))) return bail(s);
  if (cfg->update_all) {  // F4: chains over every slot, started from a snapshot
    float *xs = nullptr, *es = nullptr;
    if ((s = dalloc(c, &r.cdest, n))) return bail(s);
    if ((s = dalloc(c, &r.cpar, n))) return bail(s);
    if ((s = dalloc(c, &xs, static_cast<size_t>(n) * c->dp))) return bail(s);
    if ((s = dalloc(c, &es, n))) return bail(s);
    r.Xs = xs;
    r.Es = es;
  } else {
    r.cdest = r.dest_gid;
    r.cpar = r.parent_gid;
    r.Xs = r.X;
    r.Es = r.E;
  }
  size_t P = 1;
  while (P < static_cast<size_t>(n)) P <<= 1;
  if ((s = dalloc(c, &r.sort_scratch, P + static_cast<size_t>(n)))) return bail(s);
  if ((s = dalloc(c, &r.sel_scratch, 2 * static_cast<size_t>(k)))) return bail(s);
  if ((s = dalloc(c, &r.lx_prev, R + 1))) return bail(s);
  if ((s = dalloc(c, &r.lx_cur, R + 1))) return bail(s);
  if ((s = dalloc(c, &r.lz, R + 1))) return bail(s);
  if ((s = dalloc(c, &r.st, 1))) return bail(s);
  if ((s = dalloc(c, &c->summary, R + 3))) return bail(s);
  c->bps = metric_blocks(r.n, d);
  const int nent = d * (d + 1) / 2 + d + 1;
  if ((s = dalloc(c, &c->partials, static_cast<size_t>(kSegs * c->bps + 1) * nent))) return bail(s);  // + the reduced row
  {
    // the metric's first shift: the prior's centre (k_metric.cu)
    std::vector<double> ctr(d);
    for (int i = 0; i < d; ++i)
      ctr[i] = prior->kind == NSS_PRIOR_BOX ? 0.5 * (prior->lo[i] + prior->hi[i]) : prior->mean[i];
    if ((s = dalloc(c, &r.mshift, d))) return bail(s);
    if (cudaMemcpyAsync(r.mshift, ctr.data(), d * sizeof(double), cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
      return bail(NSS_ERR_CUDA);
  }
  if ((s = dalloc(c, &c->ticket, 1))) return bail(s);
  {
    std::vector<double> ninf(R + 1, -INFINITY);
    if (cudaMemcpyAsync(r.lz, ninf.data(), (R + 1) * sizeof(double), cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
      return bail(NSS_ERR_CUDA);
  }
  ip("alloc");
  // ---- multi-GPU ----
  r.world = 1;
  r.rank = 0;
  r.rank_lo[0] = 0;
  r.rank_lo[1] = r.n;
  if (sharded) {
    // the sharded live set: this rank's segments and gids,
    // the exchange block, the communicator and the peer tables
    const int W = dist->world, q = dist->rank;
    c->rank = q;
    c->world = W;
    r.world = W;
    r.rank = q;
    for (int j = 0; j <= W; ++j) r.rank_lo[j] = seg_lo(r.n, j * (kSegs / W));
    c->seg0 = q * (kSegs / W);
    c->nseg = kSegs / W;
    c->own_max = 0;
    for (int j = 0; j < W; ++j) c->own_max = std::max(c->own_max, r.rank_lo[j + 1] - r.rank_lo[j]);
    c->kc_cap = static_cast<int>(std::min<long long>(k, c->own_max));
    c->blk_bytes = shard_block_bytes(static_cast<int>(k), c->own_max, W, d);
    c->met_off = shard_metric_offset(static_cast<int>(k), c->own_max);
    r.c0 = 0;  // grid bound only: the chains run are those of crange
    r.c1 = static_cast<int>(std::min<long long>(k, r.rank_lo[q + 1] - r.rank_lo[q]));
    if ((s = dalloc(c, &c->crange, 2))) return bail(s);
    r.crange = c->crange;
    if ((s = dalloc(c, &c->shard_sums, static_cast<size_t>(nent)))) return bail(s);
    float **tbl = nullptr;
    if ((s = dalloc(c, &tbl, 2 * static_cast<size_t>(W)))) return bail(s);
    r.peerX = tbl;
    r.peerE = tbl + W;
    if (group) {
      c->gather = group->gather;
      c->live_buf = group->live;  // the peer tables are filled by nss_group_init
    } else {
      if ((s = dalloc(c, &c->gather, c->blk_bytes * W))) return bail(s);
      if ((s = dalloc(c, &c->live_buf, static_cast<size_t>(W) * c->own_max * (c->dp + 2)))) return bail(s);
      std::string err;
      if (!nccl_comm_init(&c->comm, W, dist->nccl_uid, q, &err)) {
        c->err = err;
        return bail(NSS_ERR_COMM);
      }
      void *mine[2] = {r.X, r.E};
      std::vector<void *> peers(2 * W);
      if (!ipc_exchange(c->comm, W, q, mine, 2, peers.data(), &c->ipc_open, c->stream, &err)) {
        c->err = err;
        return bail(NSS_ERR_COMM);
      }
      if (cudaMemcpyAsync(tbl, peers.data(), 2 * W * sizeof(void *), cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
        return bail(NSS_ERR_CUDA);
      if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(NSS_ERR_CUDA);
    }
  } else if (dist && dist->nccl_uid) {  // F3 SMC: replicated state, chains split
    c->rank = dist->rank;
    c->world = dist->world;
    c->kc = static_cast<int>((nch + c->world - 1) / c->world);
    r.c0 = static_cast<int>(std::min<long long>(nch, static_cast<long long>(c->rank) * c->kc));
    r.c1 = static_cast<int>(std::min<long long>(nch, r.c0 + static_cast<long long>(c->kc)));
    const size_t row = static_cast<size_t>(c->dp) + 1;
    if ((s = dalloc(c, &c->xbuf, static_cast<size_t>(c->kc) * row))) return bail(s);
    if ((s = dalloc(c, &c->xall, static_cast<size_t>(c->world) * c->kc * row))) return bail(s);
    std::string err;
    if (!nccl_comm_init(&c->comm, c->world, dist->nccl_uid, c->rank, &err)) {
      c->err = err;
      return bail(NSS_ERR_CUDA);
    }
  }
  // ---- init: prior draws (R-20), then the first metric ----
  LaunchCtx lc = lctx(c);
  // energies with a batched tensor-core / Cholesky implementation initialise
  // through it (the n prior draws are one batch), the rest per warp
  if (en.kind == NSS_E_GP_ARD || (en.kind == NSS_E_LOGREG && c->lr_ok)) {
    if ((s = init_batched(c))) return bail(s);
  } else {
    launch_init(r, pr, en, lc);
  }
  ip("comm");
  if (sharded) {
    // every rank drew all n initial points (same draws); the first metric is
    // formed from the ranks' segments in the first iteration
    c->metric_pending = true;
    c->live_gathered = true;
    c->use_graph = group == nullptr;
  } else {
    launch_metric(r, cfg->metric_reg, cfg->width_rule, cfg->width, 0, c->partials, c->ticket, c->bps, lc);
  }
  if (cudaGetLastError() != cudaSuccess) return bail(NSS_ERR_CUDA);
  if ((s = pull_state(c))) return bail(s);
  if ((s = device_error(c))) return bail(s);
  ip("kernels");
  *out = c;
  return NSS_OK;
}

NSS_API nss_status nss_init(const nss_prior *prior, const nss_energy *energy, const nss_config *cfg,
                            const nss_dist *dist, nss_ctx **out) {
  NvtxRange nvtx_("nss_init");
  return init_impl(prior, energy, cfg, dist, false, nullptr, out);
}

NSS_API nss_status nss_step(nss_ctx *c, nss_step_info *info) {
  NvtxRange nvtx_("nss_step");
  nss_status s = check_usable(c);
  if (s) return s;
  if (c->host_finalised) return fail(c, NSS_ERR_STATE, "run already finalised");
  if ((s = enqueue_iteration(c, info != nullptr))) return s;
  if (info) {
    if ((s = pull_state(c))) return s;
    if ((s = device_error(c))) return s;
    fill_info(c, info);
  }
  return NSS_OK;
}

NSS_API nss_status nss_steps(nss_ctx *c, int64_t count) {
  NvtxRange nvtx_("nss_steps");
  nss_status s = check_usable(c);
  if (s) return s;
  if (c->host_finalised) return fail(c, NSS_ERR_STATE, "run already finalised");
  for (int64_t i = 0; i < count; ++i)
    if ((s = enqueue_iteration(c))) return s;
  return NSS_OK;
}

// Sharded live set: every rank's rows (x, E, birth) into every rank's arrays
// (one NCCL all-gather; collective).
nss_status shard_gather_live(nss_ctx *c) {
  if (c->live_gathered) return NSS_OK;
  if (c->group) return fail(c, NSS_ERR_STATE, "in-process group member: call nss_group_gather_live");
  LaunchCtx lc = lctx(c);
  const size_t row = static_cast<size_t>(c->dp) + 2, cap = static_cast<size_t>(c->own_max);
  launch_shard_pack_live(c->r, c->live_buf + static_cast<size_t>(c->r.rank) * cap * row, lc);
  std::string err;
  if (!nccl_allgather_inplace(c->comm, c->live_buf, cap * row * sizeof(float), c->r.rank, c->stream, &err)) {
    c->poisoned = true;
    return fail(c, NSS_ERR_COMM, err);
  }
  launch_shard_unpack_live(c->r, c->live_buf, static_cast<long long>(cap), lc);
  CK(cudaGetLastError());
  c->live_gathered = true;
  return NSS_OK;
}

NSS_API nss_status nss_finalise(nss_ctx *c) {
  NvtxRange nvtx_("nss_finalise");
  nss_status s = check_usable(c);
  if (s) return s;
  if (c->host_finalised) return NSS_OK;
  if (c->sharded && (s = shard_gather_live(c))) return s;
  LaunchCtx lc = lctx(c);
  launch_finalise_sort(c->r, lc);
  if (c->sharded) launch_shard_mask_rows(c->r, lc);  // dead rows stay with their owner
  launch_evidence(c->r, 1, lc);
  CK(cudaMemcpyAsync(&c->r.st->finalised, c->h_one, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CK(cudaGetLastError());
  if ((s = pull_state(c))) return s;
  if ((s = device_error(c))) return s;
  c->host_finalised = 1;
  return NSS_OK;
}

NSS_API nss_status nss_run(nss_ctx *c, int64_t max_iters, nss_step_info *info) {
  NvtxRange nvtx_("nss_run");
  nss_status s = check_usable(c);
  if (s) return s;
  if (c->host_finalised) return fail(c, NSS_ERR_STATE, "run already finalised");
  if ((s = pull_state(c))) return s;
  const long long start = c->h_st->iter;
  long long enq = 0;
  int batch = 4;
  while (enq < max_iters && !c->h_st->terminated) {
    const long long todo = std::min<long long>(batch, max_iters - enq);
    for (long long i = 0; i < todo; ++i)
      if ((s = enqueue_iteration(c))) return s;
    enq += todo;
    if ((s = pull_state(c))) return s;
    if ((s = device_error(c))) return s;
    if (c->h_st->iter - start >= max_iters) break;
    batch = std::min(batch * 2, 64);
  }
  if ((s = nss_finalise(c))) return s;
  if (info) {
    if ((s = pull_state(c))) return s;
    fill_info(c, info);
  }
  return NSS_OK;
}

NSS_API nss_status nss_evidence_reps(nss_ctx *c, double *reps) {
  NvtxRange nvtx_("nss_evidence_reps");
  nss_status s = check_usable(c);
  if (s) return s;
  if ((s = pull_state(c))) return s;
  if (c->h_st->n_dead == 0) return fail(c, NSS_ERR_STATE, "no dead points yet");
  LaunchCtx lc = lctx(c);
  launch_evidence_summary(c->r, c->summary, lc);
  CK(cudaGetLastError());
  if (reps) CK(cudaMemcpyAsync(reps, c->summary + 2, (c->r.R + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return NSS_OK;
}

NSS_API nss_status nss_evidence(nss_ctx *c, double *log_z, double *log_z_err) {
  nss_status s = nss_evidence_reps(c, nullptr);
  if (s) return s;
  double ms[2];
  CK(cudaMemcpy(ms, c->summary, 2 * sizeof(double), cudaMemcpyDeviceToHost));
  if (log_z) *log_z = ms[0];
  if (log_z_err) *log_z_err = ms[1];
  return NSS_OK;
}

NSS_API nss_status nss_samples(nss_ctx *c, double *x, double *log_w, int64_t cap, int64_t *n_out) {
  NvtxRange nvtx_("nss_samples");
  nss_status s = check_usable(c);
  if (s) return s;
  if (!n_out) return NSS_ERR_INVALID_ARG;
  if ((s = pull_state(c))) return s;
  const long long N = c->h_st->n_dead;
  *n_out = N;
  if (N == 0) return fail(c, NSS_ERR_STATE, "no dead points yet");
  if (!x && !log_w) return NSS_OK;
  if (cap < N) return fail(c, NSS_ERR_CAPACITY, "output buffer smaller than the dead store");
  const int d = c->d, dp = c->dp;
  if (x) {
    std::vector<float> tmp(static_cast<size_t>(N) * dp);
    CK(cudaMemcpy(tmp.data(), c->r.dX, tmp.size() * sizeof(float), cudaMemcpyDeviceToHost));
    for (long long i = 0; i < N; ++i)
      for (int j = 0; j < d; ++j) x[i * d + j] = tmp[static_cast<size_t>(i) * dp + j];
  }
  if (log_w) {
    const int chunk = 1 << 16;
    double *logw = nullptr, *scratch = nullptr;
    CK(cudaMalloc(&logw, N * sizeof(double)));
    CK(cudaMalloc(&scratch, (static_cast<size_t>(c->r.R) * (chunk + 3)) * sizeof(double)));
    launch_samples(c->r, N, logw, scratch, chunk, lctx(c), 1.0, nullptr);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(log_w, logw, N * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(logw);
    cudaFree(scratch);
    if (e != cudaSuccess) {
      c->poisoned = true;
      return fail(c, NSS_ERR_CUDA, cudaGetErrorString(e));
    }
  }
  return NSS_OK;
}

// F2 posterior products: weights at inverse
// temperature beta re-simulated on the device; optional equal-weight draws.
static nss_status posterior_impl(nss_ctx *c, double beta, double *log_z, double *log_z_err, double *ess,
                                 double *log_w, int64_t cap, int64_t m, uint64_t seed, int64_t *idx, double *x) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (!std::isfinite(beta) || beta < 0.0) return NSS_ERR_INVALID_ARG;
  if ((s = pull_state(c))) return s;
  const long long N = c->h_st->n_dead;
  if (N == 0) return fail(c, NSS_ERR_STATE, "no dead points yet");
  if (log_w && cap < N) return fail(c, NSS_ERR_CAPACITY, "output buffer smaller than the dead store");
  const int chunk = 1 << 16, R = c->r.R;
  double *logw = nullptr, *scratch = nullptr, *zacc = nullptr, *cum = nullptr, *xd = nullptr;
  long long *idxd = nullptr;
  cudaError_t e = cudaMalloc(&logw, N * sizeof(double));
  if (!e) e = cudaMalloc(&scratch, (static_cast<size_t>(R) * (chunk + 3)) * sizeof(double));
  if (!e) e = cudaMalloc(&zacc, (2 * static_cast<size_t>(R) + 4) * sizeof(double));
  if (!e && m > 0) e = cudaMalloc(&cum, N * sizeof(double));
  if (!e && m > 0) e = cudaMalloc(&idxd, m * sizeof(long long));
  if (!e && m > 0) e = cudaMalloc(&xd, static_cast<size_t>(m) * c->d * sizeof(double));
  double summary[3] = {0, 0, 0};
  if (!e) {
    launch_samples(c->r, N, logw, scratch, chunk, lctx(c), beta, zacc);
    if (m > 0) launch_resample(c->r, N, logw, cum, m, seed, idxd, xd, lctx(c));
    e = cudaGetLastError();
  }
  if (!e) e = cudaMemcpyAsync(summary, zacc + 2 * R, 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  if (!e && log_w) e = cudaMemcpyAsync(log_w, logw, N * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  if (!e && idx) e = cudaMemcpyAsync(idx, idxd, m * sizeof(long long), cudaMemcpyDeviceToHost, c->stream);
  if (!e && x) e = cudaMemcpyAsync(x, xd, static_cast<size_t>(m) * c->d * sizeof(double), cudaMemcpyDeviceToHost,
                                   c->stream);
  if (!e) e = cudaStreamSynchronize(c->stream);
  cudaFree(logw);
  cudaFree(scratch);
  cudaFree(zacc);
  cudaFree(cum);
  cudaFree(idxd);
  cudaFree(xd);
  if (e != cudaSuccess) {
    c->poisoned = true;
    return fail(c, NSS_ERR_CUDA, cudaGetErrorString(e));
  }
  if (log_z) *log_z = summary[0];
  if (log_z_err) *log_z_err = summary[1];
  if (ess) *ess = summary[2];
  return NSS_OK;
}

NSS_API nss_status nss_posterior(nss_ctx *c, double beta, double *log_z, double *log_z_err, double *ess,
                                 double *log_w, int64_t cap) {
  NvtxRange nvtx_("nss_posterior");
  return posterior_impl(c, beta, log_z, log_z_err, ess, log_w, cap, 0, 0, nullptr, nullptr);
}

NSS_API nss_status nss_resample(nss_ctx *c, double beta, int64_t m, uint64_t seed, int64_t *idx, double *x) {
  if (!c || m < 1 || (!idx && !x)) return NSS_ERR_INVALID_ARG;
  return posterior_impl(c, beta, nullptr, nullptr, nullptr, nullptr, 0, m, seed, idx, x);
}

NSS_API nss_status nss_info(nss_ctx *c, nss_step_info *info) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (!info) return NSS_ERR_INVALID_ARG;
  if ((s = pull_state(c))) return s;
  fill_info(c, info);
  return device_error(c);
}

NSS_API nss_status nss_sync(nss_ctx *c) {
  nss_status s = check_usable(c);
  if (s) return s;
  if ((s = pull_state(c))) return s;
  return device_error(c);
}

NSS_API nss_status nss_destroy(nss_ctx *c) {
  if (!c) return NSS_ERR_INVALID_ARG;
  if (c->side) cudaStreamSynchronize(c->side);
  if (c->side2) cudaStreamSynchronize(c->side2);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graph(c);
  if (c->lr.Xb) lr_free(c->lr);
  if (c->gp) gp_free(c->gp);
  for (void *p : c->ipc_open) cudaIpcCloseMemHandle(p);
  if (c->comm) nccl_comm_free(c->comm);
  for (void *p : c->raw_allocs) cudaFree(p);

  // every stream is idle: the blocks go back to the pool in stream order
  for (void *p : c->allocs) cudaFreeAsync(p, c->stream);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto e : c->ev_free) cudaEventDestroy(e);
  for (auto &t : c->ev_pending) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  if (c->h_block) pinned_release(c->h_block);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_sel) cudaEventDestroy(c->ev_sel);
  if (c->ev_evid) cudaEventDestroy(c->ev_evid);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_met) cudaEventDestroy(c->ev_met);
  if (c->side2) cudaStreamDestroy(c->side2);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (nss_group *g = c->group) {
    if (--g->alive == 0) {
      cudaStreamSynchronize(g->stream);
      cudaFree(g->gather);
      cudaFree(g->live);
      cudaStreamDestroy(g->stream);
      delete g;
    }
  }
  delete c;
  return NSS_OK;
}

NSS_API const char *nss_last_error(const nss_ctx *c) { return c ? c->err.c_str() : "null context"; }

// ---- parity hooks ----
NSS_API nss_status nss_set_live(nss_ctx *c, const float *x, const float *e, int64_t next_iteration) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (!x || !e || next_iteration < 1) return NSS_ERR_INVALID_ARG;
  if (c->host_finalised) return fail(c, NSS_ERR_STATE, "run already finalised");
  const int n = c->r.n, d = c->d, dp = c->dp;
  std::vector<float> tmp(static_cast<size_t>(n) * dp, 0.f);
  for (int g = 0; g < n; ++g)
    for (int j = 0; j < d; ++j) tmp[static_cast<size_t>(g) * dp + j] = x[static_cast<size_t>(g) * d + j];
  CK(cudaMemcpyAsync(c->r.X, tmp.data(), tmp.size() * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->r.E, e, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  if ((s = pull_state(c))) return s;
  c->h_st->iter = static_cast<int>(next_iteration - 1);
  c->h_st->terminated = 0;
  CK(cudaMemcpyAsync(c->r.st, c->h_st, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
  launch_metric(c->r, c->cfg.metric_reg, c->cfg.width_rule, c->cfg.width, 0, c->partials, c->ticket, c->bps, lctx(c));
  c->metric_pending = false;
  c->term_stale = false;
  c->live_gathered = true;
  CK(cudaGetLastError());
  if ((s = pull_state(c))) return s;
  return NSS_OK;
}

NSS_API nss_status nss_get_live(nss_ctx *c, float *x, float *e) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (c->sharded && !c->group && (s = shard_gather_live(c))) return s;
  const int n = c->r.n, d = c->d, dp = c->dp;
  CK(cudaStreamSynchronize(c->stream));
  if (x) {
    std::vector<float> tmp(static_cast<size_t>(n) * dp);
    CK(cudaMemcpy(tmp.data(), c->r.X, tmp.size() * sizeof(float), cudaMemcpyDeviceToHost));
    for (int g = 0; g < n; ++g)
      for (int j = 0; j < d; ++j) x[static_cast<size_t>(g) * d + j] = tmp[static_cast<size_t>(g) * dp + j];
  }
  if (e) CK(cudaMemcpy(e, c->r.E, n * sizeof(float), cudaMemcpyDeviceToHost));
  return NSS_OK;
}

NSS_API nss_status nss_get_metric(nss_ctx *c, double *chol, double *width) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (c->metric_pending) {  // the deferred A5 of the last iteration
    if (c->sharded && !c->live_gathered) return fail(c, NSS_ERR_STATE, "sharded: metric formed in the next iteration");
    launch_metric(c->r, c->cfg.metric_reg, c->cfg.width_rule, c->cfg.width, 0, c->partials, c->ticket, c->bps,
                  lctx(c));
    c->metric_pending = false;
  }
  CK(cudaStreamSynchronize(c->stream));
  if (chol) CK(cudaMemcpy(chol, c->r.L64, static_cast<size_t>(c->d) * c->d * sizeof(double), cudaMemcpyDeviceToHost));
  if (width) {
    if ((s = pull_state(c))) return s;
    *width = c->h_st->width;
  }
  return NSS_OK;
}

NSS_API nss_status nss_get_trace(nss_ctx *c, int32_t *dead_gid, int32_t *dest_gid, int32_t *parent_gid,
                                 uint8_t *counts, float *e_star) {
  nss_status s = check_usable(c);
  if (s) return s;
  CK(cudaStreamSynchronize(c->stream));
  const size_t k = c->r.k, nch = c->r.nch;
  if (dead_gid) CK(cudaMemcpy(dead_gid, c->r.dead_gid, k * sizeof(int), cudaMemcpyDeviceToHost));
  if (dest_gid) CK(cudaMemcpy(dest_gid, c->r.cdest, nch * sizeof(int), cudaMemcpyDeviceToHost));
  if (parent_gid) CK(cudaMemcpy(parent_gid, c->r.cpar, nch * sizeof(int), cudaMemcpyDeviceToHost));
  if (counts) {
    const size_t p = c->cfg.steps > 0 ? c->cfg.steps : 1;
    CK(cudaMemcpy(counts, c->r.counts, nch * p * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  }
  if (e_star) {
    if ((s = pull_state(c))) return s;
    *e_star = c->h_st->e_star;
  }
  return NSS_OK;
}

NSS_API nss_status nss_dead(nss_ctx *c, float *e, int32_t *n_live, float *birth, int32_t *gid, float *x,
                            int64_t cap, int64_t *n_out) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (!n_out) return NSS_ERR_INVALID_ARG;
  if ((s = pull_state(c))) return s;
  const long long N = c->h_st->n_dead;
  *n_out = N;
  if (!e && !n_live && !birth && !gid && !x) return NSS_OK;
  if (cap < N) return fail(c, NSS_ERR_CAPACITY, "output buffer smaller than the dead store");
  if (e) CK(cudaMemcpy(e, c->r.dE, N * sizeof(float), cudaMemcpyDeviceToHost));
  if (n_live) CK(cudaMemcpy(n_live, c->r.dnlive, N * sizeof(int), cudaMemcpyDeviceToHost));
  if (birth) CK(cudaMemcpy(birth, c->r.dbirth, N * sizeof(float), cudaMemcpyDeviceToHost));
  if (gid) CK(cudaMemcpy(gid, c->r.dgid, N * sizeof(int), cudaMemcpyDeviceToHost));
  if (x) {
    std::vector<float> tmp(static_cast<size_t>(N) * c->dp);
    CK(cudaMemcpy(tmp.data(), c->r.dX, tmp.size() * sizeof(float), cudaMemcpyDeviceToHost));
    for (long long i = 0; i < N; ++i)
      for (int j = 0; j < c->d; ++j) x[i * c->d + j] = tmp[static_cast<size_t>(i) * c->dp + j];
  }
  return NSS_OK;
}

NSS_API nss_status nss_volume_reps(nss_ctx *c, double *log_x) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (!log_x) return NSS_ERR_INVALID_ARG;
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(log_x, c->r.lx_cur, (c->r.R + 1) * sizeof(double), cudaMemcpyDeviceToHost));
  return NSS_OK;
}

NSS_API nss_status nss_set_kernel_timing(nss_ctx *c, int32_t enable) {
  nss_status s = check_usable(c);
  if (s) return s;
  CK(cudaStreamSynchronize(c->stream));
  if ((s = collect_timing(c))) return s;
  c->timing = enable != 0;
  for (int i = 0; i < kPhases; ++i) {
    c->time_ms[i] = 0.0;
    c->timed[i] = 0;
  }
  return NSS_OK;
}

NSS_API nss_status nss_kernel_time(nss_ctx *c, double *ms, int64_t *launches) {
  nss_status s = check_usable(c);
  if (s) return s;
  CK(cudaStreamSynchronize(c->stream));
  if ((s = collect_timing(c))) return s;
  if (ms) *ms = c->time_ms[0];
  if (launches) *launches = c->timed[0];
  return NSS_OK;
}

NSS_API nss_status nss_set_hrss_engine(nss_ctx *c, int32_t engine) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (engine < NSS_ENGINE_AUTO || engine > NSS_ENGINE_BATCH) return NSS_ERR_INVALID_ARG;
  drop_graph(c);
  c->r.engine = engine;
  return NSS_OK;
}

NSS_API nss_status nss_get_hrss_engine(nss_ctx *c, int32_t *engine) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (!engine) return NSS_ERR_INVALID_ARG;
  const int e = resolve_engine(c);
  *engine = e == 2 ? NSS_ENGINE_BATCH : (e == 1 ? NSS_ENGINE_LANE : NSS_ENGINE_WARP);
  return NSS_OK;
}

NSS_API nss_status nss_phase_times(nss_ctx *c, double *ms, int64_t *launches) {
  nss_status s = check_usable(c);
  if (s) return s;
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaStreamSynchronize(c->side));
  if ((s = collect_timing(c))) return s;
  for (int i = 0; i < kPhases; ++i) {
    if (ms) ms[i] = c->time_ms[i];
    if (launches) launches[i] = c->timed[i];
  }
  return NSS_OK;
}

NSS_API nss_status nss_set_overlap(nss_ctx *c, int32_t overlap) {
  nss_status s = check_usable(c);
  if (s) return s;
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaStreamSynchronize(c->side));
  drop_graph(c);
  c->serial_evidence = overlap == 0;
  return NSS_OK;
}

NSS_API nss_status nss_set_graph(nss_ctx *c, int32_t enable) {
  nss_status s = check_usable(c);
  if (s) return s;
  CK(cudaStreamSynchronize(c->stream));
  drop_graph(c);
  c->use_graph = enable != 0;
  return NSS_OK;
}

NSS_API nss_status nss_debug_stamps(nss_ctx *c, uint64_t *stamps) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (!stamps) return NSS_ERR_INVALID_ARG;
  if ((s = pull_state(c))) return s;
  for (int i = 0; i < 16; ++i) stamps[i] = c->h_st->stamp[i];
  return NSS_OK;
}

NSS_API nss_status nss_lr_energy_batch(const double *X, const double *y, int64_t N, int32_t d, const double *theta,
                                       int64_t P, double *E_out) {
  if (!X || !y || !theta || !E_out || N < 1 || d < 1 || d > 128 || P < 1) return NSS_ERR_INVALID_ARG;
  bool exact = true;
  if (!lr_data_ok(X, N * d, d, &exact)) return NSS_ERR_UNSUPPORTED;
  LrEngine L;
  if (lr_setup(L, X, y, N, d, static_cast<int>(P)) != cudaSuccess) {
    lr_free(L);
    return NSS_ERR_CUDA;
  }
  std::vector<float> pt(static_cast<size_t>(P) * d);
  for (size_t i = 0; i < pt.size(); ++i) pt[i] = static_cast<float>(theta[i]);
  float *dP = nullptr, *dE = nullptr;
  int *dn = nullptr;
  const int np = static_cast<int>(P);
  long long launches = 0;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaError_t e = cudaMalloc(&dP, pt.size() * sizeof(float));
  if (!e) e = cudaMalloc(&dE, P * sizeof(float));
  if (!e) e = cudaMalloc(&dn, sizeof(int));
  if (!e) e = cudaMemcpy(dP, pt.data(), pt.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(dn, &np, sizeof(int), cudaMemcpyHostToDevice);
  if (!e) {
    lr_energies(L, dP, d, dn, dE, LaunchCtx{st, &launches});
    e = cudaGetLastError();
    if (const char *rp = getenv("NSS_LR_REPS")) {  // measurement hook: time R repeats of the energy pass
      const int reps = atoi(rp);
      cudaEvent_t ea, eb;
      cudaEventCreate(&ea);
      cudaEventCreate(&eb);
      cudaEventRecord(ea, st);
      for (int q = 0; q < reps; ++q) lr_energies(L, dP, d, dn, dE, LaunchCtx{st, &launches});
      cudaEventRecord(eb, st);
      cudaEventSynchronize(eb);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ea, eb);
      fprintf(stderr, "lr_energies x%d: %.3f us each\n", reps, 1000.f * ms / reps);
    }
  }
  std::vector<float> Ef(P);
  if (!e) e = cudaStreamSynchronize(st);
  if (!e) e = cudaMemcpy(Ef.data(), dE, P * sizeof(float), cudaMemcpyDeviceToHost);
  for (int64_t i = 0; i < P; ++i) E_out[i] = Ef[i];
  cudaFree(dP);
  cudaFree(dE);
  cudaFree(dn);
  cudaStreamDestroy(st);
  lr_free(L);
  return e ? NSS_ERR_CUDA : NSS_OK;
}

NSS_API nss_status nss_gp_energy_batch(const double *X, const double *y, int64_t N, int32_t d_in, double jitter,
                                       const double *phi, int64_t P, double *E_out) {
  if (!X || !y || !phi || !E_out || N < 1 || d_in < 1 || d_in + 2 > NSS_MAX_DIM || P < 1 || P > (1 << 24))
    return NSS_ERR_INVALID_ARG;
  void *gp = nullptr;
  if (!gp_setup(&gp, X, y, static_cast<int>(N), d_in, jitter)) {
    gp_free(gp);
    return gp ? NSS_ERR_UNSUPPORTED : NSS_ERR_OOM;
  }
  const int d = d_in + 2, dp = (d + 3) & ~3, np = static_cast<int>(P);
  std::vector<float> pt(static_cast<size_t>(P) * dp, 0.f);
  for (int64_t i = 0; i < P; ++i)
    for (int j = 0; j < d; ++j) pt[i * dp + j] = static_cast<float>(phi[i * d + j]);
  BatchDev b{};
  b.dp = dp;
  b.max_rows = np;
  b.p_stride = np;
  float *dP = nullptr, *dE = nullptr;
  double *dE64 = nullptr;
  int *dn = nullptr;
  long long launches = 0;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaError_t e = cudaMalloc(&dP, pt.size() * sizeof(float));
  if (!e) e = cudaMalloc(&dE, P * sizeof(float));
  if (!e) e = cudaMalloc(&dE64, P * sizeof(double));
  if (!e) e = cudaMalloc(&dn, 2 * sizeof(int));
  if (!e) e = cudaMemcpy(dP, pt.data(), pt.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(dn, &np, sizeof(int), cudaMemcpyHostToDevice);
  if (!e) {
    b.P[0] = b.P[1] = dP;
    b.partial[0] = b.partial[1] = dE;
    b.n_probe = dn;
    gp_set_out64(gp, dE64);
    gp_energy_pass(gp, b, 0, LaunchCtx{st, &launches});
    e = cudaGetLastError();
  }
  if (!e) e = cudaStreamSynchronize(st);
  if (!e) e = cudaMemcpy(E_out, dE64, P * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(dP);
  cudaFree(dE);
  cudaFree(dE64);
  cudaFree(dn);
  cudaStreamDestroy(st);
  gp_free(gp);
  return e ? NSS_ERR_CUDA : NSS_OK;
}

NSS_API nss_status nss_set_chain_range(nss_ctx *c, int32_t c0, int32_t c1) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (c->comm) return fail(c, NSS_ERR_STATE, "chain range is fixed by the NCCL rank");
  if (c0 < 0 || c1 < c0 || c1 > c->r.nch) return NSS_ERR_INVALID_ARG;
  CK(cudaStreamSynchronize(c->stream));
  drop_graph(c);
  c->r.c0 = c0;
  c->r.c1 = c1;
  return NSS_OK;
}

// ---- F3: adaptive tempered SMC with the HRSS kernel (SMC-SS) ----
NSS_API nss_status nss_smc_init(const nss_prior *prior, const nss_energy *energy, const nss_config *cfg, double rho,
                                const nss_dist *dist, nss_ctx **out) {
  if (!out || !cfg || !(rho > 0.0 && rho < 1.0)) return NSS_ERR_INVALID_ARG;
  if (energy && energy->kind == NSS_E_GP_ARD) return NSS_ERR_UNSUPPORTED;
  if (cfg->update_all || cfg->mutation != NSS_MUT_HRSS) return NSS_ERR_INVALID_ARG;
  nss_status s = init_impl(prior, energy, cfg, dist, true, nullptr, out);
  if (s) return s;
  nss_ctx *c = *out;
  const int n = c->r.n;
  int *ident = nullptr;
  auto bail = [&](nss_status st) {
    nss_destroy(c);
    *out = nullptr;
    return st;
  };
  if ((s = dalloc(c, &c->smc_cum, n))) return bail(s);
  if ((s = dalloc(c, &c->smc_par, n))) return bail(s);
  if ((s = dalloc(c, &c->smc_xs, static_cast<size_t>(n) * c->dp))) return bail(s);
  if ((s = dalloc(c, &c->smc_es, n))) return bail(s);
  if ((s = dalloc(c, &ident, n))) return bail(s);
  uint32_t *counts = nullptr;  // per-particle HRSS counts (nss_init sized them for k chains)
  if ((s = dalloc(c, &counts, static_cast<size_t>(n) * (cfg->steps > 0 ? cfg->steps : 1)))) return bail(s);
  c->r.counts = counts;
  std::vector<int> id(n);
  for (int i = 0; i < n; ++i) id[i] = i;
  if (cudaMemcpyAsync(ident, id.data(), n * sizeof(int), cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
    return bail(NSS_ERR_CUDA);
  c->smc = true;
  c->smc_rho = rho;
  RunDev &r = c->r;
  r.tempered = 1;
  r.engine = NSS_ENGINE_WARP;
  r.nch = n;
  r.cdest = ident;
  r.cpar = ident;
  r.Xs = r.X;
  r.Es = r.E;
  r.c0 = 0;
  r.c1 = n;
  if (c->comm) {
    c->kc = (n + c->world - 1) / c->world;
    r.c0 = std::min(n, c->rank * c->kc);
    r.c1 = std::min(n, r.c0 + c->kc);
    const size_t row = static_cast<size_t>(c->dp) + 1;
    if ((s = dalloc(c, &c->xbuf, static_cast<size_t>(c->kc) * row))) return bail(s);
    if ((s = dalloc(c, &c->xall, static_cast<size_t>(c->world) * c->kc * row))) return bail(s);
  }
  return NSS_OK;
}

NSS_API nss_status nss_smc_stage(nss_ctx *c) {
  NvtxRange nvtx_("nss_smc_stage");
  nss_status s = check_usable(c);
  if (s) return s;
  if (!c->smc) return fail(c, NSS_ERR_STATE, "not an SMC context");
  if ((s = ensure_vpre(c))) return s;
  LaunchCtx lc = lctx(c);
  launch_smc_stage(c->r, c->smc_rho, c->smc_cum, c->smc_par, c->smc_xs, c->smc_es, lc);
  launch_metric(c->r, c->cfg.metric_reg, c->cfg.width_rule, c->cfg.width, 0, c->partials, c->ticket, c->bps, lc);
  launch_hrss(c->r, c->pr, c->en, lc);
  if ((s = exchange(c))) return s;
  CK(cudaGetLastError());
  return NSS_OK;
}

NSS_API nss_status nss_smc_state(nss_ctx *c, double *beta, double *log_z, int64_t *stage, int32_t *parents) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (!c->smc) return fail(c, NSS_ERR_STATE, "not an SMC context");
  c->term_stale = false;  // no NS termination probe in SMC mode
  if ((s = pull_state(c))) return s;
  if ((s = device_error(c))) return s;
  if (beta) *beta = c->h_st->smc_beta;
  if (log_z) *log_z = c->h_st->smc_logz;
  if (stage) *stage = c->h_st->iter;
  if (parents) CK(cudaMemcpy(parents, c->smc_par, c->r.n * sizeof(int), cudaMemcpyDeviceToHost));
  return NSS_OK;
}

NSS_API nss_status nss_smc_run(nss_ctx *c, int64_t max_stages, double *log_z) {
  nss_status s = check_usable(c);
  if (s) return s;
  if (!c->smc) return fail(c, NSS_ERR_STATE, "not an SMC context");
  double beta = 0.0;
  for (int64_t t = 0; t < max_stages; ++t) {
    if ((s = nss_smc_state(c, &beta, nullptr, nullptr, nullptr))) return s;
    if (beta >= 1.0) break;
    if ((s = nss_smc_stage(c))) return s;
  }
  return nss_smc_state(c, nullptr, log_z, nullptr, nullptr);
}

NSS_API nss_status nss_launch_count(nss_ctx *c, int64_t *launches) {
  if (!c || !launches) return NSS_ERR_INVALID_ARG;
  nss_status s;
  if (c->loop_graph && (s = pull_state(c))) return s;  // + the device-side loops' kernels
  *launches = c->launches + static_cast<int64_t>(c->h_st->dev_launches);
  return NSS_OK;
}

// ---- in-process group: the ranks of one sharded run on one GPU ----
NSS_API nss_status nss_group_init(const nss_prior *prior, const nss_energy *energy, const nss_config *cfg,
                                  int32_t world, nss_ctx **out) {
  NvtxRange nvtx_("nss_group_init");
  if (!out || world < 1 || kSegs % world != 0 || !cfg || !prior) return NSS_ERR_INVALID_ARG;
  for (int q = 0; q < world; ++q) out[q] = nullptr;
  if (!validate(prior, energy, cfg)) return NSS_ERR_INVALID_ARG;
  nss_group *g = new nss_group();
  g->world = world;
  const int n = static_cast<int>(cfg->n_live), d = prior->d, dp = (d + 3) & ~3;
  int own_max = 0;
  for (int q = 0; q < world; ++q)
    own_max = std::max(own_max, seg_lo(n, (q + 1) * (kSegs / world)) - seg_lo(n, q * (kSegs / world)));
  const size_t blk = shard_block_bytes(static_cast<int>(cfg->k), own_max, world, d);
  const size_t live = static_cast<size_t>(world) * own_max * (dp + 2) * sizeof(float);
  if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&g->gather, blk * world) != cudaSuccess || cudaMemset(g->gather, 0, blk * world) != cudaSuccess ||
      cudaMalloc(&g->live, live) != cudaSuccess) {
    cudaFree(g->gather);
    cudaFree(g->live);
    if (g->stream) cudaStreamDestroy(g->stream);
    delete g;
    return NSS_ERR_OOM;
  }
  nss_status s = NSS_OK;
  for (int q = 0; q < world && s == NSS_OK; ++q) {
    nss_dist dd{q, world, nullptr, g->stream};
    s = init_impl(prior, energy, cfg, &dd, false, g, &out[q]);
    if (s == NSS_OK) ++g->alive;
  }
  if (s == NSS_OK) {
    std::vector<float *> tbl(2 * world);
    for (int q = 0; q < world; ++q) {
      tbl[q] = out[q]->r.X;
      tbl[world + q] = out[q]->r.E;
    }
    for (int q = 0; q < world && s == NSS_OK; ++q)
      if (cudaMemcpy(const_cast<float **>(out[q]->r.peerX), tbl.data(), tbl.size() * sizeof(float *),
                     cudaMemcpyHostToDevice) != cudaSuccess)
        s = NSS_ERR_CUDA;
  }
  if (s != NSS_OK) {
    const bool none = g->alive == 0;
    for (int q = 0; q < world; ++q)
      if (out[q]) {
        nss_destroy(out[q]);
        out[q] = nullptr;
      }
    if (none) {
      cudaFree(g->gather);
      cudaFree(g->live);
      cudaStreamDestroy(g->stream);
      delete g;
    }
    return s;
  }
  return NSS_OK;
}

static nss_status group_check(nss_ctx **ctx, int32_t world) {
  if (!ctx || world < 1) return NSS_ERR_INVALID_ARG;
  for (int q = 0; q < world; ++q) {
    nss_status s = check_usable(ctx[q]);
    if (s) return s;
    if (!ctx[q]->group || ctx[q]->group != ctx[0]->group || ctx[q]->r.rank != q || ctx[q]->group->world != world)
      return NSS_ERR_INVALID_ARG;
    if (ctx[q]->host_finalised) return fail(ctx[q], NSS_ERR_STATE, "run already finalised");
  }
  return NSS_OK;
}

NSS_API nss_status nss_group_step(nss_ctx **ctx, int32_t world, int64_t count) {
  NvtxRange nvtx_("nss_group_step");
  nss_status s = group_check(ctx, world);
  if (s) return s;
  for (int64_t i = 0; i < count; ++i) {
    for (int q = 0; q < world; ++q)
      if ((s = enqueue_iteration(ctx[q], false, kPre))) return s;
    for (int q = 0; q < world; ++q)
      if ((s = enqueue_iteration(ctx[q], false, kPost))) return s;
  }
  return NSS_OK;
}

NSS_API nss_status nss_group_gather_live(nss_ctx **ctx, int32_t world) {
  NvtxRange nvtx_("nss_group_gather_live");
  nss_status s = group_check(ctx, world);
  if (s) return s;
  for (int q = 0; q < world; ++q) {
    nss_ctx *c = ctx[q];
    const size_t row = static_cast<size_t>(c->dp) + 2, cap = static_cast<size_t>(c->own_max);
    launch_shard_pack_live(c->r, c->live_buf + static_cast<size_t>(q) * cap * row, lctx(c));
  }
  for (int q = 0; q < world; ++q) {
    nss_ctx *c = ctx[q];
    launch_shard_unpack_live(c->r, c->live_buf, static_cast<long long>(c->own_max), lctx(c));
    c->live_gathered = true;
    nss_ctx *cc = c;
    if (cudaGetLastError() != cudaSuccess) return fail(cc, NSS_ERR_CUDA, "group gather");
  }
  return NSS_OK;
}
