/*
 * include/nss.h -- C ABI of the B200-native Nested Slice Sampling hot path
 * (arXiv 2601.23252).  Shared library: paper_2601_23252_b200/libnss.so.
 *
 * "P:n" cites /root/reference/PAPER.md line n; "R-n" cites a reading in
 * DESIGN.md section 2 where the paper is silent or ambiguous.
 *
 * Conventions (all entry points):
 *  - Every call returns nss_status; nothing throws across the ABI.
 *  - All pointers are HOST pointers unless stated otherwise.  Input arrays are
 *    copied during the call; the caller keeps ownership and may free them when
 *    the call returns.  Output arrays are caller-owned host buffers.
 *  - The context owns all device memory (allocated in nss_init, released in
 *    nss_destroy) and runs every kernel on one CUDA stream (nss_dist.cuda_stream
 *    or a stream it creates).  Calls are asynchronous unless they return data.
 *  - A CUDA failure poisons the context: every later call except nss_destroy and
 *    nss_last_error returns NSS_ERR_CUDA.
 *  - One host thread per context; several contexts may coexist.
 *  - Positions and energies are fp32 on the device; covariance, Cholesky and
 *    evidence accumulators are fp64 (R-22).
 */
#ifndef NSS_H
#define NSS_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NSS_OK = 0,
  NSS_ERR_INVALID_ARG = 1,   /* bad config / null pointer / unknown kind          */
  NSS_ERR_PRIOR_SUPPORT = 2, /* init: no finite energy within 100 n prior draws (R-20) */
  NSS_ERR_NAN = 3,           /* an energy evaluation returned NaN                 */
  NSS_ERR_CUDA = 4,          /* CUDA runtime failure (context poisoned)           */
  NSS_ERR_COMM = 5,          /* inter-rank communication failure                  */
  NSS_ERR_OOM = 6,           /* device allocation failed                          */
  NSS_ERR_STATE = 7,         /* call not valid in the current state               */
  NSS_ERR_CAPACITY = 8,      /* dead store full (R-26) or output buffer too small */
  NSS_ERR_UNSUPPORTED = 9    /* configuration not implemented on this device path */
} nss_status;

/* ---- reference density Pi ---- */
typedef enum { NSS_PRIOR_BOX = 0, NSS_PRIOR_GAUSS_DIAG = 1 } nss_prior_kind;
typedef struct {
  int32_t kind;             /* nss_prior_kind                                    */
  int32_t d;                /* dimension, 1 <= d <= NSS_MAX_DIM                  */
  const double *lo, *hi;    /* BOX: d each, lo < hi; log Pi = -sum log(hi-lo)    */
  const double *mean, *sd;  /* GAUSS_DIAG: d each, sd > 0                        */
} nss_prior;

#define NSS_MAX_DIM 128

/* ---- energy E(x) = -log L(x) ---- */
typedef enum {
  NSS_E_GAUSS = 0,      /* 1/2 sum_i ((x_i-mu_i)/sigma_i)^2 + c                          */
  NSS_E_MOG = 1,        /* -log sum_j w_j N(x; mu_j, diag sigma_j^2)       */
  NSS_E_CORR_GAUSS = 2, /* 1/2 (x-mu)^T P (x-mu) + c           */
  NSS_E_FUNNEL = 3,     /* -log N(x_0;0,sy^2) - sum_{n>=1} log N(x_n;0,e^{x_0}) (R-23) */
  NSS_E_LOGREG = 4,     /* sum_r softplus(a_r.x) - y_r a_r.x                             */
  NSS_E_GP_ARD = 5,     /* GP ARD-RBF negative log marginal likelihood       */
  NSS_E_FLAT = 6        /* E = c (level-set / flat-likelihood tests)                     */
} nss_energy_kind;
typedef struct {
  int32_t kind;         /* nss_energy_kind                                  */
  int32_t d;            /* must equal the prior's d                         */
  int32_t n_comp;       /* MOG: number of components K (1..16)              */
  int64_t n_data;       /* LOGREG / GP: rows N                              */
  int32_t d_in;         /* GP: inputs per row; d = d_in + 2                 */
  const double *w;      /* MOG: K weights                                   */
  const double *mu;     /* GAUSS, CORR_GAUSS: d;  MOG: K*d row-major        */
  const double *sigma;  /* GAUSS: d;  MOG: K*d                              */
  const double *prec;   /* CORR_GAUSS: d*d row-major symmetric precision    */
  const double *data_x; /* LOGREG: N*d;  GP: N*d_in (row-major)             */
  const double *data_y; /* LOGREG: N labels in {0,1};  GP: N targets        */
  double c;             /* GAUSS / CORR_GAUSS / FLAT additive constant      */
  double sigma_y;       /* FUNNEL: standard deviation of x_0                */
  double jitter;        /* GP: added to sigma_n^2 on the diagonal           */
} nss_energy;

typedef enum { NSS_W_OPTIMAL = 0, NSS_W_FIXED = 1 } nss_width_rule;       /* R-7 */
typedef enum { NSS_DIR_MAHALANOBIS = 0, NSS_DIR_EUCLIDEAN = 1 } nss_dir_norm; /* R-6 */
typedef enum { NSS_Q_TRAPEZOID = 0, NSS_Q_RECTANGLE = 1 } nss_quadrature;  /* R-16 */

typedef struct {
  int64_t n_live;        /* m, >= 2                                        */
  int64_t k;             /* deleted per iteration, 1 <= k <= n_live-1      */
  int32_t steps;         /* p HRSS steps per replacement, >= 0             */
  int32_t width_rule;    /* nss_width_rule                                         */
  double width;          /* FIXED: w;  OPTIMAL: scale c on 4 kappa sqrt(2/(pi mu d)) */
  int32_t dir_norm;      /* nss_dir_norm                                           */
  int32_t max_stepout;   /* expansions per side, 10 in the paper           */
  int32_t max_shrink;    /* shrink proposals, 100 in the paper             */
  int32_t quadrature;    /* nss_quadrature                                         */
  double metric_reg;     /* ridge * mean diag (R-8), 1e-6                          */
  double term_log_ratio; /* termination threshold, -3 (R-19)                */
  int32_t n_volume_sims; /* R volume replicas, >= 2                       */
  int64_t max_dead;      /* dead-store capacity in records, >= n_live (R-26)       */
  uint64_t seed;         /* Philox key                          */
  int32_t update_all;    /* F4: 1 = every live point runs p HRSS steps each
                            iteration (deleted slots from their parent, survivors
                            from themselves); 0 = the k replacements only          */
  int32_t mutation;      /* F1: NSS_MUT_HRSS (the paper's method) or NSS_MUT_RW, the
                            constrained Gaussian random walk baseline (P:301-302,
                            P:765): `steps` proposals x + c 2.38/sqrt(d) L z per
                            replacement, c = `width`; Metropolis on the prior,
                            rejected outside E < E*                                 */
} nss_config;

typedef enum { NSS_MUT_HRSS = 0, NSS_MUT_RW = 1 } nss_mutation;

/* Multi-GPU: one process per GPU, world in {1, 2, 4, 8}.
 * The live set is SHARDED: rank q owns the gids of 8/world of the 8 fixed gid
 * segments [floor(s n / 8), floor((s + 1) n / 8)) (P:264-283's particles are
 * independent units).  Each iteration, every rank forms its local top-k
 * candidates (ord(E), gid keys) and the moment sums of its segments, one NCCL
 * all-gather exchanges them, and every rank then takes the same decisions
 * (threshold, dead records, parents, metric, evidence, termination) from the
 * same bytes; each rank runs the HRSS chains whose destination it owns and
 * reads parent rows another rank owns straight from that rank's memory over
 * NVLink (CUDA IPC).  A multi-GPU run is bit-identical to a one-GPU run with
 * the same seed.  NS with update_all = 1 is UNSUPPORTED sharded.
 * Per-rank data: nss_info counters (probes, evals, ...) are this rank's (sum
 * over ranks; init_evals is the same on every rank); the dead store's
 * positions (nss_dead x, nss_samples x) hold the rows of the points this rank
 * owned and zeros elsewhere (sum over ranks); every other output is
 * replicated.  Collective calls (every rank, same order): nss_step, nss_steps,
 * nss_run, nss_finalise, nss_get_live.  F3 SMC contexts instead replicate the
 * particles and split their chains (one all-gather of the new rows).
 * Pass NULL for a single GPU.  nccl_uid NULL: no communicator (single GPU). */
typedef struct {
  int32_t rank, world;
  const uint8_t *nccl_uid; /* 128 bytes from nss_get_unique_id on rank 0      */
  void *cuda_stream;       /* cudaStream_t to run on, or NULL for a new stream */
} nss_dist;

typedef struct {
  int64_t iteration;      /* outer iterations completed                         */
  double e_star;          /* threshold E* of the last iteration         */
  int64_t probes;         /* slice-membership tests (R-11)                      */
  int64_t energy_evals;   /* energies evaluated inside HRSS (R-11)              */
  int64_t expansions;     /* stepping-out expansions (N_out)                    */
  int64_t shrinks;        /* shrink proposals (N_shrink)                        */
  int64_t null_moves;     /* steps that hit the shrink cap              */
  int64_t init_evals;     /* energies evaluated by nss_init                     */
  double log_z_det;       /* replica-0 accumulated log Z                        */
  double log_z_live;      /* -min E_live + log X (replica 0)            */
  int32_t terminated;     /* termination criterion met (R-19)                   */
  int32_t finalised;      /* live set appended to the dead store (R-18)         */
} nss_step_info;

typedef struct nss_ctx nss_ctx;

/* Rank 0 of a multi-GPU run: fills 128 bytes (an NCCL unique id) to
 * broadcast to the other ranks.  UNSUPPORTED if NCCL cannot be loaded. */
nss_status nss_get_unique_id(uint8_t out[128]);

/* Validate, allocate, upload prior/energy data, draw the n initial live points
 * from the prior with rejection (R-20) and compute the first metric.
 * Errors: INVALID_ARG (k not in [1,n-1], d out of range, steps < 0, caps < 1,
 * R < 2, max_dead < n, unknown kind), PRIOR_SUPPORT, NAN, OOM, CUDA,
 * UNSUPPORTED. */
nss_status nss_init(const nss_prior *prior, const nss_energy *energy, const nss_config *cfg,
                    const nss_dist *dist, nss_ctx **out);

/* One outer iteration: delete, record dead, resample, p HRSS steps,
 * replace, metric, evidence, termination flag.  Asynchronous when info == NULL;
 * a non-NULL info synchronises and reports.  A call after termination is a
 * no-op on the device.  Errors: STATE (finalised), CAPACITY, NAN, CUDA. */
nss_status nss_step(nss_ctx *ctx, nss_step_info *info);

/* Enqueue `count` iterations without synchronising (benchmark / driver loop). */
nss_status nss_steps(nss_ctx *ctx, int64_t count);

/* Iterate until the termination criterion (R-19) or max_iters, then finalise. */
nss_status nss_run(nss_ctx *ctx, int64_t max_iters, nss_step_info *info);

/* Append the live set to the dead store and close the quadrature (R-18). */
nss_status nss_finalise(nss_ctx *ctx);

/* log Z = mean of log Z^(r), r=1..R; err = their sample std (R-17).
 * Errors: STATE when the dead store is empty. */
nss_status nss_evidence(nss_ctx *ctx, double *log_z, double *log_z_err);
/* All R+1 replica values (replica 0 deterministic). */
nss_status nss_evidence_reps(nss_ctx *ctx, double *log_z_reps /* R+1 */);

/* Dead points with normalised geometric-mean log weights.
 * Two-call pattern: x == NULL and log_w == NULL -> only *n_out.  x: n_out*d
 * row-major fp64.  Errors: STATE (empty), CAPACITY (cap < n_out). */
nss_status nss_samples(nss_ctx *ctx, double *x, double *log_w, int64_t cap, int64_t *n_out);

nss_status nss_info(nss_ctx *ctx, nss_step_info *info);   /* synchronises */
nss_status nss_sync(nss_ctx *ctx);
nss_status nss_destroy(nss_ctx *ctx);
const char *nss_last_error(const nss_ctx *ctx);

/* ---- parity hooks (exported for the tests; not on the user path) ---- */
/* Inject a live set (n*d fp32 positions, n fp32 energies); the next nss_step
 * is iteration `next_iteration`.  Recomputes the metric from x. */
/* F3 adaptive tempered SMC with the HRSS kernel (SMC-SS, P:635-681,
 * P:710-713), the paper's closest control.  nss_smc_init draws n_live
 * particles from the prior (as nss_init; k is unused, give 1) and returns a
 * context whose particles move through pi_beta ~ Pi exp(-beta E): each
 * nss_smc_stage picks beta_{t+1} by bisection on ESS = rho m (to 1e-10,
 * S:357-366), adds log mean exp(-(beta_{t+1} - beta_t) E_i) to log Z,
 * resamples multinomially (uniform 0 of Philox stream (stage, j, SMC = 7, 0)),
 * recomputes the metric from the resampled particles and applies `steps`
 * tempered HRSS steps per particle (slice of Pi exp(-beta E), no threshold;
 * warp engine).  Particles are read with nss_get_live; nss_smc_state gives
 * beta, log Z, the stage count and the last resampling parents (n, nullable).
 * Multi-GPU (dist): the particles' HRSS chains are split as for NS.
 * Errors: INVALID_ARG (rho not in (0,1), update_all or RW mutation),
 * UNSUPPORTED (GP energy), STATE (not an SMC context). */
nss_status nss_smc_init(const nss_prior *prior, const nss_energy *energy, const nss_config *cfg, double rho,
                        const nss_dist *dist, nss_ctx **out);
nss_status nss_smc_stage(nss_ctx *ctx);
nss_status nss_smc_state(nss_ctx *ctx, double *beta, double *log_z, int64_t *stage, int32_t *parents);
/* Stages until beta = 1 (at most max_stages); log_z nullable. */
nss_status nss_smc_run(nss_ctx *ctx, int64_t max_stages, double *log_z);

/* F2 posterior products at inverse temperature beta >= 0 (the
 * same dead points reweighted, w_i^(r)(beta) = exp(-beta E_i) dX_i^(r);
 * log Z(beta) mean and std (ddof 1) over the R volume replicas,
 * geometric-mean weights w~_i = exp(mean_r log w_i^(r)), Kish
 * ESS = (sum w~)^2 / sum w~^2).  log_w (nullable, cap >= n_dead) receives
 * the normalised log w~_i in death order.  beta = 1 reproduces
 * nss_evidence and nss_samples.  Errors: INVALID_ARG (beta < 0 or not
 * finite), STATE (no dead points), CAPACITY. */
nss_status nss_posterior(nss_ctx *ctx, double beta, double *log_z, double *log_z_err, double *ess,
                         double *log_w, int64_t cap);
/* Equal-weight posterior samples: m multinomial draws from the
 * normalised beta-weights; draw j uses uniform 0 of the Philox stream
 * (iteration 0, j, POSTERIOR = 5, 0) under key `seed` and takes the first dead
 * point whose cumulative weight exceeds it.  idx (m dead-store indices)
 * and/or x (m*d positions) may be NULL, not both. */
nss_status nss_resample(nss_ctx *ctx, double beta, int64_t m, uint64_t seed, int64_t *idx, double *x);

nss_status nss_set_live(nss_ctx *ctx, const float *x, const float *e, int64_t next_iteration);
nss_status nss_get_live(nss_ctx *ctx, float *x, float *e);
nss_status nss_get_metric(nss_ctx *ctx, double *chol /* d*d lower, fp64 */, double *width);
/* Last iteration: dead gids (key-descending), destination gids (ascending),
 * parent gid per destination, per (chain, step) counts packed as bytes
 * {n_left, n_right, n_shrink, accepted}, E*. Any pointer may be NULL. */
nss_status nss_get_trace(nss_ctx *ctx, int32_t *dead_gid, int32_t *dest_gid, int32_t *parent_gid,
                         uint8_t *counts /* k*p*4 */, float *e_star);
nss_status nss_dead(nss_ctx *ctx, float *e, int32_t *n_live, float *birth, int32_t *gid, float *x,
                    int64_t cap, int64_t *n_out);
nss_status nss_volume_reps(nss_ctx *ctx, double *log_x /* R+1 */);

/* HRSS engine.  AUTO picks BATCH (round-synchronous
 * chains feeding one batched energy kernel: tensor cores for logistic
 * regression with bf16-exact data, batched Cholesky for GP) for the
 * expensive energies, LANE (one probe per lane, speculative rounds) when
 * d <= 32 and the energy is cheap, WARP (warp-cooperative energy, one probe at
 * a time) otherwise.  Forcing an engine that does not apply falls back to WARP
 * (LANE) or to a generic warp-per-probe batched energy (BATCH).  All engines
 * compute the same algorithm with the same draws. */
typedef enum { NSS_ENGINE_AUTO = 0, NSS_ENGINE_WARP = 1, NSS_ENGINE_LANE = 2, NSS_ENGINE_BATCH = 3 } nss_hrss_engine;
nss_status nss_set_hrss_engine(nss_ctx *ctx, int32_t engine);
/* The engine the next iteration will use (resolved: WARP, LANE or BATCH). */
nss_status nss_get_hrss_engine(nss_ctx *ctx, int32_t *engine);

/* Parity hook: run only HRSS chains [c0, c1) (ordinals into the ascending
 * destination list) from the next iteration on, without a communicator --
 * what rank r of a multi-GPU run computes.  STATE if the
 * context has an NCCL communicator. */
nss_status nss_set_chain_range(nss_ctx *ctx, int32_t c0, int32_t c1);

/* Kernel check: logistic-regression energies E(theta_p) = sum_r softplus(a_rp)
 * - y_r a_rp, a = X theta (P:466 shape), for P probe points theta (P*d
 * row-major), computed by the tcgen05 tensor-core kernel the sampler uses.
 * X (N*d) must be bf16-exact, else NSS_ERR_UNSUPPORTED.
 * E_out: P values. */
nss_status nss_lr_energy_batch(const double *X, const double *y, int64_t N, int32_t d, const double *theta,
                               int64_t P, double *E_out);
/* (Measurement: with NSS_LR_REPS=R in the environment the call also times R
 * repeats of the energy pass with CUDA events and prints the mean to stderr.) */

/* Kernel check: GP ARD-RBF negative log marginal likelihoods (P:935-962
 * shape; DESIGN R-22) for P hyperparameter points phi (P*(d_in+2) row-major,
 * phi = log l_1..l_{d_in}, log sigma_f, log sigma_n), computed in fp64 by the
 * batched-Cholesky kernel the sampler uses (phi is rounded to fp32 first, as
 * in the sampler's state).  X: N*d_in, y: N.  E_out: P values, +inf where K
 * is not numerically positive definite. */
nss_status nss_gp_energy_batch(const double *X, const double *y, int64_t N, int32_t d_in, double jitter,
                               const double *phi, int64_t P, double *E_out);

/* ---- measurement hooks ---- */
/* When enabled, the HRSS kernel launch of every iteration is bracketed by CUDA
 * events on the context's stream; nss_kernel_time returns the summed elapsed
 * milliseconds and the number of launches since the last reset. */
nss_status nss_set_kernel_timing(nss_ctx *ctx, int32_t enable);
nss_status nss_kernel_time(nss_ctx *ctx, double *ms, int64_t *launches);
/* Per-phase totals of the same timing mode: ms[5] and launches[5] for
 * {HRSS, select/dead/resample, evidence, metric+termination, batched energy
 * passes}.  The last is the batch engine's energy kernels alone (also
 * counted inside HRSS); zero for the warp and lane engines. */
nss_status nss_phase_times(nss_ctx *ctx, double *ms /* 5 */, int64_t *launches /* 5 */);
/* overlap != 0 (default): the evidence kernel runs on a side stream
 * concurrently with HRSS; 0: all kernels in sequence on one stream. */
nss_status nss_set_overlap(nss_ctx *ctx, int32_t overlap);
/* enable != 0 (default): each iteration is replayed from a captured CUDA
 * graph; 0: kernels are launched one by one (timing mode always does). */
nss_status nss_set_graph(nss_ctx *ctx, int32_t enable);
/* Device %globaltimer stamps (ns) written at phase boundaries of the select
 * (0-6) and metric (8-13) kernels during the last iteration. */
nss_status nss_debug_stamps(nss_ctx *ctx, uint64_t *stamps /* 16 */);
/* Kernels launched by this context since creation (all kinds, including
 * those of device-side round loops; synchronises when there are any). */
nss_status nss_launch_count(nss_ctx *ctx, int64_t *launches);

/* ---- in-process rank emulation (tests) ----
 * The `world` ranks of ONE sharded run as `world` contexts on the current GPU
 * in this process: same partition, kernels and decisions as the NCCL path, the
 * members share one stream and the exchange buffer, and the peer tables point
 * at the other members' arrays (no kernel ever waits on another).  out: world
 * contexts (rank q = out[q]), each freed with nss_destroy.  Errors as nss_init;
 * INVALID_ARG unless world divides 8. */
nss_status nss_group_init(const nss_prior *prior, const nss_energy *energy, const nss_config *cfg, int32_t world,
                          nss_ctx **out);
/* `count` iterations of the group (all members; asynchronous). */
nss_status nss_group_step(nss_ctx **ctx, int32_t world, int64_t count);
/* Every member's live-set arrays completed with the other members' rows (then
 * nss_get_live, nss_finalise and nss_get_metric work on any member). */
nss_status nss_group_gather_live(nss_ctx **ctx, int32_t world);

#ifdef __cplusplus
}
#endif
#endif
