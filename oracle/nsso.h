/*
 * oracle/nsso.h -- fp64 single-threaded CPU reference ("oracle") for Nested
 * Slice Sampling (arXiv 2601.23252).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA product
 * path (paper_2601_23252_b200/csrc, include/nss.h); the two are written
 * independently from PAPER.md and the contract in DESIGN.md section 3.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (LaTeX source).
 *
 * Every call returns an nsso_status (0 = OK).  All input arrays are copied; the
 * caller keeps ownership of everything it passes in and of every output buffer.
 */
#ifndef NSSO_H
#define NSSO_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NSSO_OK = 0,
  NSSO_ERR_INVALID_ARG = 1,
  NSSO_ERR_PRIOR_SUPPORT = 2,
  NSSO_ERR_NAN = 3,
  NSSO_ERR_STATE = 7,
  NSSO_ERR_CAPACITY = 8
} nsso_status;

/* Reference density Pi. */
enum { NSSO_PRIOR_BOX = 0, NSSO_PRIOR_GAUSS_DIAG = 1 };
typedef struct {
  int32_t kind;
  int32_t d;
  const double *lo, *hi;   /* BOX: d each, lo < hi                       */
  const double *mean, *sd; /* GAUSS_DIAG: d each, sd > 0                 */
} nsso_prior;

/* Energy E(x) = -log L(x). */
enum {
  NSSO_E_GAUSS = 0,      /* 1/2 sum((x-mu)/sigma)^2 + c                           */
  NSSO_E_MOG = 1,        /* -log sum_j w_j N(x; mu_j, diag sigma_j^2)             */
  NSSO_E_CORR_GAUSS = 2, /* 1/2 (x-mu)^T P (x-mu) + c                              */
  NSSO_E_FUNNEL = 3,     /* -log N(x0;0,sy^2) - sum_n log N(x_n;0,exp(x0))   */
  NSSO_E_LOGREG = 4,     /* sum_i softplus(a_i.x) - y_i a_i.x                     */
  NSSO_E_GP_ARD = 5,     /* GP ARD-RBF negative log marginal likelihood            */
  NSSO_E_FLAT = 6        /* E = c everywhere (level-set / flat-likelihood pins)    */
};
typedef struct {
  int32_t kind;
  int32_t d;
  int32_t n_comp;       /* MOG: K                                                  */
  int64_t n_data;       /* LOGREG / GP: N rows                                     */
  int32_t d_in;         /* GP: input dimension (d = d_in + 2)                      */
  const double *w;      /* MOG: K weights (sum to 1)                               */
  const double *mu;     /* GAUSS, CORR_GAUSS: d; MOG: K*d                          */
  const double *sigma;  /* GAUSS: d; MOG: K*d                                      */
  const double *prec;   /* CORR_GAUSS: d*d row-major precision P                   */
  const double *data_x; /* LOGREG: N*d rows a_i; GP: N*d_in inputs                 */
  const double *data_y; /* LOGREG: N labels in {0,1}; GP: N targets                */
  double c;             /* GAUSS / CORR_GAUSS / FLAT additive constant            */
  double sigma_y;       /* FUNNEL: sd of x0 (3 in P:885)                           */
  double jitter;        /* GP: diagonal jitter added to sigma_n^2                  */
} nsso_energy;

enum { NSSO_W_OPTIMAL = 0, NSSO_W_FIXED = 1 };
enum { NSSO_DIR_MAHALANOBIS = 0, NSSO_DIR_EUCLIDEAN = 1 };
enum { NSSO_Q_TRAPEZOID = 0, NSSO_Q_RECTANGLE = 1 };

typedef struct {
  int64_t n_live;          /* m in the paper                     */
  int64_t k;               /* deleted per iteration, 1 <= k <= n-1       */
  int32_t steps;           /* p HRSS steps per replacement       */
  int32_t width_rule;      /* NSSO_W_*                                   */
  double width;            /* FIXED: w;  OPTIMAL: scale c on w*          */
  int32_t dir_norm;        /* NSSO_DIR_*                                 */
  int32_t max_stepout;     /* 10                                 */
  int32_t max_shrink;      /* 100                                */
  int32_t quadrature;      /* NSSO_Q_*                                   */
  double metric_reg;       /* 1e-6                                       */
  double term_log_ratio;   /* -3                                 */
  int32_t n_volume_sims;   /* R = 100                           */
  int64_t max_dead;        /* dead-store capacity                        */
  uint64_t seed;
  int32_t update_all;      /* F4: 1 = mutate all n live points each iteration */
  int32_t mutation;        /* F1: NSSO_MUT_HRSS (default) or NSSO_MUT_RW */
} nsso_config;

enum { NSSO_MUT_HRSS = 0, NSSO_MUT_RW = 1 };

typedef struct {
  int64_t iteration;       /* iterations completed                       */
  double e_star;           /* threshold of the last iteration            */
  int64_t probes, energy_evals, expansions, shrinks, null_moves, init_evals;
  double log_z_det;        /* replica 0 accumulated log Z                */
  double log_z_live;       /* -min E_live + log X (replica 0)            */
  int32_t terminated;
  int32_t finalised;
} nsso_step_info;

typedef struct nsso_ctx nsso_ctx;

/* ---- sampler (same call set as include/nss.h, prefix nsso_) ---- */
int nsso_init(const nsso_prior *prior, const nsso_energy *energy,
              const nsso_config *cfg, nsso_ctx **out);
/* Same, but draw_live = 0 skips the prior draws: the live set is all zeros
 * until nsso_set_live (for full-size parity cases whose energies are too
 * slow to draw n of in the oracle). */
int nsso_init_ex(const nsso_prior *prior, const nsso_energy *energy,
                 const nsso_config *cfg, int draw_live, nsso_ctx **out);
int nsso_step(nsso_ctx *ctx, nsso_step_info *info);

/* ---- F3: adaptive tempered SMC with the HRSS kernel (SMC-SS) ----
 * A context whose n_live particles start as prior draws (as nsso_init) and
 * move through pi_beta ~ Pi exp(-beta E): each stage picks the next beta by
 * bisection on ESS = rho m (nsso_smc_next_beta), adds log mean w to log Z,
 * resamples multinomially (uniform 0 of stream (stage, j, SMC = 7, 0)),
 * recomputes the metric from the resampled particles and applies `steps`
 * tempered HRSS steps per particle (slice of Pi exp(-beta E), no threshold).
 * k is unused (give 1). nsso_smc_stage returns STATE once beta = 1. */
int nsso_smc_init(const nsso_prior *prior, const nsso_energy *energy, const nsso_config *cfg, double rho,
                  nsso_ctx **out);
int nsso_smc_stage(nsso_ctx *ctx);
int nsso_smc_state(nsso_ctx *ctx, double *beta, double *log_z, int64_t *stage, int32_t *parents /* n */);
int nsso_smc_next_beta(const double *E, int64_t m, double beta_t, double rho, double *beta_next);
int nsso_run(nsso_ctx *ctx, int64_t max_iters, nsso_step_info *info);
int nsso_finalise(nsso_ctx *ctx);
int nsso_evidence(nsso_ctx *ctx, double *log_z, double *log_z_err);
int nsso_evidence_reps(nsso_ctx *ctx, double *log_z_reps /* R+1 */);
int nsso_samples(nsso_ctx *ctx, double *x, double *log_w, int64_t cap, int64_t *n_out);
/* F2 posterior products at inverse temperature beta: log Z(beta) mean/std over
 * the R replicas, Kish ESS of the geometric-mean weights, normalised log
 * weights (nullable, cap >= n_dead). */
int nsso_posterior(nsso_ctx *ctx, double beta, double *log_z, double *log_z_err, double *ess,
                   double *log_w, int64_t cap);
/* m equal-weight multinomial draws from the beta-weights; idx and/or x (m*d). */
int nsso_resample(nsso_ctx *ctx, double beta, int64_t m, uint64_t seed, int64_t *idx, double *x);
int nsso_info(nsso_ctx *ctx, nsso_step_info *info);
int nsso_should_terminate(nsso_ctx *ctx, int32_t *flag);
void nsso_destroy(nsso_ctx *ctx);

/* ---- parity hooks ---- */
int nsso_set_live(nsso_ctx *ctx, const double *x, const double *e, int64_t next_iteration);
int nsso_get_live(nsso_ctx *ctx, double *x, double *e);
int nsso_get_metric(nsso_ctx *ctx, double *chol /* d*d lower */, double *width);
/* Restrict the next nsso_step's HRSS to a subset of chains (ordinals into the
 * ascending destination list); count < 0 restores "all chains". */
int nsso_set_chain_subset(nsso_ctx *ctx, const int32_t *chains, int64_t count);
/* Trace of the last iteration: dead gids (key-descending), destinations
 * (ascending gid; all n gids when update_all), parent gid per destination
 * (itself for a surviving slot), per (chain, step) counts
 * packed as {n_left, n_right, n_shrink, accepted} and the smallest relative
 * decision margin seen in that step. Any pointer may be NULL. */
int nsso_get_trace(nsso_ctx *ctx, int32_t *dead_gid, int32_t *dest_gid, int32_t *parent_gid,
                   uint8_t *counts /* k*p*4 */, double *min_margin /* k*p */, double *e_star);
/* Current log X of every volume replica r = 0..R (replica 0 deterministic). */
int nsso_volume_reps(nsso_ctx *ctx, double *log_x /* R+1 */);
/* HRSS direction of stream (iter, gid, HRSS, step) under the current metric. */
int nsso_direction(nsso_ctx *ctx, uint32_t iter, uint32_t gid, uint32_t step, double *v);
int nsso_dead(nsso_ctx *ctx, double *e, int32_t *n_live, double *birth, int32_t *gid,
              double *x, int64_t cap, int64_t *n_out);

/* ---- unit hooks for the pins ---- */
void nsso_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint32_t nsso_draw_u32(uint64_t seed, uint32_t iter, uint32_t gid, uint32_t phase,
                       uint32_t sub, uint32_t q);
double nsso_draw_uniform(uint64_t seed, uint32_t iter, uint32_t gid, uint32_t phase,
                         uint32_t sub, uint32_t q);
void nsso_draw_normals(uint64_t seed, uint32_t iter, uint32_t gid, uint32_t phase,
                       uint32_t sub, int32_t d, double *z);
double nsso_energy_at(nsso_ctx *ctx, const double *x);
double nsso_log_prior_at(nsso_ctx *ctx, const double *x);
/* One HRSS step from x0 along the given direction v with width w
 * under threshold e_star, drawing u_h, u_b and shrink uniforms from stream
 * (iter, gid, HRSS, step).  counts = {n_left, n_right, n_shrink, accepted}. */
/* One constrained Gaussian random-walk proposal (F1):
 * x' = x0 + sigma L z with sigma = c 2.38 / sqrt(d) (c = cfg.width), z from
 * the normals of stream (iter, gid, RW = 6, step); accepted iff x' is in the
 * prior support, ln u < log Pi(x') - log Pi(x0) (u = draw h = 2 ceil(d/2))
 * and E(x') < E*; the energy is evaluated only if the prior test passes.
 * counts = {0, 0, evaluated, accepted}. */
int nsso_rw_step(nsso_ctx *ctx, const double *x0, double e0, double e_star, uint32_t iter, uint32_t gid,
                 uint32_t step, double *x_out, double *e_out, int32_t counts[4]);
int nsso_slice_step(nsso_ctx *ctx, const double *x0, double e0, const double *v, double w,
                    double e_star, uint32_t iter, uint32_t gid, uint32_t step,
                    double *x_out, double *e_out, int32_t counts[4]);

#ifdef __cplusplus
}
#endif
#endif
