/*
 * oracle/nsso.c -- plain, slow, fp64, single-threaded Nested Slice Sampling.
 *
 * TEST INFRASTRUCTURE ONLY (see nsso.h).  Written from PAPER.md in the paper's
 * order and notation; no blocking, fusion or reordering.  "P:n" cites
 * /root/reference/PAPER.md line n; "DESIGN R-n" cites a reading recorded in
 * DESIGN.md section 2 where the paper is silent or ambiguous.
 *
 * Parity status of each function is listed in DESIGN.md section 4.  The GP
 * and logistic-regression energies are pinned only on tiny cases (brute-force
 * quadrature, closed forms), at full scale they are "parity unpinned".
 */
#include "nsso.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PI_D 3.14159265358979323846
#define LN2PI_D 1.83787706640934548356
/* kappa_infinity as printed in the paper, P:2125 ("kappa_infty ~ 1.3035"). */
#define KAPPA_INF_PAPER 1.3035

enum { PH_INIT = 1, PH_RESAMPLE = 2, PH_HRSS = 3, PH_VOLUME = 4, PH_POSTERIOR = 5, PH_RW = 6, PH_SMC = 7 };

/* ------------------------------------------------------------------------ */
/* Counter-based RNG: Philox4x32-10 (Salmon et al. 2011). */
/* ------------------------------------------------------------------------ */
void nsso_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Draw #q of stream (iter, gid, phase, sub): word q&3 of block q>>2. */
uint32_t nsso_draw_u32(uint64_t seed, uint32_t iter, uint32_t gid, uint32_t phase,
                       uint32_t sub, uint32_t q) {
  uint32_t ctr[4] = {q >> 2, (phase << 24) | (sub & 0xFFFFFFu), gid, iter};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t out[4];
  nsso_philox(ctr, key, out);
  return out[q & 3];
}

/* u = ((r >> 9) + 1/2) * 2^-23 = (2 (r>>9) + 1) * 2^-24: a 24-bit odd integer
 * times 2^-24, strictly inside (0, 1) and exact in fp32. */
double nsso_draw_uniform(uint64_t seed, uint32_t iter, uint32_t gid, uint32_t phase,
                         uint32_t sub, uint32_t q) {
  uint32_t r = nsso_draw_u32(seed, iter, gid, phase, sub, q);
  return ((double)(r >> 9) + 0.5) * (1.0 / 8388608.0);
}

/* Box-Muller on draws (2i, 2i+1). */
void nsso_draw_normals(uint64_t seed, uint32_t iter, uint32_t gid, uint32_t phase,
                       uint32_t sub, int32_t d, double *z) {
  for (int32_t i = 0; 2 * i < d; ++i) {
    double u1 = nsso_draw_uniform(seed, iter, gid, phase, sub, (uint32_t)(2 * i));
    double u2 = nsso_draw_uniform(seed, iter, gid, phase, sub, (uint32_t)(2 * i + 1));
    double r = sqrt(-2.0 * log(u1));
    z[2 * i] = r * cos(2.0 * PI_D * u2);
    if (2 * i + 1 < d) z[2 * i + 1] = r * sin(2.0 * PI_D * u2);
  }
}

/* ------------------------------------------------------------------------ */
/* Context                                                                   */
/* ------------------------------------------------------------------------ */
struct nsso_ctx {
  int d;
  int64_t n, k;
  nsso_config cfg;
  /* prior */
  int prior_kind;
  double *lo, *hi, *pmean, *psd;
  /* energy (copied) */
  nsso_energy en;
  double *e_w, *e_mu, *e_sigma, *e_prec, *e_x, *e_y;
  /* live set */
  double *X, *E, *birth;
  /* metric: Sigma = L L^T (DESIGN R-5) and the slice width */
  double *L;
  double w;
  int64_t iter;   /* iterations completed; the next one has index iter+1 */
  /* dead store */
  int64_t n_dead;
  double *dE, *dbirth, *dX;
  int32_t *dnlive, *dgid, *dord;
  int64_t *diter;
  /* evidence replicas r = 0..R */
  int R;
  double *lx_prev, *lx_cur, *lz;
  double pend_e;
  int has_pend;
  int finalised;
  /* counters */
  int64_t probes, evals, expansions, shrinks, nulls, init_evals;
  double e_star;
  /* trace of the last iteration */
  int32_t *t_dead, *t_dest, *t_parent;
  uint8_t *t_counts;
  double *t_margin;
  int32_t *subset;
  int64_t n_subset; /* -1 = all */
  int nan_seen;
  /* F3 tempered SMC-SS: particles are X/E, beta, accumulated log Z */
  int smc;
  double smc_rho, beta, smc_logz;
  int32_t *smc_par; /* resampled parent of every particle, last stage */
};

static void *xcalloc(size_t n, size_t sz) { return calloc(n ? n : 1, sz); }
static double *dup_d(const double *src, size_t n) {
  if (!src) return NULL;
  double *p = (double *)xcalloc(n, sizeof(double));
  memcpy(p, src, n * sizeof(double));
  return p;
}

/* ------------------------------------------------------------------------ */
/* Reference density Pi and energy E                                          */
/* ------------------------------------------------------------------------ */
/* log Pi(x); -inf outside the support. */
static double log_prior(const nsso_ctx *c, const double *x) {
  int d = c->d;
  if (c->prior_kind == NSSO_PRIOR_BOX) {
    double lp = 0.0;
    for (int i = 0; i < d; ++i) {
      if (!(x[i] >= c->lo[i] && x[i] <= c->hi[i])) return -INFINITY;
      lp -= log(c->hi[i] - c->lo[i]);
    }
    return lp;
  }
  double lp = 0.0;
  for (int i = 0; i < d; ++i) {
    double t = (x[i] - c->pmean[i]) / c->psd[i];
    lp += -0.5 * t * t - log(c->psd[i]) - 0.5 * LN2PI_D;
  }
  return lp;
}

static double softplus(double a) { return a > 0 ? a + log1p(exp(-a)) : log1p(exp(a)); }

/* E(x) = -log L(x). */
static double energy(const nsso_ctx *c, const double *x) {
  const nsso_energy *en = &c->en;
  int d = c->d;
  switch (en->kind) {
    case NSSO_E_FLAT:
      return en->c;
    case NSSO_E_GAUSS: {
      double s = 0.0;
      for (int i = 0; i < d; ++i) {
        double t = (x[i] - c->e_mu[i]) / c->e_sigma[i];
        s += t * t;
      }
      return 0.5 * s + en->c;
    }
    case NSSO_E_MOG: {
      /* -log sum_j w_j prod_i N(x_i; mu_ji, sigma_ji^2) via log-sum-exp */
      int K = en->n_comp;
      double *lj = (double *)xcalloc((size_t)K, sizeof(double));
      double m = -INFINITY;
      for (int j = 0; j < K; ++j) {
        double s = log(c->e_w[j]);
        for (int i = 0; i < d; ++i) {
          double sg = c->e_sigma[j * d + i];
          double t = (x[i] - c->e_mu[j * d + i]) / sg;
          s += -0.5 * t * t - log(sg) - 0.5 * LN2PI_D;
        }
        lj[j] = s;
        if (s > m) m = s;
      }
      double acc = 0.0;
      for (int j = 0; j < K; ++j) acc += exp(lj[j] - m);
      free(lj);
      return -(m + log(acc));
    }
    case NSSO_E_CORR_GAUSS: {
      double q = 0.0;
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
          q += (x[i] - c->e_mu[i]) * c->e_prec[i * d + j] * (x[j] - c->e_mu[j]);
      return 0.5 * q + en->c;
    }
    case NSSO_E_FUNNEL: {
      /* N(y|0,3) prod_n N(x_n|0, exp(y/2)), second argument = sd
       * (DESIGN R-23); y = x[0]. */
      double y = x[0], sy = en->sigma_y;
      double e = 0.5 * (y / sy) * (y / sy) + log(sy) + 0.5 * LN2PI_D;
      for (int i = 1; i < d; ++i) e += 0.5 * x[i] * x[i] * exp(-y) + 0.5 * y + 0.5 * LN2PI_D;
      return e;
    }
    case NSSO_E_LOGREG: {
      double e = 0.0;
      for (int64_t r = 0; r < en->n_data; ++r) {
        double a = 0.0;
        for (int i = 0; i < d; ++i) a += c->e_x[r * d + i] * x[i];
        e += softplus(a) - c->e_y[r] * a;
      }
      return e;
    }
    case NSSO_E_GP_ARD: {
      /* phi = (log l_1..l_D, log sigma_f, log sigma_n).
       * K_ab = sf^2 exp(-1/2 sum_j ((X_aj - X_bj)/l_j)^2) + (sn^2 + jitter) delta_ab
       * E = 1/2 y^T K^-1 y + 1/2 log|K| + N/2 log 2pi. */
      int D = en->d_in;
      int64_t N = en->n_data;
      double sf2 = exp(2.0 * x[D]), sn2 = exp(2.0 * x[D + 1]);
      double *il = (double *)xcalloc((size_t)D, sizeof(double));
      for (int j = 0; j < D; ++j) il[j] = exp(-x[j]);
      double *K = (double *)xcalloc((size_t)(N * N), sizeof(double));
      for (int64_t a = 0; a < N; ++a)
        for (int64_t b = 0; b < N; ++b) {
          double s = 0.0;
          for (int j = 0; j < D; ++j) {
            double t = (c->e_x[a * D + j] - c->e_x[b * D + j]) * il[j];
            s += t * t;
          }
          K[a * N + b] = sf2 * exp(-0.5 * s) + (a == b ? sn2 + en->jitter : 0.0);
        }
      /* Cholesky K = G G^T, lower, in place (textbook Cholesky-Banachiewicz) */
      double logdet = 0.0;
      for (int64_t i = 0; i < N; ++i) {
        for (int64_t j = 0; j <= i; ++j) {
          double s = K[i * N + j];
          for (int64_t t = 0; t < j; ++t) s -= K[i * N + t] * K[j * N + t];
          if (i == j) {
            if (!(s > 0.0)) { free(K); free(il); return INFINITY; }
            K[i * N + i] = sqrt(s);
            logdet += 2.0 * log(K[i * N + i]);
          } else {
            K[i * N + j] = s / K[j * N + j];
          }
        }
      }
      /* alpha = G^-1 y; y^T K^-1 y = |alpha|^2 */
      double quad = 0.0;
      double *al = (double *)xcalloc((size_t)N, sizeof(double));
      for (int64_t i = 0; i < N; ++i) {
        double s = c->e_y[i];
        for (int64_t t = 0; t < i; ++t) s -= K[i * N + t] * al[t];
        al[i] = s / K[i * N + i];
        quad += al[i] * al[i];
      }
      free(al); free(K); free(il);
      return 0.5 * quad + 0.5 * logdet + 0.5 * (double)N * LN2PI_D;
    }
  }
  return NAN;
}

double nsso_energy_at(nsso_ctx *c, const double *x) { return energy(c, x); }
double nsso_log_prior_at(nsso_ctx *c, const double *x) { return log_prior(c, x); }

/* ------------------------------------------------------------------------ */
/* Metric: empirical covariance of the live set with ridge regularisation    */
/* (DESIGN R-5, R-8), Cholesky, and the slice width rule          */
/* (DESIGN R-7).                                                  */
/* ------------------------------------------------------------------------ */
static int cholesky_lower(const double *A, double *G, int d) {
  memset(G, 0, sizeof(double) * (size_t)d * (size_t)d);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = A[i * d + j];
      for (int t = 0; t < j; ++t) s -= G[i * d + t] * G[j * d + t];
      if (i == j) {
        if (!(s > 0.0) || !isfinite(s)) return 0;
        G[i * d + i] = sqrt(s);
      } else {
        G[i * d + j] = s / G[j * d + j];
      }
    }
  return 1;
}

static void compute_metric(nsso_ctx *c) {
  int d = c->d;
  int64_t n = c->n;
  double *mean = (double *)xcalloc((size_t)d, sizeof(double));
  double *S = (double *)xcalloc((size_t)d * d, sizeof(double));
  for (int64_t g = 0; g < n; ++g)
    for (int i = 0; i < d; ++i) mean[i] += c->X[g * d + i];
  for (int i = 0; i < d; ++i) mean[i] /= (double)n;
  for (int64_t g = 0; g < n; ++g)
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j)
        S[i * d + j] += (c->X[g * d + i] - mean[i]) * (c->X[g * d + j] - mean[j]);
  for (int i = 0; i < d * d; ++i) S[i] /= (double)(n - 1);
  double md = 0.0;
  for (int i = 0; i < d; ++i) md += S[i * d + i];
  md /= (double)d;
  for (int i = 0; i < d; ++i) S[i * d + i] += c->cfg.metric_reg * md;
  if (!cholesky_lower(S, c->L, d)) {
    /* fallback: diagonal of the sample variances (1 where a variance is 0) */
    memset(c->L, 0, sizeof(double) * (size_t)d * d);
    for (int i = 0; i < d; ++i) c->L[i * d + i] = S[i * d + i] > 0.0 ? sqrt(S[i * d + i]) : 1.0;
  }
  /* width */
  if (c->cfg.width_rule == NSSO_W_FIXED) {
    c->w = c->cfg.width;
  } else {
    double mu;
    if (c->cfg.dir_norm == NSSO_DIR_MAHALANOBIS) {
      /* whitened live set has covariance I: uniform ball of radius sqrt(d+2),
       * A = I/(d+2), mu = 1/(d+2)  (DESIGN R-7) */
      mu = 1.0 / (double)(d + 2);
    } else {
      /* A = Sigma^-1/(d+2), mu = tr(Sigma^-1)/(d(d+2)); tr(Sigma^-1) = |L^-1|_F^2 */
      double *Li = (double *)xcalloc((size_t)d * d, sizeof(double));
      for (int col = 0; col < d; ++col)
        for (int i = 0; i < d; ++i) {
          double s = (i == col) ? 1.0 : 0.0;
          for (int t = 0; t < i; ++t) s -= c->L[i * d + t] * Li[t * d + col];
          Li[i * d + col] = s / c->L[i * d + i];
        }
      double tr = 0.0;
      for (int i = 0; i < d * d; ++i) tr += Li[i] * Li[i];
      free(Li);
      mu = tr / ((double)d * (double)(d + 2));
    }
    /* w* = 4 kappa_inf sqrt(2/(pi mu d)) */
    c->w = c->cfg.width * 4.0 * KAPPA_INF_PAPER * sqrt(2.0 / (PI_D * mu * (double)d));
  }
  free(mean);
  free(S);
}

/* ------------------------------------------------------------------------ */
/* Hit-and-Run Slice Sampling step (Thm P:1861-1925)    */
/* ------------------------------------------------------------------------ */
typedef struct {
  nsso_ctx *c;
  const double *x;   /* current point */
  const double *v;   /* direction */
  double log_y;      /* slice height */
  double e_star;
  double *xp;        /* scratch: x + t v */
  double e_last;     /* energy at the last in() point that passed the prior */
  double min_margin; /* smallest relative decision margin seen */
  int64_t probes, evals;
  int tempered;      /* F3: slice of Pi exp(-beta E), no hard threshold */
  double beta;
} slice_ctx;

static double fabs_max1(double a) { a = fabs(a); return a > 1.0 ? a : 1.0; }

/* in(t): x+tv in the support, log Pi(x+tv) >= log y and E(x+tv) < E*.
 * E is evaluated only if the prior tests pass (DESIGN R-11). */
static int in_slice(slice_ctx *s, double t) {
  nsso_ctx *c = s->c;
  int d = c->d;
  s->probes++;
  for (int i = 0; i < d; ++i) s->xp[i] = s->x[i] + t * s->v[i];
  if (c->prior_kind == NSSO_PRIOR_BOX) {
    for (int i = 0; i < d; ++i) {
      double span = c->hi[i] - c->lo[i];
      double m = fmin(s->xp[i] - c->lo[i], c->hi[i] - s->xp[i]) / span;
      if (fabs(m) < s->min_margin) s->min_margin = fabs(m);
    }
  }
  double lp = log_prior(c, s->xp);
  if (s->tempered) {
    /* F3: x + t v in the support and log Pi - beta E >= log y */
    if (!(lp > -INFINITY)) return 0;
    double e = energy(c, s->xp);
    s->evals++;
    if (isnan(e)) { c->nan_seen = 1; return 0; }
    double f = lp - s->beta * e;
    double m = (f - s->log_y) / fabs_max1(s->log_y);
    if (fabs(m) < s->min_margin) s->min_margin = fabs(m);
    s->e_last = e;
    return f >= s->log_y;
  }
  if (c->prior_kind == NSSO_PRIOR_GAUSS_DIAG) {
    double m = (lp - s->log_y) / fabs_max1(s->log_y);
    if (fabs(m) < s->min_margin) s->min_margin = fabs(m);
  }
  if (!(lp >= s->log_y)) return 0;
  double e = energy(c, s->xp);
  s->evals++;
  if (isnan(e)) { c->nan_seen = 1; return 0; }
  double m = (s->e_star - e) / fabs_max1(s->e_star);
  if (fabs(m) < s->min_margin) s->min_margin = fabs(m);
  s->e_last = e;
  return e < s->e_star;
}

/* One HRSS step along direction v with width w.  Draw map of stream
 * (iter, gid, HRSS, step): h = 2*ceil(d/2) -> u_h (slice height), h+1 -> u_b
 * (bracket offset), h+2+i -> i-th shrink uniform. */
static int slice_step(nsso_ctx *c, const double *x0, double e0, const double *v, double w,
                      double e_star, uint32_t iter, uint32_t gid, uint32_t step,
                      double *x_out, double *e_out, int32_t counts[4], double *min_margin) {
  int d = c->d;
  uint64_t seed = c->cfg.seed;
  uint32_t h = (uint32_t)(2 * ((d + 1) / 2));
  slice_ctx s;
  s.c = c; s.x = x0; s.v = v; s.e_star = e_star;
  s.xp = (double *)xcalloc((size_t)d, sizeof(double));
  s.min_margin = INFINITY; s.probes = 0; s.evals = 0; s.e_last = NAN;
  s.tempered = c->smc; s.beta = c->beta;
  /* slice height: log y = log Pi(x) + ln u_h  (DESIGN R-9); tempered
   * (F3): log y = log Pi(x) - beta E(x) + ln u_h */
  double u_h = nsso_draw_uniform(seed, iter, gid, PH_HRSS, step, h);
  s.log_y = log_prior(c, x0) - (s.tempered ? s.beta * e0 : 0.0) + log(u_h);
  /* randomised initial bracket of width w around t = 0:
   * [-U, w - U], U = w u_b */
  double u_b = nsso_draw_uniform(seed, iter, gid, PH_HRSS, step, h + 1);
  double lft = -w * u_b;
  double rgt = lft + w;
  /* linear stepping-out, capped at max_stepout per side */
  int nl = 0, nr = 0;
  while (nl < c->cfg.max_stepout && in_slice(&s, lft)) { lft -= w; nl++; }
  while (nr < c->cfg.max_stepout && in_slice(&s, rgt)) { rgt += w; nr++; }
  /* shrinkage, capped at max_shrink; null move when the cap is hit */
  int accepted = 0, ns = 0;
  double e_new = e0;
  for (int i = 0; i < c->cfg.max_shrink; ++i) {
    double u = nsso_draw_uniform(seed, iter, gid, PH_HRSS, step, h + 2 + (uint32_t)i);
    double t = lft + u * (rgt - lft);
    ns++;
    if (in_slice(&s, t)) {
      for (int q = 0; q < d; ++q) x_out[q] = s.xp[q];
      e_new = s.e_last;
      accepted = 1;
      break;
    }
    if (t < 0.0) lft = t; else rgt = t;  /* DESIGN R-13 */
  }
  if (!accepted) {
    for (int q = 0; q < d; ++q) x_out[q] = x0[q];
    e_new = e0;
  }
  *e_out = e_new;
  counts[0] = nl; counts[1] = nr; counts[2] = ns; counts[3] = accepted;
  c->probes += s.probes;
  c->evals += s.evals;
  c->expansions += nl + nr;
  c->shrinks += ns;
  c->nulls += accepted ? 0 : 1;
  if (min_margin) *min_margin = s.min_margin;
  free(s.xp);
  return NSSO_OK;
}

/* F1 constrained random walk ("constrained Gaussian random-walk
 * baseline"; "Gaussian proposal with covariance matched to the target
 * and scaled optimally, rejecting proposals that violate the constraint"):
 * proposal covariance (c 2.38)^2/d Sigma_hat (Roberts-Gelman-Gilks scaling
 * with the live-set covariance as the matched covariance), Metropolis
 * acceptance for the prior restricted to E < E*. */
static int rw_step(nsso_ctx *c, const double *x0, double e0, double e_star, uint32_t iter, uint32_t gid,
                   uint32_t step, double *x_out, double *e_out, int32_t counts[4], double *min_margin) {
  int d = c->d;
  uint32_t h = (uint32_t)(2 * ((d + 1) / 2));
  double *z = (double *)xcalloc((size_t)d + 1, sizeof(double));
  double *xp = (double *)xcalloc((size_t)d, sizeof(double));
  nsso_draw_normals(c->cfg.seed, iter, gid, PH_RW, step, d, z);
  double u = nsso_draw_uniform(c->cfg.seed, iter, gid, PH_RW, step, h);
  double sigma = c->cfg.width * 2.38 / sqrt((double)d);
  for (int i = 0; i < d; ++i) {
    double s = 0.0;
    for (int j = 0; j <= i; ++j) s += c->L[i * d + j] * z[j];
    xp[i] = x0[i] + sigma * s;
  }
  c->probes++;
  double lp0 = log_prior(c, x0), lpp = log_prior(c, xp);
  double mm = INFINITY;
  int evaluated = 0, accepted = 0;
  double en = NAN;
  if (c->prior_kind == NSSO_PRIOR_BOX) {
    for (int i = 0; i < d; ++i) {
      double span = c->hi[i] - c->lo[i];
      double m = fmin(xp[i] - c->lo[i], c->hi[i] - xp[i]) / span;
      if (fabs(m) < mm) mm = fabs(m);
    }
  } else {
    double m = (lpp - lp0 - log(u)) / fabs_max1(lp0);
    if (fabs(m) < mm) mm = fabs(m);
  }
  if (lpp > -INFINITY && log(u) < lpp - lp0) {
    en = energy(c, xp);
    evaluated = 1;
    c->evals++;
    if (isnan(en)) c->nan_seen = 1;
    else {
      double m = (e_star - en) / fabs_max1(e_star);
      if (fabs(m) < mm) mm = fabs(m);
      accepted = en < e_star;
    }
  }
  if (accepted) {
    memcpy(x_out, xp, sizeof(double) * (size_t)d);
    *e_out = en;
  } else {
    memcpy(x_out, x0, sizeof(double) * (size_t)d);
    *e_out = e0;
    c->nulls++;
  }
  counts[0] = 0; counts[1] = 0; counts[2] = evaluated; counts[3] = accepted;
  if (min_margin) *min_margin = mm;
  free(z); free(xp);
  return NSSO_OK;
}

int nsso_rw_step(nsso_ctx *c, const double *x0, double e0, double e_star, uint32_t iter, uint32_t gid,
                 uint32_t step, double *x_out, double *e_out, int32_t counts[4]) {
  if (!c) return NSSO_ERR_INVALID_ARG;
  return rw_step(c, x0, e0, e_star, iter, gid, step, x_out, e_out, counts, NULL);
}

int nsso_slice_step(nsso_ctx *c, const double *x0, double e0, const double *v, double w,
                    double e_star, uint32_t iter, uint32_t gid, uint32_t step,
                    double *x_out, double *e_out, int32_t counts[4]) {
  return slice_step(c, x0, e0, v, w, e_star, iter, gid, step, x_out, e_out, counts, NULL);
}

/* Direction v = L z / |z| (Mahalanobis, DESIGN R-6) or L z / |L z| (Euclidean),
 * z ~ N(0, I_d) from stream (iter, gid, HRSS, step) draws 0..2ceil(d/2)-1. */
static void direction(nsso_ctx *c, uint32_t iter, uint32_t gid, uint32_t step, double *z,
                      double *v) {
  int d = c->d;
  nsso_draw_normals(c->cfg.seed, iter, gid, PH_HRSS, step, d, z);
  double zz = 0.0;
  for (int i = 0; i < d; ++i) zz += z[i] * z[i];
  double vv = 0.0;
  for (int i = 0; i < d; ++i) {
    double s = 0.0;
    for (int j = 0; j <= i; ++j) s += c->L[i * d + j] * z[j];
    v[i] = s;
    vv += s * s;
  }
  double nrm = c->cfg.dir_norm == NSSO_DIR_MAHALANOBIS ? sqrt(zz) : sqrt(vv);
  for (int i = 0; i < d; ++i) v[i] /= nrm;
}

/* ------------------------------------------------------------------------ */
/* Evidence: unrolled batch deaths, simulated shrinkage         */
/* (P:1208-1227), trapezoid or rectangle quadrature  */
/* ------------------------------------------------------------------------ */
static double lse2(double a, double b) {
  if (a == -INFINITY) return b;
  if (b == -INFINITY) return a;
  double m = a > b ? a : b;
  return m + log(exp(a - m) + exp(b - m));
}
/* log(1 - exp(a)), a < 0 */
static double log1mexp(double a) { return a > -0.6931471805599453 ? log(-expm1(a)) : log1p(-exp(a)); }

/* Log-volume increment of a single death with n_live live points:
 * replica 0 uses E[log t] = -1/n_live; replica r >= 1 draws t ~ Beta(n_live, 1),
 * log t = ln(u)/n_live with u = draw 0 of stream (iter, ordinal, VOLUME, r). */
static double dlogx(const nsso_ctx *c, int r, int64_t nlive, uint32_t iter, uint32_t ord) {
  if (r == 0) return -1.0 / (double)nlive;
  double u = nsso_draw_uniform(c->cfg.seed, iter, ord, PH_VOLUME, (uint32_t)r, 0);
  return log(u) / (double)nlive;
}

/* Feed one death (energy e) into every replica's quadrature. */
static void evidence_death(nsso_ctx *c, double e, int64_t nlive, uint32_t iter, uint32_t ord) {
  for (int r = 0; r <= c->R; ++r) {
    double lx_new = c->lx_cur[r] + dlogx(c, r, nlive, iter, ord);
    if (c->cfg.quadrature == NSSO_Q_RECTANGLE) {
      /* Delta X_i = X_{i-1} - X_i */
      double term = -e + c->lx_cur[r] + log1mexp(lx_new - c->lx_cur[r]);
      c->lz[r] = lse2(c->lz[r], term);
    } else if (c->has_pend) {
      /* dX_i = (X_{i-1} - X_{i+1}) / 2 for the pending point i */
      double term = -c->pend_e + c->lx_prev[r] + log1mexp(lx_new - c->lx_prev[r]) - log(2.0);
      c->lz[r] = lse2(c->lz[r], term);
    }
    c->lx_prev[r] = c->lx_cur[r];
    c->lx_cur[r] = lx_new;
  }
  c->pend_e = e;
  c->has_pend = 1;
}

/* log Z of replica r with the pending trapezoid point closed by X_{N+1} = 0. */
static double closed_logz(const nsso_ctx *c, int r) {
  if (c->cfg.quadrature == NSSO_Q_RECTANGLE || !c->has_pend) return c->lz[r];
  return lse2(c->lz[r], -c->pend_e + c->lx_prev[r] - log(2.0));
}

/* ------------------------------------------------------------------------ */
/* Init (DESIGN R-20): rejection from the prior until E is finite            */
/* ------------------------------------------------------------------------ */
static int prior_draw(nsso_ctx *c, uint32_t gid, uint32_t attempt, double *x) {
  int d = c->d;
  if (c->prior_kind == NSSO_PRIOR_BOX) {
    for (int i = 0; i < d; ++i) {
      double u = nsso_draw_uniform(c->cfg.seed, 0, gid, PH_INIT, attempt, (uint32_t)i);
      x[i] = c->lo[i] + u * (c->hi[i] - c->lo[i]);
    }
  } else {
    nsso_draw_normals(c->cfg.seed, 0, gid, PH_INIT, attempt, d, x);
    for (int i = 0; i < d; ++i) x[i] = c->pmean[i] + c->psd[i] * x[i];
  }
  return 0;
}

static int validate(const nsso_prior *p, const nsso_energy *e, const nsso_config *cfg) {
  if (!p || !e || !cfg) return 0;
  int d = p->d;
  if (d < 1 || e->d != d) return 0;
  if (cfg->n_live < 2 || cfg->k < 1 || cfg->k > cfg->n_live - 1) return 0;
  if (cfg->steps < 0 || cfg->max_stepout < 1 || cfg->max_shrink < 1) return 0;
  if (cfg->n_volume_sims < 2) return 0;
  if (!(cfg->width > 0.0)) return 0;
  if (cfg->max_dead < cfg->n_live) return 0;
  if (cfg->update_all != 0 && cfg->update_all != 1) return 0;
  if (cfg->mutation != NSSO_MUT_HRSS && cfg->mutation != NSSO_MUT_RW) return 0;
  if (p->kind == NSSO_PRIOR_BOX) {
    if (!p->lo || !p->hi) return 0;
    for (int i = 0; i < d; ++i) if (!(p->lo[i] < p->hi[i])) return 0;
  } else if (p->kind == NSSO_PRIOR_GAUSS_DIAG) {
    if (!p->mean || !p->sd) return 0;
    for (int i = 0; i < d; ++i) if (!(p->sd[i] > 0.0)) return 0;
  } else {
    return 0;
  }
  switch (e->kind) {
    case NSSO_E_FLAT: case NSSO_E_FUNNEL: break;
    case NSSO_E_GAUSS: if (!e->mu || !e->sigma) return 0; break;
    case NSSO_E_MOG: if (e->n_comp < 1 || !e->w || !e->mu || !e->sigma) return 0; break;
    case NSSO_E_CORR_GAUSS: if (!e->mu || !e->prec) return 0; break;
    case NSSO_E_LOGREG: if (e->n_data < 1 || !e->data_x || !e->data_y) return 0; break;
    case NSSO_E_GP_ARD:
      if (e->n_data < 1 || e->d_in < 1 || d != e->d_in + 2 || !e->data_x || !e->data_y) return 0;
      break;
    default: return 0;
  }
  return 1;
}

int nsso_init(const nsso_prior *p, const nsso_energy *e, const nsso_config *cfg, nsso_ctx **out) {
  return nsso_init_ex(p, e, cfg, 1, out);
}

int nsso_init_ex(const nsso_prior *p, const nsso_energy *e, const nsso_config *cfg, int draw_live,
                 nsso_ctx **out) {
  if (!out) return NSSO_ERR_INVALID_ARG;
  *out = NULL;
  if (!validate(p, e, cfg)) return NSSO_ERR_INVALID_ARG;
  nsso_ctx *c = (nsso_ctx *)xcalloc(1, sizeof(nsso_ctx));
  int d = p->d;
  c->d = d; c->n = cfg->n_live; c->k = cfg->k; c->cfg = *cfg;
  c->prior_kind = p->kind;
  c->lo = dup_d(p->lo, (size_t)d); c->hi = dup_d(p->hi, (size_t)d);
  c->pmean = dup_d(p->mean, (size_t)d); c->psd = dup_d(p->sd, (size_t)d);
  c->en = *e;
  int K = e->n_comp > 0 ? e->n_comp : 1;
  if (e->kind == NSSO_E_MOG) {
    c->e_w = dup_d(e->w, (size_t)K);
    c->e_mu = dup_d(e->mu, (size_t)K * d);
    c->e_sigma = dup_d(e->sigma, (size_t)K * d);
  } else if (e->kind == NSSO_E_GAUSS) {
    c->e_mu = dup_d(e->mu, (size_t)d); c->e_sigma = dup_d(e->sigma, (size_t)d);
  } else if (e->kind == NSSO_E_CORR_GAUSS) {
    c->e_mu = dup_d(e->mu, (size_t)d); c->e_prec = dup_d(e->prec, (size_t)d * d);
  } else if (e->kind == NSSO_E_LOGREG) {
    c->e_x = dup_d(e->data_x, (size_t)(e->n_data * d)); c->e_y = dup_d(e->data_y, (size_t)e->n_data);
  } else if (e->kind == NSSO_E_GP_ARD) {
    c->e_x = dup_d(e->data_x, (size_t)(e->n_data * e->d_in));
    c->e_y = dup_d(e->data_y, (size_t)e->n_data);
  }
  int64_t n = c->n, k = c->k;
  c->X = (double *)xcalloc((size_t)(n * d), sizeof(double));
  c->E = (double *)xcalloc((size_t)n, sizeof(double));
  c->birth = (double *)xcalloc((size_t)n, sizeof(double));
  c->L = (double *)xcalloc((size_t)d * d, sizeof(double));
  int64_t cap = cfg->max_dead;
  c->dE = (double *)xcalloc((size_t)cap, sizeof(double));
  c->dbirth = (double *)xcalloc((size_t)cap, sizeof(double));
  c->dX = (double *)xcalloc((size_t)(cap * d), sizeof(double));
  c->dnlive = (int32_t *)xcalloc((size_t)cap, sizeof(int32_t));
  c->dgid = (int32_t *)xcalloc((size_t)cap, sizeof(int32_t));
  c->dord = (int32_t *)xcalloc((size_t)cap, sizeof(int32_t));
  c->diter = (int64_t *)xcalloc((size_t)cap, sizeof(int64_t));
  c->R = cfg->n_volume_sims;
  c->lx_prev = (double *)xcalloc((size_t)c->R + 1, sizeof(double));
  c->lx_cur = (double *)xcalloc((size_t)c->R + 1, sizeof(double));
  c->lz = (double *)xcalloc((size_t)c->R + 1, sizeof(double));
  for (int r = 0; r <= c->R; ++r) c->lz[r] = -INFINITY;
  c->t_dead = (int32_t *)xcalloc((size_t)k, sizeof(int32_t));
  int64_t nch = cfg->update_all ? n : k; /* chains per iteration */
  c->t_dest = (int32_t *)xcalloc((size_t)nch, sizeof(int32_t));
  c->t_parent = (int32_t *)xcalloc((size_t)nch, sizeof(int32_t));
  c->t_counts = (uint8_t *)xcalloc((size_t)(nch * (cfg->steps > 0 ? cfg->steps : 1) * 4), 1);
  c->t_margin = (double *)xcalloc((size_t)(nch * (cfg->steps > 0 ? cfg->steps : 1)), sizeof(double));
  c->n_subset = -1;
  c->e_star = INFINITY;
  /* prior draws with rejection, budget 100 n attempts in total */
  int64_t budget = 100 * n, used = 0;
  for (int64_t g = 0; g < (draw_live ? n : 0); ++g) {
    uint32_t a = 0;
    for (;;) {
      if (used >= budget) { nsso_destroy(c); return NSSO_ERR_PRIOR_SUPPORT; }
      prior_draw(c, (uint32_t)g, a, &c->X[g * d]);
      used++;
      double en = energy(c, &c->X[g * d]);
      c->init_evals++;
      if (isnan(en)) { nsso_destroy(c); return NSSO_ERR_NAN; }
      if (isfinite(en)) { c->E[g] = en; break; }
      a++;
    }
    c->birth[g] = INFINITY;
  }
  compute_metric(c);
  *out = c;
  return NSSO_OK;
}

void nsso_destroy(nsso_ctx *c) {
  if (!c) return;
  free(c->smc_par);
  free(c->lo); free(c->hi); free(c->pmean); free(c->psd);
  free(c->e_w); free(c->e_mu); free(c->e_sigma); free(c->e_prec); free(c->e_x); free(c->e_y);
  free(c->X); free(c->E); free(c->birth); free(c->L);
  free(c->dE); free(c->dbirth); free(c->dX); free(c->dnlive); free(c->dgid); free(c->dord);
  free(c->diter);
  free(c->lx_prev); free(c->lx_cur); free(c->lz);
  free(c->t_dead); free(c->t_dest); free(c->t_parent); free(c->t_counts); free(c->t_margin);
  free(c->subset);
  free(c);
}

/* ------------------------------------------------------------------------ */
/* One outer iteration (steps (i)-(iv))                           */
/* ------------------------------------------------------------------------ */
static const nsso_ctx *g_sort_ctx;
/* key order: larger E first; among equal E the larger gid first (DESIGN R-1) */
static int cmp_key_desc(const void *a, const void *b) {
  int32_t ga = *(const int32_t *)a, gb = *(const int32_t *)b;
  double ea = g_sort_ctx->E[ga], eb = g_sort_ctx->E[gb];
  if (ea > eb) return -1;
  if (ea < eb) return 1;
  return ga > gb ? -1 : (ga < gb ? 1 : 0);
}
static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static void fill_info(nsso_ctx *c, nsso_step_info *info);

int nsso_should_terminate(nsso_ctx *c, int32_t *flag) {
  /* P:155-156, P:686 and DESIGN R-19: remaining-evidence bound with the best
   * live energy and the deterministic volume (replica 0). */
  *flag = 0;
  if (c->n_dead == 0) return NSSO_OK;
  double emin = INFINITY;
  for (int64_t g = 0; g < c->n; ++g) if (c->E[g] < emin) emin = c->E[g];
  double lz_live = -emin + c->lx_cur[0];
  *flag = (lz_live - lse2(c->lz[0], lz_live)) < c->cfg.term_log_ratio;
  return NSSO_OK;
}

int nsso_step(nsso_ctx *c, nsso_step_info *info) {
  if (!c) return NSSO_ERR_INVALID_ARG;
  if (c->finalised) return NSSO_ERR_STATE;
  int d = c->d;
  int64_t n = c->n, k = c->k;
  int p = c->cfg.steps;
  /* keep room for the n closing records of nsso_finalise */
  if (c->n_dead + k + n > c->cfg.max_dead) return NSSO_ERR_CAPACITY;
  uint32_t it = (uint32_t)(c->iter + 1);

  /* (i) delete: the k largest keys; E* is the k-th worst energy */
  int32_t *order = (int32_t *)xcalloc((size_t)n, sizeof(int32_t));
  for (int64_t g = 0; g < n; ++g) order[g] = (int32_t)g;
  g_sort_ctx = c;
  qsort(order, (size_t)n, sizeof(int32_t), cmp_key_desc);
  double e_star = c->E[order[k - 1]];
  c->e_star = e_star;
  /* record dead with n_live = n - j in key-descending order */
  for (int64_t j = 0; j < k; ++j) {
    int32_t g = order[j];
    int64_t q = c->n_dead + j;
    c->dE[q] = c->E[g];
    c->dbirth[q] = c->birth[g];
    c->dnlive[q] = (int32_t)(n - j);
    c->dgid[q] = g;
    c->dord[q] = (int32_t)j;
    c->diter[q] = it;
    memcpy(&c->dX[q * d], &c->X[g * d], sizeof(double) * (size_t)d);
    evidence_death(c, c->E[g], n - j, it, (uint32_t)j);
    c->t_dead[j] = g;
  }
  c->n_dead += k;

  /* (ii) resample: survivors S ascending; destinations D ascending; parent of
   * destination s is S[floor(u32 (n-k) / 2^32)] (DESIGN R-3/R-4) */
  char *is_dead = (char *)xcalloc((size_t)n, 1);
  for (int64_t j = 0; j < k; ++j) is_dead[order[j]] = 1;
  int32_t *S = (int32_t *)xcalloc((size_t)(n - k), sizeof(int32_t));
  int64_t ns = 0;
  for (int64_t g = 0; g < n; ++g) if (!is_dead[g]) S[ns++] = (int32_t)g;
  memcpy(c->t_dest, order, sizeof(int32_t) * (size_t)k);
  qsort(c->t_dest, (size_t)k, sizeof(int32_t), cmp_i32);
  for (int64_t cidx = 0; cidx < k; ++cidx) {
    uint32_t s = (uint32_t)c->t_dest[cidx];
    uint32_t u32 = nsso_draw_u32(c->cfg.seed, it, s, PH_RESAMPLE, 0, 0);
    uint64_t rank = ((uint64_t)u32 * (uint64_t)(n - k)) >> 32;
    c->t_parent[cidx] = S[rank];
  }
  /* F4 "applying updates to all m particles": every live slot runs a
   * chain, in ascending gid order; a deleted slot starts from its resampled
   * parent, a surviving slot from its own point; all start from the
   * pre-mutation live set and use the destination-keyed RNG stream. */
  if (c->cfg.update_all) {
    int32_t *par_of = (int32_t *)xcalloc((size_t)n, sizeof(int32_t));
    for (int64_t g = 0; g < n; ++g) par_of[g] = (int32_t)g;
    for (int64_t cidx = 0; cidx < k; ++cidx) par_of[c->t_dest[cidx]] = c->t_parent[cidx];
    for (int64_t g = 0; g < n; ++g) {
      c->t_dest[g] = (int32_t)g;
      c->t_parent[g] = par_of[g];
    }
    free(par_of);
    k = n; /* chains below */
  }

  /* (iii) mutate: p HRSS steps from each duplicated parent;
   * (iv) replace: write into the destination slot */
  char *run = (char *)xcalloc((size_t)k, 1);
  if (c->n_subset < 0) memset(run, 1, (size_t)k);
  else for (int64_t q = 0; q < c->n_subset; ++q)
    if (c->subset[q] >= 0 && c->subset[q] < k) run[c->subset[q]] = 1;
  double *x = (double *)xcalloc((size_t)d, sizeof(double));
  double *xn = (double *)xcalloc((size_t)d, sizeof(double));
  double *z = (double *)xcalloc((size_t)d + 1, sizeof(double));
  double *v = (double *)xcalloc((size_t)d, sizeof(double));
  memset(c->t_counts, 0, (size_t)(k * (p > 0 ? p : 1) * 4));
  for (int64_t q = 0; q < k * (p > 0 ? p : 1); ++q) c->t_margin[q] = INFINITY;
  double *Xnew = (double *)xcalloc((size_t)(k * d), sizeof(double));
  double *Enew = (double *)xcalloc((size_t)k, sizeof(double));
  for (int64_t cidx = 0; cidx < k; ++cidx) {
    if (!run[cidx]) continue;
    uint32_t s = (uint32_t)c->t_dest[cidx];
    int32_t par = c->t_parent[cidx];
    memcpy(x, &c->X[(int64_t)par * d], sizeof(double) * (size_t)d);
    double e = c->E[par];
    for (int j = 0; j < p; ++j) {
      int32_t cnt[4];
      double mm;
      double en;
      if (c->cfg.mutation == NSSO_MUT_RW) {
        rw_step(c, x, e, e_star, it, s, (uint32_t)j, xn, &en, cnt, &mm);
      } else {
        direction(c, it, s, (uint32_t)j, z, v);
        slice_step(c, x, e, v, c->w, e_star, it, s, (uint32_t)j, xn, &en, cnt, &mm);
      }
      memcpy(x, xn, sizeof(double) * (size_t)d);
      e = en;
      uint8_t *tc = &c->t_counts[(cidx * p + j) * 4];
      tc[0] = (uint8_t)cnt[0]; tc[1] = (uint8_t)cnt[1]; tc[2] = (uint8_t)cnt[2]; tc[3] = (uint8_t)cnt[3];
      c->t_margin[cidx * p + j] = mm;
    }
    memcpy(&Xnew[cidx * d], x, sizeof(double) * (size_t)d);
    Enew[cidx] = e;
  }
  for (int64_t cidx = 0; cidx < k; ++cidx) {
    if (!run[cidx]) continue;
    int32_t s = c->t_dest[cidx];
    memcpy(&c->X[(int64_t)s * d], &Xnew[cidx * d], sizeof(double) * (size_t)d);
    c->E[s] = Enew[cidx];
    if (c->t_parent[cidx] != s) c->birth[s] = e_star; /* a moved survivor keeps its birth level */
  }
  free(Xnew); free(Enew);
  free(x); free(xn); free(z); free(v); free(run); free(is_dead); free(S); free(order);
  c->iter++;
  /* adaptive metric from the post-replacement live set */
  compute_metric(c);
  if (c->nan_seen) return NSSO_ERR_NAN;
  if (info) fill_info(c, info);
  return NSSO_OK;
}

/* AMB-18 / DESIGN R-18: append the live set in key-descending order with
 * n_live = n, n-1, ..., 1, then close the quadrature with X_{N+1} = 0. */
int nsso_finalise(nsso_ctx *c) {
  if (!c) return NSSO_ERR_INVALID_ARG;
  if (c->finalised) return NSSO_OK;
  int d = c->d;
  int64_t n = c->n;
  if (c->n_dead + n > c->cfg.max_dead) return NSSO_ERR_CAPACITY;
  uint32_t it = (uint32_t)(c->iter + 1);
  int32_t *order = (int32_t *)xcalloc((size_t)n, sizeof(int32_t));
  for (int64_t g = 0; g < n; ++g) order[g] = (int32_t)g;
  g_sort_ctx = c;
  qsort(order, (size_t)n, sizeof(int32_t), cmp_key_desc);
  for (int64_t j = 0; j < n; ++j) {
    int32_t g = order[j];
    int64_t q = c->n_dead + j;
    c->dE[q] = c->E[g];
    c->dbirth[q] = c->birth[g];
    c->dnlive[q] = (int32_t)(n - j);
    c->dgid[q] = g;
    c->dord[q] = (int32_t)j;
    c->diter[q] = it;
    memcpy(&c->dX[q * d], &c->X[g * d], sizeof(double) * (size_t)d);
    evidence_death(c, c->E[g], n - j, it, (uint32_t)j);
  }
  c->n_dead += n;
  free(order);
  for (int r = 0; r <= c->R; ++r) c->lz[r] = closed_logz(c, r);
  c->has_pend = 0;
  c->finalised = 1;
  return NSSO_OK;
}

int nsso_run(nsso_ctx *c, int64_t max_iters, nsso_step_info *info) {
  if (!c) return NSSO_ERR_INVALID_ARG;
  for (int64_t i = 0; i < max_iters; ++i) {
    int32_t flag;
    nsso_should_terminate(c, &flag);
    if (flag) break;
    int st = nsso_step(c, NULL);
    if (st != NSSO_OK) return st;
  }
  int st = nsso_finalise(c);
  if (st != NSSO_OK) return st;
  if (info) fill_info(c, info);
  return NSSO_OK;
}

/* log Z point estimate and its error: mean and sample std of {log Z^(r)},
 * r = 1..R (DESIGN R-17). */
int nsso_evidence(nsso_ctx *c, double *log_z, double *log_z_err) {
  if (!c) return NSSO_ERR_INVALID_ARG;
  if (c->n_dead == 0) return NSSO_ERR_STATE;
  double s = 0.0;
  for (int r = 1; r <= c->R; ++r) s += closed_logz(c, r);
  double mean = s / c->R;
  double v = 0.0;
  for (int r = 1; r <= c->R; ++r) {
    double t = closed_logz(c, r) - mean;
    v += t * t;
  }
  if (log_z) *log_z = mean;
  if (log_z_err) *log_z_err = sqrt(v / (c->R - 1));
  return NSSO_OK;
}

int nsso_evidence_reps(nsso_ctx *c, double *reps) {
  if (!c || !reps) return NSSO_ERR_INVALID_ARG;
  if (c->n_dead == 0) return NSSO_ERR_STATE;
  for (int r = 0; r <= c->R; ++r) reps[r] = closed_logz(c, r);
  return NSSO_OK;
}

/* Posterior weights: geometric mean over R of w_i^(r) = exp(-E_i) dX_i^(r)
 * (P:1243-1247), normalised.  Re-simulates every trajectory from the dead
 * store in death order (same draws as the streamed accumulators). */
int nsso_samples(nsso_ctx *c, double *x, double *log_w, int64_t cap, int64_t *n_out) {
  if (!c || !n_out) return NSSO_ERR_INVALID_ARG;
  if (c->n_dead == 0) return NSSO_ERR_STATE;
  int64_t N = c->n_dead;
  *n_out = N;
  if (!x && !log_w) return NSSO_OK;
  if (cap < N) return NSSO_ERR_CAPACITY;
  int d = c->d;
  if (x) memcpy(x, c->dX, sizeof(double) * (size_t)(N * d));
  if (!log_w) return NSSO_OK;
  double *acc = (double *)xcalloc((size_t)N, sizeof(double));
  double *lx = (double *)xcalloc((size_t)N + 2, sizeof(double)); /* log X_0..X_N */
  for (int r = 1; r <= c->R; ++r) {
    lx[0] = 0.0;
    for (int64_t i = 0; i < N; ++i)
      lx[i + 1] = lx[i] + dlogx(c, r, c->dnlive[i], (uint32_t)c->diter[i], (uint32_t)c->dord[i]);
    for (int64_t i = 1; i <= N; ++i) {
      double ldx;
      if (c->cfg.quadrature == NSSO_Q_RECTANGLE)
        ldx = lx[i - 1] + log1mexp(lx[i] - lx[i - 1]);           /* X_{i-1} - X_i        */
      else if (i < N)
        ldx = lx[i - 1] + log1mexp(lx[i + 1] - lx[i - 1]) - log(2.0); /* (X_{i-1}-X_{i+1})/2 */
      else
        ldx = lx[i - 1] - log(2.0);                               /* X_{N+1} = 0          */
      acc[i - 1] += ldx;
    }
  }
  double m = -INFINITY;
  for (int64_t i = 0; i < N; ++i) {
    log_w[i] = acc[i] / c->R - c->dE[i];
    if (log_w[i] > m) m = log_w[i];
  }
  double s = 0.0;
  for (int64_t i = 0; i < N; ++i) s += exp(log_w[i] - m);
  double lz = m + log(s);
  for (int64_t i = 0; i < N; ++i) log_w[i] -= lz;
  free(acc);
  free(lx);
  return NSSO_OK;
}

/* ------------------------------------------------------------------------ */
/* Posterior products at inverse temperature beta (F2; P:123-132 reweighting, */
/* P:1225-1255 weights, geometric-mean collapse and Kish ESS).                */
/* ------------------------------------------------------------------------ */
/* w_i^(r)(beta) = exp(-beta E_i) dX_i^(r) over the dead points in death order,
 * Z^(r)(beta) = sum_i w_i^(r)(beta); log Z reported as mean and
 * std (ddof 1) over r = 1..R; geometric-mean weights
 * w~_i = exp(mean_r log w_i^(r)), normalised; Kish
 * ESS = (sum w~)^2 / sum w~^2.  Before finalisation the last
 * dead point closes with X_{N+1} = 0, as nsso_samples does (R-27). */
int nsso_posterior(nsso_ctx *c, double beta, double *log_z, double *log_z_err, double *ess, double *log_w,
                   int64_t cap) {
  if (!c) return NSSO_ERR_INVALID_ARG;
  if (c->n_dead == 0) return NSSO_ERR_STATE;
  int64_t N = c->n_dead;
  if (log_w && cap < N) return NSSO_ERR_CAPACITY;
  double *acc = (double *)xcalloc((size_t)N, sizeof(double));
  double *lx = (double *)xcalloc((size_t)N + 2, sizeof(double));
  double *term = (double *)xcalloc((size_t)N, sizeof(double));
  double *lzr = (double *)xcalloc((size_t)c->R + 1, sizeof(double));
  for (int r = 1; r <= c->R; ++r) {
    lx[0] = 0.0;
    for (int64_t i = 0; i < N; ++i)
      lx[i + 1] = lx[i] + dlogx(c, r, c->dnlive[i], (uint32_t)c->diter[i], (uint32_t)c->dord[i]);
    double m = -INFINITY;
    for (int64_t i = 1; i <= N; ++i) {
      double ldx;
      if (c->cfg.quadrature == NSSO_Q_RECTANGLE)
        ldx = lx[i - 1] + log1mexp(lx[i] - lx[i - 1]);
      else if (i < N)
        ldx = lx[i - 1] + log1mexp(lx[i + 1] - lx[i - 1]) - log(2.0);
      else
        ldx = lx[i - 1] - log(2.0);
      acc[i - 1] += ldx;
      term[i - 1] = -beta * c->dE[i - 1] + ldx; /* log w_i^(r)(beta) */
      if (term[i - 1] > m) m = term[i - 1];
    }
    double s = 0.0;
    for (int64_t i = 0; i < N; ++i) s += exp(term[i] - m);
    lzr[r] = m + log(s);
  }
  double mean = 0.0;
  for (int r = 1; r <= c->R; ++r) mean += lzr[r];
  mean /= c->R;
  double var = 0.0;
  for (int r = 1; r <= c->R; ++r) var += (lzr[r] - mean) * (lzr[r] - mean);
  if (log_z) *log_z = mean;
  if (log_z_err) *log_z_err = sqrt(var / (c->R - 1));
  /* geometric-mean weights, normalised in log space */
  double m = -INFINITY;
  for (int64_t i = 0; i < N; ++i) {
    term[i] = acc[i] / c->R - beta * c->dE[i];
    if (term[i] > m) m = term[i];
  }
  double s = 0.0;
  for (int64_t i = 0; i < N; ++i) s += exp(term[i] - m);
  double lse = m + log(s);
  double s2 = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    term[i] -= lse;
    s2 += exp(2.0 * term[i]);
  }
  if (ess) *ess = 1.0 / s2;
  if (log_w) memcpy(log_w, term, sizeof(double) * (size_t)N);
  free(acc); free(lx); free(term); free(lzr);
  return NSSO_OK;
}

/* Equal-weight posterior samples (F2; "resampling"):
 * m multinomial draws from the normalised weights w_bar(beta): draw j takes
 * u_j = uniform 0 of stream (iteration 0, j, POSTERIOR, 0) under key `seed`
 * and returns the first dead point i with u_j < sum_{l <= i} w_bar_l
 * (the last point if rounding leaves u_j above the total). */
int nsso_resample(nsso_ctx *c, double beta, int64_t m, uint64_t seed, int64_t *idx, double *x) {
  if (!c || m < 1 || (!idx && !x)) return NSSO_ERR_INVALID_ARG;
  if (c->n_dead == 0) return NSSO_ERR_STATE;
  int64_t N = c->n_dead;
  double *lw = (double *)xcalloc((size_t)N, sizeof(double));
  double *cum = (double *)xcalloc((size_t)N, sizeof(double));
  int st = nsso_posterior(c, beta, NULL, NULL, NULL, lw, N);
  if (st) { free(lw); free(cum); return st; }
  double run = 0.0;
  for (int64_t i = 0; i < N; ++i) { run += exp(lw[i]); cum[i] = run; }
  for (int64_t j = 0; j < m; ++j) {
    double u = nsso_draw_uniform(seed, 0, (uint32_t)j, PH_POSTERIOR, 0, 0);
    int64_t lo = 0, hi = N - 1; /* first i with u < cum[i] */
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (u < cum[mid]) hi = mid; else lo = mid + 1;
    }
    if (idx) idx[j] = lo;
    if (x) memcpy(x + j * c->d, c->dX + lo * c->d, sizeof(double) * (size_t)c->d);
  }
  free(lw); free(cum);
  return NSSO_OK;
}

/* ------------------------------------------------------------------------ */
/* F3: adaptive tempered SMC with the HRSS kernel (SMC-SS,        */
/* P:710-713)                                                     */
/* ------------------------------------------------------------------------ */
/* ESS of the normalised incremental weights exp(-db E_i),
 * computed with the weights shifted by min E (exact ratio). */
static double smc_ess(const double *E, int64_t m, double db, double emin) {
  double s = 0.0, s2 = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double w = exp(-db * (E[i] - emin));
    s += w;
    s2 += w * w;
  }
  return s * s / s2;
}

/* Next temperature: bisection on db in (0, 1 - beta_t] for
 * ESS = rho m, to 1e-10 in db; the whole remaining step when ESS stays above
 * rho m. */
int nsso_smc_next_beta(const double *E, int64_t m, double beta_t, double rho, double *beta_next) {
  if (!E || m < 1 || !beta_next || !(rho > 0.0 && rho < 1.0) || !(beta_t < 1.0)) return NSSO_ERR_INVALID_ARG;
  double emin = INFINITY;
  for (int64_t i = 0; i < m; ++i) if (E[i] < emin) emin = E[i];
  double hi = 1.0 - beta_t;
  if (smc_ess(E, m, hi, emin) >= rho * (double)m) { *beta_next = 1.0; return NSSO_OK; }
  double lo = 0.0;
  while (hi - lo > 1e-10) {
    double mid = 0.5 * (lo + hi);
    if (smc_ess(E, m, mid, emin) >= rho * (double)m) lo = mid; else hi = mid;
  }
  *beta_next = beta_t + lo;
  return NSSO_OK;
}

int nsso_smc_init(const nsso_prior *p, const nsso_energy *e, const nsso_config *cfg, double rho, nsso_ctx **out) {
  if (!(rho > 0.0 && rho < 1.0)) return NSSO_ERR_INVALID_ARG;
  int st = nsso_init(p, e, cfg, out);
  if (st) return st;
  (*out)->smc = 1;
  (*out)->smc_rho = rho;
  (*out)->beta = 0.0;
  (*out)->smc_logz = 0.0;
  (*out)->smc_par = (int32_t *)xcalloc((size_t)cfg->n_live, sizeof(int32_t));
  /* parity hook: per-particle, per-step counts and decision margins of the
   * last stage (every particle runs a chain) */
  size_t np_ = (size_t)(cfg->n_live * (cfg->steps > 0 ? cfg->steps : 1));
  free((*out)->t_counts);
  free((*out)->t_margin);
  (*out)->t_counts = (uint8_t *)xcalloc(np_ * 4, 1);
  (*out)->t_margin = (double *)xcalloc(np_, sizeof(double));
  free((*out)->t_dest);
  free((*out)->t_parent);
  (*out)->t_dest = (int32_t *)xcalloc((size_t)cfg->n_live, sizeof(int32_t));
  (*out)->t_parent = (int32_t *)xcalloc((size_t)cfg->n_live, sizeof(int32_t));
  for (int64_t j = 0; j < cfg->n_live; ++j) (*out)->t_dest[j] = (*out)->t_parent[j] = (int32_t)j;
  return NSSO_OK;
}

/* One SMC stage t = iter + 1: next temperature, log Z += log mean w
 * (P:663-668), multinomial resampling by the normalised weights (u_j =
 * uniform 0 of stream (t, j, SMC = 7, 0)), metric of the resampled particles,
 * p tempered HRSS steps per particle (stream (t, j, HRSS, step)). */
int nsso_smc_stage(nsso_ctx *c) {
  if (!c || !c->smc) return NSSO_ERR_INVALID_ARG;
  if (c->beta >= 1.0) return NSSO_ERR_STATE;
  int d = c->d;
  int64_t m = c->n;
  int p = c->cfg.steps;
  uint32_t t = (uint32_t)(c->iter + 1);
  double bn;
  int st = nsso_smc_next_beta(c->E, m, c->beta, c->smc_rho, &bn);
  if (st) return st;
  double db = bn - c->beta;
  double emin = INFINITY;
  for (int64_t i = 0; i < m; ++i) if (c->E[i] < emin) emin = c->E[i];
  double *cum = (double *)xcalloc((size_t)m, sizeof(double));
  double s = 0.0;
  for (int64_t i = 0; i < m; ++i) s += exp(-db * (c->E[i] - emin));
  c->smc_logz += -db * emin + log(s) - log((double)m);
  double run = 0.0;
  for (int64_t i = 0; i < m; ++i) { run += exp(-db * (c->E[i] - emin)) / s; cum[i] = run; }
  c->beta = bn;
  double *X0 = dup_d(c->X, (size_t)(m * d)), *E0 = dup_d(c->E, (size_t)m);
  for (int64_t j = 0; j < m; ++j) {
    double u = nsso_draw_uniform(c->cfg.seed, t, (uint32_t)j, PH_SMC, 0, 0);
    int64_t lo = 0, hi = m - 1;
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (u < cum[mid]) hi = mid; else lo = mid + 1; }
    memcpy(&c->X[j * d], &X0[lo * d], sizeof(double) * (size_t)d);
    c->E[j] = E0[lo];
    c->smc_par[j] = (int32_t)lo;
  }
  free(X0); free(E0); free(cum);
  compute_metric(c);
  double *x = (double *)xcalloc((size_t)d, sizeof(double));
  double *xn = (double *)xcalloc((size_t)d, sizeof(double));
  double *z = (double *)xcalloc((size_t)d + 1, sizeof(double));
  double *v = (double *)xcalloc((size_t)d, sizeof(double));
  for (int64_t j = 0; j < m; ++j) {
    memcpy(x, &c->X[j * d], sizeof(double) * (size_t)d);
    double e = c->E[j];
    for (int q = 0; q < p; ++q) {
      int32_t cnt[4];
      double mm, en;
      direction(c, t, (uint32_t)j, (uint32_t)q, z, v);
      slice_step(c, x, e, v, c->w, INFINITY, t, (uint32_t)j, (uint32_t)q, xn, &en, cnt, &mm);
      for (int b = 0; b < 4; ++b) c->t_counts[(j * p + q) * 4 + b] = (uint8_t)cnt[b];
      c->t_margin[j * p + q] = mm;
      memcpy(x, xn, sizeof(double) * (size_t)d);
      e = en;
    }
    memcpy(&c->X[j * d], x, sizeof(double) * (size_t)d);
    c->E[j] = e;
  }
  free(x); free(xn); free(z); free(v);
  c->iter++;
  if (c->nan_seen) return NSSO_ERR_NAN;
  return NSSO_OK;
}

int nsso_smc_state(nsso_ctx *c, double *beta, double *log_z, int64_t *stage, int32_t *parents) {
  if (!c || !c->smc) return NSSO_ERR_INVALID_ARG;
  if (parents) memcpy(parents, c->smc_par, sizeof(int32_t) * (size_t)c->n);
  if (beta) *beta = c->beta;
  if (log_z) *log_z = c->smc_logz;
  if (stage) *stage = c->iter;
  return NSSO_OK;
}


static void fill_info(nsso_ctx *c, nsso_step_info *info) {
  memset(info, 0, sizeof(*info));
  info->iteration = c->iter;
  info->e_star = c->e_star;
  info->probes = c->probes;
  info->energy_evals = c->evals;
  info->expansions = c->expansions;
  info->shrinks = c->shrinks;
  info->null_moves = c->nulls;
  info->init_evals = c->init_evals;
  info->log_z_det = c->lz[0];
  double emin = INFINITY;
  for (int64_t g = 0; g < c->n; ++g) if (c->E[g] < emin) emin = c->E[g];
  info->log_z_live = -emin + c->lx_cur[0];
  int32_t f = 0;
  nsso_should_terminate(c, &f);
  info->terminated = f;
  info->finalised = c->finalised;
}

int nsso_info(nsso_ctx *c, nsso_step_info *info) {
  if (!c || !info) return NSSO_ERR_INVALID_ARG;
  fill_info(c, info);
  return NSSO_OK;
}

/* ------------------------------------------------------------------------ */
/* Parity hooks                                                              */
/* ------------------------------------------------------------------------ */
int nsso_set_live(nsso_ctx *c, const double *x, const double *e, int64_t next_iteration) {
  if (!c || !x || !e || next_iteration < 1) return NSSO_ERR_INVALID_ARG;
  memcpy(c->X, x, sizeof(double) * (size_t)(c->n * c->d));
  memcpy(c->E, e, sizeof(double) * (size_t)c->n);
  c->iter = next_iteration - 1;
  compute_metric(c);
  return NSSO_OK;
}

int nsso_get_live(nsso_ctx *c, double *x, double *e) {
  if (!c) return NSSO_ERR_INVALID_ARG;
  if (x) memcpy(x, c->X, sizeof(double) * (size_t)(c->n * c->d));
  if (e) memcpy(e, c->E, sizeof(double) * (size_t)c->n);
  return NSSO_OK;
}

int nsso_get_metric(nsso_ctx *c, double *chol, double *width) {
  if (!c) return NSSO_ERR_INVALID_ARG;
  if (chol) memcpy(chol, c->L, sizeof(double) * (size_t)c->d * c->d);
  if (width) *width = c->w;
  return NSSO_OK;
}

int nsso_set_chain_subset(nsso_ctx *c, const int32_t *chains, int64_t count) {
  if (!c) return NSSO_ERR_INVALID_ARG;
  free(c->subset);
  c->subset = NULL;
  c->n_subset = -1;
  if (count < 0 || !chains) return NSSO_OK;
  c->subset = (int32_t *)xcalloc((size_t)count, sizeof(int32_t));
  memcpy(c->subset, chains, sizeof(int32_t) * (size_t)count);
  c->n_subset = count;
  return NSSO_OK;
}

int nsso_get_trace(nsso_ctx *c, int32_t *dead_gid, int32_t *dest_gid, int32_t *parent_gid,
                   uint8_t *counts, double *min_margin, double *e_star) {
  if (!c) return NSSO_ERR_INVALID_ARG;
  int64_t k = c->k, nch = (c->cfg.update_all || c->smc) ? c->n : c->k;
  int p = c->cfg.steps > 0 ? c->cfg.steps : 1;
  if (dead_gid) memcpy(dead_gid, c->t_dead, sizeof(int32_t) * (size_t)k);
  if (dest_gid) memcpy(dest_gid, c->t_dest, sizeof(int32_t) * (size_t)nch);
  if (parent_gid) memcpy(parent_gid, c->t_parent, sizeof(int32_t) * (size_t)nch);
  if (counts) memcpy(counts, c->t_counts, (size_t)(nch * p * 4));
  if (min_margin) memcpy(min_margin, c->t_margin, sizeof(double) * (size_t)(nch * p));
  if (e_star) *e_star = c->e_star;
  return NSSO_OK;
}

int nsso_dead(nsso_ctx *c, double *e, int32_t *n_live, double *birth, int32_t *gid, double *x,
              int64_t cap, int64_t *n_out) {
  if (!c || !n_out) return NSSO_ERR_INVALID_ARG;
  int64_t N = c->n_dead;
  *n_out = N;
  if (!e && !n_live && !birth && !gid && !x) return NSSO_OK;
  if (cap < N) return NSSO_ERR_CAPACITY;
  if (e) memcpy(e, c->dE, sizeof(double) * (size_t)N);
  if (n_live) memcpy(n_live, c->dnlive, sizeof(int32_t) * (size_t)N);
  if (birth) memcpy(birth, c->dbirth, sizeof(double) * (size_t)N);
  if (gid) memcpy(gid, c->dgid, sizeof(int32_t) * (size_t)N);
  if (x) memcpy(x, c->dX, sizeof(double) * (size_t)(N * c->d));
  return NSSO_OK;
}

int nsso_volume_reps(nsso_ctx *c, double *log_x) {
  if (!c || !log_x) return NSSO_ERR_INVALID_ARG;
  for (int r = 0; r <= c->R; ++r) log_x[r] = c->lx_cur[r];
  return NSSO_OK;
}

int nsso_direction(nsso_ctx *c, uint32_t iter, uint32_t gid, uint32_t step, double *v) {
  if (!c || !v) return NSSO_ERR_INVALID_ARG;
  double *z = (double *)xcalloc((size_t)c->d + 1, sizeof(double));
  direction(c, iter, gid, step, z, v);
  free(z);
  return NSSO_OK;
}
