"""Seeded synthetic workloads (inputs only).

This module generates the problem data -- priors, likelihood parameters,
datasets -- and the run configurations for the five configurations named in
BASELINE.json (DESIGN.md section 5 gives the recipe).  It holds none of the
method's arithmetic: no energies, no slice sampling, no evidence.  Both the
CUDA binding (`paper_2601_23252_b200.nss`) and the oracle binding
(in the test-only oracle package) consume the same `Problem` objects, so they never share
generation code with each other.

Shapes follow the paper's workloads (P:760 kappa=100 Gaussian, P:836-840
mixture, P:883-887 funnel, P:466 logistic regression, P:935-962 GP), with the
sizes BASELINE.json fixes.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Optional

import numpy as np

PRIOR_BOX = 0
PRIOR_GAUSS_DIAG = 1

E_GAUSS = 0
E_MOG = 1
E_CORR_GAUSS = 2
E_FUNNEL = 3
E_LOGREG = 4
E_GP_ARD = 5
E_FLAT = 6

W_OPTIMAL = 0
W_FIXED = 1
DIR_MAHALANOBIS = 0
DIR_EUCLIDEAN = 1
Q_TRAPEZOID = 0
Q_RECTANGLE = 1
MUT_HRSS = 0
MUT_RW = 1

LN2PI = math.log(2.0 * math.pi)


@dataclasses.dataclass
class Problem:
    name: str
    d: int
    prior_kind: int
    energy_kind: int
    lo: Optional[np.ndarray] = None
    hi: Optional[np.ndarray] = None
    mean: Optional[np.ndarray] = None
    sd: Optional[np.ndarray] = None
    # energy parameters (fp64 host arrays)
    w: Optional[np.ndarray] = None
    mu: Optional[np.ndarray] = None
    sigma: Optional[np.ndarray] = None
    prec: Optional[np.ndarray] = None
    data_x: Optional[np.ndarray] = None
    data_y: Optional[np.ndarray] = None
    c: float = 0.0
    sigma_y: float = 3.0
    jitter: float = 1e-6
    n_comp: int = 0
    d_in: int = 0
    # generator-side facts (not used by either implementation)
    meta: Dict = dataclasses.field(default_factory=dict)

    @property
    def n_data(self) -> int:
        return 0 if self.data_y is None else int(self.data_y.shape[0])


def config(n_live: int, k: int, steps: int, *, seed: int = 1, width_rule: int = W_OPTIMAL,
           width: float = 1.0, dir_norm: int = DIR_MAHALANOBIS, max_stepout: int = 10,
           max_shrink: int = 100, quadrature: int = Q_TRAPEZOID, metric_reg: float = 1e-6,
           term_log_ratio: float = -3.0, n_volume_sims: int = 100,
           max_dead: Optional[int] = None, update_all: int = 0, mutation: int = 0) -> Dict:
    """Run configuration (P:684-686 defaults)."""
    if max_dead is None:
        max_dead = n_live + k * 1000
    return dict(n_live=int(n_live), k=int(k), steps=int(steps), width_rule=int(width_rule),
                width=float(width), dir_norm=int(dir_norm), max_stepout=int(max_stepout),
                max_shrink=int(max_shrink), quadrature=int(quadrature),
                metric_reg=float(metric_reg), term_log_ratio=float(term_log_ratio),
                n_volume_sims=int(n_volume_sims), max_dead=int(max_dead), seed=int(seed),
                update_all=int(update_all), mutation=int(mutation))


# --------------------------------------------------------------------------
# C1: d=2 isotropic Gaussian likelihood under U[-5,5]^2
# --------------------------------------------------------------------------
def gauss(d: int = 2, half_width: float = 5.0, sigma: float = 1.0, mu=None) -> Problem:
    mu = np.zeros(d) if mu is None else np.asarray(mu, dtype=np.float64)
    sig = np.full(d, float(sigma))
    # normalised likelihood N(x; mu, sigma^2 I): c = sum log sigma + d/2 log 2 pi
    c = float(np.sum(np.log(sig)) + 0.5 * d * LN2PI)
    return Problem(name=f"gauss{d}", d=d, prior_kind=PRIOR_BOX, energy_kind=E_GAUSS,
                   lo=np.full(d, -half_width), hi=np.full(d, half_width), mu=mu, sigma=sig, c=c)


# --------------------------------------------------------------------------
# C2: d=10 well-separated 4-component Gaussian mixture under U[-10,10]^10
# --------------------------------------------------------------------------
def mog(d: int = 10, n_comp: int = 4, seed: int = 1002, half_width: float = 10.0,
        mean_box: float = 6.0, min_sep: float = 8.0) -> Problem:
    rng = np.random.Generator(np.random.PCG64(seed))
    means = []
    while len(means) < n_comp:
        cand = rng.uniform(-mean_box, mean_box, size=d)
        if all(np.linalg.norm(cand - m) >= min_sep for m in means):
            means.append(cand)
    sigma = rng.uniform(0.5, 1.0, size=(n_comp, d))
    w = np.full(n_comp, 1.0 / n_comp)
    return Problem(name=f"mog{d}", d=d, prior_kind=PRIOR_BOX, energy_kind=E_MOG,
                   lo=np.full(d, -half_width), hi=np.full(d, half_width), w=w,
                   mu=np.array(means), sigma=sigma, n_comp=n_comp)


# --------------------------------------------------------------------------
# C3a: d=100 correlated Gaussian (kappa = 100) under N(0, 5^2 I)
# --------------------------------------------------------------------------
def corr_gauss(d: int = 100, seed: int = 1003, prior_sd: float = 5.0, kappa: float = 100.0,
               box: Optional[float] = None) -> Problem:
    rng = np.random.Generator(np.random.PCG64(seed))
    lam = np.logspace(-math.log10(kappa), 0.0, d)  # eigenvalues of Sigma_L in [1/kappa, 1]
    a = rng.standard_normal((d, d))
    q, r = np.linalg.qr(a)
    q = q * np.sign(np.diag(r))                     # Haar-distributed orthogonal
    sigma_l = (q * lam) @ q.T
    prec = (q / lam) @ q.T
    prec = 0.5 * (prec + prec.T)
    mu = rng.standard_normal(d)
    c = float(0.5 * (d * LN2PI + np.sum(np.log(lam))))
    if box is None:
        pk, lo, hi, mean, sd = PRIOR_GAUSS_DIAG, None, None, np.zeros(d), np.full(d, prior_sd)
    else:
        pk, lo, hi, mean, sd = PRIOR_BOX, np.full(d, -box), np.full(d, box), None, None
    return Problem(name=f"corrgauss{d}", d=d, prior_kind=pk, energy_kind=E_CORR_GAUSS,
                   lo=lo, hi=hi, mean=mean, sd=sd, mu=mu, prec=prec, c=c,
                   meta=dict(sigma_l=sigma_l, lam=lam))


# --------------------------------------------------------------------------
# C3b: Neal's funnel under U[-20,20]^d
# --------------------------------------------------------------------------
def funnel(d: int = 100, half_width: float = 20.0, sigma_y: float = 3.0) -> Problem:
    return Problem(name=f"funnel{d}", d=d, prior_kind=PRIOR_BOX, energy_kind=E_FUNNEL,
                   lo=np.full(d, -half_width), hi=np.full(d, half_width), sigma_y=sigma_y)


# --------------------------------------------------------------------------
# C4: Bayesian logistic regression, N rows, d weights, prior N(0, I)
# --------------------------------------------------------------------------
def fp16_round(a: np.ndarray) -> np.ndarray:
    """Round to the nearest fp16 value (ties to even): features stored in
    half precision, exact in fp16, fp32 and fp64 (DESIGN R-28)."""
    return np.asarray(a, dtype=np.float64).astype(np.float16).astype(np.float64)


def logreg(d: int = 100, n_data: int = 10_000, seed: int = 1005, half_exact: bool = True) -> Problem:
    """X_rj ~ N(0, 1/d) (rounded to fp16 when half_exact: the tensor-core path
    then needs one X term; any finite data within the fp16 range works with
    two), theta* ~ N(0, I), y_r ~ Bernoulli(sigmoid(x_r . theta*))."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((n_data, d)) / math.sqrt(d)
    if half_exact:
        x = fp16_round(x)
    theta = rng.standard_normal(d)
    logits = x @ theta
    y = (rng.uniform(size=n_data) < 1.0 / (1.0 + np.exp(-logits))).astype(np.float64)
    return Problem(name=f"logreg{d}", d=d, prior_kind=PRIOR_GAUSS_DIAG, energy_kind=E_LOGREG,
                   mean=np.zeros(d), sd=np.ones(d), data_x=x, data_y=y,
                   meta=dict(theta_true=theta))


# --------------------------------------------------------------------------
# C5: GP ARD-RBF hyperparameters (P:935-962 shape), d = d_in + 2, prior N(0, I)
# --------------------------------------------------------------------------
def gp_ard(d_in: int = 6, n_data: int = 1024, seed: int = 1006,
           lengthscales=(0.2, 0.3, 0.5, 0.8, 1.2, 2.0), sigma_f: float = 1.0,
           sigma_n: float = 0.1) -> Problem:
    rng = np.random.Generator(np.random.PCG64(seed))
    ls = np.asarray(lengthscales[:d_in], dtype=np.float64)
    x = rng.uniform(size=(n_data, d_in))
    diff = (x[:, None, :] - x[None, :, :]) / ls
    k = sigma_f ** 2 * np.exp(-0.5 * np.sum(diff * diff, axis=-1))
    k[np.diag_indices(n_data)] += sigma_n ** 2 + 1e-8
    f = np.linalg.cholesky(k) @ rng.standard_normal(n_data)
    y = f
    y = (y - y.mean()) / y.std()  # standardised targets
    d = d_in + 2
    return Problem(name=f"gp{d}", d=d, prior_kind=PRIOR_GAUSS_DIAG, energy_kind=E_GP_ARD,
                   mean=np.zeros(d), sd=np.ones(d), data_x=x, data_y=y, d_in=d_in, jitter=1e-6)


def flat(d: int, half_width: float = 1.0, c: float = 0.0) -> Problem:
    """Constant energy under a box: level-set and flat-likelihood pins."""
    return Problem(name=f"flat{d}", d=d, prior_kind=PRIOR_BOX, energy_kind=E_FLAT,
                   lo=np.full(d, -half_width), hi=np.full(d, half_width), c=c)


# --------------------------------------------------------------------------
# The BASELINE.json configurations
# --------------------------------------------------------------------------
CONFIGS = {
    "C1": dict(problem=lambda: gauss(2), n_live=200, k=20, steps=10),
    "C2": dict(problem=lambda: mog(10), n_live=2000, k=200, steps=10),
    # p = 3d at d = 100: the paper's setting for its d ~ 100 problems; at p = d the
    # chains under-mix and log Z comes out 3-5 sigma high (profiles/r01_accuracy.md)
    "C3a": dict(problem=lambda: corr_gauss(100), n_live=10_000, k=1000, steps=300),
    "C3b": dict(problem=lambda: funnel(100), n_live=10_000, k=1000, steps=300),
    "C4": dict(problem=lambda: logreg(100, 10_000), n_live=20_000, k=10_000, steps=100),
    "C5": dict(problem=lambda: gp_ard(6, 1024), n_live=4096, k=2048, steps=8),
}


def workload(name: str, seed: int = 1, **over):
    spec = CONFIGS[name]
    prob = spec["problem"]()
    kw = dict(n_live=spec["n_live"], k=spec["k"], steps=spec["steps"], seed=seed)
    kw.update(over)
    return prob, config(**kw)
