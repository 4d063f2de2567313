"""Full-run pins for the oracle: energies against library densities, and
log Z against closed forms / brute-force quadrature (north_star; P14-P19).

Each run's |log Z - truth| must stay within max(3 sigma_NS, 0.05)-style
bounds, and the weighted dead points must reproduce posterior moments.
"""
import math

import numpy as np
import pytest
from scipy import integrate, special, stats

from paper_2601_23252_b200 import workloads as W


def _ctx(oracle_lib, p, **cfg):
    base = dict(n_live=50, k=5, steps=2)
    base.update(cfg)
    return oracle_lib.Oracle(p, W.config(**base))


# ---------------------------------------------------------------- energies --
def test_energy_gauss_vs_scipy(oracle_lib):
    p = W.gauss(3, mu=[0.3, -1.0, 2.0], sigma=1.5)
    o = _ctx(oracle_lib, p)
    rng = np.random.default_rng(1)
    for x in rng.uniform(-5, 5, (20, 3)):
        ref = -stats.multivariate_normal(p.mu, 1.5 ** 2 * np.eye(3)).logpdf(x)
        assert abs(o.energy(x) - ref) < 1e-12 * max(1, abs(ref))
        assert abs(o.log_prior(x) - (-3 * math.log(10.0))) < 1e-14


def test_energy_mog_vs_scipy(oracle_lib):
    p = W.mog(5, n_comp=3, seed=3, mean_box=4.0, min_sep=3.0)
    o = _ctx(oracle_lib, p)
    rng = np.random.default_rng(2)
    for x in rng.uniform(-8, 8, (20, 5)):
        comps = [math.log(p.w[j]) + stats.norm(p.mu[j], p.sigma[j]).logpdf(x).sum() for j in range(3)]
        ref = -special.logsumexp(comps)
        assert abs(o.energy(x) - ref) < 1e-11 * max(1, abs(ref))
    assert o.log_prior(np.full(5, 10.5)) == -np.inf


def test_energy_corr_gauss_vs_scipy(oracle_lib):
    p = W.corr_gauss(6, seed=4)
    o = _ctx(oracle_lib, p)
    rng = np.random.default_rng(3)
    mvn = stats.multivariate_normal(p.mu, p.meta["sigma_l"])
    for x in rng.standard_normal((10, 6)):
        ref = -mvn.logpdf(x)
        assert abs(o.energy(x) - ref) < 1e-9 * max(1, abs(ref))
        lp = stats.norm(0, 5).logpdf(x).sum()
        assert abs(o.log_prior(x) - lp) < 1e-12


def test_energy_funnel(oracle_lib):
    p = W.funnel(10)
    o = _ctx(oracle_lib, p)
    # log density at the origin, d = 10: -(ln 3 + 1/2 ln 2pi) + 9 (-1/2 ln 2pi)
    assert abs(o.energy(np.zeros(10)) - 10.288) < 5e-4
    rng = np.random.default_rng(4)
    for x in rng.uniform(-3, 3, (10, 10)):
        ref = -(stats.norm(0, 3).logpdf(x[0]) + stats.norm(0, math.exp(x[0] / 2)).logpdf(x[1:]).sum())
        assert abs(o.energy(x) - ref) < 1e-11 * max(1, abs(ref))


def test_energy_logreg(oracle_lib):
    p = W.logreg(7, n_data=40, seed=5)
    o = _ctx(oracle_lib, p)
    assert abs(o.energy(np.zeros(7)) - 40 * math.log(2)) < 1e-12   # softplus(0) = ln 2
    rng = np.random.default_rng(5)
    for th in rng.standard_normal((10, 7)) * 3:
        a = p.data_x @ th
        ref = np.sum(np.logaddexp(0.0, a) - p.data_y * a)
        assert abs(o.energy(th) - ref) < 1e-11 * max(1, abs(ref))


def _gp_nll_numpy(p, phi):
    D = p.d_in
    ls, sf2, sn2 = np.exp(phi[:D]), math.exp(2 * phi[D]), math.exp(2 * phi[D + 1])
    diff = (p.data_x[:, None, :] - p.data_x[None, :, :]) / ls
    K = sf2 * np.exp(-0.5 * np.sum(diff ** 2, -1)) + (sn2 + p.jitter) * np.eye(p.n_data)
    return -stats.multivariate_normal(np.zeros(p.n_data), K).logpdf(p.data_y)


def test_energy_gp(oracle_lib):
    p = W.gp_ard(d_in=3, n_data=30, seed=6, lengthscales=(0.3, 0.6, 1.0))
    o = _ctx(oracle_lib, p)
    rng = np.random.default_rng(6)
    for phi in rng.standard_normal((6, 5)) * 0.7:
        ref = _gp_nll_numpy(p, phi)
        assert abs(o.energy(phi) - ref) < 1e-8 * max(1, abs(ref))


# -------------------------------------------------------------- full runs --
def _runs(oracle_lib, p, seeds, **cfg):
    out = []
    for s in seeds:
        o = _ctx(oracle_lib, p, seed=s, **cfg)
        o.run()
        out.append((o.evidence(), o))
    return out


def _check_logz(runs, truth, per_run_sigmas=4.0):
    lz = np.array([r[0][0] for r in runs])
    sig = np.array([r[0][1] for r in runs])
    assert np.all(np.abs(lz - truth) < np.maximum(per_run_sigmas * sig, 0.05)), (lz, sig, truth)
    n = len(runs)
    assert abs(lz.mean() - truth) < max(3 * sig.mean() / math.sqrt(n), 0.05), (lz.mean(), truth)


def test_run_c1_gauss2_analytic(oracle_lib):
    """P14: normalised N(0, I_2) likelihood under U[-5,5]^2:
    log Z = 2 ln erf(5/sqrt 2) - 2 ln 10."""
    truth = 2 * math.log(math.erf(5 / math.sqrt(2))) - 2 * math.log(10)
    assert abs(truth + 4.605171332594708) < 1e-12
    p = W.gauss(2)
    runs = _runs(oracle_lib, p, range(1, 9), n_live=200, k=20, steps=10)
    _check_logz(runs, truth)
    # P19: posterior mean 0 and variance ~1 from the weighted dead points
    o = runs[0][1]
    x, lw = o.samples()
    w = np.exp(lw)
    ess = 1 / np.sum(w ** 2)
    m = w @ x
    assert np.all(np.abs(m) < 4 / math.sqrt(ess))
    assert np.all(np.abs(w @ (x - m) ** 2 - 1) < 0.25)


def test_run_gauss_times_gauss(oracle_lib):
    """P15: Gaussian likelihood under a Gaussian prior:
    log Z = log N(mu_L; 0, Sigma_L + s0^2 I); posterior mean closed form."""
    p = W.corr_gauss(3, seed=8, prior_sd=2.0, kappa=10.0)
    S0 = 4.0 * np.eye(3)
    truth = stats.multivariate_normal(np.zeros(3), p.meta["sigma_l"] + S0).logpdf(p.mu)
    runs = _runs(oracle_lib, p, range(1, 7), n_live=300, k=30, steps=6)
    _check_logz(runs, truth)
    Sl_inv = np.linalg.inv(p.meta["sigma_l"])
    post_cov = np.linalg.inv(Sl_inv + np.linalg.inv(S0))
    post_mean = post_cov @ (Sl_inv @ p.mu)
    x, lw = runs[0][1].samples()
    w = np.exp(lw)
    ess = 1 / np.sum(w ** 2)
    m = w @ x
    assert np.all(np.abs(m - post_mean) < 4 * np.sqrt(np.diag(post_cov) / ess) + 0.02)


def test_run_mog_erf_products(oracle_lib):
    """P16: MoG under a box: log Z = log sum_j w_j prod_i [Phi(hi) - Phi(lo)] - log|box|."""
    p = W.mog(4, n_comp=3, seed=12, half_width=6.0, mean_box=3.0, min_sep=4.0)
    mass = [p.w[j] * np.prod(stats.norm(p.mu[j], p.sigma[j]).cdf(p.hi) -
                              stats.norm(p.mu[j], p.sigma[j]).cdf(p.lo)) for j in range(3)]
    truth = math.log(sum(mass)) - np.sum(np.log(p.hi - p.lo))
    runs = _runs(oracle_lib, p, range(1, 7), n_live=400, k=40, steps=4)
    _check_logz(runs, truth)


def test_run_funnel_quadrature(oracle_lib):
    """P17: funnel under U[-a,a]^d: Z = (2a)^-d int N(y;0,3^2) erf(a/(sqrt2 e^{y/2}))^(d-1) dy."""
    d, a = 3, 8.0
    p = W.funnel(d, half_width=a)
    f = lambda y: stats.norm(0, 3).pdf(y) * math.erf(a / (math.sqrt(2) * math.exp(y / 2))) ** (d - 1)
    truth = math.log(integrate.quad(f, -a, a, limit=200, epsabs=0, epsrel=1e-12)[0]) - d * math.log(2 * a)
    runs = _runs(oracle_lib, p, range(1, 7), n_live=500, k=50, steps=6)
    _check_logz(runs, truth)


def test_run_logreg_quadrature(oracle_lib):
    """P18: logistic regression with 2 weights, prior N(0, I): Gauss-Hermite
    tensor quadrature of Z = E_prior[exp(-E)]."""
    p = W.logreg(2, n_data=30, seed=21)
    t, wq = np.polynomial.hermite_e.hermegauss(120)
    wq = wq / math.sqrt(2 * math.pi)
    T1, T2 = np.meshgrid(t, t, indexing="ij")
    th = np.stack([T1.ravel(), T2.ravel()], 1)
    a = th @ p.data_x.T
    loglik = -np.sum(np.logaddexp(0.0, a) - p.data_y * a, axis=1)
    truth = special.logsumexp(loglik + np.log(np.outer(wq, wq).ravel()))
    runs = _runs(oracle_lib, p, range(1, 7), n_live=300, k=30, steps=4)
    _check_logz(runs, truth)


def test_run_gp_quadrature(oracle_lib):
    """P18: GP ARD with one input (3 hyperparameters), prior N(0, I_3):
    Gauss-Hermite tensor quadrature with a numpy GP likelihood."""
    p = W.gp_ard(d_in=1, n_data=12, seed=31, lengthscales=(0.3,))
    t, wq = np.polynomial.hermite_e.hermegauss(36)
    wq = wq / math.sqrt(2 * math.pi)
    G = np.stack(np.meshgrid(t, t, t, indexing="ij"), -1).reshape(-1, 3)
    W3 = np.einsum("i,j,k->ijk", wq, wq, wq).ravel()
    ls, sf2, sn2 = np.exp(G[:, 0]), np.exp(2 * G[:, 1]), np.exp(2 * G[:, 2])
    diff2 = (p.data_x[:, None, 0] - p.data_x[None, :, 0]) ** 2
    K = sf2[:, None, None] * np.exp(-0.5 * diff2[None] / ls[:, None, None] ** 2)
    K = K + (sn2 + p.jitter)[:, None, None] * np.eye(p.n_data)[None]
    lam, V = np.linalg.eigh(K)
    proj = np.einsum("bij,i->bj", V, p.data_y)
    quad = np.sum(proj ** 2 / lam, axis=1)
    logdet = np.sum(np.log(np.abs(lam)), axis=1)
    loglik = -0.5 * quad - 0.5 * logdet - 0.5 * p.n_data * math.log(2 * math.pi)
    # nodes whose kernel matrix is numerically singular carry negligible prior mass
    loglik[lam[:, 0] < 1e-12 * lam[:, -1]] = -np.inf
    truth = special.logsumexp(loglik + np.log(W3))
    runs = _runs(oracle_lib, p, range(1, 5), n_live=200, k=20, steps=3)
    _check_logz(runs, truth)
