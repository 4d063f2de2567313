"""Pins of the oracle's posterior products (F2: nsso_posterior, nsso_resample;
P:123-132 reweighting to any inverse temperature, P:1225-1255 geometric-mean
weights and Kish ESS, S:310-316 equal-weight resampling)."""
import math

import numpy as np
import pytest
from scipy import special, stats

from paper_2601_23252_b200 import workloads as W


def _run(prob, cfg):
    from oracle import nsso
    o = nsso.Oracle(prob, cfg)
    o.run(5000)
    return o


def _gauss_box_logz(beta, d=2, a=5.0):
    """log Z(beta) = log int N(x; 0, I)^beta dU[-a, a]^d, closed form."""
    return (-d * math.log(2 * a) - 0.5 * beta * d * math.log(2 * math.pi)
            + d * (0.5 * math.log(2 * math.pi / beta) + math.log(special.erf(a * math.sqrt(beta / 2)))))


@pytest.fixture(scope="module")
def c1_run():
    return _run(W.gauss(2), W.config(n_live=400, k=40, steps=10, seed=5))


@pytest.mark.parametrize("beta", [0.5, 1.0, 2.0, 4.0])
def test_tempered_evidence_matches_closed_form(c1_run, beta):
    lz, err, ess = c1_run.posterior(beta)
    truth = _gauss_box_logz(beta)
    assert abs(lz - truth) <= max(3 * err, 0.05), (beta, lz, truth, err)
    assert 1.0 <= ess <= c1_run.info()["iteration"] * 40 + 400


def test_beta_one_is_the_evidence_and_the_sample_weights(c1_run):
    lz, err, ess, lw = c1_run.posterior(1.0, weights=True)
    lz0, err0 = c1_run.evidence()
    assert abs(lz - lz0) < 1e-10 and abs(err - err0) < 1e-10
    _, lw_s = c1_run.samples()
    assert np.allclose(lw, lw_s, rtol=0, atol=1e-12)
    # Kish: (sum w)^2 / sum w^2 of the unnormalised weights
    w = np.exp(lw - lw.max()) * 7.5
    assert abs(ess - w.sum() ** 2 / (w * w).sum()) < 1e-8 * ess


def test_beta_zero_rectangle_is_total_prior_mass():
    """Rectangle quadrature: sum_i (X_{i-1} - X_i) = 1 - X_N in every replica,
    so log Z^(r)(0) = log(1 - X_N^(r))."""
    from oracle import nsso
    o = nsso.Oracle(W.gauss(2), W.config(n_live=100, k=10, steps=5, seed=2, quadrature=W.Q_RECTANGLE))
    for _ in range(30):
        o.step()
    lz, err, _ = o.posterior(0.0)
    lx = o.volume_reps()[1:]
    per = np.log1p(-np.exp(lx))
    assert abs(lz - per.mean()) < 1e-10
    assert abs(err - per.std(ddof=1)) < 1e-10


def test_flat_likelihood_factorises():
    """E = c: log Z(beta) = -beta c + log Z(0) exactly."""
    from oracle import nsso
    prob = W.flat(3, c=2.5)
    o = nsso.Oracle(prob, W.config(n_live=64, k=8, steps=2, seed=4))
    for _ in range(12):
        o.step()
    z0, e0, s0 = o.posterior(0.0)
    for beta in (0.3, 1.0, 3.0):
        zb, eb, sb = o.posterior(beta)
        assert abs(zb - (-beta * 2.5 + z0)) < 1e-10
        assert abs(eb - e0) < 1e-10 and abs(sb - s0) < 1e-8 * s0


def test_cold_limit_concentrates_on_the_best_point(c1_run):
    lz, err, ess, lw = c1_run.posterior(1e9, weights=True)
    e = c1_run.dead()["e"]
    assert ess < 1.01 and np.argmax(lw) == np.argmin(e)
    idx, x = c1_run.resample(50, seed=9, beta=1e9)
    assert np.all(idx == np.argmin(e))


def test_resample_frequencies_follow_the_weights(c1_run):
    _, _, _, lw = c1_run.posterior(1.0, weights=True)
    m = 200_000
    idx, x = c1_run.resample(m, seed=11)
    p = np.exp(lw)
    counts = np.bincount(idx, minlength=p.size)
    order = np.argsort(p)[::-1]
    # chi-square over bins grouped to expected >= 50
    groups, cur_o, cur_e = [], 0, 0.0
    for i in order:
        cur_o += counts[i]
        cur_e += m * p[i]
        if cur_e >= 50:
            groups.append((cur_o, cur_e))
            cur_o, cur_e = 0, 0.0
    o_, e_ = np.array([g[0] for g in groups], float), np.array([g[1] for g in groups])
    chi2 = ((o_ - e_) ** 2 / e_).sum()
    assert stats.chi2.sf(chi2, len(groups) - 1) > 1e-4
    dx = c1_run.dead()["x"]
    assert np.array_equal(x, dx[idx])
    # posterior mean of N(0, I) under the box ~ 0, variance ~ 1
    assert np.all(np.abs(x.mean(axis=0)) < 0.1) and np.all(np.abs(x.var(axis=0) - 1) < 0.15)
