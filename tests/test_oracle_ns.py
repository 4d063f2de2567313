"""Pins for the oracle's outer NS iteration, volume bookkeeping, quadrature,
termination and metric (SPEC worked examples).

P3/P4 worked deletion examples, ties (DESIGN R-1), P11/P12 shrinkage order
statistics, P13 single-point trapezoid, flat-likelihood quadrature identities,
P21 termination, metric, directions, P20 determinism.
"""
import math

import numpy as np
import pytest
from scipy import special

from paper_2601_23252_b200 import workloads as W


def flat_ctx(oracle_lib, n, k, d=1, c=0.0, steps=1, **cfg):
    p = W.flat(d, half_width=1.0, c=c)
    return oracle_lib.Oracle(p, W.config(n_live=n, k=k, steps=steps, **cfg))


def test_worked_example_m5_k2(oracle_lib):
    """m=5, k=2, E=[1,2,3,4,5] -> E*=4; dead (5, n=5), (4, n=4); survivors {1,2,3}."""
    o = flat_ctx(oracle_lib, 5, 2, c=0.0)
    x = np.linspace(-0.5, 0.5, 5)[:, None]
    o.set_live(x, np.array([1.0, 2.0, 3.0, 4.0, 5.0]), 1)
    o.step()
    tr = o.trace()
    assert tr["e_star"] == 4.0
    assert list(tr["dead_gid"]) == [4, 3]
    assert list(tr["dest_gid"]) == [3, 4]
    assert set(tr["parent_gid"]) <= {0, 1, 2}
    dead = o.dead()
    assert list(dead["e"]) == [5.0, 4.0]
    assert list(dead["n_live"]) == [5, 4]
    assert np.allclose(dead["x"][:, 0], [x[4, 0], x[3, 0]])


def test_k1_is_classic_ns(oracle_lib):
    """k = 1 -> n_live = m for every record."""
    o = flat_ctx(oracle_lib, 7, 1)
    rng = np.random.default_rng(0)
    o.set_live(rng.uniform(-1, 1, (7, 1)), rng.uniform(0, 1, 7), 1)
    for _ in range(5):
        o.step()
    assert list(o.dead()["n_live"]) == [7] * 5


def test_ties_larger_gid_dies_first(oracle_lib):
    o = flat_ctx(oracle_lib, 6, 3)
    o.set_live(np.zeros((6, 1)), np.array([2.0, 2.0, 1.0, 2.0, 0.5, 2.0]), 1)
    o.step()
    tr = o.trace()
    assert list(tr["dead_gid"]) == [5, 3, 1]
    assert tr["e_star"] == 2.0
    assert set(tr["parent_gid"]) <= {0, 2, 4}


def test_parent_draw_is_multiply_high(oracle_lib):
    """Parent of destination s: S[floor(u32 (n-k) / 2^32)] (DESIGN R-4)."""
    n, k, seed = 50, 20, 77
    o = flat_ctx(oracle_lib, n, k, seed=seed)
    e = np.arange(n, dtype=float)[::-1].copy()        # gid 0..19 have the largest E
    o.set_live(np.zeros((n, 1)), e, 3)
    o.step()
    tr = o.trace()
    surv = np.arange(20, 50)
    for s, par in zip(tr["dest_gid"], tr["parent_gid"]):
        u32 = oracle_lib.draw_u32(seed, 3, int(s), 2, 0, 0)
        assert par == surv[(u32 * (n - k)) >> 32]


def test_unrolled_shrinkage_beta(oracle_lib):
    """P11: one batch at (n=10, k=3): replica 0 gets
    -(1/10+1/9+1/8); the simulated replicas have mean psi(8)-psi(11) and
    variance psi1(8)-psi1(11) (Beta(8,3) contraction)."""
    vals = []
    for seed in range(1, 401):
        o = flat_ctx(oracle_lib, 10, 3, seed=seed, steps=0)
        o.set_live(np.zeros((10, 1)), np.arange(10, dtype=float), 1)
        o.step()
        lx = o.volume_reps()
        assert abs(lx[0] + (1 / 10 + 1 / 9 + 1 / 8)) < 1e-15
        vals.append(lx[1:])
    v = np.concatenate(vals)
    mean, var = special.digamma(8) - special.digamma(11), special.polygamma(1, 8) - special.polygamma(1, 11)
    assert abs(mean - (-0.336111)) < 1e-6
    assert abs(v.mean() - mean) < 4 * math.sqrt(var / v.size)
    assert abs(v.var() / var - 1) < 0.05


def test_500_single_deaths(oracle_lib):
    """P12: 500 deaths at n=100 -> log X mean -5.0, sd sqrt(500)/100."""
    o = flat_ctx(oracle_lib, 100, 1, steps=0, n_volume_sims=2000, max_dead=700)
    for _ in range(500):
        o.step()
    lx = o.volume_reps()
    assert abs(lx[0] + 5.0) < 1e-12
    sims = lx[1:]
    assert abs(sims.mean() + 5.0) < 4 * 0.2236 / math.sqrt(sims.size)
    assert abs(sims.std() - math.sqrt(500) / 100) < 0.02


def test_single_point_trapezoid(oracle_lib):
    """P13: one dead point with E = 0 -> log Z = -ln 2 for every replica."""
    o = flat_ctx(oracle_lib, 2, 1, steps=0)
    o.set_live(np.zeros((2, 1)), np.array([0.0, -1.0]), 1)
    o.step()
    reps = o.evidence_reps()
    assert np.allclose(reps, -math.log(2.0), rtol=0, atol=1e-15)


@pytest.mark.parametrize("quad", [W.Q_TRAPEZOID, W.Q_RECTANGLE])
def test_flat_likelihood_quadrature_identity(oracle_lib, quad):
    """E = c everywhere: the trapezoid sum telescopes to e^-c (1 + X_1 - X_N)/2 and
    the rectangle sum to e^-c (1 - X_N); replica 0."""
    n, k, c = 20, 4, 1.7
    o = flat_ctx(oracle_lib, n, k, c=c, steps=1, quadrature=quad)
    for _ in range(6):
        o.step()
    o.finalise()
    lz0 = o.evidence_reps()[0]
    lxn = o.volume_reps()[0]
    x1 = math.exp(-1.0 / n)
    if quad == W.Q_TRAPEZOID:
        expect = -c + math.log((1 + x1 - math.exp(lxn)) / 2)
    else:
        expect = -c + math.log(1 - math.exp(lxn))
    assert abs(lz0 - expect) < 1e-12
    # replica 0's final log X is -sum over all deaths of 1/n_live
    total = sum(1.0 / (n - j) for j in range(k)) * 6 + sum(1.0 / (n - j) for j in range(n))
    assert abs(lxn + total) < 1e-12


def test_flat_likelihood_terminates_at_e_minus_3(oracle_lib):
    """P21: flat likelihood stops once the remaining volume X < ~e^-3."""
    o = flat_ctx(oracle_lib, 100, 10, steps=1)
    while not o.should_terminate():
        o.step()
        assert o.info()["iteration"] < 100
    lx = o.volume_reps()[0]
    per_iter = -(sum(1.0 / (100 - j) for j in range(10)))
    assert -3.0 + per_iter - 0.05 < lx < -3.0 + 0.05


def test_metric_covariance(oracle_lib):
    """metric = sample covariance (+ reg * mean diag) as L L^T."""
    rng = np.random.default_rng(4)
    n = 100_000
    x = rng.standard_normal((n, 2)) * np.array([1.0, 2.0])
    p = W.gauss(2, half_width=100.0)
    o = oracle_lib.Oracle(p, W.config(n_live=n, k=1, steps=1, metric_reg=0.0, max_dead=2 * n))
    o.set_live(x, np.zeros(n), 1)
    L, _ = o.metric()
    S = L @ L.T
    assert np.allclose(S, np.cov(x.T), rtol=1e-9, atol=1e-12)
    assert np.allclose(np.diag(S), [1.0, 4.0], rtol=0.05)
    assert np.allclose(np.triu(L, 1), 0.0)


def test_metric_degenerate_clouds(oracle_lib):
    p = W.gauss(2, half_width=100.0)
    o = oracle_lib.Oracle(p, W.config(n_live=2, k=1, steps=1))
    o.set_live(np.zeros((2, 2)), np.zeros(2), 1)              # two copies of the origin
    assert np.array_equal(o.metric()[0], np.eye(2))
    o = oracle_lib.Oracle(p, W.config(n_live=50, k=1, steps=1))
    t = np.linspace(-1, 1, 50)
    o.set_live(np.stack([t, 2 * t], 1), np.zeros(50), 1)        # points on a line
    L, _ = o.metric()
    assert np.all(np.diag(L) > 0) and np.all(np.isfinite(L))
    assert np.all(np.linalg.eigvalsh(L @ L.T) > 0)


def test_directions(oracle_lib):
    """v = L z / |z|: unit Mahalanobis norm, uniform on the sphere when L = I,
    stretched along the high-variance axis (DESIGN R-6)."""
    rng = np.random.default_rng(2)
    n = 20_000
    p = W.gauss(2, half_width=100.0)
    o = oracle_lib.Oracle(p, W.config(n_live=n, k=1, steps=1, metric_reg=0.0, max_dead=2 * n))
    o.set_live(rng.standard_normal((n, 2)) * [10.0, 1.0], np.zeros(n), 1)
    L, _ = o.metric()
    Li = np.linalg.inv(L)
    vs = np.array([o.direction(1, g, 0) for g in range(5000)])
    assert np.allclose(np.linalg.norm(vs @ Li.T, axis=1), 1.0, atol=1e-12)
    assert np.mean(vs[:, 0] ** 2) > 10 * np.mean(vs[:, 1] ** 2)
    o2 = oracle_lib.Oracle(W.gauss(3, half_width=100.0), W.config(n_live=n, k=1, steps=1, metric_reg=0.0, max_dead=2 * n))
    o2.set_live(rng.standard_normal((n, 3)), np.zeros(n), 1)
    v3 = np.array([o2.direction(1, g, 0) for g in range(20000)])
    assert np.all(np.abs(v3.mean(0)) < 4 * math.sqrt(1 / 3 / 20000) * 1.05)


def test_euclidean_direction_and_width(oracle_lib):
    rng = np.random.default_rng(8)
    n = 5000
    p = W.gauss(3, half_width=100.0)
    o = oracle_lib.Oracle(p, W.config(n_live=n, k=1, steps=1, dir_norm=W.DIR_EUCLIDEAN, metric_reg=0.0, max_dead=2 * n))
    o.set_live(rng.standard_normal((n, 3)) * [3.0, 1.0, 0.5], np.zeros(n), 1)
    v = o.direction(1, 5, 0)
    assert abs(np.linalg.norm(v) - 1) < 1e-12
    L, w = o.metric()
    sig_inv = np.linalg.inv(L @ L.T)
    mu = np.trace(sig_inv) / (3 * 5)
    assert abs(w - 4 * 1.3035 * math.sqrt(2 / (math.pi * mu * 3))) < 1e-10 * w


def test_determinism(oracle_lib):
    """P20: identical seed and config -> bit-identical dead list."""
    p = W.mog(4, n_comp=3, seed=5, half_width=10.0, mean_box=5.0, min_sep=4.0)
    cfg = W.config(n_live=100, k=10, steps=4, seed=9)
    a = oracle_lib.Oracle(p, cfg)
    b = oracle_lib.Oracle(p, cfg)
    for _ in range(15):
        a.step()
        b.step()
    da, db = a.dead(), b.dead()
    for key in da:
        assert np.array_equal(da[key], db[key])
    assert np.array_equal(a.evidence_reps(), b.evidence_reps())


def test_invalid_args(oracle_lib):
    p = W.flat(2)
    for bad in (dict(n_live=5, k=5, steps=1), dict(n_live=5, k=0, steps=1),
                dict(n_live=5, k=1, steps=-1), dict(n_live=5, k=1, steps=1, n_volume_sims=1),
                dict(n_live=5, k=1, steps=1, max_shrink=0)):
        with pytest.raises(oracle_lib.OracleError) as ei:
            oracle_lib.Oracle(p, W.config(**bad))
        assert ei.value.code == 1


def test_capacity_and_state_errors(oracle_lib):
    o = flat_ctx(oracle_lib, 10, 5, max_dead=12)
    with pytest.raises(oracle_lib.OracleError) as ei:
        o.evidence()
    assert ei.value.code == 7
    with pytest.raises(oracle_lib.OracleError) as ei:
        o.step()
        o.step()
    assert ei.value.code == 8


def test_samples_weights_normalised(oracle_lib):
    p = W.gauss(2)
    o = oracle_lib.Oracle(p, W.config(n_live=100, k=10, steps=4, seed=2))
    o.run()
    x, lw = o.samples()
    assert x.shape[0] == lw.shape[0] == o.dead()["e"].shape[0]
    assert abs(special.logsumexp(lw)) < 1e-10
    # geometric-mean weights: recomputed trajectories agree with the streamed
    # replicas -> weighted mean of exp(-E) dX reproduces log Z within its spread
    lz, err = o.evidence()
    assert err > 0


def test_prior_support_error(oracle_lib):
    """Init rejection budget 100 n: energy +inf everywhere -> error."""
    p = W.gauss(2, half_width=1.0)
    p.c = float("inf")
    with pytest.raises(oracle_lib.OracleError) as ei:
        oracle_lib.Oracle(p, W.config(n_live=10, k=1, steps=1))
    assert ei.value.code == 2
