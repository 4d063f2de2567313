"""Pins for the oracle's HRSS step against what the
paper's theory fixes (App. D).

P5 cost theorem on a fixed slice (Thm P:1861-1876), P6 exactness on an
interval and on a ball, P7 the width constants u* and kappa_inf, the
ellipsoid width law (Thm P:2115-2126), null moves, constraint
preservation (north_star).
"""
import math

import numpy as np
import pytest
from scipy import integrate, optimize, stats

from paper_2601_23252_b200 import workloads as W


def phi(u):
    return ((1 + u) * math.log1p(u) - u) / u


def flat_box(oracle_lib, lo, hi, c=0.0, **cfg):
    p = W.flat(len(lo))
    p.lo, p.hi, p.c = np.asarray(lo, float), np.asarray(hi, float), c
    base = dict(n_live=4, k=1, steps=1)
    base.update(cfg)
    return oracle_lib.Oracle(p, W.config(**base))


def ball(oracle_lib, d, **cfg):
    # E = |x|^2 (GAUSS with sigma = 1/sqrt2, c = 0); slice {E < 1} = unit ball
    p = W.gauss(d, half_width=1.5, sigma=1 / math.sqrt(2.0))
    p.c = 0.0
    base = dict(n_live=4, k=1, steps=1)
    base.update(cfg)
    return oracle_lib.Oracle(p, W.config(**base))


@pytest.mark.parametrize("w", [2.0, 5.0, 10.0, 13.57677, 20.0, 40.0])
def test_cost_theorem_fixed_slice(oracle_lib, w):
    """E[N_out + N_shrink | l] = l/w + 1 + 2 phi(w/l), l = 10."""
    ell = 10.0
    o = flat_box(oracle_lib, [0.0], [ell])
    rng = np.random.default_rng(7)
    x0s = rng.uniform(0, ell, 100_000)
    tot = 0
    for i, x0 in enumerate(x0s):
        _, _, cnt = o.slice_step([x0], 0.0, [1.0], w, 1.0, 1, i, 0)
        tot += cnt[0] + cnt[1] + cnt[2]
        assert cnt[3] == 1
    expect = ell / w + 1 + 2 * phi(w / ell)
    assert abs(tot / x0s.size - expect) < 0.02 * expect


def test_exact_on_interval(oracle_lib):
    """One step from a fixed interior start is uniform on the slice."""
    ell = 10.0
    o = flat_box(oracle_lib, [0.0], [ell])
    out = np.array([o.slice_step([3.0], 0.0, [1.0], 4.0, 1.0, 2, i, 0)[0][0]
                    for i in range(100_000)])
    assert out.min() >= 0.0 and out.max() <= ell
    assert stats.kstest(out / ell, "uniform").pvalue > 1e-3


def test_ball_second_moment(oracle_lib):
    """Uniform in the unit d-ball: E|x|^2 = d/(d+2), d = 5."""
    d = 5
    o = ball(oracle_lib, d)
    rng = np.random.default_rng(3)
    x = np.zeros(d)
    e = 0.0
    r2 = []
    for i in range(60_000):
        v = rng.standard_normal(d)
        v /= np.linalg.norm(v)
        x, e, cnt = o.slice_step(x, e, v, 1.0, 1.0, 3, i % 50_000, i // 50_000)
        assert e < 1.0 and abs(e - x @ x) < 1e-12
        r2.append(x @ x)
    r2 = np.array(r2[1000:])
    batches = r2[: (r2.size // 100) * 100].reshape(100, -1).mean(axis=1)
    se = batches.std(ddof=1) / math.sqrt(batches.size)
    assert abs(r2.mean() - d / (d + 2)) < 3 * se + 1e-3


def test_null_move_on_empty_slice(oracle_lib):
    """E* below every energy: shrinkage cap reached, the start is returned."""
    o = flat_box(oracle_lib, [-1.0, -1.0], [1.0, 1.0], c=5.0)
    x, e, cnt = o.slice_step([0.1, 0.2], 0.5, [1.0, 0.0], 1.0, 1.0, 1, 0, 0)
    assert cnt == [0, 0, 100, 0]
    assert list(x) == [0.1, 0.2] and e == 0.5


def test_stepout_cap(oracle_lib):
    """Stepping-out is capped at max_stepout expansions per side."""
    o = flat_box(oracle_lib, [-1e6], [1e6], max_stepout=3)
    for i in range(200):
        _, _, cnt = o.slice_step([0.0], 0.0, [1.0], 1.0, 1.0, 1, i, 0)
        assert cnt[0] == 3 and cnt[1] == 3 and cnt[3] == 1


def test_u_star_and_fixed_slice_minimum(oracle_lib):
    """u* solves u - ln(1+u) = 1/2; paper prints 1.357676674."""
    u = optimize.brentq(lambda t: t - math.log1p(t) - 0.5, 0.1, 5.0, xtol=1e-14)
    assert abs(u - 1.357676674) < 1e-8
    # the theorem's cost is minimised there; the oracle's MC agrees on the side
    ell = 10.0
    o = flat_box(oracle_lib, [0.0], [ell])
    rng = np.random.default_rng(11)
    x0s = rng.uniform(0, ell, 40_000)

    def mc(w):
        return np.mean([sum(o.slice_step([x0], 0.0, [1.0], w, 1.0, 5, i, 0)[2][:3])
                        for i, x0 in enumerate(x0s)])
    c_opt, c_lo, c_hi = mc(u * ell), mc(0.4 * u * ell), mc(3.0 * u * ell)
    assert c_opt < c_lo and c_opt < c_hi


def kappa_inf():
    """kappa = 1/2 + E[R ln(1 + kappa/R)], R = Q^1/2 / E[Q^1/2], Q ~ Gamma(3/2, 2)
    (P:2150-2181), by fixed-point iteration with adaptive quadrature."""
    eq = 2 * math.sqrt(2 / math.pi)
    dens = stats.gamma(a=1.5, scale=2.0).pdf

    def f(k):
        g = lambda s: math.sqrt(s) * math.log1p(k * eq / math.sqrt(s)) * dens(s)
        return integrate.quad(g, 0, np.inf, limit=200)[0] / eq

    k = 1.0
    for _ in range(200):
        k_new = 0.5 + f(k)
        if abs(k_new - k) < 1e-12:
            break
        k = k_new
    return k_new


def test_kappa_inf_and_width_rule(oracle_lib):
    eq = integrate.quad(lambda s: math.sqrt(s) * stats.gamma(a=1.5, scale=2.0).pdf(s), 0, np.inf)[0]
    assert abs(eq - 2 * math.sqrt(2 / math.pi)) < 1e-9
    k = kappa_inf()
    assert abs(k - 1.3035) < 1e-3
    # OPTIMAL width with Mahalanobis directions: whitened live set ~ ball of
    # radius sqrt(d+2), ball corollary w* = 4 kappa R sqrt(2/(pi d))
    for d in (2, 10):
        o = ball(oracle_lib, d, n_live=50, k=5)
        _, w = o.metric()
        expect = 4 * 1.3035 * math.sqrt(d + 2) * math.sqrt(2 / (math.pi * d))
        assert abs(w - expect) < 1e-12 * expect
        o2 = ball(oracle_lib, d, n_live=50, k=5, width=0.5)
        assert abs(o2.metric()[1] - 0.5 * expect) < 1e-12 * expect


def _uniform_ball(rng, n, d):
    g = rng.standard_normal((n, d))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    return g * rng.uniform(size=(n, 1)) ** (1.0 / d)


@pytest.mark.parametrize("d", [16])
def test_ellipsoid_width_law(oracle_lib, d):
    """MC cost-vs-w in a unit ball is minimised near 4 kappa sqrt(2/(pi d))
    (Thm P:2115-2126; SPEC acceptance 4), and the cost std there is O(1)."""
    o = ball(oracle_lib, d)
    rng = np.random.default_rng(5)
    n = 12_000
    xs = _uniform_ball(rng, n, d)
    vs = rng.standard_normal((n, d))
    vs /= np.linalg.norm(vs, axis=1, keepdims=True)
    wstar = 4 * 1.3035 * math.sqrt(2 / (math.pi * d))
    grid = wstar * np.array([0.4, 0.6, 0.8, 1.0, 1.25, 1.6, 2.4])
    means, stds = [], []
    for gi, w in enumerate(grid):
        c = np.array([sum(o.slice_step(xs[i], xs[i] @ xs[i], vs[i], w, 1.0, 7, i, gi)[2][:3])
                      for i in range(n)])
        means.append(c.mean())
        stds.append(c.std())
    lw = np.log(grid)
    a, b, _ = np.polyfit(lw, means, 2)
    w_min = math.exp(-b / (2 * a))
    assert abs(w_min / wstar - 1) < 0.15
    assert 0.5 < stds[3] < 3.0


def test_constraint_preservation(oracle_lib):
    """Every accepted point satisfies E < E* and lies in the support (north_star)."""
    p = W.mog(4, n_comp=3, seed=5, half_width=10.0, mean_box=5.0, min_sep=4.0)
    o = oracle_lib.Oracle(p, W.config(n_live=100, k=10, steps=4, seed=3))
    for _ in range(20):
        o.step()
        x, e = o.get_live()
        tr = o.trace()
        for s in tr["dest_gid"]:
            assert e[s] < tr["e_star"]
            assert np.all(x[s] >= p.lo) and np.all(x[s] <= p.hi)
            assert abs(o.energy(x[s]) - e[s]) <= 1e-12 * max(1.0, abs(e[s]))
