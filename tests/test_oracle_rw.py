"""Pins of the oracle's constrained random-walk mutation (F1, P:301-302,
P:765): its stationary law is the prior restricted to E < E* (checked by
KS against the closed-form restricted law in 1-D for a box and a Gaussian
prior), accepted points obey the constraint, and an NS run with RW
replacements reaches the analytic evidence."""
import math

import numpy as np
from scipy import stats

from paper_2601_23252_b200 import workloads as W


def _chain(prob, e_star, x0, steps, width=1.0):
    from oracle import nsso
    o = nsso.Oracle(prob, W.config(n_live=8, k=1, steps=1, mutation=W.MUT_RW, width=width))
    cloud = np.linspace(-1.5, 1.5, 8)[:, None] * np.ones((1, prob.d))  # metric: L from this cloud
    o.set_live(cloud, np.array([o.energy(q) for q in cloud]), 1)
    x, e = np.array(x0, float), o.energy(x0)
    xs, acc = [], 0
    for j in range(steps):
        x, e, cnt = o.rw_step(x, e, e_star, 1, 0, j)
        acc += cnt[3]
        assert e < e_star and cnt[3] <= cnt[2]
        xs.append(x[0])
    return np.array(xs), acc / steps


def test_rw_stationary_uniform_on_constrained_interval():
    """Box prior U[-10, 10], E = x^2/2: the constrained law is U(-a, a), a = sqrt(2 E*)."""
    prob = W.gauss(1, half_width=10.0)  # E = x^2/2 + const
    from oracle import nsso
    o = nsso.Oracle(prob, W.config(n_live=8, k=1, steps=1))
    c = o.energy(np.zeros(1))
    e_star = c + 2.0  # a = 2
    xs, acc = _chain(prob, e_star, np.array([0.3]), 60_000)
    xs = xs[1000::25]
    assert 0.05 < acc < 0.95
    assert stats.kstest(xs, stats.uniform(loc=-2, scale=4).cdf).pvalue > 1e-3


def test_rw_stationary_gaussian_prior_truncated():
    """Gaussian prior N(0, 1), flat likelihood below the threshold: the chain
    samples N(0, 1) (E* above the constant energy)."""
    prob = W.flat(1, c=0.0)
    prob = W.Problem(name="flatg", d=1, prior_kind=W.PRIOR_GAUSS_DIAG, energy_kind=W.E_FLAT,
                     mean=np.zeros(1), sd=np.ones(1), c=0.0)
    xs, acc = _chain(prob, 1.0, np.array([0.2]), 60_000)
    xs = xs[1000::25]
    assert stats.kstest(xs, stats.norm().cdf).pvalue > 1e-3


def test_rw_full_run_reaches_analytic_evidence():
    from oracle import nsso
    truth = 2 * math.log(math.erf(5 / math.sqrt(2))) - 2 * math.log(10)
    ok = []
    for seed in (1, 2):
        o = nsso.Oracle(W.gauss(2), W.config(n_live=200, k=20, steps=20, seed=seed, mutation=W.MUT_RW))
        o.run(5000)
        lz, sig = o.evidence()
        ok.append(abs(lz - truth) <= max(3 * sig, 0.05))
        info = o.info()
        assert info["expansions"] == 0 and info["shrinks"] == 0
    assert all(ok)
