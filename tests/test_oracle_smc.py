"""Pins of the oracle's adaptive tempered SMC-SS (F3):
the temperature rule against its closed-form example and invariants, the
constant-energy special case, and the tempered evidence against the analytic
value on C1."""
import math

import numpy as np

from paper_2601_23252_b200 import workloads as W


def test_next_beta_closed_form_and_limits():
    from oracle import nsso
    # m = 2, E = {0, 1}, rho = 0.9: (1 + x)^2 / (1 + x^2) = 1.8 -> x = 1/2 -> db = ln 2
    assert abs(nsso.smc_next_beta([0.0, 1.0], 0.0, 0.9) - math.log(2)) < 1e-9
    assert nsso.smc_next_beta(np.full(50, 3.7), 0.2, 0.9) == 1.0  # equal energies: ESS = m always
    rng = np.random.default_rng(1)
    e = rng.exponential(3.0, 500)
    prev = 2.0
    for rho in (0.5, 0.7, 0.9, 0.95, 0.99):  # larger rho never gives a larger step
        b = nsso.smc_next_beta(e, 0.0, rho)
        assert 0.0 < b <= prev
        w = np.exp(-b * (e - e.min()))
        ess = w.sum() ** 2 / (w * w).sum()
        assert abs(ess - rho * e.size) <= 1e-6 * e.size
        prev = b


def test_constant_energy_single_stage():
    from oracle import nsso
    o = nsso.Oracle(W.flat(3, c=1.25), W.config(n_live=64, k=1, steps=2, seed=3), smc_rho=0.9)
    b, lz, t, _ = o.smc_run()
    assert b == 1.0 and t == 1 and abs(lz + 1.25) < 1e-12


def test_ladder_and_ess_per_stage():
    from oracle import nsso
    o = nsso.Oracle(W.gauss(2), W.config(n_live=300, k=1, steps=6, seed=4), smc_rho=0.9)
    betas = [0.0]
    while betas[-1] < 1.0:
        x, e = o.get_live()
        b_next = nsso.smc_next_beta(e, betas[-1], 0.9)
        o.smc_stage()
        b, lz, t, par = o.smc_state()
        assert b == b_next and b > betas[-1]
        if b < 1.0:
            w = np.exp(-(b - betas[-1]) * (e - e.min()))
            assert abs(w.sum() ** 2 / (w * w).sum() / 300 - 0.9) < 0.01
        betas.append(b)
    assert betas[-1] == 1.0 and len(betas) < 40


def test_tempered_evidence_matches_analytic_c1():
    from oracle import nsso
    truth = 2 * math.log(math.erf(5 / math.sqrt(2))) - 2 * math.log(10)
    lz = []
    for seed in range(1, 7):
        o = nsso.Oracle(W.gauss(2), W.config(n_live=400, k=1, steps=10, seed=seed), smc_rho=0.9)
        lz.append(o.smc_run()[1])
    lz = np.array(lz)
    assert abs(lz.mean() - truth) < 3 * lz.std(ddof=1) / math.sqrt(lz.size) + 0.02, (lz, truth)
