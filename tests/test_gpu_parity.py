"""CUDA path vs fp64 oracle, through the C ABI (needs a B200).

Single-iteration parity on every energy / prior / option, metric and evidence
parity, init parity, full-run log Z against the analytic values, error paths.
"""
import math

import numpy as np
import pytest
from scipy import special, stats

from paper_2601_23252_b200 import workloads as W
from tests.parity_util import check_subset, compare_iteration, inject_pair, prior_scale

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_23252_b200 import nss
    nss.lib()


def _mog_small(d=6, K=3):
    return W.mog(d, n_comp=K, seed=17, half_width=8.0, mean_box=4.0, min_sep=4.0)


CASES = {
    # name: (problem factory, config kwargs, warm iterations)
    "c1_gauss2": (lambda: W.gauss(2), dict(n_live=200, k=20, steps=10), 5),
    "c2_mog10": (lambda: W.mog(10), dict(n_live=2000, k=200, steps=10), 3),
    "mog_ragged": (_mog_small, dict(n_live=777, k=91, steps=5), 2),
    "corr_gauss_d40": (lambda: W.corr_gauss(40, seed=5), dict(n_live=600, k=60, steps=8), 2),
    "corr_gauss_d100": (lambda: W.corr_gauss(100, seed=5), dict(n_live=1000, k=100, steps=6), 0),
    "funnel_d16": (lambda: W.funnel(16), dict(n_live=500, k=50, steps=6), 2),
    "funnel_d100": (lambda: W.funnel(100), dict(n_live=800, k=80, steps=4), 0),
    "logreg_small": (lambda: W.logreg(5, n_data=300, seed=3), dict(n_live=300, k=30, steps=5), 2),
    "logreg_split_data": (lambda: W.logreg(20, n_data=700, seed=3, half_exact=False), dict(n_live=300, k=30, steps=4),
                          2),
    "flat_d1": (lambda: W.flat(1), dict(n_live=64, k=7, steps=3), 1),
    "d33_ragged_lanes": (lambda: W.gauss(33, half_width=4.0), dict(n_live=333, k=33, steps=3), 1),
    "k_n_minus_1": (lambda: W.gauss(3), dict(n_live=50, k=49, steps=3), 0),
    "k1": (lambda: W.gauss(3), dict(n_live=50, k=1, steps=3), 2),
    "p0": (lambda: W.gauss(3), dict(n_live=50, k=5, steps=0), 2),
    "euclidean": (lambda: W.corr_gauss(8, seed=2), dict(n_live=300, k=30, steps=5, dir_norm=W.DIR_EUCLIDEAN), 2),
    "fixed_width": (lambda: W.mog(4, n_comp=2, seed=4, mean_box=3.0, min_sep=3.0),
                    dict(n_live=300, k=30, steps=5, width_rule=W.W_FIXED, width=1.0), 2),
    "width_scale_quarter": (lambda: W.gauss(5), dict(n_live=300, k=30, steps=5, width=0.25), 2),
    "stepout_cap": (lambda: W.gauss(2, half_width=50.0, sigma=20.0),
                    dict(n_live=100, k=10, steps=4, width_rule=W.W_FIXED, width=0.05, max_stepout=3), 0),
    "shrink_cap": (lambda: W.gauss(4), dict(n_live=100, k=10, steps=4, max_shrink=2), 2),
    "d128_max": (lambda: W.gauss(128, half_width=4.0), dict(n_live=300, k=30, steps=2), 0),
    "select_large": (lambda: W.gauss(2), dict(n_live=100_000, k=50_000, steps=1, max_dead=400_000), 0),
    # large-n thresholding paths of k_select: 32-bit ordinals on chip + chunked
    # bitonic dead-order sort; keys in global memory
    "select_ord32": (lambda: W.gauss(3), dict(n_live=20_000, k=9_000, steps=2), 0),
    "select_global": (lambda: W.gauss(2), dict(n_live=30_000, k=10_000, steps=1), 0),
}


@pytest.mark.parametrize("engine", ["warp", "lane", "batch"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_single_iteration_parity(name, engine):
    make, kw, warm = CASES[name]
    prob = make()
    cfg = W.config(seed=11, **kw)
    gpu, ref = inject_pair(prob, cfg, warm_iters=warm, engine=engine)
    if engine != "warp" and gpu.engine() != engine:
        pytest.skip(f"{engine} engine does not apply to this case")
    # metric from the same injected cloud
    Lg, wg = gpu.metric()
    Lr, wr = ref.metric()
    assert np.allclose(Lg, Lr, rtol=1e-5, atol=1e-7 * np.abs(Lr).max())
    assert abs(wg - wr) <= 1e-6 * wr
    st = compare_iteration(gpu, ref, prob, f"{name} {engine}")
    if name == "shrink_cap":
        assert (st["counts_g"][:, :, 3] == 0).any()  # some null moves happened
    if name == "stepout_cap":
        assert (st["counts_g"][:, :, 0] == 3).any()
    # dead records identical
    dg, dr = gpu.dead(), ref.dead()
    assert np.array_equal(dg["n_live"], dr["n_live"])
    assert np.array_equal(dg["gid"], dr["gid"])
    assert np.array_equal(dg["e"].astype(np.float64), dr["e"])
    assert np.array_equal(dg["x"].astype(np.float64), dr["x"])
    # evidence replicas after one iteration (same dead energies, same draws)
    assert np.allclose(gpu.volume_reps(), ref.volume_reps(), rtol=0, atol=1e-12)
    assert np.allclose(gpu.evidence_reps(), ref.evidence_reps(), rtol=0, atol=1e-10)
    gpu.close()


def test_several_iterations_teacher_forced():
    """Re-inject the oracle state every iteration (SURVEY C-9 T3) for 6 iterations of C2."""
    prob = W.mog(10)
    cfg = W.config(n_live=2000, k=200, steps=10, seed=5)
    from oracle import nsso
    ref = nsso.Oracle(prob, cfg)
    from paper_2601_23252_b200 import nss
    gpu = nss.Sampler(prob, cfg)
    for it in range(1, 7):
        x, _ = ref.get_live()
        x32 = x.astype(np.float32)
        e32 = np.array([ref.energy(xi.astype(np.float64)) for xi in x32]).astype(np.float32)
        ref.set_live(x32.astype(np.float64), e32.astype(np.float64), it)
        gpu.set_live(x32, e32, it)
        compare_iteration(gpu, ref, prob, f"C2 teacher-forced it {it}")


def test_init_parity():
    for prob, kw in ((W.gauss(2), dict(n_live=200, k=20, steps=2)),
                     (W.mog(10), dict(n_live=500, k=50, steps=2)),
                     (W.corr_gauss(12, seed=3), dict(n_live=300, k=30, steps=2)),
                     (W.logreg(4, n_data=100, seed=2), dict(n_live=100, k=10, steps=2))):
        from oracle import nsso
        from paper_2601_23252_b200 import nss
        cfg = W.config(seed=21, **kw)
        ref = nsso.Oracle(prob, cfg)
        gpu = nss.Sampler(prob, cfg)
        xg, eg = gpu.get_live()
        xr, er = ref.get_live()
        scale = 1.0 if prob.prior_kind == W.PRIOR_BOX else 5.0
        assert np.allclose(xg, xr, rtol=1e-6, atol=1e-6 * scale)
        assert np.allclose(eg, er, rtol=1e-5, atol=1e-5)
        assert gpu.info()["init_evals"] == ref.info()["init_evals"]
        gpu.close()


def test_evidence_and_weights_exact_on_flat():
    """Flat energy, p = 0: both sides hold identical dead lists, so every replica's
    log Z, log X and the posterior weights must agree to fp64 rounding."""
    from oracle import nsso
    from paper_2601_23252_b200 import nss
    for quad in (W.Q_TRAPEZOID, W.Q_RECTANGLE):
        prob = W.flat(2, c=0.7)
        cfg = W.config(n_live=97, k=13, steps=0, seed=4, quadrature=quad, n_volume_sims=50)
        ref = nsso.Oracle(prob, cfg)
        gpu = nss.Sampler(prob, cfg)
        x, e = ref.get_live()
        e = (np.arange(97, dtype=np.float64)[::-1] * 0.01).astype(np.float32).astype(np.float64)
        ref.set_live(x.astype(np.float32).astype(np.float64), e, 1)
        gpu.set_live(x.astype(np.float32), e.astype(np.float32), 1)
        for _ in range(9):
            gpu.step()
            ref.step()
        assert np.allclose(gpu.evidence_reps(), ref.evidence_reps(), rtol=0, atol=1e-10)
        gpu.finalise()
        ref.finalise()
        assert np.allclose(gpu.volume_reps(), ref.volume_reps(), rtol=0, atol=1e-10)
        assert np.allclose(gpu.evidence_reps(), ref.evidence_reps(), rtol=0, atol=1e-10)
        lg, sg = gpu.evidence()
        lr, sr = ref.evidence()
        assert abs(lg - lr) < 1e-10 and abs(sg - sr) < 1e-10
        xg, wg = gpu.samples()
        xr, wr = ref.samples()
        assert np.allclose(wg, wr, rtol=0, atol=1e-9)
        assert np.allclose(xg, xr, rtol=0, atol=0)
        gpu.close()


def _run_logz(prob, kw, seeds):
    from paper_2601_23252_b200 import nss
    out = []
    for s in seeds:
        g = nss.Sampler(prob, W.config(seed=s, **kw))
        info = g.run()
        out.append(g.evidence() + (info,))
        g.close()
    return out


def test_full_run_c1_analytic():
    """north_star: |log Z - analytic| <= max(3 sigma, 0.05) on C1 (P14)."""
    truth = 2 * math.log(math.erf(5 / math.sqrt(2))) - 2 * math.log(10)
    res = _run_logz(W.gauss(2), dict(n_live=200, k=20, steps=10), range(1, 9))
    lz = np.array([r[0] for r in res])
    sig = np.array([r[1] for r in res])
    assert np.all(np.abs(lz - truth) <= np.maximum(3 * sig, 0.05)), (lz, sig)
    assert abs(lz.mean() - truth) <= max(3 * sig.mean() / math.sqrt(len(lz)), 0.05)
    assert all(r[2]["terminated"] and r[2]["finalised"] for r in res)


def test_full_run_c2_analytic():
    prob = W.mog(10)
    mass = [prob.w[j] * np.prod(stats.norm(prob.mu[j], prob.sigma[j]).cdf(prob.hi) -
                                 stats.norm(prob.mu[j], prob.sigma[j]).cdf(prob.lo)) for j in range(4)]
    truth = math.log(sum(mass)) - np.sum(np.log(prob.hi - prob.lo))
    res = _run_logz(prob, dict(n_live=2000, k=200, steps=10), range(1, 4))
    for lz, sig, info in res:
        assert abs(lz - truth) <= max(3 * sig, 0.05), (lz, sig, truth)


def test_full_run_c3a_analytic_p3d():
    """C3a at full size (d = 100, kappa = 100, n = 1e4, k = 1e3) run to
    termination with p = 3d HRSS steps (the paper's high-d setting):
    log N(mu_L; 0, Sigma_L + 25 I) within max(3 sigma, 0.05).  (At p = d the
    chains under-mix and log Z comes out 3-5 sigma high,
    profiles/r01_accuracy.md.)"""
    from scipy import stats as st
    prob, cfg = W.workload("C3a")
    truth = st.multivariate_normal(np.zeros(prob.d), prob.meta["sigma_l"] + np.diag(prob.sd ** 2)).logpdf(
        prob.mu - prob.mean)
    res = _run_logz(prob, dict(n_live=cfg["n_live"], k=cfg["k"], steps=3 * prob.d,
                               max_dead=cfg["n_live"] + cfg["k"] * 8000), [1])
    for lz, sig, info in res:
        assert info["terminated"]
        assert abs(lz - truth) <= max(3 * sig, 0.05), (lz, sig, truth)


def _vs_oracle(prob, kw, seeds, oracle_runs=None):
    """Same configuration and seed on both sides, full runs to termination:
    |log Z_GPU - log Z_oracle| <= max(3 sigma, 0.05) per run (north_star,
    SURVEY C-9 T4), sigma = the two runs' replica spreads combined
    (sqrt(sg^2 + so^2): the two trajectories are independent draws of the same
    estimator once fp32 and fp64 decisions part).  oracle_runs: stored oracle
    results (tests/golden, scripts/golden_oracle_fullruns.py) per seed."""
    from oracle import nsso
    out = []
    for s in seeds:
        if oracle_runs is None:
            o = nsso.Oracle(prob, W.config(seed=s, **kw))
            o.run()
            lr, sr = o.evidence()
            o.close()
        else:
            lr, sr = oracle_runs[s]
        (lg, sg, info), = _run_logz(prob, kw, [s])
        assert info["terminated"]
        bound = max(3 * math.hypot(sg, sr), 0.05)
        out.append((s, lg, sg, lr, sr))
        assert abs(lg - lr) <= bound, (s, lg, sg, lr, sr)
    return out


def test_full_run_gpu_vs_oracle_c1():
    _vs_oracle(W.gauss(2), dict(n_live=200, k=20, steps=10), range(1, 7))


def test_full_run_gpu_vs_oracle_c2():
    """C2 (d = 10 MoG, n = 2000, k = 200, p = 10) at full size, 3 seeds."""
    _vs_oracle(W.mog(10), dict(n_live=2000, k=200, steps=10), range(1, 4))


@pytest.mark.parametrize("name", ["C3a", "C3b"])
def test_full_run_gpu_vs_oracle_c3_reduced(name):
    """C3 at reduced n (SURVEY C-9 T4: n = 1000, k = 100; d = 100, p = 3d):
    the oracle's full runs take 0.5-1.5 h of one core, so their results are
    stored by scripts/golden_oracle_fullruns.py (oracle only) in
    tests/golden/oracle_fullrun_<cfg>_s<seed>.json."""
    import glob
    import json
    import os
    runs = {}
    for path in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", f"oracle_fullrun_{name}_s*.json"))):
        g = json.load(open(path))
        runs[g["seed"]] = (g["log_z"], g["log_z_err"])
        cfg = g["cfg"]
    assert runs, "golden oracle runs missing"
    prob, _ = W.workload(name)
    kw = {k: cfg[k] for k in ("n_live", "k", "steps", "max_dead")}
    _vs_oracle(prob, kw, sorted(runs), oracle_runs=runs)


@pytest.mark.parametrize("name", ["logreg", "logreg_split", "gp"])
def test_full_run_gpu_vs_oracle_batch_engines(name):
    """Full runs through the batch engine's tensor-core logistic regression
    (fp16-exact and split data, R-28) and the fused fp64 GP chains, against
    the oracle's full runs with the same seeds (no analytic log Z exists)."""
    probs = {"logreg": (lambda: W.logreg(5, n_data=300, seed=3), dict(n_live=300, k=30, steps=5)),
             "logreg_split": (lambda: W.logreg(8, n_data=200, seed=6, half_exact=False), dict(n_live=300, k=30, steps=8)),
             "gp": (lambda: W.gp_ard(2, 40, seed=3), dict(n_live=200, k=20, steps=4))}
    make, kw = probs[name]
    prob = make()
    from paper_2601_23252_b200 import nss
    g = nss.Sampler(prob, W.config(seed=1, **kw))
    assert g.engine() == "batch"
    g.close()
    _vs_oracle(prob, kw, range(1, 4))


def _funnel_log_z(d, a, sigma_y):
    """P17 (SURVEY C-8): Z = (2a)^-d int_{-a}^{a} N(y; 0, sigma_y^2)
    erf(a / (sqrt 2 e^{y/2}))^(d-1) dy for the funnel under U[-a, a]^d
    (x_n ~ N(0, sd e^{y/2}), R-23), by adaptive quadrature."""
    from scipy import integrate

    def f(y):
        return stats.norm.pdf(y, 0.0, sigma_y) * special.erf(a / (math.sqrt(2.0) * math.exp(y / 2))) ** (d - 1)
    z, _ = integrate.quad(f, -a, a, points=[-10, -5, 0, 5], limit=400, epsabs=0, epsrel=1e-12)
    return math.log(z) - d * math.log(2 * a)


def test_funnel_log_z_quadrature_pin():
    """The funnel truth itself: d = 10, a = 20 gives -36.946."""
    assert abs(_funnel_log_z(10, 20.0, 3.0) - (-36.946)) < 5e-4


def test_full_run_c3b_funnel_analytic():
    """C3b at full size (funnel d = 100 under U[-20, 20]^100, n = 1e4, k = 1e3,
    p = 3d) to termination: |log Z - (-368.985)| <= max(3 sigma, 0.05) per run
    (P17)."""
    prob, cfg = W.workload("C3b")
    truth = _funnel_log_z(prob.d, float(prob.hi[0]), prob.sigma_y)
    assert abs(truth - (-368.985)) < 1e-3
    res = _run_logz(prob, dict(n_live=cfg["n_live"], k=cfg["k"], steps=cfg["steps"],
                               max_dead=cfg["n_live"] + cfg["k"] * 8000), [1, 2])
    for lz, sig, info in res:
        assert info["terminated"]
        assert abs(lz - truth) <= max(3 * sig, 0.05), (lz, sig, truth)


def test_posterior_weights_c1():
    from paper_2601_23252_b200 import nss
    g = nss.Sampler(W.gauss(2), W.config(n_live=200, k=20, steps=10, seed=3))
    g.run()
    x, lw = g.samples()
    assert abs(special.logsumexp(lw)) < 1e-9
    w = np.exp(lw)
    ess = 1 / np.sum(w ** 2)
    m = w @ x
    assert np.all(np.abs(m) < 4 / math.sqrt(ess))
    assert np.all(np.abs(w @ (x - m) ** 2 - 1) < 0.25)


def test_determinism_gpu():
    from paper_2601_23252_b200 import nss
    prob = W.mog(10)
    cfg = W.config(n_live=2000, k=200, steps=10, seed=8)
    a, b = nss.Sampler(prob, cfg), nss.Sampler(prob, cfg)
    a.steps(20)
    b.steps(20)
    da, db = a.dead(), b.dead()
    for key in da:
        assert np.array_equal(da[key], db[key])
    assert np.array_equal(a.evidence_reps(), b.evidence_reps())


def test_determinism_recycled_memory():
    """Device buffers come from a stream-ordered pool that keeps freed blocks
    (nss_init in well under a millisecond): a run on memory recycled from a
    context that left NaNs everywhere equals the same run made first."""
    from paper_2601_23252_b200 import nss
    prob = W.mog(10)
    cfg = W.config(n_live=2000, k=200, steps=10, seed=9)
    a = nss.Sampler(prob, cfg)
    a.steps(20)
    da, ra = a.dead(), a.evidence_reps()
    a.close()
    dirty = nss.Sampler(prob, dict(cfg, seed=123))
    nan_x = np.full((cfg["n_live"], prob.d), np.nan, dtype=np.float32)
    dirty.set_live(nan_x, np.full(cfg["n_live"], np.nan, dtype=np.float32), 1)
    try:
        dirty.step()
    except nss.NssError:
        pass  # NaN energies raise NSS_ERR_NAN; the buffers are dirty either way
    dirty.close()
    b = nss.Sampler(prob, cfg)
    b.steps(20)
    db, rb = b.dead(), b.evidence_reps()
    b.close()
    for key in da:
        assert np.array_equal(da[key], db[key]), key
    assert np.array_equal(ra, rb)


def test_termination_flat_matches_oracle():
    from oracle import nsso
    from paper_2601_23252_b200 import nss
    prob = W.flat(2)
    cfg = W.config(n_live=100, k=10, steps=1, seed=2)
    g = nss.Sampler(prob, cfg)
    o = nsso.Oracle(prob, cfg)
    ig, io = g.run(), o.run()
    assert ig["iteration"] == io["iteration"]
    assert ig["terminated"] == io["terminated"] == 1


def test_errors():
    from paper_2601_23252_b200 import nss
    with pytest.raises(nss.NssError) as ei:
        nss.Sampler(W.gauss(2), W.config(n_live=10, k=10, steps=1))
    assert ei.value.code == 1
    with pytest.raises(nss.NssError) as ei:  # rank outside the world
        nss.Sampler(W.gauss(2), W.config(n_live=10, k=1, steps=1), dist=(2, 2, bytes(128)))
    assert ei.value.code == 1
    g0 = nss.Sampler(W.gauss(2), W.config(n_live=10, k=3, steps=1))
    with pytest.raises(nss.NssError) as ei:  # chain range outside [0, k]
        g0.set_chain_range(1, 4)
    assert ei.value.code == 1
    p = W.gauss(2, half_width=1.0)
    p.c = float("inf")
    with pytest.raises(nss.NssError) as ei:
        nss.Sampler(p, W.config(n_live=10, k=1, steps=1))
    assert ei.value.code == 2
    p = W.gauss(2)
    p.c = float("nan")
    with pytest.raises(nss.NssError) as ei:
        nss.Sampler(p, W.config(n_live=10, k=1, steps=1))
    assert ei.value.code == 3
    g = nss.Sampler(W.gauss(2), W.config(n_live=10, k=5, steps=1, max_dead=14))
    with pytest.raises(nss.NssError) as ei:
        g.step()
    assert ei.value.code == 8
    g2 = nss.Sampler(W.gauss(2), W.config(n_live=10, k=5, steps=1))
    with pytest.raises(nss.NssError) as ei:
        g2.evidence()
    assert ei.value.code == 7
    g2.run()
    with pytest.raises(nss.NssError) as ei:
        g2.step()
    assert ei.value.code == 7


def test_c4_full_size_iteration_subset():
    """C4 at full size (n=2e4, k=1e4, p=100, N=1e4, d=100) through the tensor-core
    batch engine; the oracle replays 6 chains of the same iteration."""
    import numpy as np
    from oracle import nsso
    from paper_2601_23252_b200 import nss
    prob, cfg = W.workload("C4", seed=3)
    gpu = nss.Sampler(prob, cfg)
    assert gpu.engine() == "batch"
    rng = np.random.default_rng(44)  # seeded prior draws, energies by numpy (not the GPU)
    x0 = (prob.mean + prob.sd * rng.standard_normal((cfg["n_live"], prob.d))).astype(np.float32)
    a = x0.astype(np.float64) @ prob.data_x.T
    e32 = np.sum(np.logaddexp(0.0, a) - prob.data_y * a, axis=1).astype(np.float32)
    gpu.set_live(x0, e32, 1)
    ref = nsso.Oracle(prob, cfg, draw_live=False)
    ref.set_live(x0.astype(np.float64), e32.astype(np.float64), 1)
    chains = [0, 1, 2, 777, 2500, 5000, 6001, 7777, 9000, 9998, 9999, 4242]
    ref.set_chain_subset(chains)
    gpu.step()
    ref.step()
    check_subset(gpu, ref, prob, chains, "C4 full-size subset")
    info = gpu.info()
    assert info["null_moves"] == 0 and info["energy_evals"] > 1e6


UPDATE_ALL_CASES = {
    "lane_mog": (lambda: W.mog(4, n_comp=2, seed=4, mean_box=3.0, min_sep=3.0), dict(n_live=150, k=15, steps=4),
                 "lane"),
    "warp_corr": (lambda: W.corr_gauss(12, seed=2), dict(n_live=200, k=20, steps=3), "warp"),
    "batch_logreg": (lambda: W.logreg(5, n_data=300, seed=3), dict(n_live=120, k=12, steps=2), "batch"),
}


@pytest.mark.parametrize("name", sorted(UPDATE_ALL_CASES))
def test_update_all_single_iteration_parity(name):
    """F4: every live slot runs a chain; same bar as the standard iteration."""
    make, kw, engine = UPDATE_ALL_CASES[name]
    prob = make()
    cfg = W.config(seed=11, update_all=1, **kw)
    gpu, ref = inject_pair(prob, cfg, warm_iters=1, engine=engine)
    if gpu.engine() != engine:
        pytest.skip(f"{engine} engine does not apply")
    st = compare_iteration(gpu, ref, prob, f"update-all {name}")
    tg = gpu.trace()
    assert tg["dest_gid"].size == kw["n_live"]
    dg, dr = gpu.dead(), ref.dead()
    assert np.array_equal(dg["gid"], dr["gid"])


RW_CASES = {
    "mog_box": (lambda: W.mog(4, n_comp=2, seed=4, mean_box=3.0, min_sep=3.0), dict(n_live=150, k=15, steps=20)),
    "corr_gauss_prior": (lambda: W.corr_gauss(12, seed=2), dict(n_live=200, k=20, steps=12)),
    "funnel": (lambda: W.funnel(16), dict(n_live=200, k=20, steps=16)),
    "logreg": (lambda: W.logreg(5, n_data=300, seed=3), dict(n_live=120, k=12, steps=10)),
    "update_all": (lambda: W.gauss(3), dict(n_live=100, k=10, steps=6, update_all=1)),
}


@pytest.mark.parametrize("name", sorted(RW_CASES))
def test_rw_single_iteration_parity(name):
    """F1 constrained random walk: same bar as HRSS."""
    make, kw = RW_CASES[name]
    prob = make()
    cfg = W.config(seed=13, mutation=W.MUT_RW, **kw)
    gpu, ref = inject_pair(prob, cfg, warm_iters=1)
    st = compare_iteration(gpu, ref, prob, f"rw {name}")
    c = st["counts_g"]
    assert np.all(c[..., 0] == 0) and np.all(c[..., 1] == 0)
    assert 0 < c[..., 3].mean() < 1  # some proposals accepted, some rejected
    assert gpu.info()["expansions"] == 0


def _full_size_subset(name, chains, seed=3):
    """A BASELINE configuration at full size through the engine bench.py times;
    the oracle replays a subset of the chains of the same iteration.  Live
    points: seeded prior draws (numpy), energies from the oracle (not the GPU)."""
    from oracle import nsso
    from paper_2601_23252_b200 import nss
    prob, cfg = W.workload(name, seed=seed)
    rng = np.random.default_rng(101)
    n, d = cfg["n_live"], prob.d
    if prob.prior_kind == W.PRIOR_BOX:
        x0 = (prob.lo + (prob.hi - prob.lo) * rng.random((n, d))).astype(np.float32)
    else:
        x0 = (prob.mean + prob.sd * rng.standard_normal((n, d))).astype(np.float32)
    ref = nsso.Oracle(prob, cfg, draw_live=False)
    e0 = np.array([ref.energy(q) for q in x0.astype(np.float64)]).astype(np.float32)
    ref.set_live(x0.astype(np.float64), e0.astype(np.float64), 1)
    gpu = nss.Sampler(prob, cfg)
    gpu.set_live(x0, e0, 1)
    ref.set_chain_subset(chains)
    gpu.step()
    ref.step()
    check_subset(gpu, ref, prob, chains, f"{name} full-size subset")
    return gpu


@pytest.mark.parametrize("name", ["C3a", "C3b"])
def test_c3_full_size_iteration_subset(name):
    """C3a / C3b at full size (n=1e4, k=1e3, p=300, d=100): warp engine with
    precomputed directions, chains 0, 1, 499, 998, 999 replayed by the oracle."""
    gpu = _full_size_subset(name, [0, 1, 2, 3, 100, 250, 499, 500, 640, 777, 998, 999])
    assert gpu.engine() == "warp"
