"""The fp64 batched-Cholesky GP marginal-likelihood kernel (k_gp.cu) against
the fp64 oracle energy and an independent numpy/LAPACK evaluation, then the
GP workload (C5 shape) through the batch engine against the oracle."""
import numpy as np
import pytest

from paper_2601_23252_b200 import workloads as W
from tests.parity_util import check_subset, compare_iteration, inject_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _np_energy(prob, phi):
    """E(phi) = 1/2 y^T K^-1 y + 1/2 log|K| + N/2 log 2 pi by LAPACK (dpotrf,
    dtrsv), rows evaluated on a thread pool."""
    from concurrent.futures import ThreadPoolExecutor
    import os
    from scipy import linalg
    D = prob.d_in
    X, y = prob.data_x, prob.data_y
    d2 = [(X[:, None, j] - X[None, :, j]) ** 2 for j in range(D)]

    def one(ph):
        s = np.zeros_like(d2[0])
        for j in range(D):
            s += d2[j] * np.exp(-2.0 * ph[j])
        K = np.exp(2 * ph[D]) * np.exp(-0.5 * s)
        K[np.diag_indices(len(y))] += np.exp(2 * ph[D + 1]) + prob.jitter
        G = linalg.cholesky(K, lower=True)
        al = linalg.solve_triangular(G, y, lower=True)
        return 0.5 * al @ al + np.sum(np.log(np.diag(G))) + 0.5 * len(y) * np.log(2 * np.pi)

    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        return np.array(list(ex.map(one, list(phi))))


@pytest.mark.parametrize("d_in,n_data,P", [(6, 1024, 6), (2, 40, 300), (3, 77, 149), (6, 33, 1), (1, 5, 3)])
def test_gp_energy_batch(d_in, n_data, P):
    from oracle import nsso
    from paper_2601_23252_b200 import nss
    prob = W.gp_ard(d_in, n_data, seed=7 + n_data)
    rng = np.random.default_rng(n_data + P)
    phi = rng.standard_normal((P, d_in + 2)).astype(np.float32).astype(np.float64)
    e_gpu = nss.gp_energy_batch(prob.data_x, prob.data_y, prob.jitter, phi)
    e_np = _np_energy(prob, phi[: min(P, 40)])
    assert np.allclose(e_gpu[: len(e_np)], e_np, rtol=1e-9, atol=1e-9)
    o = nsso.Oracle(prob, W.config(n_live=8, k=1, steps=1))
    for i in range(min(P, 2)):
        eo = o.energy(phi[i])
        assert abs(e_gpu[i] - eo) <= 1e-9 * max(1.0, abs(eo)), (e_gpu[i], eo)
    o.close()


def test_gp_energy_not_positive_definite():
    """sigma_n -> 0 with coincident inputs: K is singular, E = +inf (as in the oracle)."""
    from paper_2601_23252_b200 import nss
    X = np.zeros((8, 2))
    y = np.arange(8.0)
    phi = np.array([[0.0, 0.0, 0.0, -40.0]])
    e = nss.gp_energy_batch(X, y, 0.0, phi)
    assert np.isinf(e[0]) and e[0] > 0


GP_CASES = {
    "gp_d4": (lambda: W.gp_ard(2, 40, seed=3), dict(n_live=64, k=16, steps=3), 1),
    "gp_ragged": (lambda: W.gp_ard(3, 77, seed=4), dict(n_live=100, k=33, steps=2), 1),
    "gp_k_half": (lambda: W.gp_ard(6, 64, seed=5), dict(n_live=128, k=64, steps=8), 0),
}


def _gp_mode(monkeypatch, mode):
    """GP chains run fused (one CTA per chain, default) or round-synchronous
    (NSS_GP_ROUNDS, read by nss_init)."""
    if mode == "rounds":
        monkeypatch.setenv("NSS_GP_ROUNDS", "1")
    else:
        monkeypatch.delenv("NSS_GP_ROUNDS", raising=False)


@pytest.mark.parametrize("mode", ["fused", "rounds"])
@pytest.mark.parametrize("name", sorted(GP_CASES))
def test_gp_single_iteration_parity(name, mode, monkeypatch):
    _gp_mode(monkeypatch, mode)
    make, kw, warm = GP_CASES[name]
    prob = make()
    cfg = W.config(seed=11, **kw)
    gpu, ref = inject_pair(prob, cfg, warm_iters=warm, engine="batch")
    assert gpu.engine() == "batch"
    compare_iteration(gpu, ref, prob, f"gp {name} {mode}")
    dg, dr = gpu.dead(), ref.dead()
    assert np.array_equal(dg["gid"], dr["gid"])
    assert np.array_equal(dg["e"].astype(np.float64), dr["e"])


def test_gp_init_parity():
    """Batched prior draws (R-20) equal the oracle's init draws and energies."""
    from oracle import nsso
    from paper_2601_23252_b200 import nss
    prob = W.gp_ard(2, 30, seed=9)
    cfg = W.config(seed=5, n_live=96, k=8, steps=2)
    gpu = nss.Sampler(prob, cfg)
    ref = nsso.Oracle(prob, cfg)
    xg, eg = gpu.get_live()
    xr, er = ref.get_live()
    assert np.allclose(xg, xr, rtol=1e-6, atol=1e-6)
    assert np.allclose(eg, er, rtol=1e-5)
    ig, ir = gpu.info(), ref.info()
    assert ig["init_evals"] == ir["init_evals"] == 96


def test_c5_full_size_iteration_subset():
    """C5 at full size (n=4096, k=2048, p=8, N=1024, d=8) through the batch
    engine; the oracle replays 3 chains of the same iteration.  Live points
    are seeded prior draws, their energies come from LAPACK (not the GPU)."""
    from oracle import nsso
    from paper_2601_23252_b200 import nss
    prob, cfg = W.workload("C5", seed=3)
    rng = np.random.default_rng(55)
    x0 = rng.standard_normal((cfg["n_live"], prob.d)).astype(np.float32)
    e0 = _np_energy(prob, x0.astype(np.float64)).astype(np.float32)
    gpu = nss.Sampler(prob, cfg)
    assert gpu.engine() == "batch"
    gpu.set_live(x0, e0, 1)
    ref = nsso.Oracle(prob, cfg, draw_live=False)
    ref.set_live(x0.astype(np.float64), e0.astype(np.float64), 1)
    chains = [0, 1, 511, 1024, 1500, 2047]
    ref.set_chain_subset(chains)
    gpu.step()
    ref.step()
    check_subset(gpu, ref, prob, chains, "C5 full-size subset")


@pytest.mark.parametrize("d_in,n_data,n_live,k,steps", [(6, 64, 128, 64, 8), (2, 40, 1024, 600, 3)])
def test_gp_fused_equals_rounds(monkeypatch, d_in, n_data, n_live, k, steps):
    """The fused chain kernel and the round-synchronous engine run the same
    state machine on the same energies: two iterations from one injected
    state give bit-identical traces, live sets and dead stores.  The second
    case has more chains (600) than the fused kernel has CTAs (296), so CTAs
    take several chains from the queue."""
    from paper_2601_23252_b200 import nss
    prob = W.gp_ard(d_in, n_data, seed=5)
    cfg = W.config(seed=11, n_live=n_live, k=k, steps=steps)
    rng = np.random.default_rng(7)
    x0 = rng.standard_normal((cfg["n_live"], prob.d)).astype(np.float32)
    e0 = _np_energy(prob, x0.astype(np.float64)).astype(np.float32)
    out = {}
    for mode in ("fused", "rounds"):
        _gp_mode(monkeypatch, mode)
        g = nss.Sampler(prob, cfg)
        g.set_live(x0, e0, 1)
        g.step()
        g.step()
        out[mode] = (g.trace(), g.get_live(), g.dead())
        g.close()
    (tf, (xf, ef), df), (tr, (xr, er), dr) = out["fused"], out["rounds"]
    for key in ("dead_gid", "dest_gid", "parent_gid", "counts"):
        assert np.array_equal(tf[key], tr[key]), key
    assert np.array_equal(xf, xr) and np.array_equal(ef, er)
    assert np.array_equal(df["gid"], dr["gid"]) and np.array_equal(df["e"], dr["e"])
