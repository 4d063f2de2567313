"""The tcgen05 logistic-regression energy kernel against the fp64 oracle's
energy (through the C ABI kernel-check hook), on the C4 shape and ragged
edge cases (partial probe tiles, partial data tiles, d < 128), for fp16-exact
data (one X term) and general fp32 data (X = Xhi + Xlo, three MMAs), R-28."""
import numpy as np
import pytest

from paper_2601_23252_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ref_energy(prob, theta):
    a = theta @ prob.data_x.T
    return np.sum(np.logaddexp(0.0, a) - prob.data_y * a, axis=1)


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("d,n_data,P", [(100, 10_000, 1000), (100, 10_000, 1), (5, 300, 130), (33, 1000, 257),
                                        (112, 129, 128), (128, 300, 200)])
def test_lr_energy_batch(d, n_data, P, exact):
    from oracle import nsso
    from paper_2601_23252_b200 import nss
    prob = W.logreg(d, n_data=n_data, seed=7, half_exact=exact)
    rng = np.random.default_rng(d + P)
    theta = rng.standard_normal((P, d)) * 0.7
    e_gpu = nss.lr_energy_batch(prob.data_x, prob.data_y, theta)
    e_ref = _ref_energy(prob, theta)
    assert np.all(np.abs(e_gpu - e_ref) <= 1e-5 * np.maximum(1.0, np.abs(e_ref))), np.max(np.abs(e_gpu - e_ref))
    # the oracle agrees with the numpy reference (so the kernel matches the oracle)
    o = nsso.Oracle(prob, W.config(n_live=8, k=1, steps=1))
    for i in range(min(P, 3)):
        assert abs(o.energy(theta[i]) - e_ref[i]) < 1e-9 * max(1, abs(e_ref[i]))


@pytest.mark.parametrize("bn", ["128", "160", "256"])
@pytest.mark.parametrize("n_data,P", [(10_000, 300), (1000, 129)])
def test_lr_energy_batch_tile_widths(bn, n_data, P, monkeypatch):
    """Every data-tile width of the tcgen05 pass (N = 256 default, 128 and 160
    via NSS_LR_BN, read when the engine is set up) against the fp64 reference,
    including a ragged last data tile (1000 = 3 x 256 + 232)."""
    from paper_2601_23252_b200 import nss
    monkeypatch.setenv("NSS_LR_BN", bn)
    prob = W.logreg(100, n_data=n_data, seed=11)
    theta = np.random.default_rng(P).standard_normal((P, 100)) * 0.7
    e_gpu = nss.lr_energy_batch(prob.data_x, prob.data_y, theta)
    e_ref = _ref_energy(prob, theta)
    assert np.all(np.abs(e_gpu - e_ref) <= 1e-5 * np.maximum(1.0, np.abs(e_ref))), np.max(np.abs(e_gpu - e_ref))


@pytest.mark.parametrize("exact", [True, False])
def test_lr_energy_precision_fp32_level(exact):
    """theta in two fp16 terms (22 significant bits) and X exact or split: the
    energies sit at the fp32 level of the fp64 reference, well inside the
    1e-5 parity bar (prior-scale and posterior-scale theta)."""
    from paper_2601_23252_b200 import nss
    prob = W.logreg(100, n_data=10_000, seed=13, half_exact=exact)
    rng = np.random.default_rng(5)
    theta = np.concatenate([rng.standard_normal((256, 100)), prob.meta["theta_true"] + 0.05 * rng.standard_normal((256, 100))])
    e_gpu = nss.lr_energy_batch(prob.data_x, prob.data_y, theta)
    e_ref = _ref_energy(prob, theta)
    rel = np.abs(e_gpu - e_ref) / np.abs(e_ref)
    assert rel.max() <= 3e-6, rel.max()


def test_lr_energy_rejects_data_outside_fp16_range():
    from paper_2601_23252_b200 import nss
    prob = W.logreg(4, n_data=50, seed=1)
    x = prob.data_x.copy()
    x[3, 2] = 1e5
    with pytest.raises(nss.NssError) as ei:
        nss.lr_energy_batch(x, prob.data_y, np.zeros((2, 4)))
    assert ei.value.code == 9


def test_lr_energy_independent_of_batch():
    """Every per-tile value is added to the row's fp64 accumulator exactly, so a
    probe's energy is the same bits whatever batch it is evaluated in (batch
    sizes change the kernel's tile ranges); the sharded runs rely on it."""
    from paper_2601_23252_b200 import nss
    prob = W.logreg(100, n_data=10_000, seed=21)
    theta = np.random.default_rng(3).standard_normal((3000, 100))
    full = nss.lr_energy_batch(prob.data_x, prob.data_y, theta)
    for lo, hi in ((0, 1), (5, 133), (1000, 1001), (2047, 3000)):
        part = nss.lr_energy_batch(prob.data_x, prob.data_y, theta[lo:hi])
        assert np.array_equal(part, full[lo:hi]), (lo, hi)
