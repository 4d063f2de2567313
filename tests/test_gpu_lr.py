"""The tcgen05 logistic-regression energy kernel against the fp64 oracle's
energy (through the C ABI kernel-check hook), on the C4 shape and ragged
edge cases (partial probe tiles, partial data tiles, d < 112)."""
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


@pytest.mark.parametrize("d,n_data,P", [(100, 10_000, 1000), (100, 10_000, 1), (5, 300, 130), (33, 1000, 257),
                                        (112, 129, 128)])
def test_lr_energy_batch(d, n_data, P):
    from oracle import nsso
    from paper_2601_23252_b200 import nss
    prob = W.logreg(d, n_data=n_data, seed=7)
    rng = np.random.default_rng(d + P)
    theta = rng.standard_normal((P, d)) * 0.7
    e_gpu = nss.lr_energy_batch(prob.data_x, prob.data_y, theta)
    e_ref = _ref_energy(prob, theta)
    assert np.all(np.abs(e_gpu - e_ref) <= 1e-5 * np.maximum(1.0, np.abs(e_ref))), np.max(np.abs(e_gpu - e_ref))
    # the oracle agrees with the numpy reference (so the kernel matches the oracle)
    o = nsso.Oracle(prob, W.config(n_live=8, k=1, steps=1))
    for i in range(min(P, 3)):
        assert abs(o.energy(theta[i]) - e_ref[i]) < 1e-9 * max(1, abs(e_ref[i]))


@pytest.mark.parametrize("bn", ["128", "256"])
@pytest.mark.parametrize("n_data,P", [(10_000, 300), (1000, 129)])
def test_lr_energy_batch_tile_widths(bn, n_data, P, monkeypatch):
    """Both data-tile widths of the tcgen05 pass (N = 256 default, 128 via
    NSS_LR_BN, read when the engine is set up) against the fp64 reference,
    including a ragged last data tile (1000 = 3 x 256 + 232)."""
    from paper_2601_23252_b200 import nss
    monkeypatch.setenv("NSS_LR_BN", bn)
    prob = W.logreg(100, n_data=n_data, seed=11)
    theta = np.random.default_rng(P).standard_normal((P, 100)) * 0.7
    e_gpu = nss.lr_energy_batch(prob.data_x, prob.data_y, theta)
    e_ref = _ref_energy(prob, theta)
    assert np.all(np.abs(e_gpu - e_ref) <= 1e-5 * np.maximum(1.0, np.abs(e_ref))), np.max(np.abs(e_gpu - e_ref))


def test_lr_energy_rejects_non_bf16_data():
    from paper_2601_23252_b200 import nss
    prob = W.logreg(4, n_data=50, seed=1)
    x = prob.data_x + 1e-3
    with pytest.raises(nss.NssError) as ei:
        nss.lr_energy_batch(x, prob.data_y, np.zeros((2, 4)))
    assert ei.value.code == 9
