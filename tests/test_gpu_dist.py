"""The multi-GPU path on one B200: (1) a world-1 NCCL
communicator runs the pack / all-gather / scatter exchange every iteration
and must leave the run bit-identical to a plain one-GPU run; (2) two contexts
restricted to the two chain blocks of a world-2 run (no communicator, run one
after the other, the host doing the exchange) reproduce the full run bit for
bit on every engine."""
import numpy as np
import pytest

from paper_2601_23252_b200 import dist as D
from paper_2601_23252_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CASES = {
    "lane_mog10": (lambda: W.mog(10), dict(n_live=2000, k=200, steps=10), "auto"),
    "warp_corr": (lambda: W.corr_gauss(40, seed=5), dict(n_live=600, k=61, steps=4), "warp"),
    "batch_logreg": (lambda: W.logreg(5, n_data=300, seed=3), dict(n_live=300, k=31, steps=3), "batch"),
    "batch_gp": (lambda: W.gp_ard(2, 40, seed=3), dict(n_live=64, k=17, steps=2), "batch"),
}


def _state(s):
    x, e = s.get_live()
    return x.copy(), e.copy()


@pytest.mark.parametrize("name", sorted(CASES))
def test_world1_nccl_path_is_identity(name):
    from paper_2601_23252_b200 import nss
    make, kw, engine = CASES[name]
    prob, cfg = make(), W.config(seed=5, **kw)
    a = nss.Sampler(prob, cfg)
    b = nss.Sampler(prob, cfg, dist=(0, 1, D.nccl_unique_id()))
    for s in (a, b):
        s.set_engine(engine)
        s.steps(3)
        s.sync()
    xa, ea = _state(a)
    xb, eb = _state(b)
    assert np.array_equal(xa, xb) and np.array_equal(ea, eb)
    assert np.array_equal(a.trace()["counts"], b.trace()["counts"])
    assert a.info()["energy_evals"] == b.info()["energy_evals"]


@pytest.mark.parametrize("name", sorted(CASES))
def test_two_chain_blocks_reproduce_full_iteration(name):
    from paper_2601_23252_b200 import nss
    make, kw, engine = CASES[name]
    prob, cfg = make(), W.config(seed=9, **kw)
    full = nss.Sampler(prob, cfg)
    ranks = [nss.Sampler(prob, cfg) for _ in range(2)]
    for r, s in enumerate(ranks):
        s.set_chain_range(*D.chain_range(cfg["k"], r, 2))
    for s in [full, *ranks]:
        s.set_engine(engine)
    evals = 0
    for it in range(1, 4):
        full.step()
        parts = []
        for r, s in enumerate(ranks):
            s.step()
            x, e = _state(s)
            dest = s.trace()["dest_gid"]
            c0, c1 = D.chain_range(cfg["k"], r, 2)
            parts.append([(int(dest[c]), x[dest[c]], e[dest[c]]) for c in range(c0, c1)])
        # host all-gather: both ranks apply every rank's rows
        for s in ranks:
            x, e = _state(s)
            for part in parts:
                for g, xg, eg in part:
                    x[g], e[g] = xg, eg
            s.set_live(x, e, it + 1)
        xf, ef = _state(full)
        for s in ranks:
            x, e = _state(s)
            assert np.array_equal(x, xf) and np.array_equal(e, ef), f"iteration {it}"
    evals = sum(s.info()["energy_evals"] for s in ranks)
    assert evals == full.info()["energy_evals"]


def test_sharded_sampler_through_torch_distributed_world1():
    """The torch.distributed plumbing of dist.py on the GPU box: an NCCL process
    group of one rank, rank 0's NCCL id broadcast, a sharded sampler whose run
    equals the plain one."""
    import socket

    import torch
    import torch.distributed as td
    from paper_2601_23252_b200 import nss
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    td.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                          device_id=torch.device("cuda", 0))
    try:
        prob, cfg = W.gauss(3), W.config(n_live=300, k=30, steps=4, seed=8)
        a = D.sharded_sampler(prob, cfg)
        b = nss.Sampler(prob, cfg)
        for s in (a, b):
            s.steps(5)
        xa, ea = a.get_live()
        xb, eb = b.get_live()
        assert np.array_equal(xa, xb) and np.array_equal(ea, eb)
        tot = D.job_totals(a.info())
        assert tot["energy_evals"] == b.info()["energy_evals"]
    finally:
        td.destroy_process_group()
