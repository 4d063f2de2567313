"""Multi-process host logic of the multi-GPU path on CPU
with gloo, world size 2: the chain partition, the NCCL-id broadcast, counter
totals, and the decomposition itself -- two ranks of the fp64 oracle, each
running only its chain block and exchanging new rows by all-gather, reproduce
the one-process oracle bit for bit over several iterations."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2601_23252_b200 import dist as D
from paper_2601_23252_b200 import workloads as W


def test_chain_range_partition():
    for k in (1, 2, 7, 200, 1000, 10_000):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                c0, c1 = D.chain_range(k, r, world)
                assert 0 <= c0 <= c1 <= k
                assert c1 - c0 <= -(-k // world)
                seen.extend(range(c0, c1))
            assert seen == list(range(k))
    with pytest.raises(ValueError):
        D.chain_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q, args)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res = q.get(timeout=300)
        out[r] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, res in out.items():
        if isinstance(res, BaseException):
            raise res
    return out


def _entry(fn, rank, world, port, q, args):
    import torch.distributed as td
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world, *args)))
    except BaseException as e:  # report, do not hang the other rank
        q.put((rank, e))
    finally:
        td.destroy_process_group()


def _uid_worker(rank, world):
    return D.broadcast_uid(lambda: bytes(range(128)) if rank == 0 else None)


def test_uid_broadcast_gloo():
    out = _run(_uid_worker, 2)
    assert out[0] == out[1] == bytes(range(128))


def _totals_worker(rank, world):
    info = {c: (rank + 1) * 10 for c in D.COUNTERS}
    info["iteration"] = 5
    return D.job_totals(info)


def test_job_totals_gloo():
    out = _run(_totals_worker, 2)
    for r in (0, 1):
        assert all(out[r][c] == 30 for c in D.COUNTERS)
        assert out[r]["iteration"] == 5


def _oracle_shard_worker(rank, world, name, kw, iters):
    import torch.distributed as td
    from oracle import nsso
    prob = _PROBLEMS[name]()
    cfg = W.config(seed=21, **kw)
    k = cfg["k"]
    full = nsso.Oracle(prob, cfg)     # the one-process reference
    mine = nsso.Oracle(prob, cfg)     # this rank: only its chain block
    c0, c1 = D.chain_range(k, rank, world)
    for it in range(1, iters + 1):
        full.step()
        mine.set_chain_subset(list(range(c0, c1)))
        mine.step()
        tr = mine.trace()
        x, e = mine.get_live()
        dest = tr["dest_gid"]
        rows = [(int(dest[c]), x[dest[c]].copy(), float(e[dest[c]])) for c in range(c0, c1)]
        allrows = [None] * world
        td.all_gather_object(allrows, rows)
        for part in allrows:
            for g, xg, eg in part:
                x[g], e[g] = xg, eg
        mine.set_live(x, e, it + 1)
        xf, ef = full.get_live()
        tf = full.trace()
        for key in ("dead_gid", "dest_gid", "parent_gid"):
            if not np.array_equal(tr[key], tf[key]):
                return f"iteration {it}: {key} differs"
        if not (np.array_equal(x, xf) and np.array_equal(e, ef)):
            return f"iteration {it}: live set differs"
        if not np.array_equal(tr["counts"][c0:c1], tf["counts"][c0:c1]):
            return f"iteration {it}: counts differ"
    return "ok"


_PROBLEMS = {
    "mog": lambda: W.mog(4, n_comp=2, seed=4, mean_box=3.0, min_sep=3.0),
    "corr": lambda: W.corr_gauss(6, seed=2),
    "logreg": lambda: W.logreg(3, n_data=60, seed=3),
}


@pytest.mark.parametrize("name,kw", [("mog", dict(n_live=120, k=13, steps=4)),
                                     ("corr", dict(n_live=90, k=30, steps=3)),
                                     ("logreg", dict(n_live=64, k=5, steps=2))])
def test_sharded_oracle_matches_one_process(name, kw):
    out = _run(_oracle_shard_worker, 2, name, kw, 3)
    assert out[0] == "ok" and out[1] == "ok", out
