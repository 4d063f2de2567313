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


def _merge_candidates(cands, n, k, seed, it):
    """Host mirror of k_shard_merge (csrc/k_shard.cu): the k largest keys
    (E, gid) of the gathered candidates, destinations ascending, E*, and the
    parents -- survivor j = j + (first index i with D[i] - i > j)."""
    from oracle import nsso
    allc = sorted((c for part in cands for c in part), key=lambda t: (t[0], t[1]), reverse=True)
    sel = allc[:k]
    dead_order = [g for _, g in sel]
    dest = sorted(dead_order)
    e_star = sel[-1][0]
    parents = []
    for s in dest:
        u = nsso.draw_u32(seed, it, s, 2, 0, 0)  # RESAMPLE stream, draw 0
        j = (u * (n - k)) >> 32
        i = next((i for i, dg in enumerate(dest) if dg - i > j), k)
        parents.append(j + i)
    return dead_order, dest, parents, e_star


def _oracle_shard_worker(rank, world, name, kw, iters):
    """The sharded decomposition with the fp64 oracle:
    rank q owns shard_ranges(n, world)[q]; candidates = its local top-min(k,
    n_q) keys, all-gathered and merged; it runs the chains whose destination it
    owns (an ordinal range of D) and the owned new rows are all-gathered.  Must
    reproduce the one-process oracle bit for bit."""
    import torch.distributed as td
    from oracle import nsso
    prob = _PROBLEMS[name]()
    cfg = W.config(seed=21, **kw)
    n, k = cfg["n_live"], cfg["k"]
    a, b = D.shard_ranges(n, world)[rank]
    full = nsso.Oracle(prob, cfg)     # the one-process reference
    mine = nsso.Oracle(prob, cfg)     # this rank (replicated state, owned chains only)
    for it in range(1, iters + 1):
        x, e = mine.get_live()
        keys = sorted(((float(e[g]), g) for g in range(a, b)), reverse=True)[: min(k, b - a)]
        cands = [None] * world
        td.all_gather_object(cands, sorted(keys, key=lambda t: t[1]))
        dead_order, dest, parents, e_star = _merge_candidates(cands, n, k, cfg["seed"], it)
        # segment moment sums of the owned rows, folded in segment order (k_metric.cu)
        shift = x.mean(axis=0)
        segs = []
        for s in range(8):
            lo, hi = (s * n) // 8, ((s + 1) * n) // 8
            if a <= lo and hi <= b:
                y = x[lo:hi] - shift
                segs.append((s, y.sum(axis=0), y.T @ y))
        allsegs = [None] * world
        td.all_gather_object(allsegs, segs)
        segs_all = sorted(sum(allsegs, []), key=lambda t: t[0])
        assert [t[0] for t in segs_all] == list(range(8))
        S1 = sum(t[1] for t in segs_all)
        S2 = sum(t[2] for t in segs_all)
        cov = (S2 - np.outer(S1, S1) / n) / (n - 1)
        if not np.allclose(cov, np.cov(x.T), rtol=1e-10, atol=1e-12):
            return f"iteration {it}: segment moments differ"
        lo_c = next((i for i, g in enumerate(dest) if g >= a), k)
        hi_c = next((i for i, g in enumerate(dest) if g >= b), k)
        mine.set_chain_subset(list(range(lo_c, hi_c)))
        mine.step()
        full.step()
        tr, tf = mine.trace(), full.trace()
        if list(tf["dead_gid"]) != dead_order or list(tf["dest_gid"]) != dest:
            return f"iteration {it}: merged candidates differ from the oracle's select"
        if list(tf["parent_gid"]) != parents or e_star != tf["e_star"]:
            return f"iteration {it}: parents / E* differ"
        x, e = mine.get_live()
        rows = [(int(g), x[g].copy(), float(e[g])) for g in dest[lo_c:hi_c]]
        allrows = [None] * world
        td.all_gather_object(allrows, rows)
        for part in allrows:
            for g, xg, eg in part:
                x[g], e[g] = xg, eg
        mine.set_live(x, e, it + 1)
        xf, ef = full.get_live()
        if not (np.array_equal(x, xf) and np.array_equal(e, ef)):
            return f"iteration {it}: live set differs"
        if not np.array_equal(tr["counts"][lo_c:hi_c], tf["counts"][lo_c:hi_c]):
            return f"iteration {it}: counts differ"
    return "ok"


def test_shard_ranges_partition():
    for n in (2, 7, 200, 777, 2000, 20_000):
        for world in (1, 2, 4, 8):
            rs = D.shard_ranges(n, world)
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[q][1] == rs[q + 1][0] for q in range(world - 1))
            # whole segments: the union of rank q's 8/world segments
            per = 8 // world
            assert rs[1 % world][0] == (per * n) // 8 or world == 1
    with pytest.raises(ValueError):
        D.shard_ranges(100, 3)


_PROBLEMS = {
    "mog": lambda: W.mog(4, n_comp=2, seed=4, mean_box=3.0, min_sep=3.0),
    "corr": lambda: W.corr_gauss(6, seed=2),
    "logreg": lambda: W.logreg(3, n_data=60, seed=3),
}


@pytest.mark.parametrize("name,kw", [("mog", dict(n_live=120, k=13, steps=4)),
                                     ("corr", dict(n_live=90, k=30, steps=3)),
                                     ("logreg", dict(n_live=64, k=5, steps=2))])
def test_sharded_oracle_matches_one_process(name, kw):
    for world in (2, 4):
        out = _run(_oracle_shard_worker, world, name, kw, 3)
        assert all(out[r] == "ok" for r in range(world)), out
