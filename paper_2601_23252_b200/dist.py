"""Multi-GPU plumbing for NSS: one process per GPU.

NS runs shard the live set: rank q owns the gids of 8/world of the 8 fixed gid
segments (`shard_ranges`), exchanges its top-k candidates and moment sums with
one NCCL all-gather per iteration and reads parent rows other ranks own over
NVLink (csrc/k_shard.cu, csrc/dist.cu).  F3 SMC contexts split the particles'
chains in blocks of ceil(n / world) (`chain_range`) and all-gather the new
rows.  This module only does what happens once per run on the host:
broadcasting rank 0's NCCL unique id over an existing torch.distributed group
and summing per-rank counters.
"""
from __future__ import annotations

from typing import Callable, Dict, Optional, Tuple


def shard_ranges(n: int, world: int):
    """gid range [lo, hi) of every rank of a sharded NS run (include/nss.h)."""
    from .nss import shard_ranges as _sr
    return _sr(n, world)


def chain_range(k: int, rank: int, world: int) -> Tuple[int, int]:
    """Chains [c0, c1) that `rank` runs: blocks of kc = ceil(k / world)."""
    if world < 1 or not 0 <= rank < world or k < 0:
        raise ValueError("bad rank/world")
    kc = (k + world - 1) // world
    c0 = min(k, rank * kc)
    return c0, min(k, c0 + kc)


def broadcast_uid(get_uid: Callable[[], bytes], group=None) -> bytes:
    """Rank 0 calls get_uid(); every rank returns its 128 bytes."""
    import torch.distributed as td
    obj = [get_uid() if td.get_rank(group) == 0 else None]
    td.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id broadcast")
    return bytes(uid)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id from the library (include/nss.h nss_get_unique_id)."""
    import ctypes as C
    from . import nss
    buf = (C.c_uint8 * 128)()
    st = nss.lib().nss_get_unique_id(buf)
    if st != 0:
        raise nss.NssError(st, "nss_get_unique_id")
    return bytes(buf)


def sharded_sampler(problem, cfg: Dict, stream: Optional[int] = None, group=None):
    """Sampler for this process's rank of the default (or given) process
    group: this rank's shard of the live set, an NCCL communicator over all
    ranks (collective: every rank calls it)."""
    import torch.distributed as td
    from . import nss
    rank, world = td.get_rank(group), td.get_world_size(group)
    uid = broadcast_uid(nccl_unique_id, group)
    return nss.Sampler(problem, cfg, stream=stream, dist=(rank, world, uid))


COUNTERS = ("probes", "energy_evals", "expansions", "shrinks", "null_moves")


def job_totals(info: Dict, group=None) -> Dict:
    """Sum the per-rank HRSS counters of nss_info over the group (host values)."""
    import torch
    import torch.distributed as td
    t = torch.tensor([float(info[c]) for c in COUNTERS], dtype=torch.float64)
    if td.is_initialized() and td.get_world_size(group) > 1:
        if td.get_backend(group) == "nccl":
            t = t.cuda()
        td.all_reduce(t, group=group)
    out = dict(info)
    out.update({c: int(v) for c, v in zip(COUNTERS, t.cpu().tolist())})
    return out
