"""Helpers shared by the GPU parity tests (test-side only).

Protocol (SURVEY C-9): inject an identical live set into
the CUDA path and the fp64 oracle (positions rounded to fp32, energies computed
by the oracle and rounded to fp32, so both rank identical numbers), run one
iteration on each, then compare
  * deleted gids, destinations, parents, E*: bit-exact;
  * per-(chain, step) counts {n_left, n_right, n_shrink, accepted}: exact, except
    chains whose first differing step follows an oracle decision with relative
    margin < TIE (a fp32-vs-fp64 precision tie), which may be at most 1%;
  * new positions / energies of the untagged chains: within 1e-5 relative.
"""
import numpy as np

TIE = 1e-5
RTOL = 1e-5


def inject_pair(prob, cfg, warm_iters=0, it=None, engine="auto"):
    from oracle import nsso
    from paper_2601_23252_b200 import nss

    warm = nsso.Oracle(prob, cfg)
    for _ in range(warm_iters):
        warm.step()
    x, _ = warm.get_live()
    warm.close()
    ref = nsso.Oracle(prob, cfg)        # fresh: no dead records from the warm-up
    x32 = x.astype(np.float32)
    e32 = np.array([ref.energy(xi.astype(np.float64)) for xi in x32]).astype(np.float32)
    nxt = warm_iters + 1 if it is None else it
    ref.set_live(x32.astype(np.float64), e32.astype(np.float64), nxt)
    gpu = nss.Sampler(prob, cfg)
    gpu.set_engine(engine)
    gpu.set_live(x32, e32, nxt)
    return gpu, ref


def prior_scale(prob):
    if prob.prior_kind == 0:
        return np.asarray(prob.hi) - np.asarray(prob.lo)
    return np.asarray(prob.sd)


def compare_iteration(gpu, ref, prob, max_tie_frac=0.01):
    """Run one iteration on both sides and check the parity bar. Returns stats."""
    xg0, eg0 = gpu.get_live()
    gpu.step()
    ref.step()
    tg, tr = gpu.trace(), ref.trace()
    for key in ("dead_gid", "dest_gid", "parent_gid"):
        assert np.array_equal(tg[key], tr[key]), f"{key} differs"
    assert np.float32(tr["e_star"]) == np.float32(tg["e_star"]), (tg["e_star"], tr["e_star"])
    cg, cr = tg["counts"], tr["counts"]
    k, p = cg.shape[0], cg.shape[1]
    ties, bad = [], []
    same = np.zeros(k, bool)
    for c in range(k):
        diff = np.nonzero(np.any(cg[c] != cr[c], axis=1))[0]
        if diff.size == 0:
            same[c] = True
            continue
        j = diff[0]
        if np.min(tr["min_margin"][c, : j + 1]) < TIE:
            ties.append(c)
        else:
            bad.append((c, j, cg[c, j].tolist(), cr[c, j].tolist(), float(np.min(tr["min_margin"][c, : j + 1]))))
    assert not bad, f"untagged count divergences: {bad[:5]}"
    assert len(ties) <= max(1, max_tie_frac * k), f"too many precision ties: {len(ties)}/{k}"
    xg, eg = gpu.get_live()
    xr, er = ref.get_live()
    scale = prior_scale(prob)
    for c in np.nonzero(same)[0]:
        s = tg["dest_gid"][c]
        dx = np.abs(xg[s].astype(np.float64) - xr[s])
        assert np.all(dx <= RTOL * (np.abs(xr[s]) + scale)), (c, s, dx.max())
        assert abs(float(eg[s]) - er[s]) <= RTOL * max(1.0, abs(er[s])), (c, s, eg[s], er[s])
    # survivors untouched
    dest = set(tg["dest_gid"].tolist())
    keep = np.array([g for g in range(xg.shape[0]) if g not in dest], dtype=np.int64)
    assert np.array_equal(xg[keep], xg0[keep]) and np.array_equal(eg[keep], eg0[keep])
    return dict(ties=len(ties), same=int(same.sum()), k=k, counts_g=cg, counts_r=cr)
