"""Helpers shared by the GPU parity tests (test-side only).

Protocol (SURVEY C-9): inject an identical live set into
the CUDA path and the fp64 oracle (positions rounded to fp32, energies computed
by the oracle and rounded to fp32, so both rank identical numbers), run one
iteration on each, then compare
  * deleted gids, destinations, parents, E*: bit-exact;
  * per-(chain, step) counts {n_left, n_right, n_shrink, accepted}: exact, except
    chains whose first differing step follows an oracle decision with relative
    margin < TIE (a fp32-vs-fp64 precision tie, SURVEY C-9 guard band); at most
    MAX_TIE_FRAC = 0.1% of the chains of a case may be tagged (C-9: "fail if
    more than 0.1% of chains are tied"), and every tag is logged (TIE_LOG,
    printed by tests/conftest.py at the end of the session);
  * new positions / energies of the untagged chains: within 1e-5 relative.
"""
import numpy as np

TIE = 1e-5
RTOL = 1e-5
MAX_TIE_FRAC = 1e-3
TIE_LOG = []  # (case, chains, tagged ties)


def classify_chains(counts_g, counts_r, margin, case=""):
    """Split chains into count-identical ones and precision ties (C-9 guard
    band); any untagged divergence or more than MAX_TIE_FRAC tags fails.
    Returns the boolean mask of count-identical chains."""
    k = counts_g.shape[0]
    same = np.zeros(k, bool)
    ties, bad = [], []
    for c in range(k):
        diff = np.nonzero(np.any(counts_g[c] != counts_r[c], axis=1))[0]
        if diff.size == 0:
            same[c] = True
            continue
        j = diff[0]
        mm = float(np.min(margin[c, : j + 1]))
        if mm < TIE:
            ties.append(c)
        else:
            bad.append((c, int(j), counts_g[c, j].tolist(), counts_r[c, j].tolist(), mm))
    TIE_LOG.append((case, k, len(ties)))
    assert not bad, f"untagged count divergences: {bad[:5]}"
    assert len(ties) <= MAX_TIE_FRAC * k, f"too many precision ties: {len(ties)}/{k} (bar {MAX_TIE_FRAC:.1%})"
    return same


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


def compare_iteration(gpu, ref, prob, case=""):
    """Run one iteration on both sides and check the parity bar. Returns stats."""
    xg0, eg0 = gpu.get_live()
    gpu.step()
    ref.step()
    tg, tr = gpu.trace(), ref.trace()
    for key in ("dead_gid", "dest_gid", "parent_gid"):
        assert np.array_equal(tg[key], tr[key]), f"{key} differs"
    assert np.float32(tr["e_star"]) == np.float32(tg["e_star"]), (tg["e_star"], tr["e_star"])
    cg, cr = tg["counts"], tr["counts"]
    k = cg.shape[0]
    same = classify_chains(cg, cr, tr["min_margin"], case)
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
    return dict(ties=int(k - same.sum()), same=int(same.sum()), k=k, counts_g=cg, counts_r=cr)


def check_subset(gpu, ref, prob, chains, case=""):
    """After one step on both sides with the oracle replaying only `chains`
    (SURVEY C-9 T3 for the large configurations): indices bit-exact, the
    subset's counts under the guard band, values of the identical chains
    within RTOL.  Returns the number of count-identical chains."""
    tg, tr = gpu.trace(), ref.trace()
    for key in ("dead_gid", "dest_gid", "parent_gid"):
        assert np.array_equal(tg[key], tr[key]), key
    assert np.float32(tr["e_star"]) == np.float32(tg["e_star"]), (tg["e_star"], tr["e_star"])
    ch = np.asarray(chains)
    same = classify_chains(tg["counts"][ch], tr["counts"][ch], tr["min_margin"][ch], case)
    xg, eg = gpu.get_live()
    xr, er = ref.get_live()
    scale = prior_scale(prob)
    for c in ch[same]:
        s = tg["dest_gid"][c]
        assert np.all(np.abs(xg[s].astype(np.float64) - xr[s]) <= RTOL * (np.abs(xr[s]) + scale)), (case, c)
        assert abs(float(eg[s]) - er[s]) <= RTOL * max(1.0, abs(er[s])), (case, c, eg[s], er[s])
    return int(same.sum())
