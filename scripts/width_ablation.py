"""Slice-width ablation on the B200: tests the
paper's claim that HRSS costs concentrate near the optimal width (P:357-362,
P:758).  For each width setting, after `warm` untimed iterations,
`iters` iterations are run with per-launch kernel timing; from the per-chain
per-step counts of every iteration (nss_get_trace) it reports

  * evals / HRSS step (physical energy calls) and the theorem count
    (expansions + shrinks) per step: mean, std, max;
  * tail efficiency of the chain-parallel HRSS kernel: mean over chains of the
    iteration's probes per chain / the maximum (the kernel lasts as long as its
    slowest chain when all chains are resident);
  * HRSS kernel ms per iteration and evals/s inside the kernel.

    python scripts/width_ablation.py [C3a|C2|C3b] [warm] [iters]  > out.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3a"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 20
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)

settings = [("optimal c=0.25", dict(width=0.25)), ("optimal c=0.5", dict(width=0.5)),
            ("optimal c=1", dict(width=1.0)), ("optimal c=2", dict(width=2.0)),
            ("optimal c=4", dict(width=4.0)), ("fixed w=1", dict(width_rule=W.W_FIXED, width=1.0)),
            ("euclidean c=1", dict(width=1.0, dir_norm=W.DIR_EUCLIDEAN))]
rows = []
for label, over in settings:
    prob, cfg = W.workload(name, seed=3, **over)
    s = nss.Sampler(prob, cfg, stream=st.cuda_stream)
    s.steps(warm)
    s.sync()
    cap = cfg["max_stepout"]
    theo, probes_chain, nulls = [], [], 0
    i0 = s.info()
    s.set_kernel_timing(True)
    for _ in range(iters):
        s.step()
        c = s.trace()["counts"].astype(np.int64)  # k x p x {nL, nR, nS, acc}
        nl, nr, ns, acc = c[..., 0], c[..., 1], c[..., 2], c[..., 3]
        theo.append((nl + nr + ns).ravel())
        pr = nl + (nl < cap) + nr + (nr < cap) + ns
        probes_chain.append(pr.sum(axis=1))
        nulls += int((acc == 0).sum())
    i1 = s.info()
    ph = s.phase_times()
    w = s.metric()[1]
    s.close()
    theo = np.concatenate(theo)
    eff = [float(p.mean() / max(p.max(), 1)) for p in probes_chain]
    n_steps = iters * cfg["k"] * cfg["steps"]
    hrss_ms = ph["hrss"][0] / max(ph["hrss"][1], 1)
    evals = i1["energy_evals"] - i0["energy_evals"]
    rows.append(dict(config=name, setting=label, width=w, iterations=iters,
                     evals_per_step=evals / n_steps,
                     theorem_per_step_mean=float(theo.mean()), theorem_per_step_std=float(theo.std()),
                     theorem_per_step_max=int(theo.max()), null_moves=nulls,
                     tail_efficiency=float(np.mean(eff)),
                     hrss_ms_per_iter=hrss_ms, evals_per_s_in_kernel=evals / (ph["hrss"][0] / 1e3)))
    print(json.dumps(rows[-1]), flush=True)
