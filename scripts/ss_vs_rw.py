"""F1 study on the B200: slice sampling (HRSS) vs the constrained Gaussian
random walk as the NS replacement kernel (Table) on an
ill-conditioned Gaussian (kappa = 100) under a box prior, d = 10, 50, 100.

For HRSS: energy calls per HRSS step (every probe inside the box calls the
energy), mean +- std and max.  For RW: proposals per successful sample (the
gaps between accepted proposals of each chain; the paper's count, every
proposal being a likelihood call there), mean +- std and max, and the energy
calls per success (proposals leaving the box are rejected before the call).
Both: HRSS-kernel ms per iteration, evals/s inside it, tail efficiency.

    python scripts/ss_vs_rw.py [warm] [iters] > out.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 30
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)

for d in (10, 50, 100):
    prob = W.corr_gauss(d, seed=1003, box=10.0)
    for label, over in (("HRSS", dict(mutation=W.MUT_HRSS, steps=d)),
                        ("RW", dict(mutation=W.MUT_RW, steps=5 * d))):
        cfg = W.config(n_live=1000, k=100, seed=2, **over)
        s = nss.Sampler(prob, cfg, stream=st.cuda_stream)
        s.steps(warm)
        s.sync()
        i0 = s.info()
        s.set_kernel_timing(True)
        per_step, gaps, tails = [], [], []
        cap = cfg["max_stepout"]
        for _ in range(iters):
            s.step()
            c = s.trace()["counts"].astype(np.int64)  # k x p x 4
            if label == "HRSS":
                nl, nr, ns = c[..., 0], c[..., 1], c[..., 2]
                pr = nl + (nl < cap) + nr + (nr < cap) + ns
                per_step.append(pr.ravel())
                work = pr.sum(axis=1)
            else:
                ev, acc = c[..., 2], c[..., 3]
                work = ev.sum(axis=1)
                for row_e, row_a in zip(ev, acc):
                    run_e = run_p = 0
                    for e_, a_ in zip(row_e, row_a):
                        run_e += e_
                        run_p += 1
                        if a_:
                            gaps.append((run_p, run_e))
                            run_e = run_p = 0
            tails.append(work.mean() / max(work.max(), 1))
        i1 = s.info()
        ph = s.phase_times()
        s.close()
        if label == "HRSS":
            vals = np.concatenate(per_step)
        else:
            g = np.array(gaps)
            vals, evals_gap = g[:, 0], g[:, 1]
        evals = i1["energy_evals"] - i0["energy_evals"]
        row = dict(d=d, kernel=label, steps=cfg["steps"], metric=("energy calls per HRSS step" if label == "HRSS"
                                                                  else "proposals per successful sample"),
                   mean=float(vals.mean()), std=float(vals.std()), max=int(vals.max()),
                   accept_rate=(None if label == "HRSS" else float(len(gaps) / (iters * 100 * cfg["steps"]))),
                   tail_efficiency=float(np.mean(tails)),
                   energy_calls_per_success=(None if label == "HRSS" else
                                             [float(evals_gap.mean()), float(evals_gap.std())]), hrss_ms_per_iter=ph["hrss"][0] / max(ph["hrss"][1], 1),
                   evals_per_iter=evals / iters, evals_per_s=evals / (ph["hrss"][0] / 1e3))
        print(json.dumps(row), flush=True)
