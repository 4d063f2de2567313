"""C5 (GP, d = 8) full runs at p = d and p = 3d (no analytic log Z): under-mixing at p = d
would show as a log Z gap between the two settings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

prob, cfg = W.workload("C5")
print("| p | seed | log Z | sigma_NS | iterations | energy evals | wall s |")
print("|---|---|---|---|---|---|---|")
for steps in (8, 24):
    for seed in (1, 2):
        c = dict(cfg, seed=seed, steps=steps, max_dead=cfg["n_live"] + cfg["k"] * 3000)
        g = nss.Sampler(prob, c)
        t0 = time.perf_counter()
        info = g.run()
        lz, sig = g.evidence()
        dt = time.perf_counter() - t0
        g.close()
        print(f"| {steps} | {seed} | {lz:.3f} | {sig:.3f} | {info['iteration']} | {info['energy_evals']} | {dt:.1f} |",
              flush=True)
