"""C3a at full size (d = 100, kappa = 100, n = 1e4, k = 1e3, p = 3d) run to
termination on the GPU; the weighted posterior mean and variances against the
closed form of a Gaussian likelihood under a Gaussian prior (north_star: no
measurable posterior-moment bias).  z = (mean - truth) / sqrt(var_post / ESS)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

prob, cfg = W.workload("C3a")
Sl_inv = np.asarray(prob.prec, dtype=np.float64)
S0_inv = np.diag(1.0 / np.asarray(prob.sd, dtype=np.float64) ** 2)
post_cov = np.linalg.inv(Sl_inv + S0_inv)
post_mean = post_cov @ (Sl_inv @ np.asarray(prob.mu) + S0_inv @ np.asarray(prob.mean))
post_sd = np.sqrt(np.diag(post_cov))
print("| seed | ESS (Kish) | max abs z of the 100 means | rms z | max rel. error of the 100 variances |")
print("|---|---|---|---|---|")
for seed in (1, 2, 3):
    g = nss.Sampler(prob, dict(cfg, seed=seed, max_dead=cfg["n_live"] + cfg["k"] * 8000))
    g.run()
    x, lw = g.samples()
    g.close()
    w = np.exp(lw - lw.max())
    w /= w.sum()
    ess = 1.0 / np.sum(w ** 2)
    m = w @ x
    v = w @ (x - m) ** 2
    z = (m - post_mean) / (post_sd / np.sqrt(ess))
    rel_v = np.abs(v / post_sd ** 2 - 1.0)
    print(f"| {seed} | {ess:.0f} | {np.max(np.abs(z)):.2f} | {np.sqrt(np.mean(z ** 2)):.2f} | {np.max(rel_v):.3f} |",
          flush=True)
