"""F4 p-ablation (appendix "Mutation Chain Length";
SURVEY F4): HRSS steps per replacement p = 1 ... 20 on the C2 workload (d = 10
four-component Gaussian mixture, n = 2000, k = 200), full runs to the
termination rule on one B200.  Per p over `seeds` runs:

  * log Z bias against the analytic value (erf products in the box, P16) in
    units of the runs' replica sigma, and the rms of the per-run z;
  * posterior-moment bias (P19): the weighted posterior mean of x against the
    closed form sum_j m_j mu_j (m_j = posterior component masses) and the
    component masses themselves (nearest-mean assignment); z = (mean over the
    seeds - truth) / (seed-to-seed sd / sqrt(seeds)) -- the NS estimate of a
    mode's mass fluctuates with the live points' split between modes, which
    the Kish ESS of one run does not see, so the spread is taken over runs;
  * energy evaluations per iteration and per run, iterations, wall seconds.

The paper's metric is MMD to reference samples (out of scope here, SURVEY
F4): |dlogZ| and the moment z-scores stand in for it.

    python scripts/p_ablation.py [seeds] > profiles/r02_p_ablation.json
"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from scipy import stats  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 6
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)

prob = W.mog(10)
mass = np.array([prob.w[j] * np.prod(stats.norm(prob.mu[j], prob.sigma[j]).cdf(prob.hi) -
                                      stats.norm(prob.mu[j], prob.sigma[j]).cdf(prob.lo)) for j in range(4)])
truth = math.log(mass.sum()) - float(np.sum(np.log(prob.hi - prob.lo)))
m_true = mass / mass.sum()
mean_true = m_true @ prob.mu

rows = []
for p in (1, 2, 3, 4, 5, 6, 8, 10, 12, 15, 20):
    zs, bias, sigs, evals, iters, secs, means, masses = [], [], [], [], [], [], [], []
    for s in range(1, seeds + 1):
        cfg = W.config(n_live=2000, k=200, steps=p, seed=s)
        t0 = time.perf_counter()
        g = nss.Sampler(prob, cfg, stream=st.cuda_stream)
        info = g.run()
        lz, sig = g.evidence()
        secs.append(time.perf_counter() - t0)
        x, lw = g.samples()
        g.close()
        w = np.exp(lw - lw.max())
        w /= w.sum()
        means.append(w @ x)
        comp = np.argmin(((x[:, None, :] - prob.mu[None]) ** 2).sum(-1), axis=1)
        masses.append(np.array([w[comp == j].sum() for j in range(4)]))
        zs.append((lz - truth) / sig)
        bias.append(lz - truth)
        sigs.append(sig)
        evals.append(info["energy_evals"])
        iters.append(info["iteration"])
    means, masses = np.array(means), np.array(masses)
    zmean = (means.mean(0) - mean_true) / (means.std(0, ddof=1) / math.sqrt(seeds))
    zmass = (masses.mean(0) - m_true) / (masses.std(0, ddof=1) / math.sqrt(seeds))
    row = dict(p=p, seeds=seeds, log_z_bias_mean=float(np.mean(bias)), log_z_bias_sd=float(np.std(bias, ddof=1)),
               sigma_ns=float(np.mean(sigs)),
               z_rms=float(np.sqrt(np.mean(np.square(zs)))), z_max=float(np.max(np.abs(zs))),
               mean_z_rms=float(np.sqrt(np.mean(zmean ** 2))), mass_z_max=float(np.max(np.abs(zmass))),
               mass_sd_between_runs=float(masses.std(0, ddof=1).mean()),
               evals_per_run=float(np.mean(evals)), iterations=float(np.mean(iters)),
               evals_per_iteration=float(np.mean(evals) / np.mean(iters)), seconds_per_run=float(np.mean(secs)))
    rows.append(row)
    print(json.dumps(row), flush=True)
