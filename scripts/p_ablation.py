"""F4 p-ablation (appendix "Mutation Chain Length";
SURVEY F4): HRSS steps per replacement p = 1 ... 20 on the C2 workload (d = 10
four-component Gaussian mixture, n = 2000, k = 200), full runs to the
termination rule on one B200.  Per p over `seeds` runs:

  * log Z bias against the analytic value (erf products in the box, P16) in
    units of the runs' replica sigma, and the rms of the per-run z;
  * posterior-moment z-scores (P19): the weighted posterior mean of x against
    the closed form sum_j m_j mu_j (m_j = posterior component masses), and the
    component masses themselves (nearest-mean assignment), each divided by its
    Kish-ESS standard error;
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
# posterior covariance (diagonal per component; truncation negligible): E[x^2] - mean^2
var_true = m_true @ (prob.sigma ** 2 + prob.mu ** 2) - mean_true ** 2

rows = []
for p in (1, 2, 3, 4, 5, 6, 8, 10, 12, 15, 20):
    zs, bias, sigs, evals, iters, secs, zmean, zmass = [], [], [], [], [], [], [], []
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
        ess = 1.0 / np.sum(w ** 2)
        m = w @ x
        zmean.append(float(np.sqrt(np.mean(((m - mean_true) / np.sqrt(var_true / ess)) ** 2))))
        comp = np.argmin(((x[:, None, :] - prob.mu[None]) ** 2).sum(-1), axis=1)
        mj = np.array([w[comp == j].sum() for j in range(4)])
        zmass.append(float(np.max(np.abs(mj - m_true) / np.sqrt(m_true * (1 - m_true) / ess))))
        zs.append((lz - truth) / sig)
        bias.append(lz - truth)
        sigs.append(sig)
        evals.append(info["energy_evals"])
        iters.append(info["iteration"])
    row = dict(p=p, seeds=seeds, log_z_bias_mean=float(np.mean(bias)), log_z_bias_sd=float(np.std(bias, ddof=1)),
               sigma_ns=float(np.mean(sigs)),
               z_rms=float(np.sqrt(np.mean(np.square(zs)))), z_max=float(np.max(np.abs(zs))),
               moment_z_rms_mean=float(np.mean(zmean)), mass_z_max=float(np.max(zmass)),
               evals_per_run=float(np.mean(evals)), iterations=float(np.mean(iters)),
               evals_per_iteration=float(np.mean(evals) / np.mean(iters)), seconds_per_run=float(np.mean(secs)))
    rows.append(row)
    print(json.dumps(row), flush=True)
