"""Time the batched GP energy kernel alone on the C5 data (N=1024, d_in=6):
P probe rows through nss_gp_energy_batch (includes setup/copies; the kernel
time is read from ncu or the printed rate for large P)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 296
prob = W.gp_ard(6, 1024)
phi = np.random.default_rng(1).standard_normal((P, 8))
nss.gp_energy_batch(prob.data_x, prob.data_y, prob.jitter, phi[:2])
t = time.time()
e = nss.gp_energy_batch(prob.data_x, prob.data_y, prob.jitter, phi)
dt = time.time() - t
print(f"GP N=1024: {P} energies in {dt * 1e3:.1f} ms -> {P / dt:.0f} evals/s; "
      f"{dt * 148 / P * 1e3:.2f} ms per matrix per SM; finite {np.isfinite(e).mean():.3f}")
