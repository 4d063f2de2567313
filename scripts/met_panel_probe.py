"""Share of the metric's Cholesky spent in the one-warp panel factorisations
(measurement build NSS_NVCC_EXTRA=-DNSS_MET_PROF: stamp 7 = ns in the panels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3b"
torch.cuda.set_device(0)
prob, cfg = W.workload(name)
s = nss.Sampler(prob, cfg)
acc = []
for i in range(20):
    s.step()
    st = s.debug_stamps().astype(np.int64)
    if i >= 5:
        acc.append((st[15] - st[14], st[7]))
a = np.median(np.array(acc), axis=0)
print(name, "factorise ns", a[0], "of which panels (incl. their barrier)", a[1])
