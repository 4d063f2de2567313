"""Phase latencies inside the select and metric kernels (device %globaltimer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
torch.cuda.set_device(0)
prob, cfg = W.workload(name)
s = nss.Sampler(prob, cfg)
acc = []
for i in range(30):
    s.step()
    st = s.debug_stamps().astype(np.int64)
    if i >= 5:
        acc.append(st)
st = np.median(np.array(acc), axis=0)
sel = np.diff(st[0:7])
met = np.diff(st[8:14])
print(name, "select phases (ns): load", sel[0], "minmax", sel[1], "radix", sel[2], "compact", sel[3], "sort", sel[4],
      "outputs", sel[5], " total", st[6] - st[0])
print(name, "metric phases (ns): load", met[0], "compute+ticket", met[1], "psum", met[2], "chol", met[3], "tail", met[4],
      " total", st[13] - st[8], " select->metric start", st[8] - st[6])
print(name, "metric chol split (ns): normalise", st[14] - st[11], "factorise", st[15] - st[14], "copies", st[12] - st[15])
