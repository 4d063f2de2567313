import os, sys
sys.path.insert(0, os.getcwd())
from paper_2601_23252_b200 import nss, workloads as W
prob, cfg = W.workload("C3a")
for k in (100, 1000):
    c = dict(cfg, n_live=10 * k, k=k)
    s = nss.Sampler(prob, c)
    s.set_kernel_timing(True)
    try:
        s.step()
        print("k", k, "ok", s.info()["iteration"])
    except Exception as e:
        print("k", k, "error", e)
    s.close()
