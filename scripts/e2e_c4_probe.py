"""One-off costs of a C4 / C3a run through the public API: nss_init, the first
step (lazy engine setup, graph capture) and the steady steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

torch.cuda.set_device(0)
st = torch.cuda.Stream()
for name in sys.argv[1:] or ["C4"]:
    prob, cfg = W.workload(name)
    for rep in range(2):
        t0 = time.perf_counter()
        s = nss.Sampler(prob, dict(cfg, seed=100 + rep), stream=st.cuda_stream)
        t1 = time.perf_counter()
        s.step(sync=True)
        t2 = time.perf_counter()
        for _ in range(5):
            s.step(sync=True)
        t3 = time.perf_counter()
        s.close()
        print(f"{name}: init {1e3 * (t1 - t0):.1f} ms | first step {1e3 * (t2 - t1):.1f} ms | steady step "
              f"{1e3 * (t3 - t2) / 5:.2f} ms")
