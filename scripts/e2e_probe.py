"""Where the end-to-end time of C2 goes: init, per-step step(info), evidence."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

torch.cuda.set_device(0)
st = torch.cuda.Stream()
prob, cfg = W.workload("C2")
for rep in range(3):
    t0 = time.perf_counter()
    s = nss.Sampler(prob, dict(cfg, seed=100 + rep), stream=st.cuda_stream)
    t1 = time.perf_counter()
    for _ in range(200):
        s.step(sync=True)
    t2 = time.perf_counter()
    for _ in range(200):
        s.step(sync=False)
    s.sync()
    t3 = time.perf_counter()
    s.evidence()
    t4 = time.perf_counter()
    s.close()
    print(f"init {1e3 * (t1 - t0):.2f} ms | step(info) {1e6 * (t2 - t1) / 200:.1f} us | step(no sync) "
          f"{1e6 * (t3 - t2) / 200:.1f} us | evidence {1e3 * (t4 - t3):.2f} ms")
