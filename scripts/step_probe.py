"""Per-step host overhead of the C2 step variants (warm): graph only, graph +
sync, graph + info (term probe + sync + info), and the ctypes call alone."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

torch.cuda.set_device(0)
st = torch.cuda.Stream()
prob, cfg = W.workload("C2")
s = nss.Sampler(prob, dict(cfg, seed=5), stream=st.cuda_stream)
for _ in range(20):
    s.step(sync=True)
L = nss.lib()
h = s._h
info = nss.nss_step_info()
N = 150


def t(fn):
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    return 1e6 * (time.perf_counter() - t0) / N


a = t(lambda: L.nss_step(h, None))
s.sync()
b = t(lambda: (L.nss_step(h, None), L.nss_sync(h)))
c = t(lambda: L.nss_step(h, C.byref(info)))
d = t(lambda: s.step(sync=True))
e = t(lambda: L.nss_info(h, C.byref(info)))
print(f"step async {a:.1f} us | step+sync {b:.1f} | step(info) raw {c:.1f} | step(info) python {d:.1f} | "
      f"nss_info {e:.1f}")

# first steps of fresh contexts (graph capture + instantiation happen in step 1)
for rep in range(3):
    s2 = nss.Sampler(prob, dict(cfg, seed=50 + rep), stream=st.cuda_stream)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        s2.step(sync=True)
        ts.append(1e6 * (time.perf_counter() - t0))
    s2.close()
    print("fresh context, first 5 steps (us):", " ".join(f"{x:.0f}" for x in ts))
