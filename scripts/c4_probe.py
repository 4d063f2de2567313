"""C4 / C3 / C5 throughput probe: iterations and energy evals per second (live)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
prob, cfg = W.workload(name)
t0 = time.time()
s = nss.Sampler(prob, cfg, stream=st.cuda_stream)
torch.cuda.synchronize()
print(f"{name}: init {time.time() - t0:.2f} s, engine {s.engine()}")
s.steps(2)
s.sync()
i0 = s.info()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
s.steps(iters)
b.record(st)
torch.cuda.synchronize()
ms = a.elapsed_time(b)
i1 = s.info()
ev = i1["energy_evals"] - i0["energy_evals"]
pr = i1["probes"] - i0["probes"]
print(f"{name}: {ms / iters:.2f} ms/iter, {ev / (ms / 1e3):.3e} evals/s, {pr / (ms / 1e3):.3e} probes/s, "
      f"evals/iter {ev / iters:.0f}, launches {s.launch_count()}")
s.set_kernel_timing(True)
s.steps(2)
pt = s.phase_times()
print(" ".join(f"{k}={v[0] / max(v[1], 1):.2f}ms" for k, v in pt.items()))
