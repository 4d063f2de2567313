"""Live per-phase kernel times (CUDA events inside the library) for a config.

    python scripts/phase_probe.py [C2] [iters]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
prob, cfg = W.workload(name)
for overlap in (True, False):
    for engine in ("auto", "warp"):
        s = nss.Sampler(prob, cfg, stream=st.cuda_stream)
        s.set_overlap(overlap)
        s.set_engine(engine)
        s.steps(3)
        s.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        s.steps(iters)
        b.record(st)
        torch.cuda.synchronize()
        tot = a.elapsed_time(b) / iters
        s.set_kernel_timing(True)
        s.steps(iters)
        pt = s.phase_times()
        s.set_kernel_timing(False)
        info = s.info()
        print(f"{name} overlap={overlap} engine={s.engine()}: step {1e3 * tot:.1f} us (untimed launches) | " +
              " ".join(f"{k}={1e3 * v[0] / max(v[1], 1):.1f}us" for k, v in pt.items()) +
              f" | iter={info['iteration']}")
        s.close()
