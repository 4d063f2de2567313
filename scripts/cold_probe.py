"""Per-kernel event times of C2 iterations with and without an L2 flush
between iterations (cold-start cost per kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_23252_b200 import nss, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
prob, cfg = W.workload(name)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for do_flush in (True, False):
    s = nss.Sampler(prob, dict(cfg, seed=7), stream=st.cuda_stream)
    s.steps(5)
    s.sync()
    s.set_kernel_timing(True)
    for _ in range(100):
        if do_flush:
            flush.zero_()
        s.step(sync=False)
    s.sync()
    pt = s.phase_times()
    print(("flushed" if do_flush else "warm   "), " ".join(f"{k}={v[0] / max(v[1], 1) * 1e3:.1f}us" for k, v in pt.items()))
    s.close()
