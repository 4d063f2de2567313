"""Measure the fp64 (and tf32) dense GEMM throughput of this B200 with
cuBLAS through torch.matmul (best of 10, CUDA events), for the roofline of
the fp64 kernels ("Not measured: FP64 and TF32")."""
import json
import sys

import torch

torch.cuda.set_device(0)
out = {}
for name, dt, n in (("fp64", torch.float64, 8192), ("tf32", torch.float32, 8192)):
    torch.backends.cuda.matmul.allow_tf32 = name == "tf32"
    a = torch.randn(n, n, dtype=dt, device="cuda")
    b = torch.randn(n, n, dtype=dt, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[f"{name}_tflops"] = 2 * n ** 3 / (best / 1e3) / 1e12
out["how"] = "torch.matmul 8192^3 (cuBLAS), best of 10, CUDA events"
print(json.dumps(out))
