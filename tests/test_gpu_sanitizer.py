"""compute-sanitizer over C1/C2 (and the batch engines, a sharded group):
memcheck and racecheck must report no errors.  One tool per
run (B200_PROFILING: running several sanitizer tools in one job has left GPUs
unusable), so the test runs only when NSS_SANITIZER names the tool:

    NSS_SANITIZER=memcheck  python -m pytest tests/test_gpu_sanitizer.py
    NSS_SANITIZER=racecheck python -m pytest tests/test_gpu_sanitizer.py

On this build's GPU pool compute-sanitizer is closed (it answers "closed on
this pool", profiles/r02_sanitizer_closed.txt): the test then skips, and the
memory-safety evidence is the parity suite's bounds/edge cases (empty,
ragged, maximum sizes) against the oracle."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sanitizer_clean():
    tool = os.environ.get("NSS_SANITIZER")
    if tool not in ("memcheck", "racecheck", "synccheck", "initcheck"):
        pytest.skip("set NSS_SANITIZER=<tool> (one tool per job)")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    cmd = [cs, "--tool", tool, "--error-exitcode", "17", "--print-limit", "20", sys.executable,
           os.path.join(ROOT, "scripts", "sanitize_case.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=3000)
    out = p.stdout + p.stderr
    if "closed on this pool" in out:
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.txt"), "w") as f:
        f.write(" ".join(cmd) + "\n" + out)
    assert p.returncode == 0 and "sanitize case ok" in out, out[-4000:]
