"""The opt-in engine variants (DESIGN 7.3, 7.6), each read once per process
from the environment, checked against the oracle by re-running the
single-iteration parity cases they change in a child pytest with the switch
set:

* NSS_WPC=4   -- four warps per chain for the factored correlated Gaussian
* NSS_MULTI=1 -- several chains per warp (warp engine, d > 32)
* NSS_GROUP=1 -- four speculative probes per warp in groups of eight lanes
* NSS_NO_PDL=1 -- the batch engine without programmatic dependent launches
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = {
    "wpc4": ({"NSS_WPC": "4"}, "warp and corr_gauss"),
    "multi": ({"NSS_MULTI": "1"}, "warp and (corr_gauss or funnel or d33 or d128)"),
    "group": ({"NSS_GROUP": "1"}, "warp and (funnel or d33 or d128)"),
    "no_pdl": ({"NSS_NO_PDL": "1"}, "batch and (logreg or corr_gauss_d40 or c2_mog10)"),
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_single_iteration_parity(name):
    env_add, sel = VARIANTS[name]
    env = dict(os.environ, **env_add)
    cmd = [sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-q", "-x",
           "-m", "gpu", "-k", f"test_single_iteration_parity and ({sel})", "-p", "no:cacheprovider"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    tail = (p.stdout + p.stderr)[-3000:]
    assert p.returncode == 0, tail
    assert " passed" in p.stdout and " failed" not in p.stdout, tail
