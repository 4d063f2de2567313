"""Write tests/golden/oracle_fullruns_<cfg>_s<seed>.json: full fp64-oracle NSS
runs (to the termination criterion R-19, then finalised, R-18) of the reduced
C3 configurations SURVEY C-9 T4 names ("C3 at reduced n": n_live = 1000,
k = 100, p = 3d = 300, d = 100).  A full oracle run there takes 0.5-1.5 h of
one host core, too long for a test, so the value is stored; this script calls
ONLY oracle/ (and the seeded input generator workloads.py) -- nothing of the
CUDA path -- so the stored numbers are the oracle's.

    python scripts/golden_oracle_fullruns.py C3a 1      # one run per process
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import nsso  # noqa: E402
from paper_2601_23252_b200 import workloads as W  # noqa: E402

REDUCED = dict(n_live=1000, k=100)


def reduced_workload(name, seed):
    prob, cfg = W.workload(name, seed=seed, **REDUCED)
    cfg["max_dead"] = cfg["n_live"] + cfg["k"] * 8000
    return prob, cfg


def main():
    name, seed = sys.argv[1], int(sys.argv[2])
    prob, cfg = reduced_workload(name, seed)
    t0 = time.time()
    o = nsso.Oracle(prob, cfg)
    info = o.run()
    lz, err = o.evidence()
    out = {"config": name, "problem": prob.name, "seed": seed, "cfg": cfg, "log_z": lz, "log_z_err": err,
           "iterations": info["iteration"], "energy_evals": info["energy_evals"],
           "terminated": info["terminated"], "oracle_seconds": time.time() - t0,
           "source": "scripts/golden_oracle_fullruns.py (oracle/nsso.c only)"}
    path = os.path.join(ROOT, "tests", "golden", f"oracle_fullrun_{name}_s{seed}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
