cd $GRAFT_REPO_ROOT
NSS_NVCC_EXTRA=-DNSS_LR_PROF python -c "from paper_2601_23252_b200 import build as b; b.build(force=True)" > gpurun_out/c41_build.log 2>&1
cat > /tmp/one_run.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2601_23252_b200 import nss, workloads as W
prob, cfg = W.workload("C4")
s = nss.Sampler(prob, dict(cfg, max_dead=cfg["n_live"] + cfg["k"] * 500))
info = s.run()
print("iterations", info["iteration"], "evals", info["energy_evals"])
s.close()
PY
timeout 600 python /tmp/one_run.py > gpurun_out/c41_run.txt 2> gpurun_out/c41_prof.txt
