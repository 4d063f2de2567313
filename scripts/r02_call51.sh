cd $GRAFT_REPO_ROOT
NSS_NVCC_EXTRA=-DNSS_MET_PROF python -c "from paper_2601_23252_b200 import build as b; b.build(force=True)" > gpurun_out/c51_build.log 2>&1
timeout 300 python scripts/met_panel_probe.py C3b > gpurun_out/c51_panel.txt 2>&1
