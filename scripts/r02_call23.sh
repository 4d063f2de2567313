cd $GRAFT_REPO_ROOT
NSS_NVCC_EXTRA=-DNSS_LR_PROF python -c "from paper_2601_23252_b200 import build as b; b.build(force=True)" > gpurun_out/c23_build.log 2>&1
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c23_bench.json 2> gpurun_out/c23_bench.err
grep lr_prof gpurun_out/c23_bench.err > gpurun_out/c23_lr_prof.txt
