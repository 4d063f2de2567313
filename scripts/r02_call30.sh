cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c30_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gp.py -q -x > gpurun_out/c30_gp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c30_gp_tests.log
NSS_GP_PROF=1 timeout 600 python bench.py --config C5 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c30_bench_C5.json 2> gpurun_out/c30_bench_C5.err
timeout 300 python scripts/gp_kernel_probe.py 2960 > gpurun_out/c30_probe.txt 2>&1
