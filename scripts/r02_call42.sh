cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c42_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gp.py -q -x > gpurun_out/c42_gp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c42_gp_tests.log
timeout 300 python scripts/gp_kernel_probe.py 2960 > gpurun_out/c42_probe.txt 2>&1
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c42_bench_C5.json 2> gpurun_out/c42_bench_C5.err
bash scripts/gp_phases.sh > gpurun_out/c42_phases.txt 2>&1
