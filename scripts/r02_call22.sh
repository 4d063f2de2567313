cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fr scripts/fp64_rates.cu && timeout 120 /tmp/fr > gpurun_out/c22_fp64_rates.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c22_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gp.py -q -x > gpurun_out/c22_gp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c22_gp_tests.log
timeout 300 python scripts/gp_kernel_probe.py 2960 > gpurun_out/c22_gp_probe.txt 2>&1
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c22_bench_C5.json 2> gpurun_out/c22_bench_C5.err
bash scripts/gp_phases.sh > gpurun_out/c22_phases.txt 2>&1
