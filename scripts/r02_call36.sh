cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c36_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lr.py tests/test_gpu_gp.py tests/test_gpu_dist.py -q -x > gpurun_out/c36_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c36_pytest.log
timeout 900 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c36_bench_C4.json 2> gpurun_out/c36_bench_C4.err
timeout 900 python bench.py --config C5 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c36_bench_C5.json 2> gpurun_out/c36_bench_C5.err
