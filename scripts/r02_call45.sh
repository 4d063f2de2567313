cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c45_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_lr.py tests/test_gpu_smc.py -q -x > gpurun_out/c45_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c45_pytest.log
for C in C3b C3a C4; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c45_bench_$C.json 2> gpurun_out/c45_bench_$C.err
done
