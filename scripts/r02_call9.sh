cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c9_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_lr.py tests/test_gpu_dist.py -q -x > gpurun_out/c9_tests.log 2>&1
for v in "X=1" "NSS_LOOP_ROUNDS=4" "NSS_LOOP_ROUNDS=32" "NSS_NO_PDL=1" "NSS_HOST_ROUNDS=1"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c9_bench_$v.json 2>&1
done
