cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c13_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_lr.py -q -x > gpurun_out/c13_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "logreg or c4 or batch" >> gpurun_out/c13_tests.log 2>&1
for v in "X=1" "NSS_ADV_WARP=1" "X=2" "NSS_ADV_WARP=2"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c13_bench_$v.json 2>&1
done
