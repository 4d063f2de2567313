cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c15_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -k "corr or C3a or c3 or warp" > gpurun_out/c15_tests.log 2>&1
echo "rc=$?" >> gpurun_out/c15_tests.log
for v in "X=1" "NSS_MULTI_NC=2" "NSS_NO_MULTI=1"; do
  env $v timeout 600 python bench.py --config C3a --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c15_bench_$v.json 2>&1
done
