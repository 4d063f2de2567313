cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c17_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -k "funnel or d33 or d128 or C3b or c3 or k1 or k_n or p0 or stepout or shrink_cap or width or flat" > gpurun_out/c17_tests.log 2>&1
echo "rc=$?" >> gpurun_out/c17_tests.log
for v in "X=1" "NSS_NO_GROUP=1"; do
  env $v timeout 600 python bench.py --config C3b --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c17_bench_C3b_$v.json 2>&1
done
