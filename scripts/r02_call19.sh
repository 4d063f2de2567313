cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c19_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "d100 or d33 or d40 or d128 or C3 or c3 or c4 or corr or funnel" > gpurun_out/c19_tests.log 2>&1
echo "rc=$?" >> gpurun_out/c19_tests.log
for C in C3b C3a C4; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c19_bench_$C.json 2>&1
done
