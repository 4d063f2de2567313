cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c20_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_lr.py tests/test_gpu_dist.py -q -x -k "logreg or lr or gp" > gpurun_out/c20_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "logreg or c4 or batch" >> gpurun_out/c20_tests.log 2>&1
echo "rc=$?" >> gpurun_out/c20_tests.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c20_bench_C4_$i.json 2>&1; done
