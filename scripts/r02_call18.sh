cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c18_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_lr.py tests/test_gpu_dist.py tests/test_gpu_gp.py -q > gpurun_out/c18_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "logreg or c4 or batch" >> gpurun_out/c18_tests.log 2>&1
echo "rc=$?" >> gpurun_out/c18_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c18_bench_C4.json 2>&1
timeout 900 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c18_bench_C5.json 2>&1
