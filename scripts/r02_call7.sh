cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c7_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_lr.py tests/test_gpu_dist.py -q > gpurun_out/c7_lr_dist.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "logreg or c4 or update_all or rw" > gpurun_out/c7_parity_lr.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c7_bench_c4.json 2> gpurun_out/c7_bench_c4.err
