cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c8_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_lr.py tests/test_gpu_dist.py tests/test_gpu_gp.py -q > gpurun_out/c8_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "logreg or c4 or batch" > gpurun_out/c8_parity.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c8_bench_c4.json 2> gpurun_out/c8_bench_c4.err
timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c8_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch_advance -s 300 -c 1 -o gpurun_out/c8_adv python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c8_ncu.log 2>&1
