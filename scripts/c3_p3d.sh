timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or full_run" 2>&1 | tail -2
python bench.py --config C3a --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c3a.json 2>&1; echo "c3a rc=$?"
python bench.py --config C3b --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c3b.json 2>&1; echo "c3b rc=$?"
