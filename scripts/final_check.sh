mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --config C3a --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c3a.json 2>&1; echo "c3a rc=$?"
python bench.py --config C3b --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c3b.json 2>&1; echo "c3b rc=$?"
python bench.py > gpurun_out/r01_bench_c2.json 2> gpurun_out/r01_bench_c2.err; echo "c2 rc=$?"
