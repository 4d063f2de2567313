mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/val_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/val_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/val_smoke.log
timeout 600 python bench.py > gpurun_out/val_bench_c2.json 2> gpurun_out/val_bench_c2.err; echo "c2 rc=$?"; cat gpurun_out/val_bench_c2.json
timeout 600 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/val_bench_c4.json 2>&1; echo "c4 rc=$?"
