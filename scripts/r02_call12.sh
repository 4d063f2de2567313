cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c12_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_lr.py -q -x -k "not c3_reduced and not funnel_analytic and not c3a_analytic" > gpurun_out/c12_tests.log 2>&1
for C in C2 C1 C4; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c12_bench_$C.json 2> gpurun_out/c12_bench_$C.err
done
for C in C3a C3b; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 > gpurun_out/c12_bench_$C.json 2> gpurun_out/c12_bench_$C.err
done
python scripts/stamp_probe.py C2 > gpurun_out/c12_stamps.txt 2>&1
python scripts/stamp_probe.py C1 >> gpurun_out/c12_stamps.txt 2>&1
