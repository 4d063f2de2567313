cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c33_build.log 2>&1
NSS_WPC=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "corr or c3" > gpurun_out/c33_wpc4.log 2>&1; echo "rc=$?" >> gpurun_out/c33_wpc4.log
for w in 4 2; do
  NSS_WPC=$w timeout 900 python bench.py --config C3a --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c33_bench_C3a_$w.json 2> gpurun_out/c33_bench_C3a_$w.err
done
