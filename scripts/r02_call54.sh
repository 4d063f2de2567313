cd $GRAFT_REPO_ROOT
for w in 2 4; do
  NSS_NVCC_EXTRA=-DNSS_ADV_WARPS=$w python -c "from paper_2601_23252_b200 import build as b; b.build(force=True)" > gpurun_out/c54_build_$w.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "batch" > gpurun_out/c54_pytest_$w.log 2>&1; echo "rc=$?" >> gpurun_out/c54_pytest_$w.log
  timeout 900 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c54_bench_C4_$w.json 2> gpurun_out/c54_bench_C4_$w.err
done
