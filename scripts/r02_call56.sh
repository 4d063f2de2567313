cd $GRAFT_REPO_ROOT
for m in 32 24; do
  NSS_NVCC_EXTRA="-DNSS_ADV_WARPS=1 -DNSS_ADV_MINB=$m" python -c "from paper_2601_23252_b200 import build as b; b.build(force=True)" > gpurun_out/c56_build_$m.log 2>&1
  grep -A2 "k_batch_advance" gpurun_out/c56_build_$m.log | grep -i "spill\|registers" | head -4 > gpurun_out/c56_regs_$m.txt
  timeout 900 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c56_bench_C4_$m.json 2> gpurun_out/c56_bench_C4_$m.err
done
