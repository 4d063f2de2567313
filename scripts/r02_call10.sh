cd $GRAFT_REPO_ROOT
for P in 4 8 2; do
  NSS_NVCC_EXTRA="-DNSS_LR_POLY=$P" python -c "from paper_2601_23252_b200 import build as b; b.build(force=True)" > gpurun_out/c10_build_$P.log 2>&1
  timeout 300 python -m pytest tests/test_gpu_lr.py -q -x > gpurun_out/c10_lr_$P.log 2>&1
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c10_bench_poly$P.json 2>&1
done
python -c "from paper_2601_23252_b200 import build as b; b.build(force=True)" > gpurun_out/c10_build_0.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c10_bench_poly0.json 2>&1
