cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c31_build.log 2>&1
NSS_LR_BN=160 timeout 600 python -m pytest tests/test_gpu_lr.py -q -x > gpurun_out/c31_lr160.log 2>&1; echo "rc=$?" >> gpurun_out/c31_lr160.log
NSS_LR_BN=160 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "logreg or batch" > gpurun_out/c31_par160.log 2>&1; echo "rc=$?" >> gpurun_out/c31_par160.log
for bn in 160 256; do
  NSS_LR_BN=$bn timeout 900 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c31_bench_C4_$bn.json 2> gpurun_out/c31_bench_C4_$bn.err
done
