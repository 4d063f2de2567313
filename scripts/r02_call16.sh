cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c16_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_lr.py -q -k "not c3_reduced and not funnel_analytic and not c3a_analytic" > gpurun_out/c16_tests.log 2>&1
echo "rc=$?" >> gpurun_out/c16_tests.log
NSS_MULTI=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "corr" >> gpurun_out/c16_tests.log 2>&1
for C in C3b C3a C4; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c16_bench_$C.json 2> gpurun_out/c16_bench_$C.err
done
NSS_HOST_ROUNDS=1 timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c16_plain.log 2>&1 && \
NSS_HOST_ROUNDS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/c16_c4_launches.csv python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c16_ncu_launch.log 2>&1
