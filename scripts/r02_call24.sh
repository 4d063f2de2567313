cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c24_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c24_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c24_pytest.log
for C in C3b C3a C4; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c24_bench_$C.json 2> gpurun_out/c24_bench_$C.err
done
NSS_HOST_ROUNDS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_dirs -c 20 --csv --log-file gpurun_out/c24_dirs.csv python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c24_ncu.log 2>&1
