cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c60_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c60_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c60_pytest.log
timeout 900 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c60_bench_C4.json 2> gpurun_out/c60_bench_C4.err
NSS_HOST_ROUNDS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_select -c 10 --csv --log-file gpurun_out/c60_select.csv python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c60_ncu.log 2>&1
