cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c49_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c49_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c49_pytest.log
for C in C3b C3a; do timeout 300 python scripts/stamp_probe.py $C >> gpurun_out/c49_stamps.txt 2>&1; done
for C in C3b C3a C4; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c49_bench_$C.json 2> gpurun_out/c49_bench_$C.err
done
