cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c57_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/c57_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c57_pytest.log
for C in C4 C1 C2 C3a C3b C5; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 > gpurun_out/c57_bench_$C.json 2> gpurun_out/c57_bench_$C.err
done
timeout 900 python bench.py --config C4 --mode shard --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c57_bench_C4_shard.json 2> gpurun_out/c57_bench_C4_shard.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/c57_ref_C4.json 2> gpurun_out/c57_ref_C4.err
NSS_HOST_ROUNDS=1 timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c57_plain.log 2>&1 && \
NSS_HOST_ROUNDS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/c57_c4_launches.csv python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c57_ncu_launch.log 2>&1
