# full GPU suite, C4/C5 bench lines, ncu launch list + full capture of k_gp_chains (C5)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01b_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r01b_gputests.log
timeout 600 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r01b_bench_c4.json 2>&1; echo "c4 rc=$?"
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/r01b_bench_c5.json 2> gpurun_out/r01b_bench_c5.err; echo "c5 rc=$?"
G="python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b_c5_launches.csv $G > gpurun_out/r01b_c5_ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_gp_chains -s 2 -c 1 -o gpurun_out/r01b_c5_gp_chains $G > gpurun_out/r01b_c5_ncu2.log 2>&1; echo "ncu2 rc=$?"
