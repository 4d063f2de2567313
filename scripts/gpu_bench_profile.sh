set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref.json 2>&1; cat gpurun_out/ref.json
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_hrss -s 10 -c 2 -o gpurun_out/prof_hrss python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
ls -la gpurun_out
