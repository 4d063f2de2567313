# usage: bash scripts/round_bench.sh <tag>   (on a GPU box via gpurun)
# bench lines for the default workload and every other config, the reference
# arm (CPU oracle), then the launch list of the default workload
tag=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err; echo "c2 rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${tag}_ref_c2.json 2>&1; echo "ref rc=$?"
python bench.py --config C1 --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_bench_c1.json 2>&1; echo "c1 rc=$?"
python bench.py --config C3a --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_c3a.json 2>&1; echo "c3a rc=$?"
python bench.py --config C3b --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_c3b.json 2>&1; echo "c3b rc=$?"
python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err; echo "c4 rc=$?"
python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err; echo "c5 rc=$?"
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c2.csv \
    python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu1.log 2>&1; echo "ncu1 rc=$?"
