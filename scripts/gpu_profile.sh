# usage: bash scripts/gpu_profile.sh <tag> <kernel-regex> [bench args...]
tag=$1; kre=$2; shift 2
python bench.py --no-cpu-baseline --steps 60 --warmup 3 "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --no-cpu-baseline --steps 60 --warmup 3 "$@" > gpurun_out/${tag}_ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:$kre -s 20 -c 2 -o gpurun_out/${tag}_prof \
    python bench.py --no-cpu-baseline --steps 60 --warmup 3 "$@" > gpurun_out/${tag}_ncu2.log 2>&1; echo "ncu2 rc=$?"
