cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c4_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pr scripts/pipe_rates.cu && /tmp/pr > gpurun_out/c4_pipe_rates.txt 2>&1
timeout 300 python bench.py --config C2 --mode shard --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c4_shard_c2.json 2> gpurun_out/c4_shard_c2.err
timeout 300 python bench.py --config C4 --mode shard --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c4_shard_c4.json 2> gpurun_out/c4_shard_c4.err
timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lr_energy -s 300 -c 1 -o gpurun_out/c4_lr python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4_ncu.log 2>&1
