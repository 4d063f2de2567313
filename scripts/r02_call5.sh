cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c5_build.log 2>&1
timeout 600 python scripts/p_ablation.py 6 > gpurun_out/c5_p_ablation.json 2> gpurun_out/c5_p_ablation.err
timeout 300 python bench.py --config C2 --mode shard --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c5_shard_c2.json 2> gpurun_out/c5_shard_c2.err
timeout 300 python bench.py --config C4 --mode shard --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c5_shard_c4.json 2> gpurun_out/c5_shard_c4.err
NSS_SANITIZER=memcheck timeout 1800 python -m pytest tests/test_gpu_sanitizer.py -q > gpurun_out/c5_memcheck.log 2>&1
