cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c6_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_lr.py -q > gpurun_out/c6_lr.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -k "not c3_reduced and not sanitizer" > gpurun_out/c6_all.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c6_bench_c4.json 2> gpurun_out/c6_bench_c4.err
timeout 600 python scripts/p_ablation.py 12 > gpurun_out/c6_p_ablation.json 2> gpurun_out/c6_p_ablation.err
