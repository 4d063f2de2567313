cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/c2_bench_c4.json 2> gpurun_out/c2_bench_c4.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/c2_bench_c2.json 2> gpurun_out/c2_bench_c2.err
