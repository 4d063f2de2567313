cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c61_build.log 2>&1
for L in 8 16 4; do
  NSS_LOOP_ROUNDS=$L timeout 900 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c61_bench_C4_$L.json 2> gpurun_out/c61_bench_C4_$L.err
done
