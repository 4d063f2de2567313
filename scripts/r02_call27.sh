cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c27_build.log 2>&1
for n in 2 1; do
  NSS_GP_CTAS=$n timeout 300 python scripts/gp_kernel_probe.py 2960 > gpurun_out/c27_probe_$n.txt 2>&1
  NSS_GP_CTAS=$n timeout 900 python bench.py --config C5 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c27_bench_C5_$n.json 2> gpurun_out/c27_bench_C5_$n.err
done
