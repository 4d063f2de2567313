cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c52_build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_metric$" -s 20 -c 2 -o gpurun_out/c52_met python bench.py --config C3b --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c52_ncu.log 2>&1
