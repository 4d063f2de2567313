cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c35_build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_hrss$" -s 3 -c 1 -o gpurun_out/c35_c3a python bench.py --config C3a --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c35_ncu.log 2>&1
