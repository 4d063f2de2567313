cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c37_build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_metric|k_select|k_hrss_lane" -s 30 -c 3 -o gpurun_out/c37_c2 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c37_ncu.log 2>&1
