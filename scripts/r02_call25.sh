cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c25_build.log 2>&1
NSS_HOST_ROUNDS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dirs -s 2 -c 1 -o gpurun_out/c25_dirs python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c25_ncu.log 2>&1
