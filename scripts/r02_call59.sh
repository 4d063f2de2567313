cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c59_build.log 2>&1
NSS_HOST_ROUNDS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lr_energy|k_batch_advance" -s 40 -c 3 -o gpurun_out/c59_c4_full python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c59_ncu_full.log 2>&1
