cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c47_build.log 2>&1
for C in C4 C3b; do timeout 300 python scripts/stamp_probe.py $C >> gpurun_out/c47_stamps.txt 2>&1; done
