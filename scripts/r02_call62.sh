cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c62_build.log 2>&1
timeout 1800 python scripts/accuracy_table.py > gpurun_out/c62_accuracy.md 2> gpurun_out/c62_accuracy.err
