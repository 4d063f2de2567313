cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c58_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -k full_size > gpurun_out/c58_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c58_pytest.log
