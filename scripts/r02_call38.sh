cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c38_build.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_options.py tests/test_gpu_lr.py -q > gpurun_out/c38_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c38_pytest.log
