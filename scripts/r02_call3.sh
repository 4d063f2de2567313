cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c3_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/c3_dist.log 2>&1
echo "rc=$?" >> gpurun_out/c3_dist.log
timeout 1500 python -m pytest tests -m gpu -q -k "not c3_reduced and not test_gpu_dist" > gpurun_out/c3_all.log 2>&1
echo "rc=$?" >> gpurun_out/c3_all.log
