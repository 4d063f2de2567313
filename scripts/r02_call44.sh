cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c44_build.log 2>&1
timeout 900 python -m pytest tests/test_bench_contract.py -q > gpurun_out/c44_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c44_pytest.log
