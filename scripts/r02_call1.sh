cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c1_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -k "not c3_reduced" > gpurun_out/c1_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/c1_pytest.log
timeout 300 python bench.py --config C4 --steps 20 --warmup 5 > gpurun_out/c1_bench_c4.log 2>&1
