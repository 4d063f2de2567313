cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c11_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/c11_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c11_pytest.log
for C in C4 C2 C1 C3a C3b C5; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 > gpurun_out/c11_bench_$C.json 2> gpurun_out/c11_bench_$C.err
done
NSS_NVCC_EXTRA="-DNSS_ADV_MINB=4" python -c "from paper_2601_23252_b200 import build as b; b.build(force=True)" > gpurun_out/c11_build_minb4.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c11_bench_minb4.json 2>&1
