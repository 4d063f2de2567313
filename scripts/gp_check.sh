mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gp.py -x -q > gpurun_out/gp6_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gp6_tests.log
python scripts/gp_kernel_probe.py 2960; python scripts/gp_kernel_probe.py 2960
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gp6_bench_c5.json 2>&1; echo "c5 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/gp6_bench_c5.json'));print(d['ms_per_step'],d['value'],d['roofline'],d['e2e'])" || tail -20 gpurun_out/gp6_bench_c5.json
bash scripts/gp_phases.sh 2>&1 | grep phases
