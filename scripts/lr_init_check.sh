timeout 900 python -m pytest tests/test_gpu_lr.py tests/test_gpu_parity.py -x -q > gpurun_out/lri_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/lri_tests.log
python scripts/e2e_c4_probe.py C4
python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/lri_c4.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/lri_c4.json'));print('C4', round(d['ms_per_step'],3), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'])"
