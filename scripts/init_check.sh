NSS_INIT_PROF=1 python scripts/e2e_probe.py 2>&1 | tail -12
python scripts/e2e_probe.py 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/init_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/init_tests.log
python bench.py --no-cpu-baseline > gpurun_out/init_c2.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/init_c2.json'));print('C2', d['ms_per_step'], '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'])"
python bench.py --config C1 --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/init_c1.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/init_c1.json'));print('C1', d['ms_per_step'], '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'])"
