timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pg_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pg_tests.log
python scripts/step_probe.py 2>&1 | tail -4
python scripts/e2e_probe.py 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/pg_c2.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/pg_c2.json'));print('C2', round(d['ms_per_step']*1e3,2), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'])"
python bench.py --config C1 --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/pg_c1.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/pg_c1.json'));print('C1', round(d['ms_per_step']*1e3,2), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'])"
