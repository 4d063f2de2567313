timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/met_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/met_tests.log
python scripts/stamp_probe.py C3b; python scripts/stamp_probe.py C2
for c in C3a C3b; do python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/met_$c.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/met_$c.json'));print('$c', round(d['ms_per_step'],4), '%.4g'%d['value'], d['phase_ms_per_step'])"; done
python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/met_C4.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/met_C4.json'));print('C4', round(d['ms_per_step'],4), '%.4g'%d['value'], d['phase_ms_per_step'])"
