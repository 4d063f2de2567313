python scripts/stamp_probe.py C3b
for c in C3a C3b; do python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/m2_$c.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/m2_$c.json'));print('$c', round(d['ms_per_step'],4), '%.4g'%d['value'], d['phase_ms_per_step']['metric'])"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
