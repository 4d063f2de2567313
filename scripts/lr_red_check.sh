timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/lrr_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/lrr_tests.log
timeout 300 python scripts/lr_kernel_probe.py 2>&1 | tail -1
timeout 600 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/lrr_c4.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/lrr_c4.json'));print('C4', round(d['ms_per_step'],3), '%.4g'%d['value'], d['roofline']['frac'], d['roofline']['kernel_ms_avg'], d['phase_ms_per_step'])"
