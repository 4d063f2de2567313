export NSS_LR_BN=256
timeout 300 python -m pytest tests/test_gpu_lr.py -x -q > gpurun_out/lr256_tests.log 2>&1; echo "tests(256) rc=$?"; tail -3 gpurun_out/lr256_tests.log
for bn in 256 128; do export NSS_LR_BN=$bn
timeout 300 python scripts/lr_kernel_probe.py 2>&1 | tail -3
timeout 600 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/lr_ab.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/lr_ab.json'));print('bn=$bn C4', round(d['ms_per_step'],3), '%.4g'%d['value'], d['roofline']['frac'], d['roofline']['kernel_ms_avg'])"
done
