python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/r01_bench_c4.json 2> gpurun_out/r01_bench_c4.err; echo "c4 rc=$?"
B="python bench.py --config C4 --steps 4 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/c4p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_lr_energy|k_batch_advance' -s 200 -c 2 \
    -o gpurun_out/r01_c4_lr $B > gpurun_out/c4p_ncu.log 2>&1; echo "c4 ncu rc=$?"
