A="python bench.py --config C3a --steps 6 --warmup 3 --no-cpu-baseline"
$A > gpurun_out/c3ap_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'^k_hrss$' -s 3 -c 1 -o gpurun_out/r01_c3a_hrss $A \
    > gpurun_out/c3ap_ncu.log 2>&1; echo "c3a ncu rc=$?"
