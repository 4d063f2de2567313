# usage: bash scripts/round_profile2.sh <tag>: full ncu captures of the dominant
# kernels of C3a (k_hrss), C4 (k_lr_energy, k_batch_advance) and C5
# (k_gp_energy), each after the same command exited 0 without ncu
tag=${1:-r01}
mkdir -p gpurun_out
A="python bench.py --config C3a --steps 6 --warmup 3 --no-cpu-baseline"
$A > gpurun_out/${tag}_c3a_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'^k_hrss$' -s 3 -c 1 -o gpurun_out/${tag}_c3a_hrss $A \
    > gpurun_out/${tag}_c3a_ncu.log 2>&1; echo "c3a rc=$?"
B="python bench.py --config C4 --steps 4 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/${tag}_c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_lr_energy|k_batch_advance' -s 200 -c 2 \
    -o gpurun_out/${tag}_c4_lr $B > gpurun_out/${tag}_c4_ncu.log 2>&1; echo "c4 rc=$?"
G="python scripts/gp_kernel_probe.py 592"
$G > gpurun_out/${tag}_c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gp -s 1 -c 1 -o gpurun_out/${tag}_c5_gp $G \
    > gpurun_out/${tag}_c5_ncu.log 2>&1; echo "c5 rc=$?"
