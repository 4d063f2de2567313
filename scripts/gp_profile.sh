# usage: bash scripts/gp_profile.sh <tag>: full ncu capture of k_gp_energy on a
# 592-matrix launch (two matrices per CTA), after the same command exits 0
tag=${1:-r01}
mkdir -p gpurun_out
G="python scripts/gp_kernel_probe.py 592"
$G > gpurun_out/${tag}_c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gp -s 1 -c 1 -o gpurun_out/${tag}_c5_gp $G \
    > gpurun_out/${tag}_c5_ncu.log 2>&1; echo "c5 rc=$?"
