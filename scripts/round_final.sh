# final round-1 measurements: every bench line, the reference arm, the C2
# launch list, full ncu captures of k_hrss (C3a) and the large-d metric (C3b)
tag=${1:-r01}
mkdir -p gpurun_out
bash scripts/round_bench.sh $tag
A="python bench.py --config C3a --steps 6 --warmup 3 --no-cpu-baseline"
$A > gpurun_out/${tag}_c3a_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'^k_hrss$' -s 3 -c 1 -o gpurun_out/${tag}_c3a_hrss $A \
    > gpurun_out/${tag}_c3a_ncu.log 2>&1; echo "c3a ncu rc=$?"
B="python bench.py --config C3b --steps 6 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/${tag}_c3b_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_metric' -s 6 -c 3 -o gpurun_out/${tag}_c3b_metric $B \
    > gpurun_out/${tag}_c3b_ncu.log 2>&1; echo "c3b ncu rc=$?"
