"""Pipe utilisation summary of every kernel in an ncu report (tensor, fp64,
FMA/ALU, XU/MUFU pipes, DRAM bytes, active lanes, divergence)."""
import csv
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor%",
    "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "fp64%",
    "SM_A.TriageCompute.sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed": "xu%",
    "TPC.TriageCompute.sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed": "alu%",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma%",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "lanes/inst",
    "smsp__sass_average_branch_targets_threads_uniform.pct": "branch_uniform%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy%",
}
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
for r in rows[2:]:
    name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    parts = []
    for m, short in WANT.items():
        if m in idx and r[idx[m]] not in ("", "n/a"):
            parts.append(f"{short}={r[idx[m]]}{units[idx[m]] if units[idx[m]] not in ('%', '') else ''}")
    print(f"{name:28s} " + " ".join(parts))
