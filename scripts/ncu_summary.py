"""Summarise ncu outputs: per-kernel launch list shares and key metrics of a full capture."""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    for d in data:
        agg[d["Kernel Name"].split("(")[0][:70]].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k:70s} n={len(v):4d} avg={sum(v) / len(v) / 1e3:9.2f}us share={sum(v) / tot:.3f}")
    return "\n".join(out)


KEYS = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Executed Ipc Active",
        "Block Size", "Grid Size", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Branch Efficiency", "Avg. Divergent Branches", "L1/TEX Hit Rate", "L2 Hit Rate"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    lines = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in KEYS:
            lines.append(f"{d['ID']:>3} {d['Kernel Name'].split('(')[0][:40]:40s} {d['Metric Name']:38s} {d['Metric Value']:>12} {d['Metric Unit']}")
    return "\n".join(lines)


def raw(rep, pats=("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active", "smsp__thread_inst_executed_per_inst_executed", "sm__inst_executed_pipe", "smsp__average_warp")):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        for h, u, v in zip(hdr, units, r):
            if any(h.startswith(p) for p in pats):
                lines.append(f"{h:70s} {v:>14} {u}")
    return "\n".join(lines)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print({"launches": launches, "details": details, "raw": raw}[mode](path))
