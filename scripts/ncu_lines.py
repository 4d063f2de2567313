"""Per-source-line hot spots of one kernel (ncu report built with -lineinfo and
--import-source on): stall samples and instructions per CUDA source line."""
import csv
import subprocess
import sys

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kname,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
path, hdr, res = "?", None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        try:
            s, ins = int(r[4]), int(r[7])
        except ValueError:
            continue
        if s or ins:
            res.append((s, ins, path, r[0], r[1].strip()[:90]))
tot = sum(x[0] for x in res) or 1
print(f"samples={tot}")
for s, ins, p, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {ins:9d} {p}:{ln:<5s} {src}")
