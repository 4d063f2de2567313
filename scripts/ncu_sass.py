"""SASS-level hot spots of the first launch of a kernel in an ncu report:
top instructions by stall samples, and instruction mix."""
import collections
import csv
import subprocess
import sys

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kname,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data, nk = None, [], 0
for r in rows:
    if r and r[0] == "Kernel Name":
        nk += 1
        if nk > 1:
            break
        continue
    if r and r[0] == "Address":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and len(r) > 5:
        data.append(r)
S = hdr["Warp Stall Sampling (All Samples)"]
I = hdr["Instructions Executed"]
tot_s = sum(int(r[S]) for r in data) or 1
tot_i = sum(int(r[I]) for r in data)
print(f"samples={tot_s} warp-instructions={tot_i}")
for idx, r in sorted(enumerate(data), key=lambda t: -int(t[1][S]))[:top]:
    print(f"{idx:5d} {100 * int(r[S]) / tot_s:5.1f}% {int(r[I]):8d}  {r[hdr['Source']][:90]}")
ops = collections.Counter()
for r in data:
    t = r[hdr["Source"]].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += int(r[I])
print(" ".join(f"{o}:{n}" for o, n in ops.most_common(24)))
