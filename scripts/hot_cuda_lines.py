"""Per-CUDA-line stall samples, executed instructions and SASS size of one
kernel from an ncu report (--import-source on): which source lines are hot
and how much code they carry (instruction-cache study).
usage: python scripts/hot_cuda_lines.py <ncu-rep> [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
f = None
hdr = None
stats = collections.defaultdict(lambda: [0, 0, 0])  # samples, executed, sass count
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ei = hdr.index("Instructions Executed")
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0] and r[0] != "-":  # a CUDA source line
        cur = (f, int(r[0]), r[1][:70])
        try:
            stats[cur][0] += int(r[si] or 0)
            stats[cur][1] += int(r[ei] or 0)
        except ValueError:
            pass
    elif r[2] and r[2] != "-" and cur:  # SASS row under the current line
        stats[cur][2] += 1
ts = sum(v[0] for v in stats.values()) or 1
te = sum(v[1] for v in stats.values()) or 1
sass_total = sum(v[2] for v in stats.values())
print(f"total SASS rows {sass_total}")
print(f"{'stall%':>6} {'exec%':>6} {'sass':>5}  line")
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/ts:6.2f} {100*v[1]/te:6.2f} {v[2]:5d}  {k[0]}:{k[1]}  {k[2]}")
