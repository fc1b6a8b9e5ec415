"""Aggregate an ncu --page source (cuda,sass) CSV to per-source-line stall
samples and executed warp instructions.  usage: ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
samples, insts = defaultdict(int), defaultdict(int)
src_text = {}
fname, line, hdr = None, None, None
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 8:
        continue
    if row[0]:
        line = (fname, int(row[0]))
        src_text[line] = row[1].strip()
    if line is None or not row[2]:
        continue
    try:
        samples[line] += int(row[4] or 0)
        insts[line] += int(row[7] or 0)
    except ValueError:
        pass
tot_s = sum(samples.values()) or 1
tot_i = sum(insts.values()) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for key in sorted(samples, key=lambda k: -samples[k])[:top]:
    print(f"{100*samples[key]/tot_s:5.1f}% smp {100*insts[key]/tot_i:5.1f}% ins  {key[0]}:{key[1]:<5} {src_text.get(key,'')[:90]}")

# ---- per-function aggregation (plan.cuh / common.cuh functions by start line) ----
import re
full = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                      capture_output=True, text=True).stdout
allsrc, cur = {}, None
for row in csv.reader(full.splitlines()):
    if row and row[0] == "File Name":
        cur = row[1].split("/")[-1]
    elif row and row[0].isdigit() and cur:
        allsrc[(cur, int(row[0]))] = row[1].strip()
starts = []
for (f, ln), txt in allsrc.items():
    m = re.match(r"(?:template <[^>]*>\s*)?(?:__host__ )?__device__ (?:__forceinline__ )?\S+ (\w+)\(", txt)
    if m or txt.startswith("__global__"):
        starts.append((f, ln, m.group(1) if m else "kernel_body"))
    m2 = re.match(r"struct (\w+)", txt)
    if m2:
        starts.append((f, ln, "struct " + m2.group(1)))
starts.sort()
func_s, func_i = defaultdict(int), defaultdict(int)
for key in samples:
    f, ln = key
    name = "?"
    for sf, sl, nm in starts:
        if sf == f and sl <= ln:
            name = nm
    func_s[f + ":" + name] += samples[key]
    func_i[f + ":" + name] += insts[key]
print("\nper function:")
for k in sorted(func_s, key=lambda k: -func_s[k])[:30]:
    print(f"{100*func_s[k]/tot_s:5.1f}% smp {100*func_i[k]/tot_i:5.1f}% ins  {k}")
