"""Summarize gpurun_out ncu artefacts of one tag into profiles/<tag>_*.txt.
usage: python scripts/profile_summary.py <tag>"""
import csv
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
out_dir = ROOT / "profiles"
out_dir.mkdir(exist_ok=True)
g = ROOT / "gpurun_out"

# launch list shares (cold-cache, serialised: compare shares, not absolutes)
lines = []
lf = g / f"launches_{tag}.csv"
if lf.exists():
    rows = list(csv.reader(lf.read_text().splitlines()))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines.append(f"# ncu launch list ({lf.name}): gpu__time_duration.sum, --clock-control none")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:45s} launches={len(v):4d} total_ms={sum(v)/1e6:9.3f} share={100*sum(v)/tot:5.1f}%")
    (out_dir / f"{tag}_launches.txt").write_text("\n".join(lines) + "\n")

want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "launch__grid_size",
        "launch__block_size", "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "sm__cycles_elapsed.avg", "launch__shared_mem_per_block_dynamic",
        "smsp__average_warp_latency_issue_stalled", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for rep in sorted(g.glob(f"*_{tag}.ncu-rep")):
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    out = [f"# {rep.name}: ncu --set full --clock-control none (one launch)"]
    for data in rows[2:]:
        out.append(f"## {data[hdr.index('Kernel Name')] if 'Kernel Name' in hdr else ''}")
        for i, n in enumerate(hdr):
            if any(n == w or n.startswith(w + ".") for w in want):
                out.append(f"{n:70s} {units[i]:12s} {data[i]}")
    lines_out = subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_lines.py"), str(rep), "30"],
                               capture_output=True, text=True).stdout
    out.append("\n# source attribution (stall samples / executed warp instructions)\n" + lines_out)
    (out_dir / f"{tag}_{rep.stem.rsplit('_', 1)[0]}.txt").write_text("\n".join(out) + "\n")
print(sorted(p.name for p in out_dir.glob(f"{tag}_*")))

# per-launch DRAM traffic of the captured kernels -> profiles/traffic.json (read by bench.py)
import json
traffic = {"source": f"ncu --set full captures *_{tag}.ncu-rep (one launch each)"}
for rep in sorted(g.glob(f"*_{tag}.ncu-rep")):
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    hdr, units, data = rows[0], rows[1], rows[2]
    def val(name):
        i = hdr.index(name)
        v = float(data[i].replace(",", ""))
        u = units[i].lower()
        return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
    kname = data[hdr.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0]
    kname = kname[len("void "):] if kname.startswith("void ") else kname
    traffic[kname] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
(out_dir / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
print(traffic)
