"""Print the per-phase SM-cycle breakdown of a -DWS_PHASES library build.
usage: WSGPU_LIB=lib/libwsgpu_phases.so python scripts/phases.py [mixtures]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_03365_b200 as ws

NAMES = {0: "place:prologue", 1: "place:wave order", 2: "place:flows_in+disp", 3: "place:candidates",
         4: "place:score", 8: "place:minloc", 5: "place:commit+flows", 6: "place:restore", 7: "place:emit",
         10: "sched:graph", 11: "sched:fit+valid", 12: "sched:alloc", 13: "sched:schedule", 14: "sched:writeback"}
# argument: a mixture count (sweep prefix), or family:tasks:devices for one
# BASELINE scenario plan (single-plan latency)
arg = sys.argv[1] if len(sys.argv) > 1 else "100000"
ps = ws.ProblemSet()
if ":" in arg:
    fam, t, d = arg.split(":")
    ps.add_scenario(fam, int(t), int(d), 0)
    n = 1
elif arg.startswith("mix"):  # one sweep mixture, e.g. mix37617
    ps.add_sweep(int(arg[3:]), 1)
    n = 1
else:
    n = int(arg)
    ps.add_sweep(0, n)
ps.encode(pinned=True)
pl = ws.Planner(0)
f = ws.lib.ws_debug_phase_cycles
f.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 32)()
pl.stage(ps)
pl.plan_staged()
pl.fetch(ps)
f(buf, 32)
pl.plan_staged()
pl.fetch(ps)
f(buf, 32)
tot_p = sum(buf[i] for i in range(0, 10)) or 1
tot_s = sum(buf[i] for i in range(10, 15)) or 1
for i, name in NAMES.items():
    tot = tot_p if i < 10 else tot_s
    print(f"{name:24s} {buf[i] / n:12.0f} cycles/plan  {100 * buf[i] / tot:5.1f}%")
ne = buf[20] or 1
print(f"scored entries/plan {buf[20] / n:.1f}; per entry: ncand {buf[21] / ne:.1f}  n {buf[22] / ne:.1f}  "
      f"ndisp {buf[23] / ne:.1f}  nfin {buf[24] / ne:.2f}  islands {buf[25] / ne:.1f}  "
      f"lane-iters {buf[26] / ne:.2f}  N {buf[27] / ne:.1f}")
print(f"placement attempts/plan {buf[28] / n:.1f}; replayed waves/plan {buf[29] / n:.1f}; "
      f"wave placements/plan {buf[30] / n:.1f}")
