"""Tuning aid: device ms (k_sched + k_place) of given sweep mixtures planned alone.
usage: python scripts/plan_times.py i [i ...]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_03365_b200 as ws  # noqa: E402

pl = ws.Planner(0)
for i in map(int, sys.argv[1:]):
    one = ws.ProblemSet()
    one.add_sweep(i, 1)
    one.encode(pinned=True)
    pl.stage(one)
    best = (1e9, 0, 0)
    for _ in range(3):
        pl.plan_staged()
        r = pl.fetch(one)
        k = pl.kernel_ms()
        best = min(best, (k[1] + k[2], k[1], k[2]))
    print(f"mixture {i:6d} status {r.results[0].status} sched {best[1]:.3f} place {best[2]:.3f} ms", flush=True)
