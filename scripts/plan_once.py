"""Stage the 100k sweep and plan it `reps` times (an ncu target: no timing).
usage: python scripts/plan_once.py [mixtures] [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_03365_b200 as ws

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ps = ws.ProblemSet()
ps.add_sweep(0, n)
ps.encode(pinned=True)
pl = ws.Planner(0)
pl.stage(ps)
for _ in range(reps):
    pl.plan_staged()
res = pl.fetch(ps)
print("ok", sum(1 for i in range(n) if res.results[i].status == 0))
