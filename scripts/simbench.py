"""Device time of the plan evaluator k_sim over the 100k sweep (tuning aid).
usage: python scripts/simbench.py [mixtures] [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_03365_b200 as ws

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ps = ws.ProblemSet()
ps.add_sweep(0, n)
ps.encode(pinned=True)
pl = ws.Planner(0)
pl.stage(ps)
pl.plan_staged()
res = pl.fetch(ps)
out = None
ms = []
for _ in range(reps + 2):
    pl.simulate_staged()
    out = pl.fetch_sim(ps, out=out)
    ms.append(pl.sim_ms())
best = min(ms[2:])
print(f"k_sim: {best:.3f} ms per {n} plans = {n / best * 1e3:,.0f} evaluations/s; planner k_* ms = {pl.kernel_ms()}")
