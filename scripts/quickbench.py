"""Device-resident planning throughput of one library variant (tuning aid).
usage: WSGPU_LIB=path python scripts/quickbench.py [mixtures] [steps]"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_03365_b200 as ws

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ps = ws.ProblemSet()
ps.add_sweep(0, n)
ps.encode(pinned=True)
pl = ws.Planner(0)
pl.stage(ps)
for _ in range(3):
    pl.plan_staged()
res = pl.fetch(ps)
ks = []
for _ in range(steps):
    pl.plan_staged()
    pl.fetch(ps, out=res)
    ks.append(pl.kernel_ms())
tot = [sum(k) for k in ks]
best = min(tot)
print(f"{os.environ.get('WSGPU_LIB', 'default')}: {n / (best / 1000):,.0f} plans/s  "
      f"fit/sched/place ms = {min(k[0] for k in ks):.2f}/{min(k[1] for k in ks):.2f}/{min(k[2] for k in ks):.2f}")
print(f"soft-cap overflows re-planned: {pl.retry_count}")
