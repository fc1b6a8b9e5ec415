"""Tuning aid: device time of single sweep mixtures planned alone (ws_plan_staged
on a one-plan batch) -- finds the long-tail plans that bound a shard's kernel time.
usage: python scripts/slow_plans.py [n_random]"""
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_03365_b200 as ws  # noqa: E402

n_rand = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
pl = ws.Planner(0)
ps = ws.ProblemSet()
ps.add_sweep(0, 100000)
ps.encode(pinned=True)
res = pl.plan(ps)
failed = [i for i in range(100000) if res.results[i].status != 0]
sample = sorted(set(failed) | set(random.Random(1).sample(range(100000), n_rand)))
times = []
for i in sample:
    one = ws.ProblemSet()
    one.add_sweep(i, 1)
    one.encode(pinned=True)
    pl.stage(one)
    best = 1e9
    for _ in range(3):
        pl.plan_staged()
        pl.fetch(one)
        k = pl.kernel_ms()
        best = min(best, k[1] + k[2])
    times.append((best, i, i in failed))
times.sort(reverse=True)
print(f"{len(failed)} failed plans; sched+place ms of single plans (top 25):")
for t, i, f in times[:25]:
    print(f"  mixture {i:6d} rank4={i % 4} {'FAILED' if f else 'ok    '} {t:7.3f} ms")
fs = [t for t, i, f in times if f]
ok = [t for t, i, f in times if not f]
print(f"failed: mean {sum(fs) / max(len(fs), 1):.3f} ms max {max(fs, default=0):.3f}; "
      f"random ok: mean {sum(ok) / max(len(ok), 1):.3f} ms max {max(ok, default=0):.3f}")
for r in range(4):
    print(f"  rank {r} of 4: failed plans {sum(1 for i in failed if i % 4 == r)}, "
          f"sum of their ms {sum(t for t, i, f in times if f and i % 4 == r):.2f}")
