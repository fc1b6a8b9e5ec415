"""Per-strategy device kernel times over the 100k sweep (tuning aid):
k_fit / k_sched(+scoped) / k_place(+retry) ms of ws_plan_staged for each strategy.
usage: python scripts/strategy_kernels.py [count]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_03365_b200 as ws  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
pl = ws.Planner(0)
for strategy in ws.STRATEGIES:
    ps = ws.ProblemSet()
    ps.add_sweep(0, n, strategy=strategy)
    ps.encode(pinned=True)
    pl.stage(ps)
    best = None
    for _ in range(4):
        pl.plan_staged()
        res = pl.fetch(ps)
        k = pl.kernel_ms()
        best = k if best is None or sum(k) < sum(best) else best
    fails = sum(1 for i in range(n) if res.results[i].status != 0)
    print(f"{strategy:22s} fit {best[0]:7.2f}  sched {best[1]:7.2f}  place {best[2]:7.2f} ms  "
          f"({n / sum(best) / 1e3:6.2f} M plans/s, {fails} failed)", flush=True)
