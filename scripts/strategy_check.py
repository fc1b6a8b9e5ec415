"""GPU vs CPU oracle on a sweep sample for every planning strategy (dev aid):
plan text and evaluation text must be identical.
usage: python scripts/strategy_check.py [count]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import paper_2409_03365_b200 as ws  # noqa: E402
import pyoracle as po  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
pl = ws.Planner(0)
for strategy in ws.STRATEGIES:
    for seq in (0, 1):
        ps = ws.ProblemSet()
        ps.add_sweep(0, n, strategy=strategy, sequential=seq)
        ps.encode(pinned=True)
        res = pl.plan(ps)
        ores = po.plan_batch(ps)
        badp = [i for i in range(n) if ps.text(i, res.results, res.arena) != ps.text(i, ores.results, ores.arena)]
        sims = pl.simulate(ps, res)
        osims = po.simulate_batch(ps, ores)
        bads = [i for i in range(n) if ps.sim_text(i, res, sims) != ps.sim_text(i, ores, osims)]
        fails = sum(1 for i in range(n) if res.results[i].status != 0)
        print(f"{strategy:22s} seq={seq}: plan mismatches {len(badp)} {badp[:5]}, sim mismatches {len(bads)}, "
              f"failed plans {fails}", flush=True)
        if badp:
            i = badp[0]
            a, b = ps.text(i, res.results, res.arena), ps.text(i, ores.results, ores.arena)
            for x, y in zip(a.splitlines(), b.splitlines()):
                if x != y:
                    print("  gpu:", x[:200])
                    print("  cpu:", y[:200])
                    break
