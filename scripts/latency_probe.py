"""Tuning aid: where single-plan latency goes for the BASELINE configs --
device kernel ms (k_fit / k_sched / k_place) vs the host-call wall time."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_03365_b200 as ws  # noqa: E402

pl = ws.Planner(0)
for fam, t, d in (("clip-like", 4, 8), ("clip-like", 10, 64), ("ofasys-like", 7, 32), ("qwen-val-like", 3, 64)):
    one = ws.ProblemSet()
    one.add_scenario(fam, t, d, 0)
    one.encode(pinned=True)
    ro = None
    for _ in range(20):
        ro = pl.plan(one, out=ro)
    wall = []
    for _ in range(200):
        t0 = time.perf_counter()
        ro = pl.plan(one, out=ro)
        wall.append((time.perf_counter() - t0) * 1e3)
    pl.stage(one)
    ks = []
    for _ in range(50):
        pl.plan_staged()
        pl.fetch(one)
        ks.append(pl.kernel_ms())
    k = [statistics.median(x[i] for x in ks) for i in range(3)]
    print(f"{fam} {t}t/{d}d: host call {statistics.median(wall):.3f} ms; kernels fit {k[0]:.3f} sched {k[1]:.3f} "
          f"place(+retry) {k[2]:.3f} ms; launches {pl.launch_count}", flush=True)
