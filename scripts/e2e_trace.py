"""Host-side timing of the pipelined host call (WSGPU_TRACE=1 prints one line
per call on stderr): host prep, launch issue, end, device pipeline.
usage: WSGPU_TRACE=1 python scripts/e2e_trace.py [mixtures] [calls]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2409_03365_b200 as ws  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ps = ws.ProblemSet()
ps.add_sweep(0, n)
ps.encode(pinned=True)
pl = ws.Planner(0)
r = pl.plan(ps)
for _ in range(calls):
    r = pl.plan(ps, out=r)
