"""Dev aid: plan the 100k sweep through ws_plan_batch_host on a FRESH context
(first-call buffer state) and again, and compare every plan's text hash with
the reference hashes (tests/golden/sweep_hashes.txt.gz)."""
import gzip
import hashlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2409_03365_b200 as ws  # noqa: E402

hashes = gzip.open(ROOT / "tests" / "golden" / "sweep_hashes.txt.gz", "rt").read().split()
pl = ws.Planner(0)
ps = ws.ProblemSet()
ps.add_sweep(0, len(hashes))
ps.encode(pinned=True)
for tag in ("fresh", "again"):
    res = pl.plan(ps)
    bad = [i for i in range(len(hashes))
           if hashlib.sha1(ps.text(i, res.results, res.arena).encode()).hexdigest()[:16] != hashes[i]]
    print(tag, len(bad), bad[:8], flush=True)
