"""Tuning aid: ws_plan_batch_host end-to-end time over the 100k sweep for
host-pipeline shapes ($WSGPU_HOST_CHUNKS x $WSGPU_HOST_STREAMS), each checked
record-for-record against the unchunked call."""
import ctypes as C
import hashlib
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: F401
import paper_2409_03365_b200 as ws

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
# "<chunks>x<streams>" or "w<weights>x<streams>", e.g. 3x2, w1,3,3,1x2
configs = [c.rsplit("x", 1) for c in (sys.argv[2:] or ["1x1", "2x1", "2x2", "3x2", "4x2", "6x2", "8x2"])]
ps = ws.ProblemSet()
ps.add_sweep(0, n)
ps.encode(pinned=True)


def digest(res) -> list[bytes]:
    base = C.addressof(res.arena)
    out = []
    for i in range(n):
        r = res.results[i]
        h = hashlib.sha1(C.string_at(C.addressof(r), C.sizeof(r) - 16))  # header minus offset/size
        if r.status == 0:
            h.update(C.string_at(base + r.offset, r.size))
        out.append(h.digest())
    return out


ref = None
for chunks, streams in configs:
    os.environ.pop("WSGPU_HOST_WEIGHTS", None)
    if chunks.startswith("w"):
        os.environ["WSGPU_HOST_WEIGHTS"] = chunks[1:]
    else:
        os.environ["WSGPU_HOST_CHUNKS"] = chunks
    os.environ["WSGPU_HOST_STREAMS"] = streams
    pl = ws.Planner(0)
    res = pl.plan(ps)
    res = pl.plan(ps, out=res)
    times = []
    for _ in range(20):
        t0 = time.perf_counter()
        res = pl.plan(ps, out=res)
        times.append(time.perf_counter() - t0)
    d = digest(res)
    ref = ref or d
    ts = sorted(times)
    ms = ts[len(ts) // 2] * 1e3
    bad = [i for i in range(n) if d[i] != ref[i]]
    print(f"chunks={chunks} streams={streams}: median {ms:7.2f} ms  min {ts[0] * 1e3:7.2f}  p90 {ts[int(0.9 * len(ts))] * 1e3:7.2f} ms  "
          f"{n / ms * 1e3 / 1e6:5.2f} M plans/s  records "
          f"{'identical' if not bad else f'DIFFER on {len(bad)} plans, first {bad[:5]}'}", flush=True)
    pl.close()
