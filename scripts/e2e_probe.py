"""Where the end-to-end time goes (tuning aid): H2D staging, device planning,
result fetch, and the zero-copy ws_plan_batch_host call, over the 100k sweep."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2409_03365_b200 as ws

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
ps = ws.ProblemSet()
ps.add_sweep(0, n)
ps.encode(pinned=True)
pl = ws.Planner(0)
res = pl.plan(ps)
res = pl.plan(ps, out=res)
dev = torch.device("cuda", 0)


def t(f, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


blob = torch.empty(ps.encoded_bytes, dtype=torch.uint8, device=dev)
host = torch.empty(ps.encoded_bytes, dtype=torch.uint8, pin_memory=True)
print(f"encoded bytes {ps.encoded_bytes/1e6:.1f} MB; arena used {res.arena_used.value/1e6:.1f} MB")
print(f"raw H2D pinned copy        {t(lambda: blob.copy_(host, non_blocking=True)):8.2f} ms")
dres = torch.empty(res.arena_used.value, dtype=torch.uint8, device=dev)
hres = torch.empty(res.arena_used.value, dtype=torch.uint8, pin_memory=True)
print(f"raw D2H pinned copy        {t(lambda: hres.copy_(dres, non_blocking=True)):8.2f} ms")
print(f"ws_stage_batch             {t(lambda: pl.stage(ps)):8.2f} ms")
print(f"ws_plan_staged             {t(lambda: pl.plan_staged()):8.2f} ms")
out = pl.fetch(ps)
print(f"ws_fetch_results           {t(lambda: pl.fetch(ps, out=out)):8.2f} ms")
print(f"stage+plan+fetch           {t(lambda: (pl.stage(ps), pl.plan_staged(), pl.fetch(ps, out=out))):8.2f} ms")
print(f"ws_plan_batch_host         {t(lambda: pl.plan(ps, out=res)):8.2f} ms  kernels {pl.kernel_ms()}")
