# e2e (ws_plan_batch_host, 100k sweep) with/without the phase kernels
for ss in 1 0; do for es in 1 0; do
WSGPU_SCHED_SPLIT=$ss WSGPU_EMIT_SPLIT=$es python -c "
import sys,time; sys.path.insert(0,'.')
import torch, paper_2409_03365_b200 as ws
ps=ws.ProblemSet(); ps.add_sweep(0,100000); ps.encode(pinned=True); pl=ws.Planner(0); r=pl.plan(ps); r=pl.plan(ps,out=r)
best=1e9
for _ in range(6):
    torch.cuda.synchronize(); t0=time.perf_counter(); r=pl.plan(ps,out=r); best=min(best,time.perf_counter()-t0)
print('sched_split $ss emit_split $es', round(best*1e3,2), 'ms')
"
done; done
