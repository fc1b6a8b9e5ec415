# e2e of ws_plan_batch_host (100k sweep) for several chunk weightings (WSGPU_HOST_WEIGHTS)
for w in ${WEIGHTS:-1,3,3,1 1,4,4,2,1 1,2,2,1 1,3,1 1,5,5,1 1,3,3,3,1 2,3,3,2}; do
WSGPU_HOST_WEIGHTS=$w python -c "
import sys,time; sys.path.insert(0,'.')
import torch, paper_2409_03365_b200 as ws
ps=ws.ProblemSet(); ps.add_sweep(0,100000); ps.encode(pinned=True); pl=ws.Planner(0); r=pl.plan(ps); r=pl.plan(ps,out=r)
best=1e9
for _ in range(6):
    torch.cuda.synchronize(); t0=time.perf_counter(); r=pl.plan(ps,out=r); best=min(best,time.perf_counter()-t0)
print('weights $w', round(best*1e3,2), 'ms', 'pipeline', round(pl.kernel_ms()[2],2))
"
done
