"""GPU: the C-ABI multi-GPU entry points (ws_abi.h) from a C++ host with no
torch: ws_plan_batch_multi (one process, one context per GPU) and ws_best_nccl
(one rank per GPU, 16-byte min-loc over NCCL), checked against the
single-context call record for record (tests/native/multi_gpu.cpp).  On a
one-GPU box the batch is sharded over two contexts of device 0 and the NCCL
communicator has one rank."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2409_03365_b200" / "lib"


def test_multi_context_batch_and_nccl_minloc(tmp_path):
    exe = tmp_path / "multi_gpu"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
                    "-o", str(exe), str(ROOT / "tests" / "native" / "multi_gpu.cpp"), "-L", str(LIB), "-lwsgpu",
                    f"-Wl,-rpath,{LIB}", "-L/usr/local/cuda/lib64", "-lcudart", "-lnccl", "-lpthread"],
                   check=True, capture_output=True)
    r = subprocess.run([str(exe), "20000"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 mismatches" in r.stdout
    assert "all ranks agree" in r.stdout


def test_python_plan_batch_multi_matches_single():
    """The Python binding of ws_plan_batch_multi (two planners on cuda:0, or one
    per GPU) gives the single planner's plan texts; ws_best_host = k_best."""
    import torch

    import paper_2409_03365_b200 as ws
    n_gpu = max(1, torch.cuda.device_count())
    planners = [ws.Planner(i % n_gpu) for i in range(max(2, n_gpu))]
    ps = ws.ProblemSet()
    ps.add_sweep(0, 9000)
    ps.encode(pinned=True)
    single = planners[0].plan(ps)
    texts = single.texts(ps)
    multi = ws.plan_batch_multi(planners, ps)
    assert multi.texts(ps) == texts
    planners[0].stage(ps)
    planners[0].plan_staged()
    assert ws.best_host(multi, len(ps), 0) == planners[0].best(0)
