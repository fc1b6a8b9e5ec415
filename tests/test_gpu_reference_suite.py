"""GPU: the reference's OWN test sources (unit tests under a Catch2 shim, and
the acceptance suite), compiled in place in the build container with every
plan_workload call redirected to the B200 planner (oracle/ref/gpu_prelude.hpp,
include/wsgpu/wavesched_compat.hpp).  Binaries travel in oracle/_ref/."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parent.parent / "oracle" / "_ref"


def _run(name, timeout):
    exe = REF / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (make -C oracle reftests needs the reference tree)")
    return subprocess.run([str(exe)], cwd=REF, capture_output=True, text=True, timeout=timeout)


def test_reference_unit_tests_pass_on_gpu_planner():
    r = _run("unit_gpu", 900)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "95 test cases, 0 failed" in r.stdout


def test_reference_acceptance_suite_passes_on_gpu_planner():
    r = _run("acceptance_gpu", 1200)
    assert r.returncode == 0, r.stdout[-3000:]
    assert r.stdout.count("[PASS] criterion") == 10


def test_dropin_reference_types_concurrent_threads_and_batch():
    """wavesched_gpu::plan_workload (reference types in, PlannerResult out) from
    many host threads at once and wavesched_gpu::plan_workloads (one batch,
    parallel decode) give the reference planner's plans (oracle/ref/dropin_bench.cpp
    checks the 4 BASELINE configs and every 97th sweep plan)."""
    import json
    exe = REF / "dropin_bench"
    if not exe.exists():
        pytest.skip(f"{exe} not built")
    r = subprocess.run([str(exe), "20", "3000", "8"], cwd=REF, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(v["identical_plan"] for v in d["latency_ms"].values())
    t = d["throughput"]
    assert t["batched_spot_mismatches"] == 0
    assert len(set(t["errors"])) == 1  # the same infeasible plans on every path
