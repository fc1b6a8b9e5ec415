"""GPU: clusters wider than 64 devices (up to WS_MAX_DEVICES = 256) -- the
DevMask<4> instances of k_sched / k_sched_scoped / k_place / k_sim -- against
the REFERENCE on 223 cases (tests/golden/make_wide_golden.py): QWen-VAL on 256
GPUs (the paper's planner-time table), all families at
96-256 devices, sequential placement, no backtracking, drop floor, the three
baselines (decoupled-sequential, distmm-mt, task-level-optimus), tight memory
(backtracking, PlacementInfeasible) and non-contiguous islands.  Byte-identical
plan text or error, and byte-identical evaluation (simulate_plan +
validate_plan) of the planned records and of the plans read back as plan
files."""
import gzip
import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def wide_cases():
    with gzip.open(GOLDEN / "wide_cases.json.gz", "rt") as f:
        return json.load(f)


def _set(cases):
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    for c in cases:
        opts = dict(c["options"])
        if c.get("strategy"):
            opts["strategy"] = c["strategy"]
        ps.add_text(c["workload"], c["topology"], **opts)
    ps.encode(pinned=True)
    return ps


def test_wide_clusters_match_reference(wide_cases):
    import paper_2409_03365_b200 as ws
    ps = _set(wide_cases)
    pl = ws.Planner(0)
    texts = pl.plan(ps).texts(ps)
    bad = [c["name"] for c, t in zip(wide_cases, texts) if t != c["expected"]]
    assert not bad, bad[:10]
    assert any(c["name"].startswith("wide/qwen-val-like/3t/256d") for c in wide_cases)


def test_wide_clusters_evaluate_like_reference(wide_cases):
    """k_sim<DevMask<4>> on the device-resident records of the wide plans."""
    import paper_2409_03365_b200 as ws
    ps = _set(wide_cases)
    pl = ws.Planner(0)
    res = pl.plan(ps)
    sims = pl.simulate(ps, res)
    bad = [c["name"] for i, c in enumerate(wide_cases) if ps.sim_text(i, res, sims) != c["sim_expected"]]
    assert not bad, bad[:10]
    assert any(c["name"].startswith("wide-distmm/") for c in wide_cases)
    assert any(c["name"].startswith("wide-optimus/") for c in wide_cases)


def test_wide_plan_files_evaluate_like_reference(wide_cases):
    """The reference's wide plans as plan files (parse_plan, ext device words)."""
    import paper_2409_03365_b200 as ws
    cases = [c for c in wide_cases if not c["expected"].startswith("error")]
    ps = ws.PlanSet()
    for c in cases:
        ps.add_text(c["expected"])
    sims = ws.Planner(0).simulate_plans(ps)
    bad = [c["name"] for i, c in enumerate(cases) if ps.sim_text(i, sims) != c["sim_expected"]]
    assert not bad, bad[:10]


def test_wide_and_narrow_plans_in_one_batch(wide_cases, golden_cases):
    """A batch mixing <= 64-device plans with wider ones runs the wide kernels
    for all of them: the narrow plans come out unchanged."""
    import paper_2409_03365_b200 as ws
    narrow = [c for c in golden_cases if c["name"].startswith(("config/", "suite/"))][:30]
    cases = narrow + wide_cases[:40]
    ps = ws.ProblemSet()
    for c in cases:
        opts = dict(c["options"])
        if c.get("strategy"):
            opts["strategy"] = c["strategy"]
        ps.add_text(c["workload"], c["topology"], **opts)
    ps.encode(pinned=True)
    pl = ws.Planner(0)
    res = pl.plan(ps)
    texts = res.texts(ps)
    bad = [c["name"] for c, t in zip(cases, texts) if t != c["expected"]]
    assert not bad, bad[:10]
    # evaluation of the mixed batch: the narrow records keep the narrow layout
    sims = pl.simulate(ps, res)
    bad = [c["name"] for i, c in enumerate(cases) if "sim_expected" in c and
           ps.sim_text(i, res, sims) != c["sim_expected"]]
    assert not bad, bad[:10]
    alone = _set(narrow)  # the narrow plans planned and evaluated by the u64 instances
    ares = pl.plan(alone)
    asims = pl.simulate(alone, ares)
    bad = [c["name"] for i, c in enumerate(narrow)
           if ps.sim_text(i, res, sims) != alone.sim_text(i, ares, asims)]
    assert not bad, bad[:10]


def test_wide_dropin_reference_256(wide_cases):
    """The drop-in (text form) on the paper's 256-GPU QWen-VAL plan."""
    import paper_2409_03365_b200 as ws
    c = next(c for c in wide_cases if c["name"] == "wide/qwen-val-like/3t/256d/s0")
    assert ws.plan_workload(c["workload"], c["topology"]) == c["expected"]
