"""GPU: the device plan evaluator k_sim (simulate_plan + validate_plan) through
the C-ABI against the reference's outputs and the CPU oracle, bit-exact.
Run with -m gpu."""
import hashlib

import pytest

import pyoracle as po
import records as rc
from conftest import sim_groups

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def planner():
    import paper_2409_03365_b200 as ws
    return ws.Planner(0)


def test_gpu_sim_matches_reference_cases(planner, sim_cases):
    """Host records path (ws_simulate_batch_host): GPU plans, the same edits,
    then the device evaluator; broken plans included."""
    for sim, cases in sim_groups(sim_cases):
        ps = rc.build_sim_set(cases)
        res = planner.plan(ps)
        rc.apply_edits(cases, ps, res)
        sims = planner.simulate(ps, res, **sim)
        texts = [ps.sim_text(i, res, sims) for i in range(len(cases))]
        bad = [c["name"] for c, t in zip(cases, texts) if t != c["expected"]]
        assert not bad, (sim, bad[:10])
        assert planner.sim_ms() > 0.0


def test_gpu_sim_staged_equals_oracle_records(planner):
    """Device-resident path (plan_staged -> simulate_staged): result structs and
    arena records equal the oracle's byte for byte (arena offsets aside)."""
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    ps.add_sweep(3000, 600)
    ps.encode(pinned=True)
    planner.stage(ps)
    planner.plan_staged()
    planner.simulate_staged()
    res = planner.fetch(ps)
    sims = planner.fetch_sim(ps)
    ref = po.simulate_batch(ps, po.plan_batch(ps))
    for i in range(len(ps)):
        a, b = sims.results[i], ref.results[i]
        for f, _ in type(a)._fields_:
            if f in ("offset", "size"):
                continue
            assert getattr(a, f) == getattr(b, f), (i, f)
        if a.status == 0:
            assert bytes(sims.arena[a.offset:a.offset + a.size]) == bytes(ref.arena[b.offset:b.offset + b.size]), i
    assert ps.sim_text(0, res, sims).startswith("sim makespan=")


def test_gpu_sim_full_sweep_100k_matches_reference(planner, sim_sweep_hashes):
    """Every mixture of BASELINE config 5 planned and evaluated on the device:
    the evaluation text hashes to the reference's simulate/validate output."""
    import paper_2409_03365_b200 as ws
    n = len(sim_sweep_hashes)
    assert n == 100000
    ps = ws.ProblemSet()
    ps.add_sweep(0, n)
    ps.encode(pinned=True)
    planner.stage(ps)
    planner.plan_staged()
    planner.simulate_staged()
    res = planner.fetch(ps)
    sims = planner.fetch_sim(ps)
    got = [hashlib.sha1(ps.sim_text(i, res, sims).encode()).hexdigest()[:16] for i in range(n)]
    mism = [i for i in range(n) if got[i] != sim_sweep_hashes[i]]
    assert not mism, mism[:20]
    # candidate selection by simulated makespan (ws_best_staged mode 2)
    key, idx = planner.best(mode=2)
    best = min((sims.results[i].makespan, i) for i in range(n) if sims.results[i].status == 0)
    assert (key, idx) == best
