"""GPU: the baseline planners on the device against the
reference's plans and evaluations, bit-exact.  Run with -m gpu."""
import hashlib

import pytest

from conftest import build_set

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def planner():
    import paper_2409_03365_b200 as ws
    return ws.Planner(0)


def test_gpu_baselines_match_reference(planner, baseline_cases):
    ps, kept, _ = build_set(baseline_cases)
    ps.encode(pinned=True)
    res = planner.plan(ps)
    bad = [c["name"] for i, c in enumerate(kept) if ps.text(i, res.results, res.arena) != c["expected"]]
    assert not bad, bad[:10]
    sims = planner.simulate(ps, res)
    bad = [c["name"] for i, c in enumerate(kept) if ps.sim_text(i, res, sims) != c["sim_expected"]]
    assert not bad, bad[:10]


def test_gpu_baseline_full_sweep(planner, baseline_sweep_hashes):
    import paper_2409_03365_b200 as ws
    for strategy, hashes in baseline_sweep_hashes.items():
        n = len(hashes)
        ps = ws.ProblemSet()
        ps.add_sweep(0, n, strategy=strategy)
        ps.encode(pinned=True)
        res = planner.plan(ps)
        bad = [i for i in range(n)
               if hashlib.sha1(ps.text(i, res.results, res.arena).encode()).hexdigest()[:16] != hashes[i]]
        assert not bad, (strategy, bad[:20])
