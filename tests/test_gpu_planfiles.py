"""GPU: the device evaluator (k_sim) on reference-written plan files of all four
strategies, healthy and broken, equals the reference's parse_plan +
simulate_plan + validate_plan.  Run with -m gpu."""
import pytest

from conftest import sim_groups

pytestmark = pytest.mark.gpu


def test_gpu_evaluates_plan_files_like_reference(plan_files):
    import paper_2409_03365_b200 as ws
    planner = ws.Planner(0)
    for sim, cases in sim_groups(plan_files):
        ps = ws.PlanSet()
        for c in cases:
            ps.add_text(c["plan"])
        sims = planner.simulate_plans(ps, **sim)
        bad = [c["name"] for i, c in enumerate(cases) if ps.sim_text(i, sims) != c["expected"]]
        assert not bad, (sim, bad[:10])
        assert planner.sim_ms() > 0.0
