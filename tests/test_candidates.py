"""CPU: the candidate-plan search of one workload (SURVEY §8(e),
paper_2409_03365_b200.candidates): the fixed variant grid, and the oracle's
selection rule against the reference planner itself (when oracle/_ref is built)."""
from __future__ import annotations

import pytest

import pyoracle as po


def test_variant_grid():
    from paper_2409_03365_b200 import candidates as cd, make_options
    v = cd.candidate_variants()
    assert len(v) == 96
    assert len({tuple(sorted(x.items())) for x in v}) == 96
    d = make_options()  # reference PlannerOptions defaults (planner.hpp:21-27)
    x = v[56]
    assert (x["bt_depth"], x["bt_branching"], x["sequential"], x["eps"], x["drop_floor"]) == \
        (d.bt_depth, d.bt_branching, d.sequential, d.eps, d.drop_floor)


@pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("cfg", [("clip-like", 4, 8), ("clip-like", 10, 64), ("ofasys-like", 7, 32),
                                 ("qwen-val-like", 3, 64)])
def test_oracle_selection_matches_reference(cfg):
    from paper_2409_03365_b200 import candidates as cd
    w, t = po.ref_scenario(*cfg, 0)
    v = cd.candidate_variants()
    _, ref_best = po.ref_candidates_ms(w, t, v, 4)
    key, idx = po.best_candidate(cd.candidate_set(w, t, v, pinned=False), "makespan")
    assert idx == ref_best
