"""CPU: the plan-evaluation oracle (oracle/ws_sim_oracle.cpp, a restatement of
simulate_plan + validate_plan) against the reference's own outputs
(tests/golden/sim_cases.json.gz, sim_sweep_hashes.txt.gz), including broken
plans that exercise validate_plan's violation paths."""
import hashlib

import pyoracle as po
import records as rc
from conftest import sim_groups


def evaluate_with_oracle(cases, sim):
    ps = rc.build_sim_set(cases)
    res = po.plan_batch(ps)
    rc.apply_edits(cases, ps, res)
    sims = po.simulate_batch(ps, res, **sim)
    return [ps.sim_text(i, res, sims) for i in range(len(cases))]


def test_oracle_sim_matches_reference_cases(sim_cases):
    for sim, cases in sim_groups(sim_cases):
        texts = evaluate_with_oracle(cases, sim)
        bad = [c["name"] for c, t in zip(cases, texts) if t != c["expected"]]
        assert not bad, (sim, bad[:10])


def test_sim_cases_cover_every_violation_kind(sim_cases):
    text = "".join(c["expected"] for c in sim_cases)
    for needle in ("recorded span", "entry span exceeds wave duration", "allocations exceed device count",
                   "layers", "capacity exceeded", "overlapping execution intervals", "dependency", "unplaced",
                   "placed on", "assigned twice", "appears twice", "exceeds capacity"):
        assert needle in text, needle


def test_oracle_sim_sweep_sample_matches_reference(sim_sweep_hashes):
    import paper_2409_03365_b200 as ws
    idx = list(range(0, len(sim_sweep_hashes), 97))[:600]
    ps = ws.ProblemSet()
    for i in idx:
        ps.add_sweep(i, 1)
    ps.encode()
    res = po.plan_batch(ps)
    sims = po.simulate_batch(ps, res)
    bad = [i for j, i in enumerate(idx)
           if hashlib.sha1(ps.sim_text(j, res, sims).encode()).hexdigest()[:16] != sim_sweep_hashes[i]]
    assert not bad, bad[:10]
