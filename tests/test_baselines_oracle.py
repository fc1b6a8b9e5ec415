"""CPU: the oracle's baseline planners (decoupled-sequential,
baselines.hpp:104-131) against the reference's own plans and evaluations
(tests/golden/baseline_cases.json.gz, baseline_sweep_hashes.txt.gz)."""
import hashlib

import pyoracle as po
from conftest import build_set


def test_oracle_baselines_match_reference(baseline_cases):
    ps, kept, failed = build_set(baseline_cases)
    for c, msg in failed:
        assert c["expected"].startswith("error"), (c["name"], msg)
    ps.encode()
    res = po.plan_batch(ps)
    bad = [c["name"] for i, c in enumerate(kept) if ps.text(i, res.results, res.arena) != c["expected"]]
    assert not bad, bad[:10]
    sims = po.simulate_batch(ps, res)
    bad = [c["name"] for i, c in enumerate(kept) if ps.sim_text(i, res, sims) != c["sim_expected"]]
    assert not bad, bad[:10]


def test_oracle_baseline_sweep_sample(baseline_sweep_hashes):
    import paper_2409_03365_b200 as ws
    for strategy, hashes in baseline_sweep_hashes.items():
        idx = list(range(0, len(hashes), 131))[:500]
        ps = ws.ProblemSet()
        for i in idx:
            ps.add_sweep(i, 1, strategy=strategy)
        ps.encode()
        res = po.plan_batch(ps)
        bad = [i for j, i in enumerate(idx)
               if hashlib.sha1(ps.text(j, res.results, res.arena).encode()).hexdigest()[:16] != hashes[i]]
        assert not bad, (strategy, bad[:10])
