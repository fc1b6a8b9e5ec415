"""GPU: candidate-plan search -- all 96 planner variants of a
workload planned in one device batch, best selected on the device by predicted
makespan, optimality gap or simulated makespan -- equals the oracle's selection
bit for bit (key and index)."""
from __future__ import annotations

import gzip
import json

import pytest

import pyoracle as po
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _workloads():
    with gzip.open(GOLDEN / "cli_cases.json.gz", "rt") as f:
        cases = json.load(f)
    out = [(c["name"], c["inputs"]["w.txt"], c["inputs"]["t.txt"]) for c in cases
           if c["command"] == "compare" and "w.txt" in c["inputs"] and "t.txt" in c["inputs"]]
    return out[:24]


def test_best_candidate_matches_oracle():
    import paper_2409_03365_b200 as ws
    from paper_2409_03365_b200 import candidates as cd
    planner = ws.Planner(0)
    bad = []
    for name, w, t in _workloads():
        ps = cd.candidate_set(w, t)
        for key in ("makespan", "gap", "simulated"):
            got = cd.best_candidate(planner, ps, key)
            want = po.best_candidate(ps, key)
            if got[1] != want[1] or (got[1] >= 0 and got[0] != want[0]):
                bad.append((name, key, got, want))
    assert not bad, bad[:5]


def test_sharded_search_single_rank():
    import paper_2409_03365_b200 as ws
    from paper_2409_03365_b200 import candidates as cd
    name, w, t = _workloads()[0]
    planner = ws.Planner(0)
    assert cd.best_candidate_sharded(planner, w, t, key="gap") == po.best_candidate(cd.candidate_set(w, t), "gap")
