"""GPU: JSON-ingested problems (workload_from_json / topology_from_json) planned
on the device equal the reference outcomes of their text twins.  Run with -m gpu."""
import pytest

pytestmark = pytest.mark.gpu


def test_gpu_json_cases(json_cases_fixture):
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    kept = []
    for c in json_cases_fixture:
        try:
            ps.add_json(c["workload"], c["topology"], **c["options"])
            kept.append(c)
        except ws.ParseError:
            pass
    ps.encode(pinned=True)
    res = ws.Planner(0).plan(ps)
    bad = [c["name"] for i, c in enumerate(kept) if ps.text(i, res.results, res.arena) != c["expected"]]
    assert not bad, bad[:10]
