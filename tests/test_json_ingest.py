"""CPU: JSON ingestion (workload_from_json /
topology_from_json, cli.hpp:46-110): JSON workloads plan (on the oracle)
exactly like their text twins through the reference, and malformed JSON gives
the reference's error text (tests/golden/json_cases.json.gz)."""
import pyoracle as po


def test_json_cases(json_cases_fixture):
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    kept = []
    for c in json_cases_fixture:
        try:
            ps.add_json(c["workload"], c["topology"], **c["options"])
            kept.append(c)
        except ws.ParseError as e:
            assert c["expected"] == f"error Parse: {e}\n", (c["name"], str(e))
    assert len(kept) >= 600
    ps.encode()
    res = po.plan_batch(ps)
    bad = [c["name"] for i, c in enumerate(kept) if ps.text(i, res.results, res.arena) != c["expected"]]
    assert not bad, bad[:10]
    assert sum(not c["expected"].startswith("error") for c in kept) >= 500
