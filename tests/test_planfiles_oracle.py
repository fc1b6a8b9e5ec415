"""CPU: plan files of all four strategies written by the reference (SURVEY
§8(f) row 3): the host parse_plan round-trips them byte for byte, and the
evaluation oracle on the parsed plans equals the reference's
parse_plan + simulate_plan + validate_plan (tests/golden/plan_files.json.gz)."""
import pyoracle as po
from conftest import sim_groups


def test_parse_plan_round_trips_reference_files(plan_files):
    import paper_2409_03365_b200 as ws
    ps = ws.PlanSet()
    for c in plan_files:
        ps.add_text(c["plan"])
    # hand-edited broken files are not in canonical 17-digit form; the rest are write_plan output
    bad = [c["name"] for i, c in enumerate(plan_files) if "broken" not in c["name"] and ps.write(i) != c["plan"]]
    assert not bad, bad[:10]


def test_oracle_evaluates_plan_files_like_reference(plan_files):
    import paper_2409_03365_b200 as ws
    for sim, cases in sim_groups(plan_files):
        ps = ws.PlanSet()
        for c in cases:
            ps.add_text(c["plan"])
        sims = po.simulate_planset(ps, **sim)
        bad = [c["name"] for i, c in enumerate(cases) if ps.sim_text(i, sims) != c["expected"]]
        assert not bad, (sim, bad[:10])


def test_plan_files_cover_all_strategies_and_violations(plan_files):
    names = " ".join(c["name"] for c in plan_files)
    for s in ("wavefront/", "decoupled-sequential/", "task-level-optimus/", "distmm-mt/"):
        assert s in names
    text = "".join(c["expected"] for c in plan_files)
    for needle in ("exceeds capacity", "assigned twice", "recorded span", "layers", "unplaced", "capacity exceeded"):
        assert needle in text, needle


def test_parse_plan_errors_like_reference():
    import paper_2409_03365_b200 as ws
    ps = ws.PlanSet()
    for text, want in (("strategy x\n", "plan: incomplete topology"),
                       ("island 0: 0 1\nbw intra=2 inter=1\nmem 10\nend_time 1\n", "plan: missing strategy line"),
                       ("strategy x\nwave 0 start=0\n", "plan line 2: missing key 'dur'")):
        try:
            ps.add_text(text)
        except ws.ParseError as e:
            assert str(e) == want, (str(e), want)
        else:
            raise AssertionError("no ParseError for: " + text)
