"""GPU parity of strategy comparison and dynamic re-planning (SURVEY §8(f)
row 4): paper_2409_03365_b200.compare / .dynamic -- every (phase, strategy)
pair planned in one device batch and evaluated in one k_sim launch -- against
the reference's own cmd_compare / cmd_dynamic (cli.hpp:243-327): identical
printed text (or exception class + message) and byte-identical files
(compare.csv, every phase<p>.<strategy>.plan.txt, dynamic.csv, cumulative.csv),
including the partial output written before a mid-sequence error."""
from __future__ import annotations

import pytest

from cli_cases import load_cases, run_case

pytestmark = pytest.mark.gpu
CASES = load_cases()


def _run(cmd, i, t, o, **kw):
    import paper_2409_03365_b200 as ws
    try:
        return (ws.compare if cmd == "compare" else ws.dynamic)(i, t, o, **kw)
    except ws.PlannerError as e:
        return f"error {type(e).__name__}: {e}\n"


def test_commands_match_reference(tmp_path):
    bad = []
    for k, c in enumerate(CASES):
        printed, files = run_case(c, tmp_path / str(k), _run)
        if printed != c["printed"]:
            bad.append((c["name"], "printed", printed[:160], c["printed"][:160]))
        elif files != c["outputs"]:
            diff = sorted(n for n in set(files) | set(c["outputs"]) if files.get(n) != c["outputs"].get(n))
            bad.append((c["name"], "files", diff[:4]))
    assert not bad, bad[:6]


def test_plan_for_strategy_drop_in():
    import paper_2409_03365_b200 as ws
    import pyoracle as po  # noqa: F401  (oracle only as the checker)
    c = next(c for c in CASES if c["name"] == "compare/clip-like/4t/8d")
    w, t = c["inputs"]["w.txt"], c["inputs"]["t.txt"]
    for s in ("wavefront", "decoupled-sequential", "task-level-optimus", "distmm-mt"):
        assert ws.plan_for_strategy(s, w, t).startswith("# wavesched plan v1\nstrategy " + s)
    with pytest.raises(ws.ParseError, match="unknown strategy 'nope'"):
        ws.plan_for_strategy("nope", w, t)
