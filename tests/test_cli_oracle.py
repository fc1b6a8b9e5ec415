"""CPU tests of the strategy-comparison / dynamic re-planning path (SURVEY
§8(f) row 4, cli.hpp:237-327): the oracle restatement (oracle/pycli.py) against
the reference's own commands (tests/golden/cli_cases.json.gz), and the
product's command parsing through the C-ABI for every case that fails before
any planning (no GPU needed)."""
from __future__ import annotations

import pytest

from cli_cases import load_cases, run_case

CASES = load_cases()


def test_fixture_shape():
    kinds = {c["command"] for c in CASES}
    assert kinds == {"compare", "dynamic"}
    assert sum(1 for c in CASES if c["printed"].startswith("error PlacementInfeasible")) >= 3
    assert any(c["outputs"] and c["printed"].startswith("error ") for c in CASES)  # partial output before an error
    assert any("ours" in c for c in CASES)  # JSON inputs


def test_oracle_matches_reference_commands(tmp_path):
    import pycli
    bad = []
    for k, c in enumerate(CASES):
        printed, files = run_case(c, tmp_path / str(k), lambda cmd, i, t, o, **kw: pycli.oracle_cmd(cmd, i, t, o, **kw))
        if printed != c["printed"] or files != c["outputs"]:
            bad.append((c["name"], printed[:120], c["printed"][:120]))
    assert not bad, bad[:5]


EARLY = [c for c in CASES if c["printed"].startswith("error ParseError") and not c["outputs"]
         and "/error/" in c["name"]]


@pytest.mark.parametrize("case", EARLY, ids=[c["name"] for c in EARLY])
def test_early_errors_through_the_abi(case, tmp_path):
    """Load/sequence errors raise before the device is touched: same class and message."""
    import paper_2409_03365_b200 as ws

    def run(cmd, i, t, o, **kw):
        try:
            return (ws.compare if cmd == "compare" else ws.dynamic)(i, t, o, **kw)
        except ws.PlannerError as e:
            return f"error {type(e).__name__}: {e}\n"

    printed, files = run_case(case, tmp_path, run)
    assert printed == case["printed"]
    assert files == case["outputs"]


def test_abi_exports_commands():
    import paper_2409_03365_b200 as ws
    for name in ("wsx_cmd_compare", "wsx_cmd_dynamic", "wsx_plan_strategy_text"):
        assert hasattr(ws.lib, name)
