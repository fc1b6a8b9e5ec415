"""Runs a tests/golden/cli_cases.json.gz case (compare / dynamic command,
SURVEY §8(f) row 4) in a scratch directory: writes its input files, calls
`run(command, input, topology, out_dir, **opts)` from inside that directory
and returns (printed text, {file name: text} written under out/)."""
from __future__ import annotations

import gzip
import json
import os
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


def load_cases() -> list[dict]:
    with gzip.open(GOLDEN / "cli_cases.json.gz", "rt") as f:
        return json.load(f)


def run_case(case: dict, tmp: Path, run) -> tuple[str, dict]:
    src = case.get("ours", case)  # JSON cases: our command reads the .json twins
    tmp.mkdir(parents=True, exist_ok=True)
    cwd = os.getcwd()
    os.chdir(tmp)
    try:
        for name, text in src["inputs"].items():
            Path(name).parent.mkdir(parents=True, exist_ok=True)
            Path(name).write_text(text)
        printed = run(case["command"], src["input"], src["topology"], "out", **case["opts"])
        out = Path("out")
        files = {p.name: p.read_text() for p in sorted(out.iterdir())} if out.exists() else {}
    finally:
        os.chdir(cwd)
    return printed, files
