"""Shared fixtures.  `-m "not gpu"` runs on CPU (oracle vs golden fixtures,
host logic, C-ABI exports, gloo multi-process); `-m gpu` runs the parity
tests of the CUDA planner on a B200."""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA planner parity tests)")


@pytest.fixture(scope="session")
def golden_cases():
    with gzip.open(GOLDEN / "cases.json.gz", "rt") as f:
        return json.load(f)


@pytest.fixture(scope="session")
def backtrack_cases():
    with gzip.open(GOLDEN / "backtrack_cases.json.gz", "rt") as f:
        return json.load(f)


@pytest.fixture(scope="session")
def sweep_hashes():
    with gzip.open(GOLDEN / "sweep_hashes.txt.gz", "rt") as f:
        return f.read().split()


def build_set(cases):
    """ProblemSet of the parseable cases; returns (set, kept cases, parse-failed cases)."""
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    kept, failed = [], []
    for c in cases:
        try:
            ps.add_text(c["workload"], c["topology"], **c["options"])
            kept.append(c)
        except ws.ParseError as e:
            failed.append((c, str(e)))
    return ps, kept, failed


@pytest.fixture(scope="session")
def sim_cases():
    with gzip.open(GOLDEN / "sim_cases.json.gz", "rt") as f:
        return json.load(f)


@pytest.fixture(scope="session")
def sim_sweep_hashes():
    with gzip.open(GOLDEN / "sim_sweep_hashes.txt.gz", "rt") as f:
        return f.read().split()


def sim_groups(cases):
    """Cases grouped by SimulatorOptions (one evaluation call per group)."""
    groups = {}
    for c in cases:
        groups.setdefault(tuple(sorted(c["sim"].items())), []).append(c)
    return [(dict(k), v) for k, v in groups.items()]


@pytest.fixture(scope="session")
def baseline_cases():
    with gzip.open(GOLDEN / "baseline_cases.json.gz", "rt") as f:
        return json.load(f)


@pytest.fixture(scope="session")
def baseline_sweep_hashes():
    """{strategy: [sha1[:16] of the reference plan text of sweep mixture i]}"""
    out = {}
    with gzip.open(GOLDEN / "baseline_sweep_hashes.txt.gz", "rt") as f:
        for line in f:
            name, *hashes = line.split()
            out[name] = hashes
    return out


@pytest.fixture(scope="session")
def plan_files():
    with gzip.open(GOLDEN / "plan_files.json.gz", "rt") as f:
        return json.load(f)


@pytest.fixture(scope="session")
def json_cases_fixture():
    with gzip.open(GOLDEN / "json_cases.json.gz", "rt") as f:
        return json.load(f)
