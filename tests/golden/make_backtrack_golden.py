"""Golden fixtures for the placement DFS (placement.hpp:409-441) under
non-default backtracking options, generated from the REFERENCE planner
(oracle/_ref/libwsref.so, build container only).

The sweep mixtures whose placement backtracks the most (found with the CPU
restatement: most scored entries, mostly PlacementInfeasible) planned with
several (backtrack_depth, backtrack_branching) pairs, so the device DFS -- its
attempt budget, step-backs and the attempt memo that skips repeated variants
 -- is pinned outside the default depth 2 / branching 3.
Writes backtrack_cases.json.gz: inputs + the reference outcome (plan text or
"error <Class>: <what>").

usage: python tests/golden/make_backtrack_golden.py
"""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent / "oracle"))
import pyoracle as po  # noqa: E402

# the heaviest backtracking sweep mixtures (scored entries with the default options)
MIXTURES = [37617, 13857, 70359, 20331, 7914, 58308, 534, 9177, 6297, 11682, 11151, 10245, 7713, 28335,
            33642, 48774, 44985, 38943, 85218, 90174, 92334, 98271, 55434, 53988, 61377, 62277, 63894, 86931]
OPTIONS = [{}, {"bt_depth": 1, "bt_branching": 2}, {"bt_depth": 3, "bt_branching": 2},
           {"bt_depth": 2, "bt_branching": 5}, {"bt_depth": 4, "bt_branching": 3},
           {"bt_depth": 1, "bt_branching": 8}, {"bt_depth": 0}, {"bt_depth": 2, "bt_branching": 1}]


def sweep_inputs(i: int) -> tuple[str, str]:
    """Sweep mixture i as reference text inputs."""
    fam = ("clip-like", "ofasys-like", "qwen-val-like")[i % 3]
    return po.ref_scenario(fam, 2 + (i // 3) % 15, (8, 16, 32, 64)[(i // 45) % 4], i)


def main() -> None:
    if not po.ref_available():
        raise SystemExit("oracle/_ref/libwsref.so missing: run `make -C oracle ref` (needs /root/reference)")
    cases = []
    for i in MIXTURES:
        w, t = sweep_inputs(i)
        if i == MIXTURES[0]:  # the inputs are the sweep's: default options reproduce its plan
            assert po.ref_plan_text(w, t) == po.ref_sweep_plan(i)
        for o in OPTIONS:
            cases.append({"name": f"bt/{i}/" + ",".join(f"{k}={v}" for k, v in o.items()), "workload": w,
                          "topology": t, "options": o, "expected": po.ref_plan_text(w, t, **o)})
    out = HERE / "backtrack_cases.json.gz"
    with gzip.open(out, "wt") as f:
        json.dump(cases, f)
    errs = sum(1 for c in cases if c["expected"].startswith("error"))
    print(f"{out.name}: {len(cases)} cases ({errs} reference errors)")


if __name__ == "__main__":
    main()
