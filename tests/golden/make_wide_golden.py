"""Golden fixtures for clusters wider than 64 devices (up to WS_MAX_DEVICES =
256), generated from the REFERENCE planner (oracle/_ref/libwsref.so, build
container only).  The CPU oracle restatement keeps device sets in one u64
(<= 64 devices), so these cases pin the device planner to the reference
directly.  Writes wide_cases.json.gz: inputs + the reference outcome (plan
text or "error <Class>: <what>") and the reference's evaluation of that plan
(simulate_plan + validate_plan text, default simulation options; the same
text as the reference's evaluation of the plan read back as a plan file) for

  * the paper's QWen-VAL on 256 GPUs and the other
    BASELINE families at 96, 128, 192 and 256 devices, several seeds;
  * option variants: sequential placement, no backtracking, drop floor,
    the three baselines (plan_for_strategy: decoupled-sequential, distmm-mt,
    task-level-optimus);
  * tight memory (PlacementInfeasible / backtracking) and a hand-made
    topology with non-contiguous islands.

usage: python tests/golden/make_wide_golden.py
"""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent / "oracle"))
import pyoracle as po  # noqa: E402


def main() -> None:
    if not po.ref_available():
        raise SystemExit("oracle/_ref/libwsref.so missing: run `make -C oracle ref` (needs /root/reference)")
    cases = []

    def add(name, w, t, opts, strategy=None):
        expected = (po.ref_strategy_plan_text(w, t, strategy, **opts) if strategy
                    else po.ref_plan_text(w, t, **opts))
        so = dict(opts, strategy=strategy) if strategy else opts
        case = {"name": name, "workload": w, "topology": t, "options": opts, "strategy": strategy,
                "expected": expected, "sim_expected": po.ref_sim_text(w, t, {}, **so)}
        if not expected.startswith("error"):  # the plan read back as a plan file evaluates the same
            assert po.ref_sim_plan_text(expected) == case["sim_expected"], name
        cases.append(case)

    for fam, tasks in (("qwen-val-like", 3), ("clip-like", 4), ("clip-like", 10), ("clip-like", 16),
                       ("ofasys-like", 7), ("ofasys-like", 12)):
        for devices in (96, 128, 192, 256):
            for seed in (0, 1, 2):
                w, t = po.ref_scenario(fam, tasks, devices, seed)
                add(f"wide/{fam}/{tasks}t/{devices}d/s{seed}", w, t, {})
                if seed == 0:
                    add(f"wide-seq/{fam}/{tasks}t/{devices}d", w, t, {"sequential": 1})
                    add(f"wide-bt0/{fam}/{tasks}t/{devices}d", w, t, {"bt_depth": 0})
                    add(f"wide-drop/{fam}/{tasks}t/{devices}d", w, t, {"drop_floor": 0.05})
                    add(f"wide-decoupled/{fam}/{tasks}t/{devices}d", w, t, {}, "decoupled-sequential")
                    add(f"wide-distmm/{fam}/{tasks}t/{devices}d", w, t, {}, "distmm-mt")
                    add(f"wide-optimus/{fam}/{tasks}t/{devices}d", w, t, {}, "task-level-optimus")
    # tight memory: placement backtracking and PlacementInfeasible on wide clusters
    for fam, tasks in (("clip-like", 10), ("ofasys-like", 7)):
        w, t = po.ref_scenario(fam, tasks, 256, 0)
        for gib in (24, 40, 64):
            tt = "\n".join(l if not l.startswith("mem") else f"mem {gib * (1 << 30)}" for l in t.splitlines()) + "\n"
            add(f"wide-mem{gib}/{fam}/{tasks}t/256d", w, tt, {})
    # non-contiguous islands over 160 devices (shard_moves' unit-by-unit path)
    w, _ = po.ref_scenario("clip-like", 8, 160, 3)
    isl = [[d for d in range(160) if d % 5 == i] for i in range(5)]
    topo = "".join(f"island {i}: {' '.join(map(str, x))}\n" for i, x in enumerate(isl)) + \
           "bw intra=100000000000 inter=20000000000\nmem 85899345920\n"
    add("wide-noncontig/clip-like/8t/160d", w, topo, {})
    out = HERE / "wide_cases.json.gz"
    with gzip.open(out, "wt") as f:
        json.dump(cases, f)
    errs = sum(1 for c in cases if c["expected"].startswith("error"))
    print(f"{out.name}: {len(cases)} cases ({errs} reference errors)")


if __name__ == "__main__":
    main()
