"""Generate the committed plan-file fixtures (the plan
format either side of the evaluator) from the REFERENCE itself: plan files of
all four strategies written by the reference (plan_for_strategy + write_plan,
cli.hpp:163-171, plan_io.hpp:53-110), some edited into broken plans, and the
reference's parse_plan + simulate_plan + validate_plan evaluation text of each.
Build container only (oracle/_ref/libwsref.so).  Writes plan_files.json.gz.

usage: python tests/golden/make_planfile_golden.py
"""
from __future__ import annotations

import gzip
import json
import random
import re
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(HERE))
import pyoracle as po  # noqa: E402
from make_golden import CONFIGS, SUITE  # noqa: E402

STRATEGIES = ["wavefront", "decoupled-sequential", "task-level-optimus", "distmm-mt"]


def broken(text: str, kind: str, rng: random.Random) -> str | None:
    lines = text.splitlines(keepends=True)
    if kind == "memory":  # a capacity below the placed peak
        m = re.search(r"^mem (\d+)$", text, re.M)
        return re.sub(r"^mem \d+$", f"mem {int(m.group(1)) // 5}", text, flags=re.M) if m else None
    if kind == "clash":  # second entry of a wave takes the first entry's first device
        for i, ln in enumerate(lines):
            if ln.startswith("wave ") and i + 2 < len(lines) and lines[i + 1].startswith("entry") \
                    and lines[i + 2].startswith("entry") and "devices=" in lines[i + 1] and "devices=" in lines[i + 2]:
                d0 = lines[i + 1].split("devices=")[1].split(",")[0].strip()
                head, devs = lines[i + 2].rstrip("\n").split("devices=")
                rest = devs.split(",")[1:]
                if str(d0) in rest:
                    continue
                lines[i + 2] = head + "devices=" + ",".join([d0] + rest) + "\n"
                return "".join(lines)
        return None
    if kind == "span":  # a recorded span that disagrees with the curve
        idx = [i for i, ln in enumerate(lines) if ln.startswith("entry")]
        i = rng.choice(idx)
        lines[i] = re.sub(r" dur=([0-9.e+-]+)", lambda m: f" dur={float(m.group(1)) * 1.25!r}", lines[i], count=1)
        return "".join(lines)
    if kind == "layers":  # one layer too many for an entity
        idx = [i for i, ln in enumerate(lines) if ln.startswith("entry")]
        i = rng.choice(idx)
        lines[i] = re.sub(r" l=(\d+)", lambda m: f" l={int(m.group(1)) + 1}", lines[i], count=1)
        return "".join(lines)
    if kind == "unplaced":  # an entry loses its device list
        idx = [i for i, ln in enumerate(lines) if ln.startswith("entry") and "devices=" in ln]
        if not idx:
            return None
        i = rng.choice(idx)
        lines[i] = lines[i].split(" devices=")[0] + "\n"
        return "".join(lines)
    if kind == "start":  # a later wave moved onto the first wave's start
        idx = [i for i, ln in enumerate(lines) if ln.startswith("wave ")]
        if len(idx) < 2:
            return None
        s0 = re.search(r" start=(\S+)", lines[idx[0]]).group(1)
        i = rng.choice(idx[1:])
        lines[i] = re.sub(r" start=\S+", f" start={s0}", lines[i], count=1)
        return "".join(lines)
    raise ValueError(kind)


def main() -> None:
    if not po.ref_available():
        raise SystemExit("oracle/_ref/libwsref.so missing: run `make -C oracle ref` (needs /root/reference)")
    rng = random.Random(2409)
    inputs = []
    for n, t, d in CONFIGS + SUITE:
        inputs.append((f"scenario/{n}/{t}t/{d}d", *po.ref_scenario(n, t, d, 0)))
    fam, devs = ("clip-like", "ofasys-like", "qwen-val-like"), (8, 16, 32, 64)
    for i in range(0, 100000, 997):
        inputs.append((f"sweep/{i}", *po.ref_scenario(fam[i % 3], 2 + (i // 3) % 15, devs[(i // 45) % 4], i)))
    for i, (w, t) in enumerate(po.ref_fuzz(60)):
        inputs.append((f"fuzz/{i}", w, t))
    cases = []
    kinds = ["memory", "clash", "span", "layers", "unplaced", "start"]
    for name, w, t in inputs:
        for s in STRATEGIES:
            text = po.ref_strategy_plan_text(w, t, s)
            if text.startswith("error"):
                continue
            cases.append({"name": f"{s}/{name}", "plan": text, "sim": {}, "expected": po.ref_sim_plan_text(text)})
            if rng.random() < 0.3:
                kind = kinds[len(cases) % len(kinds)]
                bad = broken(text, kind, rng)
                if bad is not None:
                    cases.append({"name": f"{s}/{name}/broken-{kind}", "plan": bad, "sim": {},
                                  "expected": po.ref_sim_plan_text(bad)})
    for s in STRATEGIES:  # SimulatorOptions variants on one plan per strategy
        w, t = po.ref_scenario("ofasys-like", 7, 32, 0)
        text = po.ref_strategy_plan_text(w, t, s)
        for sim in ({"zero_volumes": True}, {"skip_sync": True}, {"backward_ratio": 3.0}):
            cases.append({"name": f"{s}/ofasys/sim{sorted(sim)}", "plan": text, "sim": sim,
                          "expected": po.ref_sim_plan_text(text, **sim)})
    with gzip.open(HERE / "plan_files.json.gz", "wt") as f:
        json.dump(cases, f)
    print(f"{len(cases)} plan files; {sum(c['name'].count('broken') for c in cases)} broken; "
          f"{sum('valid 0 ' in c['expected'] for c in cases)} with violations")


if __name__ == "__main__":
    main()
