"""Generate the committed fixtures for strategy comparison and dynamic
re-planning from the REFERENCE itself: its own
cmd_compare / cmd_dynamic (cli.hpp:243-327) run on input files in a scratch
directory, recording what each prints (or the exception run_command maps to an
exit code) and every file it writes (compare.csv; phase<p>.<strategy>.plan.txt,
dynamic.csv, cumulative.csv).  JSON inputs (".json" paths, cli.hpp:117-130) are
anchored on their text twins as in make_json_golden.py: the reference's own
JSON reader drops truth/profiles (it iterates items() of a destroyed
temporary), so the reference runs the twin .txt files and the case's "ours"
block names the .json files the builder's command reads instead.  Build container only (oracle/_ref/libwsref.so).
Writes cli_cases.json.gz.

usage: python tests/golden/make_cli_golden.py
"""
from __future__ import annotations

import gzip
import json
import os
import random
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(HERE))
import pyoracle as po  # noqa: E402
from make_golden import CONFIGS, SUITE  # noqa: E402
from make_json_golden import text_twin, topology_json, workload_json  # noqa: E402


def run_case(case: dict) -> dict:
    """Runs the reference command on the case's input files; fills printed/outputs."""
    with tempfile.TemporaryDirectory() as d:
        cwd = os.getcwd()
        os.chdir(d)
        try:
            for name, text in case["inputs"].items():
                Path(name).parent.mkdir(parents=True, exist_ok=True)
                Path(name).write_text(text)
            o = case["opts"]
            case["printed"] = po.ref_cmd(case["command"], case["input"], case["topology"], "out",
                                         eps=o.get("eps", 1e-7), bt_depth=o.get("bt_depth", 2),
                                         seed=o.get("synth_seed", 0))
            out = Path("out")
            case["outputs"] = {p.name: p.read_text() for p in sorted(out.iterdir())} if out.exists() else {}
        finally:
            os.chdir(cwd)
    return case


def compare_case(name: str, workload: str, topology: str, opts: dict | None = None, wname: str = "w.txt",
                 tname: str = "t.txt") -> dict:
    return {"name": name, "command": "compare", "inputs": {wname: workload, tname: topology}, "input": wname,
            "topology": tname, "opts": opts or {}}


def dynamic_case(name: str, phases: list[tuple[str, str | None, int | None]], topology: str,
                 opts: dict | None = None, extra_lines: str = "", sequence: str | None = None) -> dict:
    """phases: (file name, workload text or None = missing file, iters or None = default)."""
    inputs = {"topo.txt": topology}
    lines = ["# dynamic sequence", ""]
    for fname, text, iters in phases:
        if text is not None:
            inputs[fname] = text
        lines.append(f"phase workload={fname}" + (f" iters={iters}" if iters is not None else ""))
    seq = sequence if sequence is not None else "\n".join(lines) + "\n" + extra_lines
    inputs["seq.txt"] = seq
    return {"name": name, "command": "dynamic", "inputs": inputs, "input": "seq.txt", "topology": "topo.txt",
            "opts": opts or {}}


def main() -> None:
    if not po.ref_available():
        raise SystemExit("oracle/_ref/libwsref.so missing: run `make -C oracle ref` (needs /root/reference)")
    rng = random.Random(3365)
    cases = []
    # ---- compare: the BASELINE configs, the bundled suite, fuzz and sweep workloads
    for n, t, d in CONFIGS:
        w, tp = po.ref_scenario(n, t, d, 0)
        cases.append(compare_case(f"compare/{n}/{t}t/{d}d", w, tp))
        cases.append(compare_case(f"compare/{n}/{t}t/{d}d/bt0", w, tp, {"bt_depth": 0}))
        cases.append(compare_case(f"compare/{n}/{t}t/{d}d/eps", w, tp, {"eps": 1e-9}))
    for n, t, d in SUITE:
        w, tp = po.ref_scenario(n, t, d, 0)
        cases.append(compare_case(f"compare/suite/{n}/{t}t/{d}d", w, tp))
    for k, (w, tp) in enumerate(po.ref_fuzz(60)[::2]):
        cases.append(compare_case(f"compare/fuzz/{2 * k}", w, tp))
    infeasible = []
    for i in rng.sample(range(100000), 40) + [7291, 13873, 26731]:
        w, tp = po.ref_sweep_workload(i)
        cases.append(compare_case(f"compare/sweep/{i}", w, tp))
    # sweep mixtures whose wavefront plan is PlacementInfeasible (error path)
    with gzip.open(HERE / "cases.json.gz", "rt") as f:
        for c in json.load(f):
            if c["expected"].startswith("error PlacementInfeasible") and not c["options"] and \
                    len(infeasible) < 3:
                infeasible.append(c)
                cases.append(compare_case(f"compare/infeasible/{c['name']}", c["workload"], c["topology"]))
    # JSON inputs (cli.hpp:117-130: ".json" paths load through the JSON readers)
    for n, t, d in CONFIGS[:3]:
        w, tp = po.ref_scenario(n, t, d, 0)
        c = compare_case(f"compare/json/{n}/{t}t/{d}d", text_twin(w), tp)
        c["ours"] = {"inputs": {"w.json": workload_json(w), "t.json": topology_json(tp)}, "input": "w.json",
                     "topology": "t.json"}
        cases.append(c)
    # errors: missing files, unparsable workload
    w, tp = po.ref_scenario("clip-like", 4, 8, 0)
    c = compare_case("compare/error/missing-workload", w, tp)
    c["input"] = "nope.txt"
    cases.append(c)
    c = compare_case("compare/error/missing-topology", w, tp)
    c["topology"] = "nope.txt"
    cases.append(c)
    cases.append(compare_case("compare/error/bad-workload", w.replace("module ", "modul ", 1), tp))

    # ---- dynamic re-planning: phase sequences over one topology
    for fam, d, counts in (("clip-like", 8, (2, 4, 6, 8)), ("clip-like", 64, (4, 10, 16)),
                           ("ofasys-like", 32, (3, 7, 5)), ("qwen-val-like", 16, (2, 3)),
                           ("ofasys-like", 16, (2, 9, 4, 12, 6))):
        phases, topo = [], None
        for p, t in enumerate(counts):
            w, tp = po.ref_scenario(fam, t, d, p)
            topo = topo or tp
            phases.append((f"p{p}.txt", w, rng.choice([None, 1, 10, 250, 1000])))
        cases.append(dynamic_case(f"dynamic/{fam}/{d}d/{len(counts)}", phases, topo))
        cases.append(dynamic_case(f"dynamic/{fam}/{d}d/{len(counts)}/bt0", phases, topo, {"bt_depth": 0}))
    # mixed families on one cluster, repeated phases, a JSON phase
    mixed, topo = [], None
    for p, (fam, t) in enumerate((("clip-like", 4), ("ofasys-like", 7), ("qwen-val-like", 3), ("clip-like", 4))):
        w, tp = po.ref_scenario(fam, t, 32, 0)
        topo = topo or tp
        mixed.append((f"wl/{fam}-{t}.txt", w, 5 * (p + 1)))
    cases.append(dynamic_case("dynamic/mixed/32d", mixed, topo))
    for k in range(12):  # random sweep-shaped sequences at a fixed device count
        d = rng.choice([8, 16, 32, 64])
        phases, topo = [], None
        for p in range(rng.randint(1, 5)):
            fam = rng.choice(["clip-like", "ofasys-like", "qwen-val-like"])
            w, tp = po.ref_scenario(fam, rng.randint(2, 16), d, rng.randrange(1 << 30))
            topo = topo or tp
            phases.append((f"phase{p}.txt", w, rng.randint(1, 500)))
        cases.append(dynamic_case(f"dynamic/random/{k}", phases, topo))
    w1, tp = po.ref_scenario("clip-like", 4, 8, 0)
    w2, _ = po.ref_scenario("qwen-val-like", 3, 8, 1)
    w3, _ = po.ref_scenario("ofasys-like", 5, 8, 2)
    c = dynamic_case("dynamic/json", [("a.txt", text_twin(w1), 3), ("b.txt", w2, 2), ("c.txt", text_twin(w3), 1)],
                     tp)
    ours = dict(c["inputs"])
    del ours["a.txt"], ours["c.txt"]
    ours["a.json"], ours["c.json"] = workload_json(w1), workload_json(w3)
    ours["seq.txt"] = c["inputs"]["seq.txt"].replace("a.txt", "a.json").replace("c.txt", "c.json")
    c["ours"] = {"inputs": ours, "input": "seq.txt", "topology": "topo.txt"}
    cases.append(c)
    # infeasible phase in the middle (wavefront raises PlacementInfeasible after phase 0's files)
    if infeasible:
        c0 = infeasible[0]
        d = c0["topology"]
        cases.append(dynamic_case("dynamic/error/infeasible-phase",
                                  [("ok.txt", None, 1), ("bad.txt", c0["workload"], 2)], d))
        # phase 0 (filled in below) is a feasible workload on the same topology
    # sequence errors
    w, tp = po.ref_scenario("clip-like", 4, 8, 0)
    cases.append(dynamic_case("dynamic/error/missing-phase-file",
                              [("a.txt", w, 2), ("b.txt", w, 3), ("gone.txt", None, 1)], tp))
    cases.append(dynamic_case("dynamic/error/first-phase-missing", [("gone.txt", None, 1)], tp))
    cases.append(dynamic_case("dynamic/error/empty", [], tp, sequence="# nothing\n\n"))
    cases.append(dynamic_case("dynamic/error/bad-keyword", [("a.txt", w, 1)], tp,
                              sequence="phase workload=a.txt\nphaze workload=a.txt\n"))
    cases.append(dynamic_case("dynamic/error/missing-key", [("a.txt", w, 1)], tp, sequence="phase iters=3\n"))
    cases.append(dynamic_case("dynamic/error/not-kv", [("a.txt", w, 1)], tp, sequence="phase workload=a.txt 7\n"))
    cases.append(dynamic_case("dynamic/error/bad-iters", [("a.txt", w, 1)], tp,
                              sequence="phase workload=a.txt iters=lots\n"))
    cases.append(dynamic_case("dynamic/error/bad-phase-workload", [("a.txt", w, 1),
                                                                   ("b.txt", w.replace("task ", "tusk ", 1), 1)], tp))
    c = dynamic_case("dynamic/error/missing-topology", [("a.txt", w, 1)], tp)
    c["topology"] = "nope.txt"
    cases.append(c)
    c = dynamic_case("dynamic/error/missing-sequence", [("a.txt", w, 1)], tp)
    c["input"] = "nope.txt"
    cases.append(c)

    # the infeasible-phase case needs a feasible phase 0 on the infeasible mixture's topology
    for c in cases:
        if c["name"] == "dynamic/error/infeasible-phase":
            topo_text = c["inputs"]["topo.txt"]
            feasible = None
            for cand in (po.ref_scenario(f, t, n, 0) for f in ("clip-like", "qwen-val-like", "ofasys-like")
                         for t in (2, 3, 4) for n in (8, 16, 32, 64)):
                if cand[1] == topo_text:
                    feasible = cand[0]
                    break
            if feasible is None:
                cases.remove(c)
            else:
                c["inputs"]["ok.txt"] = feasible
            break

    out = [run_case(c) for c in cases]
    errs = sum(1 for c in out if c["printed"].startswith("error "))
    with gzip.open(HERE / "cli_cases.json.gz", "wt") as f:
        json.dump(out, f)
    print(f"wrote {len(out)} cases ({errs} ending in an error) to {HERE / 'cli_cases.json.gz'}")
    for c in out:
        if c["printed"].startswith("error "):
            print(" ", c["name"], "->", c["printed"].strip()[:110], "| files:", sorted(c["outputs"]))


if __name__ == "__main__":
    main()
