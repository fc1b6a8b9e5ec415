"""Generate the committed golden fixtures from the REFERENCE planner itself.

Runs only in the build container, where oracle/_ref/libwsref.so is compiled
from the reference headers (make -C oracle ref).  Writes:

  cases.json.gz       inputs + expected reference outcome (plan text or
                      "error <Class>: <what>") for the bundled acceptance suite
                      (default and sequential placement), the BASELINE configs
                      with option variants, the first 300 acceptance fuzz
                      workloads, and the hand-written edge cases (edge_cases.py)
  sweep_hashes.txt.gz sha1[:16] of the reference outcome of every SURVEY §8(d)
                      sweep mixture 0..99999 (inputs are regenerated on the GPU
                      box by the repo's scenario generator)

usage: python tests/golden/make_golden.py [--sweep N]
"""
from __future__ import annotations

import gzip
import hashlib
import json
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent / "oracle"))
sys.path.insert(0, str(HERE))
import pyoracle as po  # noqa: E402
from edge_cases import cases as edge_cases  # noqa: E402

SUITE = [(n, t, d) for n in ("clip-like", "ofasys-like") for t in (4, 7, 10) for d in (8, 16, 32)] + \
        [("qwen-val-like", 3, d) for d in (8, 16, 32)]
CONFIGS = [("clip-like", 4, 8), ("clip-like", 10, 64), ("ofasys-like", 7, 32), ("qwen-val-like", 3, 64)]
VARIANTS = {"default": {}, "bt0": {"bt_depth": 0}, "drop": {"drop_floor": 0.05, "eps": 1e-9},
            "noise": {"synth_noise": 0.02, "synth_seed": 7}, "mem": {"grad_mult": 40.0}}


def main() -> None:
    n_sweep = 100000
    if "--sweep" in sys.argv:
        n_sweep = int(sys.argv[sys.argv.index("--sweep") + 1])
    if not po.ref_available():
        raise SystemExit("oracle/_ref/libwsref.so missing: run `make -C oracle ref` (needs /root/reference)")
    cases = []

    def add(name, w, t, opts):
        cases.append({"name": name, "workload": w, "topology": t, "options": opts,
                      "expected": po.ref_plan_text(w, t, **opts)})

    for n, t, d in SUITE:
        w, tp = po.ref_scenario(n, t, d, 0)
        add(f"suite/{n}/{t}t/{d}d", w, tp, {})
        add(f"suite-seq/{n}/{t}t/{d}d", w, tp, {"sequential": 1})
    for n, t, d in CONFIGS:
        w, tp = po.ref_scenario(n, t, d, 0)
        for v, opts in VARIANTS.items():
            add(f"config/{n}/{t}t/{d}d/{v}", w, tp, opts)
    for i, (w, tp) in enumerate(po.ref_fuzz(300)):
        add(f"fuzz/{i}", w, tp, {})
    # sweep mixtures whose placement needs backtracking / ends infeasible (SURVEY §8 branch table)
    fam, devs = ("clip-like", "ofasys-like", "qwen-val-like"), (8, 16, 32, 64)
    for i in (1593, 1956, 2559, 534, 840):
        w, tp = po.ref_scenario(fam[i % 3], 2 + (i // 3) % 15, devs[(i // 45) % 4], i)
        add(f"sweep-bt/{i}", w, tp, {})
        add(f"sweep-bt/{i}/bt0", w, tp, {"bt_depth": 0})
    for name, w, tp, opts in edge_cases():
        add(f"edge/{name}", w, tp, opts)
    with gzip.open(HERE / "cases.json.gz", "wt") as f:
        json.dump(cases, f)
    print(f"{len(cases)} cases; {sum(c['expected'].startswith('error') for c in cases)} error outcomes")

    def h(i):
        return hashlib.sha1(po.ref_sweep_plan(i).encode()).hexdigest()[:16]

    with ThreadPoolExecutor(8) as ex:
        hashes = list(ex.map(h, range(n_sweep), chunksize=256))
    with gzip.open(HERE / "sweep_hashes.txt.gz", "wt") as f:
        f.write("\n".join(hashes) + "\n")
    print(f"{n_sweep} sweep hashes")


if __name__ == "__main__":
    main()
