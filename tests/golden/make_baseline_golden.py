"""Generate the committed fixtures of the baseline planners built on the device
 from the REFERENCE itself (baselines.hpp via
oracle/_ref/libwsref.so, build container only).  Writes:

  baseline_cases.json.gz        per case: inputs, strategy, the reference plan
                                text (or "error <Class>: <what>") and the
                                reference simulate/validate text of that plan
  baseline_sweep_hashes.txt.gz  sha1[:16] of the reference plan text of every
                                SURVEY §8(d) sweep mixture 0..99999 per strategy

usage: python tests/golden/make_baseline_golden.py [--sweep N]
"""
from __future__ import annotations

import gzip
import hashlib
import json
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(HERE))
import pyoracle as po  # noqa: E402
from edge_cases import cases as edge_cases  # noqa: E402
from make_golden import CONFIGS, SUITE, VARIANTS  # noqa: E402

STRATEGIES = ["decoupled-sequential", "distmm-mt", "task-level-optimus"]


def main() -> None:
    n_sweep = 100000
    if "--sweep" in sys.argv:
        n_sweep = int(sys.argv[sys.argv.index("--sweep") + 1])
    if not po.ref_available():
        raise SystemExit("oracle/_ref/libwsref.so missing: run `make -C oracle ref` (needs /root/reference)")
    cases = []

    def add(name, w, t, opts, strategy):
        o = dict(opts, strategy=strategy)
        cases.append({"name": name, "workload": w, "topology": t, "options": o,
                      "expected": po.ref_plan_text(w, t, **o),
                      "sim_expected": po.ref_sim_text(w, t, {}, **o)})

    for strategy in STRATEGIES:
        for n, t, d in SUITE:
            w, tp = po.ref_scenario(n, t, d, 0)
            add(f"{strategy}/suite/{n}/{t}t/{d}d", w, tp, {}, strategy)
        for n, t, d in CONFIGS:
            w, tp = po.ref_scenario(n, t, d, 0)
            for v, opts in VARIANTS.items():
                add(f"{strategy}/config/{n}/{t}t/{d}d/{v}", w, tp, opts, strategy)
        for i, (w, tp) in enumerate(po.ref_fuzz(300)):
            add(f"{strategy}/fuzz/{i}", w, tp, {}, strategy)
        for name, w, tp, opts in edge_cases():
            add(f"{strategy}/edge/{name}", w, tp, opts, strategy)
    with gzip.open(HERE / "baseline_cases.json.gz", "wt") as f:
        json.dump(cases, f)
    print(f"{len(cases)} cases; {sum(c['expected'].startswith('error') for c in cases)} error outcomes")

    fam, devs = ("clip-like", "ofasys-like", "qwen-val-like"), (8, 16, 32, 64)
    lines = []
    for s, strategy in enumerate(STRATEGIES, start=1):
        def h(i):
            w, tp = po.ref_scenario(fam[i % 3], 2 + (i // 3) % 15, devs[(i // 45) % 4], i)
            return hashlib.sha1(po.ref_plan_text(w, tp, strategy=s).encode()).hexdigest()[:16]

        with ThreadPoolExecutor(8) as ex:
            lines.append(strategy + " " + " ".join(ex.map(h, range(n_sweep), chunksize=256)))
    with gzip.open(HERE / "baseline_sweep_hashes.txt.gz", "wt") as f:
        f.write("\n".join(lines) + "\n")
    print(f"{n_sweep} sweep hashes per strategy")


if __name__ == "__main__":
    main()
