"""Generate the committed plan-evaluation fixtures from the REFERENCE
simulate_plan / validate_plan (simulate.hpp, validate.hpp) itself.

Runs only in the build container (oracle/_ref/libwsref.so compiled from the
reference headers, `make -C oracle ref`).  Writes:

  sim_cases.json.gz        inputs + expected canonical evaluation text
                           (csrc/host/sim_text.cpp format) for
                           * the BASELINE configs under four SimulatorOptions,
                           * the bundled suite (default and sequential placement),
                           * 150 acceptance fuzz workloads,
                           * broken plans: sweep mixtures planned by the pinned
                             oracle, edited by tests/records.py corrupt() (and a
                             lowered memory capacity), written as plan text by the
                             host decoder and evaluated by the reference's
                             parse_plan + simulate_plan + validate_plan
  sim_sweep_hashes.txt.gz  sha1[:16] of the reference evaluation text of every
                           SURVEY §8(d) sweep mixture 0..99999

usage: python tests/golden/make_sim_golden.py [--sweep N]
"""
from __future__ import annotations

import gzip
import hashlib
import json
import re
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))
import pyoracle as po  # noqa: E402
import records as rc  # noqa: E402

from make_golden import CONFIGS, SUITE  # noqa: E402

SIM_VARIANTS = {"default": {}, "zero": {"zero_volumes": True}, "nosync": {"skip_sync": True},
                "bwd3": {"backward_ratio": 3.0}}
N_BROKEN = 240
N_MEMORY = 24


def broken_cases():
    """Sweep mixtures planned by the oracle, then edited (one kind each)."""
    import paper_2409_03365_b200 as ws
    out = []
    ps = ws.ProblemSet()
    ps.add_sweep(0, N_BROKEN + N_MEMORY)
    ps.encode()
    res = po.plan_batch(ps)
    for i in range(N_BROKEN):
        kind = rc.KINDS[i % len(rc.KINDS)]
        if not rc.corrupt(res, i, kind, seed=i):
            continue
        out.append({"name": f"broken/{kind}/{i}", "sweep": i, "options": {}, "sim": {},
                    "corrupt": [kind, i], "mem_capacity": None,
                    "expected": po.ref_sim_plan_text(ps.text(i, res.results, res.arena))})
    for i in range(N_BROKEN, N_BROKEN + N_MEMORY):
        if res.results[i].status != 0:
            continue
        text = ps.text(i, res.results, res.arena)
        m = re.search(r"^mem (\d+)$", text, re.M)
        if not m:
            continue
        cap = int(m.group(1)) // 4  # well below the placed peak of most plans
        text = re.sub(r"^mem \d+$", f"mem {cap}", text, flags=re.M)
        out.append({"name": f"broken/memory/{i}", "sweep": i, "options": {}, "sim": {},
                    "corrupt": None, "mem_capacity": cap, "expected": po.ref_sim_plan_text(text)})
    return out


def main() -> None:
    n_sweep = 100000
    if "--sweep" in sys.argv:
        n_sweep = int(sys.argv[sys.argv.index("--sweep") + 1])
    if not po.ref_available():
        raise SystemExit("oracle/_ref/libwsref.so missing: run `make -C oracle ref` (needs /root/reference)")
    cases = []

    def add(name, w, t, opts, sim):
        cases.append({"name": name, "workload": w, "topology": t, "sweep": None, "options": opts, "sim": sim,
                      "corrupt": None,
                      "mem_capacity": None, "expected": po.ref_sim_text(w, t, sim, **opts)})

    for n, t, d in CONFIGS:
        w, tp = po.ref_scenario(n, t, d, 0)
        for v, sim in SIM_VARIANTS.items():
            add(f"config/{n}/{t}t/{d}d/{v}", w, tp, {}, sim)
    for n, t, d in SUITE:
        w, tp = po.ref_scenario(n, t, d, 0)
        add(f"suite/{n}/{t}t/{d}d", w, tp, {}, {})
        add(f"suite-seq/{n}/{t}t/{d}d", w, tp, {"sequential": 1}, {})
    for i, (w, tp) in enumerate(po.ref_fuzz(150)):
        add(f"fuzz/{i}", w, tp, {}, {})
    cases += broken_cases()
    with gzip.open(HERE / "sim_cases.json.gz", "wt") as f:
        json.dump(cases, f)
    nbad = sum("\nvalid 0 " in c["expected"] for c in cases)
    print(f"{len(cases)} cases; {nbad} with violations")

    def h(i):
        return hashlib.sha1(po.ref_sweep_sim(i).encode()).hexdigest()[:16]

    with ThreadPoolExecutor(8) as ex:
        hashes = list(ex.map(h, range(n_sweep), chunksize=256))
    with gzip.open(HERE / "sim_sweep_hashes.txt.gz", "wt") as f:
        f.write("\n".join(hashes) + "\n")
    print(f"{n_sweep} sweep hashes")


if __name__ == "__main__":
    main()
