"""Generate the committed JSON-ingestion fixtures (SURVEY §8(f) row 3:
workload_from_json / topology_from_json, cli.hpp:46-110) from the REFERENCE.
Each workload is converted to the JSON schema; the expected outcome is the
reference planner's outcome on the workload's TEXT twin (same content: the
JSON schema has no out_bytes), because the reference's own JSON reader drops
truth/profiles/breakpoints (it iterates items() of a destroyed temporary).
Malformed-JSON errors come from the reference's JSON readers directly.
Build container only.  Writes json_cases.json.gz.

usage: python tests/golden/make_json_golden.py
"""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(HERE))
import pyoracle as po  # noqa: E402
from make_golden import CONFIGS, SUITE  # noqa: E402

INT_KEYS = {"layers", "B", "seq", "hidden", "tp", "param_bytes", "act_bytes"}
REAL_KEYS = {"w", "c"}


def workload_json(text: str) -> str:
    """The text grammar (workload.hpp:139-210) as the JSON schema of
    workload_from_json (which has no out_bytes)."""
    mods, tasks, truth, profiles, bps = [], [], {}, {}, {}
    for line in text.splitlines():
        t = line.split()
        if not t or t[0].startswith("#"):
            continue
        kv = dict(x.split("=", 1) for x in t[2:] if "=" in x)
        if t[0] == "module":
            m = {"kind": t[1]}
            for k, v in kv.items():
                if k in INT_KEYS:
                    m[k if k != "layers" else "layers"] = int(v)
                elif k in REAL_KEYS:
                    m[k] = float(v)
                elif k == "param_group":
                    m[k] = v
            tasks_ok = True  # noqa: F841
            mods.append(m)
        elif t[0] == "task":
            tasks.append({"id": t[1], "flow": kv["flow"]})
        elif t[0] == "truth":
            n_lo, n_hi, a, bc, bw = map(float, t[3:8])
            truth.setdefault(t[1], []).append({"n_lo": n_lo, "n_hi": n_hi, "alpha": a, "beta_c": bc, "beta_w": bw})
        elif t[0] == "metaop":
            profiles.setdefault(t[1], []).append({"n": int(kv["n"]), "time": float(kv["time"]),
                                                  "config": kv.get("config", "dp")})
        elif t[0] == "breakpoints":
            bps[t[1]] = [int(x) for x in t[2:]]
    return json.dumps({"modules": mods, "tasks": tasks, "truth": truth, "profiles": profiles, "breakpoints": bps})


def text_twin(text: str) -> str:
    """The text workload with exactly the JSON schema's content (no out_bytes)."""
    out = []
    for line in text.splitlines():
        if line.startswith("module "):
            line = " ".join(x for x in line.split() if not x.startswith("out_bytes="))
        out.append(line)
    return "\n".join(out) + "\n"


def topology_json(text: str) -> str:
    islands, out = [], {}
    for line in text.splitlines():
        t = line.split()
        if not t or t[0].startswith("#"):
            continue
        if t[0] == "island":
            islands.append([int(x) for x in t[2:]])
        elif t[0] == "bw":
            kv = dict(x.split("=", 1) for x in t[1:])
            out["intra_bw"], out["inter_bw"] = float(kv["intra"]), float(kv["inter"])
        elif t[0] == "mem":
            out["mem"] = int(t[1])
    out["islands"] = islands
    return json.dumps(out)


def main() -> None:
    if not po.ref_available():
        raise SystemExit("oracle/_ref/libwsref.so missing: run `make -C oracle ref` (needs /root/reference)")
    inputs = []
    for n, t, d in CONFIGS + SUITE:
        inputs.append((f"scenario/{n}/{t}t/{d}d", *po.ref_scenario(n, t, d, 0)))
    fam, devs = ("clip-like", "ofasys-like", "qwen-val-like"), (8, 16, 32, 64)
    for i in range(0, 100000, 499):
        inputs.append((f"sweep/{i}", *po.ref_scenario(fam[i % 3], 2 + (i // 3) % 15, devs[(i // 45) % 4], i)))
    for i, (w, t) in enumerate(po.ref_fuzz(100)):
        inputs.append((f"fuzz/{i}", w, t))
    cases = []
    for name, w, t in inputs:
        wj, tj = workload_json(w), topology_json(t)
        for strategy in ("wavefront", "decoupled-sequential"):
            cases.append({"name": f"{strategy}/{name}", "workload": wj, "topology": tj,
                          "options": {"strategy": strategy},
                          "expected": po.ref_plan_text(text_twin(w), t, strategy=strategy)})
    w, t = po.ref_scenario("clip-like", 4, 8, 0)
    wj, tj = workload_json(w), topology_json(t)
    bad = [("syntax", wj[:-5], tj), ("missing-key", wj.replace('"layers"', '"layerz"', 1), tj),
           ("duplicate", wj.replace('"modules": [', '"modules": [' + json.dumps(json.loads(wj)["modules"][0]) + ", ", 1),
            tj), ("topology", wj, tj.replace('"mem"', '"memory"'))]
    for name, a, b in bad:
        cases.append({"name": f"error/{name}", "workload": a, "topology": b, "options": {},
                      "expected": po.ref_json_plan_text(a, b)})
    with gzip.open(HERE / "json_cases.json.gz", "wt") as f:
        json.dump(cases, f)
    print(f"{len(cases)} cases; {sum(c['expected'].startswith('error') for c in cases)} error outcomes")


if __name__ == "__main__":
    main()
