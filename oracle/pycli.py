"""CPU restatement of the reference's compare / dynamic commands
(cli.hpp:237-327) over the oracle planner and evaluator (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: the checker for the strategy-comparison and dynamic
re-planning path, pinned to the reference's own commands by the fixtures in
tests/golden/cli_cases.json.gz.  The product path is
paper_2409_03365_b200.compare / .dynamic (csrc/host/strategies.cpp).
"""
from __future__ import annotations

import os
import re
from pathlib import Path

import pyoracle

# all_strategies (cli.hpp:237-241), in the reference's order
STRATEGIES = ["wavefront", "decoupled-sequential", "task-level-optimus", "distmm-mt"]


class CmdError(Exception):
    """An exception the reference command raises: "<Class>: <what>"."""


def _fmt_sec(v: float) -> str:  # common.hpp:109 fmt_g(v, 9)
    return "%.9g" % v


def _read(path: str) -> str:  # read_file, cli.hpp:25-31
    try:
        with open(path, "rb") as f:
            return f.read().decode()
    except OSError:
        raise CmdError(f"ParseError: cannot open '{path}'") from None


def _write(path: str, text: str) -> None:  # write_file, cli.hpp:33-40
    Path(path).parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w") as f:
        f.write(text)


def _plan_all(ws, texts: list[tuple[str, str, bool]], opts: dict):
    """Plans (workload, topology, is_json) x STRATEGIES on the oracle and evaluates
    them; returns per problem (plan text or "error ...", (valid, makespan) or None)."""
    ps = ws.ProblemSet()
    for w, t, js in texts:
        for s in STRATEGIES:
            (ps.add_json if js else ps.add_text)(w, t, strategy=s, **opts)
    ps.encode()
    res = pyoracle.plan_batch(ps)
    sims = pyoracle.simulate_batch(ps, res)
    out = []
    for i, text in enumerate(res.texts(ps)):
        r = sims.results[i]  # copied out: the result buffers are freed with `sims`
        out.append((text, (bool(r.valid), float(r.makespan)) if not text.startswith("error ") else None))
    return out


def _load(path: str) -> tuple[str, bool]:
    """load_workload / load_topology (cli.hpp:117-130): the file text and whether
    the path selects the JSON reader."""
    return _read(path), len(path) > 5 and path.endswith(".json")


def _stoll(text: str) -> int | None:
    """std::stoll: optional leading whitespace and sign, then digits; trailing text ignored."""
    m = re.match(r"[ \t\n\v\f\r]*([+-]?\d+)", text)
    if not m or not -(1 << 63) <= int(m.group(1)) < (1 << 63):
        return None
    return int(m.group(1))


def oracle_cmd(command: str, input_path: str, topology_path: str, out_dir: str, **opts) -> str:
    """cmd_compare / cmd_dynamic restated: returns what the command prints, or
    "error <Class>: <what>\\n"; writes the same files under out_dir."""
    import paper_2409_03365_b200 as ws
    try:
        return _compare(ws, input_path, topology_path, out_dir, opts) if command == "compare" else \
            _dynamic(ws, input_path, topology_path, out_dir, opts)
    except CmdError as e:
        return f"error {e}\n"


def _parse_workload(ws, text: str, js: bool, topo: str, tjs: bool) -> None:
    """Raises the reference's load-time error of a workload (parsed against a known-good topology)."""
    ps = ws.ProblemSet()
    try:
        if js or tjs:
            ps.add_json(text, topo)
        else:
            ps.add_text(text, topo)
    except ws.PlannerError as e:
        raise CmdError(f"{type(e).__name__}: {e}") from None


def _compare(ws, wpath: str, tpath: str, out_dir: str, opts: dict) -> str:
    wtext, wjs = _load(wpath)
    ttext, tjs = _load(tpath)
    _parse_workload(ws, wtext, wjs, ttext, tjs)
    makespan = {}
    for s, (text, sim) in zip(STRATEGIES, _plan_all(ws, [(wtext, ttext, wjs or tjs)], opts)):
        if text.startswith("error "):  # plan_for_strategy throws (cli.hpp:248)
            raise CmdError(text[len("error "):].rstrip("\n"))
        valid, makespan[s] = sim
        if not valid:  # cli.hpp:249-252
            raise CmdError(f"InvariantError: strategy {s} produced an invalid plan")
    ref = makespan["decoupled-sequential"]
    table = "strategy,makespan,speedup_vs_decoupled\n"
    for s in STRATEGIES:
        table += f"{s},{_fmt_sec(makespan[s])},{_fmt_sec(ref / makespan[s])}\n"
    _write(os.path.join(out_dir, "compare.csv"), table)
    return table


def _sequence(text: str) -> list[tuple[str, int]]:
    """cmd_dynamic's sequence parser (cli.hpp:283-297)."""
    phases = []
    for lineno, line in enumerate(text.split("\n"), 1):
        if line.lstrip().startswith("#") or not line.strip():
            continue
        toks = line.split()
        where = f"sequence line {lineno}"
        if toks[0] != "phase":
            raise CmdError(f"ParseError: {where}: expected 'phase ...'")
        kv = {}
        for t in toks[1:]:
            if "=" not in t:
                raise CmdError(f"ParseError: {where}: expected key=value token, got '{t}'")
            k, v = t.split("=", 1)
            kv[k] = v
        if "workload" not in kv:
            raise CmdError(f"ParseError: {where}: missing key 'workload'")
        iters = 1
        if "iters" in kv:
            v = _stoll(kv["iters"])
            if v is None:
                raise CmdError(f"ParseError: {where}: key 'iters' is not an integer")
            iters = (v + (1 << 31)) % (1 << 32) - (1 << 31)  # static_cast<int>
        phases.append((kv["workload"], iters))
    if not phases:
        raise CmdError("ParseError: dynamic sequence declares no phases")
    return phases


def _dynamic(ws, spath: str, tpath: str, out_dir: str, opts: dict) -> str:
    ttext, tjs = _load(tpath)
    phases = _sequence(_read(spath))
    # load phases up to the first failure (the reference loads each at the top of its phase)
    loaded, failure = [], None
    for wpath, iters in phases:
        try:
            wtext, wjs = _load(wpath)
            _parse_workload(ws, wtext, wjs, ttext, tjs)
            loaded.append((wtext, wjs, iters))
        except CmdError as e:
            failure = e
            break
    planned = _plan_all(ws, [(w, ttext, js or tjs) for w, js, _ in loaded], opts) if loaded else []
    cumulative = {s: 0.0 for s in STRATEGIES}
    table = "phase,strategy,iters,iteration_time,cumulative\n"
    for p, (_, _, iters) in enumerate(loaded):
        for k, s in enumerate(STRATEGIES):
            text, sim = planned[4 * p + k]
            if text.startswith("error "):
                raise CmdError(text[len("error "):].rstrip("\n"))
            cumulative[s] += sim[1] * iters
            table += f"{p},{s},{iters},{_fmt_sec(sim[1])},{_fmt_sec(cumulative[s])}\n"
            _write(os.path.join(out_dir, f"phase{p}.{s}.plan.txt"), text)
    if failure is not None:
        raise failure
    summary = "strategy,cumulative_seconds\n" + "".join(f"{s},{_fmt_sec(cumulative[s])}\n" for s in STRATEGIES)
    _write(os.path.join(out_dir, "dynamic.csv"), table)
    _write(os.path.join(out_dir, "cumulative.csv"), summary)
    return summary
