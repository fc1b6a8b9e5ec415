"""CPU: host-side logic and the C-ABI surface (no compute calls)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_functions():
    names = set()
    for h in (ROOT / "include" / "wsgpu").glob("*.h"):
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(ws[x]?_[a-z_0-9]+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    import paper_2409_03365_b200 as ws
    lib = ctypes.CDLL(str(ws.LIB_PATH))
    missing = [n for n in sorted(declared_functions()) if not hasattr(lib, n)]
    assert not missing, missing
    assert len(declared_functions()) >= 25


def test_library_contains_sm100a_kernels():
    import subprocess
    import paper_2409_03365_b200 as ws
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(ws.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_parse_dump_round_trip(golden_cases):
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    for c in golden_cases[:60]:
        i = ps.add_text(c["workload"], c["topology"])
        w = ps.dump_workload(i)
        t = ps.dump_topology(i)
        j = ps.add_text(w, t)
        assert ps.dump_workload(j) == w
        assert ps.dump_topology(j) == t


def test_parse_errors_raise_reference_classes():
    import paper_2409_03365_b200 as ws
    topo = "island 0: 0 1\nbw intra=1e11 inter=1e10\nmem 100\n"
    ps = ws.ProblemSet()
    with pytest.raises(ws.ParseError, match="unknown module 'nope'"):
        ps.add_text("module a layers=1 B=4\ntruth a piece 1 8 0 0 1\ntask t flow=nope\n", topo)
    with pytest.raises(ws.ParseError, match="workload declares no tasks"):
        ps.add_text("module a layers=1 B=4\n", topo)
    with pytest.raises(ws.ParseError, match="duplicate task id"):
        ps.add_text("module a layers=1 B=4\ntask t flow=a\ntask t flow=a\n", topo)
    with pytest.raises(ws.ParseError, match="topology needs"):
        ps.add_text("module a layers=1 B=4\ntask t flow=a\n", "island 0: 0\n")
    with pytest.raises(ws.ParseError, match="unknown scenario"):
        ps.add_scenario("bogus", 3, 8)
    assert len(ps) == 0


def test_raise_for_text_maps_classes():
    import paper_2409_03365_b200 as ws
    with pytest.raises(ws.PlacementInfeasible, match="wave 3"):
        ws.raise_for_text("error PlacementInfeasible: placement backtrack budget exhausted at wave 3\n")
    with pytest.raises(ws.InfeasibleError):
        ws.raise_for_text("error NoValidAllocation: metaop 'm0': tp degree 16 exceeds device count 8\n")
    with pytest.raises(ws.InvariantError):
        ws.raise_for_text("error OutOfRange: eval_time: n=5 outside [1, 4]\n")
    assert ws.raise_for_text("# wavesched plan v1\n").startswith("#")


def test_options_defaults_match_reference():
    import paper_2409_03365_b200 as ws
    o = ws.make_options()
    assert (o.eps, o.max_iters, o.drop_floor, o.sequential, o.bt_depth, o.bt_branching, o.grad_mult,
            o.synth_noise, o.synth_seed) == (1e-7, 200, 0.0, 0, 2, 3, 3.0, 0.0, 0)
    with pytest.raises(TypeError):
        ws.make_options(bogus=1)


def test_encoding_is_compact_and_deterministic():
    import paper_2409_03365_b200 as ws
    a, b = ws.ProblemSet(), ws.ProblemSet()
    a.add_sweep(0, 200)
    b.add_sweep(0, 200)
    a.encode()
    b.encode()
    assert a.encoded_bytes == b.encoded_bytes
    assert a.encoded_bytes < 200 * 4096
    assert a.arena_bound() > 0


def test_empty_set_encodes():
    import paper_2409_03365_b200 as ws
    import pyoracle
    ps = ws.ProblemSet()
    ps.encode()
    res = pyoracle.plan_batch(ps)
    assert res.n == 0


def test_scenario_generator_matches_reference_texts(golden_cases):
    """The repo's generator rebuilds the reference generator's workloads."""
    import paper_2409_03365_b200 as ws
    by_name = {c["name"]: c for c in golden_cases}
    for fam, t, d in (("clip-like", 10, 64), ("ofasys-like", 7, 32), ("qwen-val-like", 3, 64)):
        ref = by_name[f"config/{fam}/{t}t/{d}d/default"]
        ps = ws.ProblemSet()
        i = ps.add_scenario(fam, t, d, 0)
        j = ps.add_text(ref["workload"], ref["topology"])
        assert ps.dump_workload(i) == ps.dump_workload(j)
        assert ps.dump_topology(i) == ps.dump_topology(j)
