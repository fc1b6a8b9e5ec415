"""Typed views of planned records (ws_abi.h arena layout) for tests: locate a
plan's sections and edit entries / waves in place, e.g. to feed deliberately
broken plans to the evaluator (validate_plan's violation paths)."""
from __future__ import annotations

import numpy as np

ENTRY = np.dtype([("span", "<f8"), ("devmask", "<u8"), ("metaop", "<i4"), ("n", "<i4"), ("layers", "<i4"),
                  ("rot", "<i4")])
WAVE = np.dtype([("start", "<f8"), ("duration", "<f8"), ("level", "<i4"), ("entry_begin", "<i4"),
                 ("n_entries", "<i4"), ("pad", "<i4")])
FLOW = np.dtype([("volume", "<u8"), ("from_wave", "<i4"), ("from_metaop", "<i4"), ("to_wave", "<i4"),
                 ("to_metaop", "<i4"), ("mode", "<i4"), ("pad", "<i4")])
PLAN_REC_BYTES = 104  # sizeof(ws_plan_rec); mem_capacity at byte 48
SIZES = {"metaop": 40, "level": 16, "piece": 40, "edge": 8, "wave": 32, "entry": 32, "flow": 32}


def _al8(v: int) -> int:
    return (v + 7) & ~7


def sections(r) -> dict[str, int]:
    """Byte offsets (inside the arena) of each section of plan result r."""
    o = int(r.offset)
    out = {}
    for name, count in (("metaop", r.n_metaops), ("level", r.n_levels), ("piece", r.n_pieces),
                        ("edge", r.n_edges), ("wave", r.n_waves), ("entry", r.n_entries), ("flow", r.n_flows)):
        out[name] = o
        o += _al8(SIZES[name] * int(count))
    return out


def arena_array(res) -> np.ndarray:
    return np.frombuffer(res.arena, dtype=np.uint8)


def entries(res, i: int) -> np.ndarray:
    r = res.results[i]
    off = sections(r)["entry"]
    return arena_array(res)[off:off + 32 * r.n_entries].view(ENTRY)


def waves(res, i: int) -> np.ndarray:
    r = res.results[i]
    off = sections(r)["wave"]
    return arena_array(res)[off:off + 32 * r.n_waves].view(WAVE)


def flows(res, i: int) -> np.ndarray:
    r = res.results[i]
    off = sections(r)["flow"]
    return arena_array(res)[off:off + 32 * r.n_flows].view(FLOW)


KINDS = ("device_clash", "span", "layers", "unplaced", "n", "start", "entity", "rot")


def corrupt(res, i: int, kind: str, seed: int) -> bool:
    """Break plan i in place (deterministically from seed); False if not applicable."""
    rng = np.random.default_rng(seed)
    if res.results[i].status != 0:
        return False
    en, wv = entries(res, i), waves(res, i)
    if len(en) == 0:
        return False
    e = int(rng.integers(len(en)))
    if kind == "device_clash":  # copy another entry's first device into this one
        multi = [w for w in range(len(wv)) if wv[w]["n_entries"] >= 2]
        if not multi:
            return False
        w = multi[int(rng.integers(len(multi)))]
        a, b = int(wv[w]["entry_begin"]), int(wv[w]["entry_begin"]) + 1
        m = int(en[b]["devmask"])
        en[a]["devmask"] = np.uint64(int(en[a]["devmask"]) | (m & -m))
    elif kind == "span":
        en[e]["span"] = en[e]["span"] * (1.5 if rng.random() < 0.5 else 0.25)
    elif kind == "layers":
        en[e]["layers"] = en[e]["layers"] + 1
    elif kind == "unplaced":
        en[e]["devmask"] = np.uint64(0)
    elif kind == "n":
        en[e]["n"] = en[e]["n"] + 1
    elif kind == "start":  # pull a later wave onto the start of the first
        if len(wv) < 2:
            return False
        w = 1 + int(rng.integers(len(wv) - 1))
        wv[w]["start"] = wv[0]["start"]
    elif kind == "entity":  # run an entry as a different (known) MetaOp
        k = int(res.results[i].n_metaops)
        if k < 2:
            return False
        en[e]["metaop"] = (int(en[e]["metaop"]) + 1) % k
    elif kind == "rot":  # a device list that wraps (sequential-ablation order)
        m = int(en[e]["devmask"])
        if bin(m).count("1") < 2:
            return False
        en[e]["rot"] = (m & -m).bit_length()  # start after the lowest device
    else:
        raise ValueError(kind)
    return True


def set_mem_capacity(pset, i: int, cap: int) -> None:
    """Overwrite ClusterTopology::mem_capacity of encoded problem i in place
    (ws_plan_rec.mem_capacity inside the encoded batch)."""
    import ctypes as C
    batch = pset.batch
    plans = C.c_void_p.from_address(batch + 56).value  # ws_batch.plans
    C.c_uint64.from_address(plans + PLAN_REC_BYTES * i + 48).value = cap


def build_sim_set(cases):
    """ProblemSet for sim golden cases (text inputs or sweep indices), edits applied
    by apply_edits() after planning."""
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    for c in cases:
        if c.get("sweep") is not None:
            ps.add_sweep(c["sweep"], 1, **c["options"])
        else:
            ps.add_text(c["workload"], c["topology"], **c["options"])
    ps.encode()
    return ps


def apply_edits(cases, ps, res) -> None:
    for j, c in enumerate(cases):
        if c.get("corrupt"):
            kind, seed = c["corrupt"]
            assert corrupt(res, j, kind, seed)
        if c.get("mem_capacity") is not None:
            set_mem_capacity(ps, j, c["mem_capacity"])
