"""GPU parity: the CUDA planner (through the C-ABI) against the reference's
outputs (golden fixtures) and the CPU oracle, bit-exact.  Run with -m gpu."""
import ctypes
import hashlib

import pytest

from conftest import build_set

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def planner():
    import paper_2409_03365_b200 as ws
    return ws.Planner(0)


def records(res, i):
    """(header without arena offset, record bytes) of plan i."""
    r = res.results[i]
    hdr = bytes(r)
    size = ctypes.sizeof(r)
    hdr = bytearray(hdr)
    off_field = type(r).offset.offset
    hdr[off_field:off_field + 8] = b"\0" * 8
    body = bytes(res.arena[r.offset:r.offset + r.size]) if r.status == 0 else b""
    return bytes(hdr[:size]), body


def test_gpu_matches_reference_golden_cases(planner, golden_cases):
    ps, kept, _ = build_set(golden_cases)
    ps.encode(pinned=True)
    texts = planner.plan(ps).texts(ps)
    bad = [c["name"] for c, t in zip(kept, texts) if t != c["expected"]]
    assert not bad, bad[:10]
    assert planner.launch_count >= 2


def test_gpu_backtracking_options_match_reference(planner, backtrack_cases):
    """The placement DFS under non-default (depth, branching), including the
    attempt memo's skipped repeats and budget exhaustion at the reference's
    wave, on the sweep's heaviest backtracking mixtures."""
    ps, kept, _ = build_set(backtrack_cases)
    ps.encode(pinned=True)
    texts = planner.plan(ps).texts(ps)
    bad = [c["name"] for c, t in zip(kept, texts) if t != c["expected"]]
    assert not bad, bad[:10]
    assert sum(1 for c in kept if "budget exhausted" in c["expected"]) >= 50


def test_gpu_full_sweep_100k_matches_reference(planner, sweep_hashes):
    """BASELINE config 5 at full size: every mixture's plan text hashes to the
    reference planner's (217 PlacementInfeasible outcomes included)."""
    import paper_2409_03365_b200 as ws
    n = len(sweep_hashes)
    assert n == 100000
    ps = ws.ProblemSet()
    ps.add_sweep(0, n)
    ps.encode(pinned=True)
    res = planner.plan(ps)
    got = [hashlib.sha1(ps.text(i, res.results, res.arena).encode()).hexdigest()[:16] for i in range(n)]
    mism = [i for i in range(n) if got[i] != sweep_hashes[i]]
    assert not mism, mism[:20]
    infeasible = sum(1 for i in range(n) if res.results[i].status != 0)
    assert infeasible == 217


def test_gpu_records_bit_identical_to_oracle(planner, golden_cases):
    import paper_2409_03365_b200 as ws
    import pyoracle
    ps, kept, _ = build_set(golden_cases)
    ps.add_sweep(0, 3000)
    ps.encode(pinned=True)
    g = planner.plan(ps)
    o = pyoracle.plan_batch(ps)
    bad = [i for i in range(len(ps)) if records(g, i) != records(o, i)]
    assert not bad, bad[:10]


def test_gpu_best_plan_minloc_matches_oracle(planner):
    import paper_2409_03365_b200 as ws
    import pyoracle
    from paper_2409_03365_b200 import parallel
    ps = ws.ProblemSet()
    ps.add_sweep(0, 4000)
    ps.encode(pinned=True)
    planner.stage(ps)
    planner.plan_staged()
    key, idx = planner.best(0)
    o = pyoracle.plan_batch(ps)
    recs = [(o.results[i].end_time / o.results[i].lower_bound, i) for i in range(len(ps)) if o.results[i].status == 0]
    assert (key, idx) == parallel.reduce_minloc(recs)
    key1, idx1 = planner.best(1)
    recs1 = [(o.results[i].end_time, i) for i in range(len(ps)) if o.results[i].status == 0]
    assert (key1, idx1) == parallel.reduce_minloc(recs1)


def test_gpu_empty_batch(planner):
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    ps.encode(pinned=True)
    res = planner.plan(ps)
    assert res.n == 0


def test_gpu_ragged_batch_and_determinism(planner, golden_cases):
    """Mixed sizes (1..64 devices, 1..22 MetaOps, error outcomes) in one batch,
    planned twice on the same context: identical records, all equal to the
    reference."""
    import paper_2409_03365_b200 as ws
    picks = [c for c in golden_cases if c["name"].startswith(("edge/", "fuzz/1", "config/"))]
    ps, kept, _ = build_set(picks[::-1])
    ps.add_sweep(99000, 500)
    ps.encode(pinned=True)
    a = planner.plan(ps)
    b = planner.plan(ps)
    assert all(records(a, i) == records(b, i) for i in range(len(ps)))
    texts = a.texts(ps)
    assert all(t == c["expected"] for c, t in zip(kept, texts))


def test_gpu_device_limit_is_loud(planner):
    """More devices than the build supports (WS_MAX_DEVICES = 256) is a reported
    LimitExceeded, not a fallback; 70 devices (the wide kernels) plan."""
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    for n in (300, 70):
        topo = "island 0: " + " ".join(str(i) for i in range(n)) + "\nbw intra=1e11 inter=1e10\nmem 100000000000\n"
        ps.add_text("module a layers=2 B=48\ntruth a piece 1 1024 0.1 0 1\ntask t flow=a\n", topo)
    ps.encode(pinned=True)
    texts = planner.plan(ps).texts(ps)
    assert texts[0].startswith("error LimitExceeded")
    assert texts[1].startswith("# wavesched plan v1") and "devices" in texts[1]


def test_gpu_dropin_plan_workload(golden_cases):
    import paper_2409_03365_b200 as ws
    c = next(c for c in golden_cases if c["name"] == "config/clip-like/10t/64d/default")
    assert ws.plan_workload(c["workload"], c["topology"]) == c["expected"]
    c = next(c for c in golden_cases if c["name"] == "edge/place/infeasible-memory")
    with pytest.raises(ws.PlacementInfeasible, match="no feasible placement for wave 0"):
        ws.plan_workload(c["workload"], c["topology"])


def test_gpu_dropin_concurrent_callers(golden_cases):
    """The drop-in is reentrant: 8 host threads planning at once
    (each on its own pooled context) get the reference's plan texts."""
    import threading

    import paper_2409_03365_b200 as ws
    cases = [c for c in golden_cases if c["name"].startswith(("config/", "sweep-bt/", "suite/", "fuzz/"))][:96]
    got = [None] * len(cases)

    def work(t):
        for i in range(t, len(cases), 8):
            c = cases[i]
            try:
                got[i] = ws.plan_workload(c["workload"], c["topology"], **c["options"])
            except ws.PlannerError as e:
                got[i] = f"error {type(e).__name__}: {e}\n"

    th = [threading.Thread(target=work, args=(t,)) for t in range(8)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    bad = [c["name"] for c, g in zip(cases, got) if g != c["expected"]]
    assert not bad, bad[:10]


def test_gpu_kernel_timing_reported(planner, monkeypatch):
    """With programmatic dependent launch (default) k_sched starts behind k_fit
    and the fit is reported inside k_sched's time; with WSGPU_PDL=0 each kernel
    has its own events."""
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    ps.add_sweep(0, 2000)
    ps.encode(pinned=True)
    planner.plan(ps)
    fit_ms, sched_ms, place_ms = planner.kernel_ms()
    assert fit_ms >= 0 and sched_ms > 0 and place_ms > 0
    monkeypatch.setenv("WSGPU_PDL", "0")
    pl = ws.Planner(0)
    pl.plan(ps)
    fit_ms, sched_ms, place_ms = pl.kernel_ms()
    assert fit_ms > 0 and sched_ms > 0 and place_ms > 0


def _tiny_soft_caps_planner(monkeypatch, **env):
    import paper_2409_03365_b200 as ws
    monkeypatch.setenv("WSGPU_TINY_SOFT_CAPS", "1")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    return ws.Planner(0)


def test_gpu_retry_pass_drains_every_overflow(monkeypatch, golden_cases):
    """Soft-cap overflows are all re-planned with the hard caps, however many
    a batch holds (no per-call cap): with soft caps below every plan
    ($WSGPU_TINY_SOFT_CAPS) a 2600-plan batch overflows > 2048 plans and still
    equals the oracle record for record -- staged path (fetch, best, simulate
    drain the rest) and the one-shot host call."""
    import paper_2409_03365_b200 as ws
    import pyoracle
    pl = _tiny_soft_caps_planner(monkeypatch)
    ps, kept, _ = build_set(golden_cases[:100])
    ps.add_sweep(0, 2500)
    ps.encode(pinned=True)
    o = pyoracle.plan_batch(ps)
    g = pl.plan(ps)
    assert pl.retry_count >= 2048
    bad = [i for i in range(len(ps)) if records(g, i) != records(o, i)]
    assert not bad, bad[:10]
    # staged: best() and simulate_staged() consume the results before any fetch
    pl.stage(ps)
    pl.plan_staged()
    key, idx = pl.best(1)
    okeys = [(o.results[i].end_time, i) for i in range(len(ps)) if o.results[i].status == 0]
    assert (key, idx) == min(okeys)
    pl.plan_staged()
    pl.simulate_staged()
    sims = pl.fetch_sim(ps)
    g2 = pl.fetch(ps)
    assert pl.retry_count >= 2048
    bad = [i for i in range(len(ps)) if records(g2, i) != records(o, i)]
    assert not bad, bad[:10]
    osims = pyoracle.simulate_batch(ps, o)
    bad = [i for i in range(len(ps)) if ps.sim_text(i, g2, sims) != ps.sim_text(i, o, osims)]
    assert not bad, bad[:10]


def test_gpu_small_batch_soft_cap_fallback(monkeypatch):
    """Host batches of <= 64 plans launch with the soft record caps; a plan
    over them sends the batch to the staged path (hard-cap retry): with soft
    caps below every plan, small batches still equal the oracle."""
    import paper_2409_03365_b200 as ws
    import pyoracle
    pl = _tiny_soft_caps_planner(monkeypatch)
    for start in (0, 500, 1000):
        ps = ws.ProblemSet()
        ps.add_sweep(start, 40)
        ps.encode(pinned=True)
        g, o = pl.plan(ps), pyoracle.plan_batch(ps)
        bad = [i for i in range(len(ps)) if records(g, i) != records(o, i)]
        assert not bad, bad[:10]


def test_gpu_retry_pass_drains_pipelined_chunks(monkeypatch):
    """The same for the chunked H2D / compute / D2H pipeline of
    ws_plan_batch_host: every chunk overflows more than one retry launch."""
    import paper_2409_03365_b200 as ws
    import pyoracle
    pl = _tiny_soft_caps_planner(monkeypatch, WSGPU_HOST_CHUNKS="2")
    ps = ws.ProblemSet()
    ps.add_sweep(0, 9000)
    ps.encode(pinned=True)
    g = pl.plan(ps)
    assert pl.retry_count >= 4096
    o = pyoracle.plan_batch(ps)
    bad = [i for i in range(len(ps)) if records(g, i) != records(o, i)]
    assert not bad, bad[:10]


def test_gpu_pipelined_host_call_matches(sweep_hashes, monkeypatch):
    """ws_plan_batch_host as a chunked H2D / compute / D2H pipeline
    ($WSGPU_HOST_CHUNKS) gives the same plans as the one-shot call."""
    import paper_2409_03365_b200 as ws
    monkeypatch.setenv("WSGPU_HOST_CHUNKS", "3")
    pl = ws.Planner(0)
    n = 30000
    ps = ws.ProblemSet()
    ps.add_sweep(0, n)
    ps.encode(pinned=True)
    res = pl.plan(ps)
    got = [hashlib.sha1(ps.text(i, res.results, res.arena).encode()).hexdigest()[:16] for i in range(n)]
    assert got == sweep_hashes[:n]
    # records stay on the device: evaluation right after the host call
    pl.simulate_staged()
    sims = pl.fetch_sim(ps)
    assert all(sims.results[i].valid for i in range(n) if res.results[i].status == 0)


def test_gpu_weak_scaling_mixtures_match_oracle(planner):
    """bench.py's weak scaling plans sweep mixtures beyond the 100k reference
    hashes (rank r: [r*100k, (r+1)*100k)); a sample of each 100k block up to 8
    GPUs equals the oracle record for record."""
    import random

    import paper_2409_03365_b200 as ws
    import pyoracle as po
    rng = random.Random(8)
    idx = sorted(rng.sample(range(100000, 800000), 2100))
    ps = ws.ProblemSet()
    for i in idx:
        ps.add_sweep(i, 1)
    ps.encode(pinned=True)
    res = planner.plan(ps)
    ores = po.plan_batch(ps)
    bad = [idx[i] for i in range(len(idx)) if records(res, i) != records(ores, i)]
    assert not bad, bad[:10]


def test_gpu_small_batches_warp_fit_match_oracle(planner, golden_cases):
    """Batches of at most kFitWarpMaxModules (4096) modules fit each curve with
    a warp per module, larger ones with a thread per module: small batches
    (golden cases one at a time, sweep mixtures in groups of 50) give records
    bit-identical to the oracle's."""
    import paper_2409_03365_b200 as ws
    import pyoracle
    bad = []
    for c in golden_cases[:40]:
        ps, kept, _ = build_set([c])
        ps.encode(pinned=True)
        g, o = planner.plan(ps), pyoracle.plan_batch(ps)
        if any(records(g, i) != records(o, i) for i in range(len(ps))):
            bad.append(c["name"])
    for start in range(0, 2000, 50):
        ps = ws.ProblemSet()
        ps.add_sweep(start, 50)
        ps.encode(pinned=True)
        g, o = planner.plan(ps), pyoracle.plan_batch(ps)
        bad += [start + i for i in range(len(ps)) if records(g, i) != records(o, i)]
    assert not bad, bad[:10]
