"""ctypes binding of the CPU oracle (oracle/liboracle.so) and, when built, the
reference bridge (oracle/_ref/libwsref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product path.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libwsref.so"

_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        if not ORACLE_LIB.exists():
            raise ImportError(f"{ORACLE_LIB} missing (make -C oracle)")
        lib = C.CDLL(str(ORACLE_LIB))
        lib.wso_plan_batch.restype = C.c_int
        lib.wso_plan_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        lib.wso_simulate_batch.restype = C.c_int
        lib.wso_simulate_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        _oracle = lib
    return _oracle


def plan_batch(pset):
    """Plan every problem of a ProblemSet on the CPU oracle; returns Results."""
    from paper_2409_03365_b200 import Results
    cap = pset.arena_bound()
    out = Results(len(pset), cap)
    oracle().wso_plan_batch(pset.batch, out.results, out.arena, cap, C.byref(out.arena_used))
    return out


def simulate_batch(pset, res, **sim_opts):
    """simulate_plan + validate_plan of planned records on the CPU oracle; returns SimResults."""
    from paper_2409_03365_b200 import SimResults, make_sim_options
    lib = oracle()
    cap = pset.sim_arena_bound()
    out = SimResults(len(pset), cap)
    lib.wso_simulate_batch(pset.batch, res.results, res.arena, C.byref(make_sim_options(**sim_opts)),
                           out.results, out.arena, cap, C.byref(out.arena_used))
    return out


def simulate_planset(plans, **sim_opts):
    """Oracle evaluation of a PlanSet (parsed plan files); returns SimResults."""
    from paper_2409_03365_b200 import SimResults, make_sim_options
    b, res, arena, _ = plans.encoded
    cap = plans.sim_arena_bound()
    out = SimResults(len(plans), cap)
    oracle().wso_simulate_batch(b, res, arena, C.byref(make_sim_options(**sim_opts)), out.results, out.arena, cap,
                                C.byref(out.arena_used))
    return out


class RefOpts(C.Structure):
    _fields_ = [("eps", C.c_double), ("max_iters", C.c_int), ("drop_floor", C.c_double),
                ("sequential", C.c_int), ("bt_depth", C.c_int), ("bt_branching", C.c_int),
                ("grad_mult", C.c_double), ("synth_noise", C.c_double), ("synth_seed", C.c_ulonglong),
                ("strategy", C.c_int)]


class RefSimOpts(C.Structure):
    _fields_ = [("backward_ratio", C.c_double), ("zero_volumes", C.c_int), ("skip_sync", C.c_int)]


def ref_sim_options(backward_ratio=2.0, zero_volumes=False, skip_sync=False) -> RefSimOpts:
    return RefSimOpts(backward_ratio, 1 if zero_volumes else 0, 1 if skip_sync else 0)


def ref_sim_text(workload: str, topology: str, sim: dict | None = None, **opts) -> str:
    """Reference plan_workload + simulate_plan + validate_plan: canonical evaluation text."""
    return _s(ref().wsref_sim_text(workload.encode(), topology.encode(), C.byref(ref_options(**opts)),
                                   C.byref(ref_sim_options(**(sim or {})))))


def ref_sim_plan_text(plan_text: str, **sim) -> str:
    """Reference simulate_plan + validate_plan of a plan file (parse_plan)."""
    return _s(ref().wsref_sim_plan_text(plan_text.encode(), C.byref(ref_sim_options(**sim))))


def ref_sweep_sim(i: int, **sim) -> str:
    return _s(ref().wsref_sweep_sim(i, C.byref(ref_sim_options(**sim))))


def ref_sweep_sim_bench(start: int, count: int, threads: int) -> float:
    return ref().wsref_sweep_sim_bench(start, count, threads)


def ref_available() -> bool:
    return REF_LIB.exists()


def ref():
    """The reference planner compiled from the reference headers (build container only)."""
    global _ref
    if _ref is None:
        lib = C.CDLL(str(REF_LIB))
        vp = C.c_void_p
        lib.wsref_plan_text.restype = vp
        lib.wsref_plan_text.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(RefOpts)]
        lib.wsref_free.argtypes = [vp]
        lib.wsref_scenario.restype = C.c_int
        lib.wsref_scenario.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_ulonglong, C.POINTER(vp), C.POINTER(vp)]
        lib.wsref_fuzz.restype = C.c_int
        lib.wsref_fuzz.argtypes = [C.c_int, C.POINTER(C.POINTER(vp)), C.POINTER(C.POINTER(vp))]
        lib.wsref_free_list.argtypes = [C.POINTER(vp), C.c_int]
        lib.wsref_sweep_plan.restype = vp
        lib.wsref_sweep_plan.argtypes = [C.c_long]
        lib.wsref_sweep_prepare.restype = vp
        lib.wsref_sweep_prepare.argtypes = [C.c_long, C.c_long, C.c_int]
        lib.wsref_sweep_free.argtypes = [vp]
        lib.wsref_sweep_run.restype = C.c_double
        lib.wsref_sweep_run.argtypes = [vp, C.c_long, C.c_long, C.c_int, C.POINTER(C.c_long)]
        lib.wsref_sweep_bench.restype = C.c_double
        lib.wsref_sweep_bench.argtypes = [C.c_long, C.c_long, C.c_int, C.POINTER(C.c_long)]
        lib.wsref_sim_text.restype = vp
        lib.wsref_sim_text.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(RefOpts), C.POINTER(RefSimOpts)]
        lib.wsref_sim_plan_text.restype = vp
        lib.wsref_sim_plan_text.argtypes = [C.c_char_p, C.POINTER(RefSimOpts)]
        lib.wsref_sweep_sim.restype = vp
        lib.wsref_sweep_sim.argtypes = [C.c_long, C.POINTER(RefSimOpts)]
        lib.wsref_sweep_sim_bench.restype = C.c_double
        lib.wsref_sweep_sim_bench.argtypes = [C.c_long, C.c_long, C.c_int]
        lib.wsref_json_plan_text.restype = vp
        lib.wsref_json_plan_text.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(RefOpts)]
        lib.wsref_strategy_plan_text.restype = vp
        lib.wsref_strategy_plan_text.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(RefOpts)]
        lib.wsref_sweep_bench_strategy.restype = C.c_double
        lib.wsref_sweep_bench_strategy.argtypes = [C.c_long, C.c_long, C.c_int, C.c_int]
        lib.wsref_cmd.restype = vp
        lib.wsref_cmd.argtypes = [C.c_int, C.c_char_p, C.c_char_p, C.c_char_p, C.c_double, C.c_int, C.c_ulonglong]
        lib.wsref_sweep_workload.restype = vp
        lib.wsref_sweep_workload.argtypes = [C.c_long, C.POINTER(vp)]
        lib.wsref_sweep_compare_bench.restype = C.c_double
        lib.wsref_sweep_compare_bench.argtypes = [C.c_long, C.c_long, C.c_int]
        lib.wsref_candidates_ms.restype = C.c_double
        lib.wsref_candidates_ms.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(RefOpts), C.c_int, C.c_int,
                                            C.POINTER(C.c_long)]
        lib.wsref_latency_ms.restype = C.c_double
        lib.wsref_latency_ms.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int]
        _ref = lib
    return _ref


def _s(ptr) -> str:
    try:
        return C.string_at(ptr).decode()
    finally:
        ref().wsref_free(ptr)


def ref_options(**kw) -> RefOpts:
    o = RefOpts(1e-7, 200, 0.0, 0, 2, 3, 3.0, 0.0, 0, 0)
    for k, v in kw.items():
        if k == "strategy" and isinstance(v, str):
            v = {"wavefront": 0, "decoupled-sequential": 1, "distmm-mt": 2, "task-level-optimus": 3}[v]
        setattr(o, k, v)
    return o


def ref_plan_text(workload: str, topology: str, **opts) -> str:
    return _s(ref().wsref_plan_text(workload.encode(), topology.encode(), C.byref(ref_options(**opts))))


def ref_scenario(name: str, tasks: int, devices: int, seed: int = 0) -> tuple[str, str]:
    w, t = C.c_void_p(), C.c_void_p()
    rc = ref().wsref_scenario(name.encode(), tasks, devices, seed, C.byref(w), C.byref(t))
    if rc != 0:
        raise ValueError(_s(w))
    return _s(w), _s(t)


def ref_fuzz(count: int) -> list[tuple[str, str]]:
    ws, ts = C.POINTER(C.c_void_p)(), C.POINTER(C.c_void_p)()
    ref().wsref_fuzz(count, C.byref(ws), C.byref(ts))
    out = [(C.string_at(ws[i]).decode(), C.string_at(ts[i]).decode()) for i in range(count)]
    ref().wsref_free_list(ws, count)
    ref().wsref_free_list(ts, count)
    return out


def ref_strategy_plan_text(workload: str, topology: str, strategy: str, **opts) -> str:
    """Reference plan_for_strategy (cli.hpp:163-171) plan text, any of the four strategies."""
    return _s(ref().wsref_strategy_plan_text(workload.encode(), topology.encode(), strategy.encode(),
                                             C.byref(ref_options(**opts))))


def ref_json_plan_text(workload_json: str, topology_json: str, **opts) -> str:
    """Reference workload_from_json + topology_from_json + planning (cli.hpp:46-110)."""
    return _s(ref().wsref_json_plan_text(workload_json.encode(), topology_json.encode(), C.byref(ref_options(**opts))))


def ref_sweep_plan(i: int) -> str:
    return _s(ref().wsref_sweep_plan(i))


def ref_sweep_bench(start: int, count: int, threads: int) -> tuple[float, int]:
    bad = C.c_long(0)
    rate = ref().wsref_sweep_bench(start, count, threads, C.byref(bad))
    return rate, bad.value


class RefSweepSet:
    """Sweep mixtures [start, start+count) generated and parsed once by the
    reference (outside any timed region); run() plans them with the reference
    plan_workload on `threads` std::threads and returns (plans/s, infeasible)."""

    def __init__(self, start: int, count: int, threads: int):
        self.count = count
        self._h = ref().wsref_sweep_prepare(start, count, threads)

    def run(self, threads: int, first: int = 0, count: int | None = None) -> tuple[float, int]:
        bad = C.c_long(0)
        n = self.count if count is None else count
        rate = ref().wsref_sweep_run(self._h, first, n, threads, C.byref(bad))
        return rate, int(bad.value)

    def __del__(self):
        if getattr(self, "_h", None):
            ref().wsref_sweep_free(self._h)
            self._h = None


def ref_sweep_bench_strategy(start: int, count: int, threads: int, strategy: str) -> float:
    sid = {"wavefront": 0, "decoupled-sequential": 1, "distmm-mt": 2, "task-level-optimus": 3}[strategy]
    return ref().wsref_sweep_bench_strategy(start, count, threads, sid)


def ref_latency_ms(name: str, tasks: int, devices: int, reps: int) -> float:
    return ref().wsref_latency_ms(name.encode(), tasks, devices, reps)


def ref_cmd(command: str, input_path: str, topology_path: str, out_dir: str, eps: float = 1e-7,
            bt_depth: int = 2, seed: int = 0) -> str:
    """The reference's own cmd_compare / cmd_dynamic (cli.hpp:243-327): what it
    prints, or "error <Class>: <what>"; files land under out_dir."""
    which = {"compare": 0, "dynamic": 1}[command]
    return _s(ref().wsref_cmd(which, input_path.encode(), topology_path.encode(), out_dir.encode(), eps, bt_depth,
                              seed))


def ref_sweep_workload(i: int) -> tuple[str, str]:
    """Workload + topology text of sweep mixture i."""
    t = C.c_void_p()
    w = ref().wsref_sweep_workload(i, C.byref(t))
    return _s(w), _s(t)


def ref_sweep_compare_bench(start: int, count: int, threads: int) -> float:
    """Reference compare loop (all strategies planned + validated + simulated) over
    sweep mixtures; workloads/s on `threads` threads."""
    return ref().wsref_sweep_compare_bench(start, count, threads)


def best_candidate(pset, key: str = "makespan") -> tuple[float, int]:
    """Oracle side of the candidate search (paper_2409_03365_b200.candidates):
    every candidate planned (and, for "simulated", evaluated) on the CPU oracle,
    then the same selection rule -- key = end_time / lower_bound ("gap"),
    end_time ("makespan") or the simulated makespan; failed plans are +inf;
    ties go to the smaller index.  Returns (key, index), (+inf, -1) if none."""
    res = plan_batch(pset)
    sims = simulate_batch(pset, res) if key == "simulated" else None
    best_k, best_i = float("inf"), -1
    for i in range(len(pset)):
        r = res.results[i]
        if r.status != 0:
            continue
        if key == "gap":
            k = r.end_time / r.lower_bound
        elif key == "makespan":
            k = r.end_time
        else:
            if sims.results[i].status != 0:
                continue
            k = sims.results[i].makespan
        if best_i < 0 or k < best_k:
            best_k, best_i = k, i
    return best_k, best_i


def ref_candidates_ms(workload: str, topology: str, variants: list[dict], threads: int) -> tuple[float, int]:
    """Reference planner over every candidate variant of one workload on `threads`
    threads: (wall ms, best candidate index by predicted makespan)."""
    arr = (RefOpts * len(variants))(*[ref_options(**v) for v in variants])
    best = C.c_long(-1)
    ms = ref().wsref_candidates_ms(workload.encode(), topology.encode(), arr, len(variants), threads, C.byref(best))
    return ms, best.value
