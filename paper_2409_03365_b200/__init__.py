"""paper_2409_03365_b200 — B200-native execution planner of Spindle (arXiv 2409.03365).

Python mirror of the reference planner interface
(/root/reference/proj/include/wavesched/planner.hpp:156 ``plan_workload``) over
the C-ABI in include/wsgpu/ws_abi.h and include/wsgpu/wsx.h.  All planning runs
in the sm_100a kernels of lib/libwsgpu.so; importing fails loudly if that
library is missing, and there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(__import__("os").environ.get("WSGPU_LIB", _PKG / "lib" / "libwsgpu.so"))

__all__ = [
    "LIB_PATH", "Options", "PlanResult", "ProblemSet", "Planner", "plan_workload", "PlannerError",
    "ParseError", "InfeasibleError", "InvariantError", "CyclicWorkload", "UnknownModule", "EmptyWorkload",
    "InsufficientProfile", "DegenerateFit", "OutOfRange", "NoValidAllocation", "EmptyLevel",
    "PlacementInfeasible", "LimitExceeded", "WS_STATUS", "raise_for_text", "SimOptions", "SimResult",
    "SimResults", "make_sim_options", "PlanSet", "STRATEGIES",
]


# ---- exception taxonomy (common.hpp:20-60) ---------------------------------
class PlannerError(RuntimeError):
    """wavesched::Error"""


class ParseError(PlannerError):
    pass


class InfeasibleError(PlannerError):
    pass


class InvariantError(PlannerError):
    pass


class CyclicWorkload(ParseError):
    pass


class UnknownModule(ParseError):
    pass


class EmptyWorkload(ParseError):
    pass


class InsufficientProfile(ParseError):
    pass


class DegenerateFit(InfeasibleError):
    pass


class OutOfRange(InvariantError):
    pass


class NoValidAllocation(InfeasibleError):
    pass


class EmptyLevel(InvariantError):
    pass


class PlacementInfeasible(InfeasibleError):
    pass


class LimitExceeded(PlannerError):
    """Input beyond the WS_MAX_* limits of this build."""


_ERRORS = {c.__name__: c for c in (
    ParseError, InfeasibleError, InvariantError, CyclicWorkload, UnknownModule, EmptyWorkload,
    InsufficientProfile, DegenerateFit, OutOfRange, NoValidAllocation, EmptyLevel, PlacementInfeasible,
    LimitExceeded)}
_ERRORS["Error"] = PlannerError

WS_STATUS = {"ok": 0, "parse": 2, "infeasible": 3, "invariant": 4, "limit": 5, "internal": 6}


def raise_for_text(text: str) -> str:
    """Return plan text, or raise the exception an ``error <Class>: <what>`` line names."""
    if text.startswith("error "):
        head, _, what = text[len("error "):].rstrip("\n").partition(": ")
        raise _ERRORS.get(head, PlannerError)(what)
    return text


# ---- C structures -------------------------------------------------------------
class Options(C.Structure):
    """PlannerOptions (planner.hpp:21-27) as ws_options (wsx.h)."""
    _fields_ = [("eps", C.c_double), ("max_iters", C.c_int32), ("sequential", C.c_int32),
                ("drop_floor", C.c_double), ("bt_depth", C.c_int32), ("bt_branching", C.c_int32),
                ("grad_mult", C.c_double), ("synth_noise", C.c_double), ("synth_seed", C.c_uint64),
                ("strategy", C.c_int32), ("pad", C.c_int32)]


class PlanResult(C.Structure):
    """ws_plan_result (ws_abi.h)."""
    _fields_ = [("status", C.c_int32), ("err_code", C.c_int32), ("err_a", C.c_int64), ("err_b", C.c_int64),
                ("err_x", C.c_double), ("err_y", C.c_double), ("n_metaops", C.c_int32), ("n_edges", C.c_int32),
                ("n_levels", C.c_int32), ("n_waves", C.c_int32), ("n_entries", C.c_int32), ("n_flows", C.c_int32),
                ("n_pieces", C.c_int32), ("n_scopes", C.c_int32), ("lower_bound", C.c_double), ("end_time", C.c_double),
                ("offset", C.c_uint64), ("size", C.c_uint64)]


class SimOptions(C.Structure):
    """SimulatorOptions (simulate.hpp:69-73) as ws_sim_opts (ws_abi.h)."""
    _fields_ = [("backward_ratio", C.c_double), ("zero_volumes", C.c_int32), ("skip_sync", C.c_int32)]


def make_sim_options(backward_ratio: float = 2.0, zero_volumes: bool = False, skip_sync: bool = False) -> SimOptions:
    return SimOptions(backward_ratio, 1 if zero_volumes else 0, 1 if skip_sync else 0)


class SimResult(C.Structure):
    """ws_sim_result (ws_abi.h): SimulationReport scalars + ValidationReport verdict."""
    _fields_ = [("status", C.c_int32), ("valid", C.c_int32), ("n_violations", C.c_int32),
                ("timeline_items", C.c_int32), ("makespan", C.c_double), ("fwd_bwd_seconds", C.c_double),
                ("param_sync_seconds", C.c_double), ("send_recv_seconds", C.c_double),
                ("fwd_bwd_fraction", C.c_double), ("param_sync_fraction", C.c_double),
                ("send_recv_fraction", C.c_double), ("total_transferred_bytes", C.c_double),
                ("total_inter_island_bytes", C.c_double), ("offset", C.c_uint64), ("size", C.c_uint64)]


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(LIB_PATH))
    vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    sig = {
        "ws_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "ws_ctx_destroy": (None, [vp]),
        "ws_ctx_last_error": (C.c_char_p, [vp]),
        "ws_plan_batch_host": (C.c_int, [vp, vp, vp, vp, u64, C.POINTER(u64), vp]),
        "ws_stage_batch": (C.c_int, [vp, vp, vp]),
        "ws_plan_staged": (C.c_int, [vp, vp]),
        "ws_fetch_results": (C.c_int, [vp, vp, vp, u64, C.POINTER(u64), vp]),
        "ws_last_launch_count": (C.c_int, [vp]),
        "ws_last_retry_count": (C.c_longlong, [vp]),
        "ws_plan_batch_multi": (C.c_int, [C.POINTER(vp), C.c_int, vp, vp, vp, u64, C.POINTER(u64)]),
        "ws_best_host": (C.c_int, [vp, i64, C.c_int, C.POINTER(C.c_double), C.POINTER(i64)]),
        "ws_last_kernel_ms": (C.c_int, [vp, C.POINTER(C.c_double), C.c_int]),
        "ws_best_staged": (C.c_int, [vp, C.c_int, C.POINTER(C.c_double), C.POINTER(i64), vp]),
        "ws_best_batch_host": (C.c_int, [vp, vp, C.c_int, C.POINTER(SimOptions), C.POINTER(C.c_double),
                                         C.POINTER(i64), vp]),
        "ws_arena_bound": (u64, [vp]),
        "wsx_default_options": (None, [C.POINTER(Options)]),
        "wsx_set_new": (vp, []),
        "wsx_set_free": (None, [vp]),
        "wsx_set_size": (i32, [vp]),
        "wsx_add_text": (i32, [vp, C.c_char_p, C.c_char_p, C.POINTER(Options)]),
        "wsx_add_json": (i32, [vp, C.c_char_p, C.c_char_p, C.POINTER(Options)]),
        "wsx_add_scenario": (i32, [vp, C.c_char_p, i32, i32, u64, C.POINTER(Options)]),
        "wsx_add_sweep": (i32, [vp, i64, i64, C.POINTER(Options)]),
        "wsx_set_error": (C.c_char_p, [vp]),
        "wsx_encode": (vp, [vp, i32]),
        "wsx_encoded_bytes": (u64, [vp]),
        "wsx_result_text": (vp, [vp, i32, vp, vp]),
        "wsx_dump_workload": (vp, [vp, i32]),
        "wsx_dump_topology": (vp, [vp, i32]),
        "wsx_free_str": (None, [vp]),
        "wsx_plan_workload_text": (vp, [C.c_char_p, C.c_char_p, C.POINTER(Options)]),
        "wsx_algorithmic_bytes": (None, [vp, vp, vp, C.POINTER(u64), C.POINTER(u64)]),
        "wsx_host_alloc": (vp, [u64]),
        "wsx_sim_text": (vp, [vp, i32, vp, vp, vp, vp]),
        "wsx_plans_new": (vp, []),
        "wsx_plans_free": (None, [vp]),
        "wsx_plans_size": (i32, [vp]),
        "wsx_plans_add_text": (i32, [vp, C.c_char_p]),
        "wsx_plans_error": (C.c_char_p, [vp]),
        "wsx_plans_encode": (vp, [vp, i32, C.POINTER(vp), C.POINTER(vp), C.POINTER(u64)]),
        "wsx_plans_write": (vp, [vp, i32]),
        "wsx_plans_sim_text": (vp, [vp, i32, vp, vp]),
        "ws_simulate_staged": (C.c_int, [vp, C.POINTER(SimOptions), vp]),
        "ws_fetch_sim": (C.c_int, [vp, vp, vp, u64, C.POINTER(u64), vp]),
        "ws_simulate_batch_host": (C.c_int, [vp, vp, vp, vp, u64, C.POINTER(SimOptions), vp, vp, u64,
                                             C.POINTER(u64), vp]),
        "ws_sim_arena_bound": (u64, [vp]),
        "ws_last_sim_ms": (C.c_double, [vp]),
        "wsx_host_free": (None, [vp]),
        "wsx_plan_strategy_text": (vp, [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(Options)]),
        "wsx_cmd_compare": (vp, [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(Options)]),
        "wsx_cmd_dynamic": (vp, [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(Options)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def _take_str(ptr: int) -> str:
    try:
        return C.string_at(ptr).decode()
    finally:
        lib.wsx_free_str(ptr)


def make_options(**kw) -> Options:
    """Options with the reference defaults, overridden by keyword (eps, max_iters,
    sequential, drop_floor, bt_depth, bt_branching, grad_mult, synth_noise, synth_seed)."""
    o = Options()
    lib.wsx_default_options(C.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown planner option {k!r}")
        if k == "strategy" and isinstance(v, str):
            if v not in STRATEGIES:
                raise ParseError(f"unknown strategy '{v}'")
            v = STRATEGIES[v]
        setattr(o, k, v)
    return o


# plan_for_strategy selectors (cli.hpp:163-171) built on the device
STRATEGIES = {"wavefront": 0, "decoupled-sequential": 1, "distmm-mt": 2, "task-level-optimus": 3}


class ProblemSet:
    """A batch of planning problems (WorkloadSpec + ClusterTopology + options)."""

    def __init__(self):
        self._h = lib.wsx_set_new()
        self._batch = None

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and lib is not None:  # module globals are gone at interpreter shutdown
            lib.wsx_set_free(h)

    def __len__(self) -> int:
        return lib.wsx_set_size(self._h)

    def _check(self, idx: int) -> int:
        if idx < 0:
            raise ParseError(lib.wsx_set_error(self._h).decode())
        self._batch = None
        return idx

    def add_text(self, workload: str, topology: str, **opts) -> int:
        return self._check(lib.wsx_add_text(self._h, workload.encode(), topology.encode(),
                                            C.byref(make_options(**opts))))

    def add_json(self, workload: str, topology: str, **opts) -> int:
        """JSON workload / topology (cli.hpp:46-110); text grammar if not starting with '{'."""
        return self._check(lib.wsx_add_json(self._h, workload.encode(), topology.encode(),
                                            C.byref(make_options(**opts))))

    def add_scenario(self, name: str, tasks: int, devices: int, seed: int = 0, **opts) -> int:
        return self._check(lib.wsx_add_scenario(self._h, name.encode(), tasks, devices, seed,
                                                C.byref(make_options(**opts))))

    def add_sweep(self, start: int, count: int, **opts) -> int:
        return self._check(lib.wsx_add_sweep(self._h, start, count, C.byref(make_options(**opts))))

    def encode(self, pinned: bool = False) -> int:
        """Encode into the ws_batch SoA format; returns the ws_batch pointer."""
        self._batch = lib.wsx_encode(self._h, 1 if pinned else 0)
        return self._batch

    @property
    def batch(self) -> int:
        return self._batch if self._batch is not None else self.encode()

    @property
    def encoded_bytes(self) -> int:
        return int(lib.wsx_encoded_bytes(self._h))

    def arena_bound(self) -> int:
        return int(lib.ws_arena_bound(self.batch))

    def text(self, i: int, results, arena) -> str:
        """write_plan() text (plan_io.hpp:53-110) of problem i, or 'error <Class>: <what>'."""
        return _take_str(lib.wsx_result_text(self._h, i, C.cast(results, C.c_void_p),
                                             C.cast(arena, C.c_void_p)))

    def sim_arena_bound(self) -> int:
        return int(lib.ws_sim_arena_bound(self.batch))

    def sim_text(self, i: int, results: "Results", sims: "SimResults") -> str:
        """Canonical simulate_plan + validate_plan text of problem i (see
        csrc/host/sim_text.cpp), or its planner error text."""
        return _take_str(lib.wsx_sim_text(self._h, i, C.cast(results.results, C.c_void_p),
                                          C.cast(results.arena, C.c_void_p), C.cast(sims.results, C.c_void_p),
                                          C.cast(sims.arena, C.c_void_p)))

    def algorithmic_bytes(self, res: "Results") -> tuple[int, int]:
        """SURVEY §8(d) compulsory (in, out) bytes of this set's plans."""
        a, b = C.c_uint64(), C.c_uint64()
        lib.wsx_algorithmic_bytes(self._h, res.results, res.arena, C.byref(a), C.byref(b))
        return a.value, b.value

    def dump_workload(self, i: int) -> str:
        return _take_str(lib.wsx_dump_workload(self._h, i))

    def dump_topology(self, i: int) -> str:
        return _take_str(lib.wsx_dump_topology(self._h, i))


class PlanSet:
    """Plan files of any strategy (parse_plan, plan_io.hpp:112-255) for the
    device evaluator: Planner.simulate_plans(PlanSet) replaces
    simulate_plan(parse_plan(text)) + validate_plan for every plan."""

    def __init__(self):
        self._h = lib.wsx_plans_new()
        self._enc = None

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and lib is not None:
            lib.wsx_plans_free(h)

    def __len__(self) -> int:
        return lib.wsx_plans_size(self._h)

    def add_text(self, plan_text: str) -> int:
        i = lib.wsx_plans_add_text(self._h, plan_text.encode())
        if i < 0:
            raise ParseError(lib.wsx_plans_error(self._h).decode())
        self._enc = None
        return i

    def encode(self, pinned: bool = False):
        """(ws_batch*, ws_plan_result*, arena*, arena bytes) of the encoded plans."""
        res, arena, nbytes = C.c_void_p(), C.c_void_p(), C.c_uint64()
        b = lib.wsx_plans_encode(self._h, 1 if pinned else 0, C.byref(res), C.byref(arena), C.byref(nbytes))
        if not b:
            raise ParseError(lib.wsx_plans_error(self._h).decode())
        self._enc = (b, res.value, arena.value, nbytes.value)
        return self._enc

    @property
    def encoded(self):
        return self._enc if self._enc is not None else self.encode()

    def sim_arena_bound(self) -> int:
        return int(lib.ws_sim_arena_bound(self.encoded[0]))

    def write(self, i: int) -> str:
        """write_plan text of parsed plan i (round trip)."""
        return _take_str(lib.wsx_plans_write(self._h, i))

    def sim_text(self, i: int, sims: "SimResults") -> str:
        return _take_str(lib.wsx_plans_sim_text(self._h, i, C.cast(sims.results, C.c_void_p),
                                                C.cast(sims.arena, C.c_void_p)))


class Results:
    """Host copy of one planning call: ws_plan_result[] + arena bytes, in
    page-locked host memory (wsx_host_alloc) so the D2H copies run at full
    PCIe/C2C speed.  Reusable across calls of the same or smaller size."""

    def __init__(self, n: int, arena_cap: int):
        self._res_ptr = lib.wsx_host_alloc(C.sizeof(PlanResult) * max(n, 1))
        self._arena_ptr = lib.wsx_host_alloc(max(arena_cap, 8))
        self.results = (PlanResult * max(n, 1)).from_address(self._res_ptr)
        self.arena = (C.c_uint8 * max(arena_cap, 8)).from_address(self._arena_ptr)
        self.arena_used = C.c_uint64(0)
        self.n = n
        self.cap_plans = max(n, 1)
        self.cap_arena = max(arena_cap, 8)

    def fits(self, n: int, arena_cap: int) -> bool:
        return n <= self.cap_plans and arena_cap <= self.cap_arena

    def __del__(self):
        for name in ("_res_ptr", "_arena_ptr"):
            ptr = getattr(self, name, None)
            if ptr and lib is not None:
                lib.wsx_host_free(ptr)
                setattr(self, name, None)

    def texts(self, pset: ProblemSet) -> list[str]:
        return [pset.text(i, self.results, self.arena) for i in range(self.n)]


class SimResults:
    """Host copy of one evaluation call: ws_sim_result[] + simulation arena
    (page-locked, reusable like Results)."""

    def __init__(self, n: int, arena_cap: int):
        self._res_ptr = lib.wsx_host_alloc(C.sizeof(SimResult) * max(n, 1))
        self._arena_ptr = lib.wsx_host_alloc(max(arena_cap, 8))
        self.results = (SimResult * max(n, 1)).from_address(self._res_ptr)
        self.arena = (C.c_uint8 * max(arena_cap, 8)).from_address(self._arena_ptr)
        self.arena_used = C.c_uint64(0)
        self.n = n
        self.cap_plans = max(n, 1)
        self.cap_arena = max(arena_cap, 8)

    def fits(self, n: int, arena_cap: int) -> bool:
        return n <= self.cap_plans and arena_cap <= self.cap_arena

    __del__ = Results.__del__

    def texts(self, pset: ProblemSet, res: Results) -> list[str]:
        return [pset.sim_text(i, res, self) for i in range(self.n)]


class Planner:
    """A ws_ctx bound to one CUDA device."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        if lib.ws_ctx_create(device, C.byref(h)) != 0:
            raise PlannerError(f"CUDA planner unavailable on device {device}")
        self._h = h

    def close(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.ws_ctx_destroy(self._h)
            self._h = None

    __del__ = close

    def _ok(self, rc: int):
        if rc != 0:
            raise PlannerError(lib.ws_ctx_last_error(self._h).decode())

    def _out(self, pset: ProblemSet, out: Results | None) -> tuple[Results, int]:
        cap = pset.arena_bound()
        if out is None or not out.fits(len(pset), cap):
            out = Results(len(pset), cap)
        out.n = len(pset)
        return out, cap

    def plan(self, pset: ProblemSet, stream: int | None = None, out: Results | None = None) -> Results:
        """Host batch in, host results out (H2D + kernels + D2H); pass `out`
        to reuse page-locked result buffers across calls."""
        out, cap = self._out(pset, out)
        self._ok(lib.ws_plan_batch_host(self._h, pset.batch, out.results, out.arena, cap,
                                        C.byref(out.arena_used), stream))
        return out

    def stage(self, pset: ProblemSet, stream: int | None = None):
        self._ok(lib.ws_stage_batch(self._h, pset.batch, stream))

    def plan_staged(self, stream: int | None = None):
        self._ok(lib.ws_plan_staged(self._h, stream))

    def fetch(self, pset: ProblemSet, stream: int | None = None, out: Results | None = None) -> Results:
        out, cap = self._out(pset, out)
        self._ok(lib.ws_fetch_results(self._h, out.results, out.arena, cap, C.byref(out.arena_used), stream))
        return out

    def best(self, mode: int = 0, stream: int | None = None) -> tuple[float, int]:
        key, idx = C.c_double(), C.c_int64()
        self._ok(lib.ws_best_staged(self._h, mode, C.byref(key), C.byref(idx), stream))
        return key.value, idx.value

    def best_of(self, pset: ProblemSet, mode: int = 0, stream: int | None = None, **sim_opts) -> tuple[float, int]:
        """Plan (and for mode 2 evaluate) a host batch and min-locate it in one
        call (ws_best_batch_host: the candidate search of one workload)."""
        key, idx = C.c_double(), C.c_int64()
        so = make_sim_options(**sim_opts)
        self._ok(lib.ws_best_batch_host(self._h, pset.batch, mode, C.byref(so), C.byref(key), C.byref(idx), stream))
        return key.value, idx.value

    def _sim_out(self, pset: ProblemSet, out: SimResults | None) -> tuple[SimResults, int]:
        cap = pset.sim_arena_bound()
        if out is None or not out.fits(len(pset), cap):
            out = SimResults(len(pset), cap)
        out.n = len(pset)
        return out, cap

    def simulate_staged(self, stream: int | None = None, **sim_opts):
        """simulate_plan + validate_plan of every record of the last plan_staged,
        on the device (results stay there until fetch_sim)."""
        self._ok(lib.ws_simulate_staged(self._h, C.byref(make_sim_options(**sim_opts)), stream))

    def fetch_sim(self, pset: ProblemSet, stream: int | None = None, out: SimResults | None = None) -> SimResults:
        out, cap = self._sim_out(pset, out)
        self._ok(lib.ws_fetch_sim(self._h, out.results, out.arena, cap, C.byref(out.arena_used), stream))
        return out

    def simulate(self, pset: ProblemSet, res: Results, stream: int | None = None, out: SimResults | None = None,
                 **sim_opts) -> SimResults:
        """Evaluate host plan records (any producer of the ws_abi.h layout)."""
        out, cap = self._sim_out(pset, out)
        self._ok(lib.ws_simulate_batch_host(self._h, pset.batch, res.results, res.arena, res.arena_used.value,
                                            C.byref(make_sim_options(**sim_opts)), out.results, out.arena, cap,
                                            C.byref(out.arena_used), stream))
        return out

    def simulate_plans(self, plans: PlanSet, stream: int | None = None, out: SimResults | None = None,
                       **sim_opts) -> SimResults:
        """simulate_plan + validate_plan of parsed plan files on the device."""
        b, res, arena, nbytes = plans.encoded
        cap = plans.sim_arena_bound()
        n = len(plans)
        if out is None or not out.fits(n, cap):
            out = SimResults(n, cap)
        out.n = n
        self._ok(lib.ws_simulate_batch_host(self._h, b, res, arena, nbytes, C.byref(make_sim_options(**sim_opts)),
                                            out.results, out.arena, cap, C.byref(out.arena_used), stream))
        return out

    def sim_ms(self) -> float:
        """Device ms of the last k_sim launch."""
        return float(lib.ws_last_sim_ms(self._h))

    @property
    def launch_count(self) -> int:
        return lib.ws_last_launch_count(self._h)

    @property
    def retry_count(self) -> int:
        """Soft-cap overflows of the last planning call, all re-planned with the hard caps."""
        return int(lib.ws_last_retry_count(self._h))

    def kernel_ms(self) -> tuple[float, float, float]:
        """Device ms of (k_fit, k_sched, k_place incl. retry) in the last call."""
        buf = (C.c_double * 3)()
        lib.ws_last_kernel_ms(self._h, buf, 3)
        return buf[0], buf[1], buf[2]


def plan_batch_multi(planners: "list[Planner]", pset: ProblemSet, out: Results | None = None) -> Results:
    """One host batch sharded over several planners (one per GPU; the same GPU
    twice is allowed) in one call: ws_plan_batch_multi, contiguous blocks of
    equal estimated cost, each on its own host thread."""
    out, cap = planners[0]._out(pset, out)
    arr = (C.c_void_p * len(planners))(*[p._h for p in planners])
    rc = lib.ws_plan_batch_multi(arr, len(planners), pset.batch, out.results, out.arena, cap, C.byref(out.arena_used))
    planners[0]._ok(rc)
    return out


def best_host(res: Results, n: int, mode: int = 0) -> tuple[float, int]:
    """min-loc over host results (ws_best_host): gap (mode 0) or makespan (1)."""
    k, i = C.c_double(0), C.c_int64(-1)
    lib.ws_best_host(res.results, n, mode, C.byref(k), C.byref(i))
    return k.value, i.value


def plan_workload(workload: str, topology: str, **opts) -> str:
    """Drop-in for wavesched::plan_workload on reference text inputs: returns the
    write_plan() text of the plan, or raises the reference's exception class."""
    return raise_for_text(_take_str(lib.wsx_plan_workload_text(workload.encode(), topology.encode(),
                                                               C.byref(make_options(**opts)))))


def plan_for_strategy(strategy: str, workload: str, topology: str, **opts) -> str:
    """Drop-in for wavesched::plan_for_strategy (cli.hpp:163-171) on reference
    text inputs: the write_plan() text of the strategy's plan, or the reference's
    exception (ParseError "unknown strategy '<s>'" for an unknown name)."""
    return raise_for_text(_take_str(lib.wsx_plan_strategy_text(workload.encode(), topology.encode(),
                                                               strategy.encode(), C.byref(make_options(**opts)))))


def compare(workload_path: str, topology_path: str, out_dir: str = "out", **opts) -> str:
    """The reference's `compare` command (cmd_compare, cli.hpp:243-264): every
    strategy planned, validated and simulated -- all four in one device batch
    and one evaluation launch.  Writes out_dir/compare.csv and returns the table
    it prints; raises the reference's exception otherwise."""
    return raise_for_text(_take_str(lib.wsx_cmd_compare(str(workload_path).encode(), str(topology_path).encode(),
                                                        str(out_dir).encode(), C.byref(make_options(**opts)))))


def dynamic(sequence_path: str, topology_path: str, out_dir: str = "out", **opts) -> str:
    """The reference's dynamic re-planning command (cmd_dynamic, cli.hpp:269-327):
    a sequence file of `phase workload=<path> iters=<k>` lines, every (phase,
    strategy) pair planned in one device batch and simulated in one launch.
    Writes phase<p>.<strategy>.plan.txt, dynamic.csv and cumulative.csv under
    out_dir and returns the cumulative table it prints."""
    return raise_for_text(_take_str(lib.wsx_cmd_dynamic(str(sequence_path).encode(), str(topology_path).encode(),
                                                        str(out_dir).encode(), C.byref(make_options(**opts)))))
