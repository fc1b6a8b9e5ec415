"""Candidate-plan search for one workload.

"Candidate plans" of a workload are the reference-supported planner variants:
PlannerOptions (planner.hpp:21-27) -- placement backtracking depth and
branching, the sequential-placement ablation, the allocator's bisection eps
and drop_floor -- each an independent plan_workload call.  All candidates are
planned in ONE device batch; the best is selected on the device (k_best,
ws_best_staged) by

  "makespan"   predicted_makespan = WavefrontSchedule end time (planner.hpp:193-194)
  "gap"        predicted_makespan / lower_bound (PAPER's optimality gap)
  "simulated"  simulate_plan(plan).makespan (simulate.hpp:322-324), via k_sim

with infeasible candidates at +inf and ties to the smaller candidate index.
Across GPUs the candidates are split strided and the per-rank bests meet in
one NCCL min-loc exchange (parallel.global_best).
"""
from __future__ import annotations

from . import parallel

KEYS = {"gap": 0, "makespan": 1, "simulated": 2}


def candidate_variants() -> list[dict]:
    """The fixed candidate grid (96 variants): backtrack depth 0-3 x branching
    2-4 x sequential off/on x eps {1e-7, 1e-9} x drop_floor {0, 0.05}.  Index 0
    is not the reference default; the default (depth 2, branching 3, parallel,
    1e-7, 0) is index 2*24 + 1*8 = 56."""
    out = []
    for bt in (0, 1, 2, 3):
        for br in (2, 3, 4):
            for seq in (0, 1):
                for eps in (1e-7, 1e-9):
                    for drop in (0.0, 0.05):
                        out.append({"bt_depth": bt, "bt_branching": br, "sequential": seq, "eps": eps,
                                    "drop_floor": drop})
    return out


def candidate_set(workload: str, topology: str, variants: list[dict] | None = None, indices=None, pinned=True):
    """ProblemSet of the workload planned under each variant (optionally only the
    given candidate indices, e.g. one rank's share)."""
    from . import ProblemSet
    variants = candidate_variants() if variants is None else variants
    ps = ProblemSet()
    for i in (range(len(variants)) if indices is None else indices):
        ps.add_json(workload, topology, **variants[i])
    ps.encode(pinned=pinned)
    return ps


def candidate_set_for_scenario(name: str, tasks: int, devices: int, seed: int = 0,
                               variants: list[dict] | None = None, pinned=True):
    """ProblemSet of a generated scenario (scenarios.hpp) under each variant."""
    from . import ProblemSet
    variants = candidate_variants() if variants is None else variants
    ps = ProblemSet()
    for v in variants:
        ps.add_scenario(name, tasks, devices, seed, **v)
    ps.encode(pinned=pinned)
    return ps


def best_candidate(planner, pset, key: str = "makespan", stream=None) -> tuple[float, int]:
    """Plan every candidate of `pset` on the device and min-locate the best:
    (key value, candidate index); (+inf, -1) when every candidate failed."""
    if key not in KEYS:
        raise ValueError(f"unknown candidate key {key!r} (one of {sorted(KEYS)})")
    return planner.best_of(pset, KEYS[key], stream)  # ws_best_batch_host: one call


def best_candidate_sharded(planner, workload: str, topology: str, variants: list[dict] | None = None,
                           key: str = "makespan", rank: int = 0, world: int = 1, device=None) -> tuple[float, int]:
    """Multi-GPU search: rank r plans candidates i with i % world == r, then one
    NCCL min-loc exchange returns the global (key, candidate index) on every rank."""
    variants = candidate_variants() if variants is None else variants
    idx = list(parallel.shard(len(variants), rank, world))
    k, li = (float("inf"), -1)
    if idx:
        k, li = best_candidate(planner, candidate_set(workload, topology, variants, idx), key)
    gi = parallel.local_to_global(li, rank, world) if li >= 0 else -1
    return parallel.global_best(k if li >= 0 else float("inf"), gi, device)
