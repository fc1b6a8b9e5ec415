"""bench.py — batched planning throughput of the B200 planner.

Workload (default): BASELINE config 5, the synthetic sweep generator (2-16
tasks, clip/ofasys/qwen families, 8-64 device cluster specs), 100k mixtures
per GPU.  The path partitions into independent plans, so ranks scale weakly
(rule: no data-path collective): rank r plans its own block of mixtures
[r*100k, (r+1)*100k); one NCCL min-loc exchange selects the global best plan.
`--scaling strong` splits one fixed 100k set strided across ranks instead
(bounded below by the slowest single plan, ~5 ms of serial backtracking).
A "step" plans every mixture of the rank's share once.

  value  plans/s with the encoded batch already resident in HBM (device-timed,
         CUDA events on the planner stream, max over ranks)
  e2e    plans/s through the C-ABI host call ws_plan_batch_host: pinned host
         batch -> H2D -> kernels -> D2H of the result headers + arena
  roofline   dominant kernel (k_place) vs the measured HBM copy bandwidth
  cpu_baseline  the reference planner (oracle/_ref, compiled from the
         reference sources) on all host cores over a bounded sweep sample
  evaluation / baselines / compare   simulate+validate (k_sim), the three
         baseline planners, and all four strategies + evaluation per mixture

usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
       [--mixtures M] [--scaling weak|strong]
Under torchrun (N>1) every rank plans its share; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

METRIC = "candidate plans evaluated/s and plan latency (ms) vs CPU ref; HBM GB/s fraction"
CONFIGS = {  # BASELINE.json configs[0..3] (single-plan latency lines)
    "clip4x8": ("clip-like", 4, 8),
    "clip10x64": ("clip-like", 10, 64),
    "ofasys7x32": ("ofasys-like", 7, 32),
    "qwen3x64": ("qwen-val-like", 3, 64),
}
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed regions: an NVML
    thread polls every 5 ms while a `with sampler.sampling():` block is open
    (the timed regions are a few hundred ms, so nvidia-smi's 100 ms loop would
    see only 1-3 samples); nvidia-smi is the fallback when NVML is missing."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        import threading
        self.sm, self.mx, self.reasons = [], [], set()
        self.active = threading.Event()
        self.stop_ev = threading.Event()
        self.thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
        except Exception:
            self.nvml = None

    def _loop(self):
        nv = self.nvml
        while not self.stop_ev.is_set():
            if not self.active.wait(0.05):
                continue
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                self.mx.append(self.max_mhz)
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, b in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def sampling(self):
        sampler = self

        class _Scope:
            def __enter__(self):
                sampler.active.set()

            def __exit__(self, *exc):
                sampler.active.clear()

        return _Scope()

    def stop(self) -> dict:
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self.stop_ev.set()
        self.active.set()
        self.thread.join()
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "how": "NVML every 5 ms inside the timed loops (device-resident, evaluation, e2e, baselines, compare)"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(n_sample: int, threads: int) -> dict:
    """Reference planner (compiled from the reference sources) on host cores."""
    import pyoracle as po
    if po.ref_available():
        rate, bad = po.ref_sweep_bench(0, n_sample, threads)
        return {"value": rate, "unit": "plans/s", "cores": threads, "kind": "reference", "cpu_model": cpu_model(),
                "sample": f"sweep mixtures 0..{n_sample - 1}, reference plan_workload, inputs pre-parsed, "
                          f"{threads} std::threads ({bad} infeasible)"}
    import paper_2409_03365_b200 as ws
    ps = ws.ProblemSet()
    ps.add_sweep(0, n_sample)
    ps.encode()
    t0 = time.perf_counter()
    po.plan_batch(ps)
    dt = time.perf_counter() - t0
    return {"value": n_sample / dt, "unit": "plans/s", "cores": 1, "kind": "port", "cpu_model": cpu_model(),
            "sample": f"sweep mixtures 0..{n_sample - 1}, oracle restatement, 1 thread"}


def workload_config(args, world: int) -> dict:
    """`config` of both arms (identical dicts: the reference arm plans the same
    workload; its threads and sample are described in its cpu_baseline)."""
    weak = args.scaling == "weak"
    return {"workload": (f"sweep (BASELINE config 5 generator: 2-16 tasks, clip/ofasys/qwen, 8-64 devices), "
                         f"{args.mixtures} mixtures " + ("per GPU" if weak else "in total")),
            "plans_per_rank": args.mixtures if weak else (args.mixtures + world - 1) // world,
            "sharding": (f"rank r plans mixtures [r*{args.mixtures}, (r+1)*{args.mixtures})" if weak
                         else "strided i % world == rank"),
            "l2": "256 MiB buffer written between timed steps (outside the timed events)",
            "parallelism": f"dp{world} (independent plans, one NCCL min-loc all_gather at the end)"}


def run_reference(args) -> None:
    """The reference planner (plan_workload compiled from the reference headers,
    -O3 -ffp-contract=off) on all host cores.  At N=1 every timed step plans
    exactly the mixtures our arm plans (sweep [0, --mixtures)); at N>1 the whole
    job (N x --mixtures per step) does not fit a few minutes of CPU, so each
    step plans rank 0's block (the N=1 set) and the rate is per plan."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import pyoracle as po
    threads = os.cpu_count() or 1
    if not po.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libwsref.so not built (needs /root/reference)"}))
        return
    n = args.ref_sample or args.mixtures
    job = args.mixtures * world if args.scaling == "weak" else args.mixtures
    n = min(n, job)
    sweep = po.RefSweepSet(0, n, threads)  # generation + parse, untimed
    for _ in range(args.warmup):  # warm-up steps: a bounded 2000-plan prefix
        sweep.run(threads, 0, min(n, 2000))
    rates, bad = [], 0
    for _ in range(args.steps):
        rate, bad = sweep.run(threads)
        rates.append(rate)
    t_total = sum(n / r for r in rates)
    value = args.steps * n / t_total
    same = n == job
    scope = "the whole job" if same else f"{n} of the job's {job} plans per step"
    line = {
        "metric": METRIC, "value": value, "unit": "plans/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * t_total / args.steps * (job / n), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "plans/s", "cores": threads, "kind": "reference", "cpu_model": cpu_model(),
                         "sample": (f"sweep mixtures 0..{n - 1} every step ({scope}), "
                                    f"reference plan_workload compiled from the reference headers "
                                    f"(-O3 -ffp-contract=off), inputs pre-parsed, {threads} std::threads, "
                                    f"{bad} PlacementInfeasible/other errors per step"),
                         "same_plans_as_ours": same},
        "e2e": {"value": value, "unit": "plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mixtures", type=int, default=100000,
                    help="sweep mixtures per rank (weak scaling) or in total (strong)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="reference-arm mixtures per step (default: --mixtures, i.e. our arm's set at N=1)")
    ap.add_argument("--cpu-sample", type=int, default=6000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--latency-reps", type=int, default=300, help="single-plan latency samples (SURVEY 8(d): >= 300)")
    ap.add_argument("--dropin-plans", type=int, default=20000, help="sweep plans of the drop-in throughput block")
    ap.add_argument("--no-dropin", action="store_true")
    ap.add_argument("--compare-mixtures", type=int, default=25000,
                    help="sweep mixtures of the strategy-comparison block (each planned by all 4 strategies)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import paper_2409_03365_b200 as ws
    from paper_2409_03365_b200 import parallel

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    # ---- inputs (untimed): this rank's shard of the sweep, encoded + pinned ----
    # weak scaling (default): every rank plans its own block of --mixtures sweep
    # mixtures (rank r: global mixtures [r*M, (r+1)*M)); strong: the fixed
    # --mixtures set split strided across ranks
    weak = args.scaling == "weak"
    idx = list(parallel.block(args.mixtures, rank) if weak else parallel.shard(args.mixtures, rank, world))
    total = args.mixtures * world if weak else args.mixtures  # plans per step, whole job

    def to_global(li: int) -> int:
        return parallel.block_to_global(li, rank, args.mixtures) if weak else parallel.local_to_global(li, rank, world)

    ps = ws.ProblemSet()
    for i in idx:
        ps.add_sweep(i, 1)
    ps.encode(pinned=True)
    in_bytes_blob = ps.encoded_bytes
    planner = ws.Planner(local)
    stream = torch.cuda.Stream(device=dev)
    sptr = stream.cuda_stream

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()

    # ---- device-resident throughput ----
    planner.stage(ps, sptr)
    for _ in range(args.warmup):
        planner.plan_staged(sptr)
    torch.cuda.synchronize(dev)
    res = planner.fetch(ps, sptr)
    launches_per_step = planner.launch_count
    clocks = ClockSampler(local)
    barrier()
    step_ms, plan_kernel_ms = [], []
    with clocks.sampling():
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            planner.plan_staged(sptr)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            plan_kernel_ms.append(planner.kernel_ms())
    barrier()
    t_local = sum(step_ms) / 1000.0
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    t_max = float(t.item())
    # per-rank device time per step (load balance of the strided shards)
    rank_t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        gathered = [torch.zeros_like(rank_t) for _ in range(world)]
        torch.distributed.all_gather(gathered, rank_t)
        rank_step_ms = [1000.0 * float(g.item()) / args.steps for g in gathered]
    else:
        rank_step_ms = [1000.0 * t_local / args.steps]
    value = total * args.steps / t_max

    # ---- correctness + global best (min-loc over ranks) ----
    planner.stage(ps, sptr)
    planner.plan_staged(sptr)
    res = planner.fetch(ps, sptr)
    key, li = planner.best(0, sptr)
    gi = to_global(li) if li >= 0 else -1
    best_key, best_idx = parallel.global_best(key if li >= 0 else float("inf"), gi, dev)
    n_ok = sum(1 for i in range(len(ps)) if res.results[i].status == 0)
    infeasible = torch.tensor([len(ps) - n_ok], dtype=torch.int64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(infeasible)
    alg_in, alg_out = ps.algorithmic_bytes(res)
    d2h_bytes = len(ps) * ctypes_sizeof_result() + int(res.arena_used.value)

    # ---- plan evaluation: simulate_plan + validate_plan
    # of every planned mixture on the device (k_sim), records already resident ----
    for _ in range(2):
        planner.simulate_staged(sptr)
    barrier()
    sim_ms = []
    with clocks.sampling():
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            planner.simulate_staged(sptr)
            e1.record(stream)
            e1.synchronize()
            sim_ms.append(e0.elapsed_time(e1))
    barrier()
    sims = planner.fetch_sim(ps, sptr)
    n_invalid = sum(1 for i in range(len(ps)) if sims.results[i].status == 0 and not sims.results[i].valid)
    skey, sli = planner.best(2, sptr)
    sgi = to_global(sli) if sli >= 0 else -1
    best_sim, best_sim_idx = parallel.global_best(skey if sli >= 0 else float("inf"), sgi, dev)
    ts = torch.tensor([sum(sim_ms) / 1000.0, float(n_invalid)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(ts[:1], op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(ts[1:], op=torch.distributed.ReduceOp.SUM)
    sim_value = total * args.steps / float(ts[0].item())
    n_invalid = int(ts[1].item())

    # ---- end to end through the C-ABI host call (page-locked host buffers) ----
    r2 = None
    for _ in range(2):
        r2 = planner.plan(ps, sptr, out=r2)
    barrier()
    e2e_ms = []
    with clocks.sampling():
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r2 = planner.plan(ps, sptr, out=r2)
            e1.record(stream)
            e1.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
    barrier()
    te = torch.tensor([sum(e2e_ms) / 1000.0], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_value = total * args.steps / float(te.item())
    # bytes the pipelined call copies back: every result header + each plan's record
    d2h_step = len(ps) * ctypes_sizeof_result() + sum(int(r2.results[i].size) for i in range(len(ps))
                                                      if r2.results[i].status == 0)

    # ---- baseline planners on the device, same shard ----
    baselines = {}
    for strategy in ("decoupled-sequential", "task-level-optimus", "distmm-mt"):
        pb = ws.ProblemSet()
        for i in idx:
            pb.add_sweep(i, 1, strategy=strategy)
        pb.encode(pinned=True)
        planner.stage(pb, sptr)
        for _ in range(2):
            planner.plan_staged(sptr)
        barrier()
        bms = []
        with clocks.sampling():
            for _ in range(args.steps):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                planner.plan_staged(sptr)
                e1.record(stream)
                e1.synchronize()
                bms.append(e0.elapsed_time(e1))
        barrier()
        tb = torch.tensor([sum(bms) / 1000.0], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(tb, op=torch.distributed.ReduceOp.MAX)
        rb = planner.fetch(pb, sptr)
        bad = torch.tensor([sum(1 for i in range(len(pb)) if rb.results[i].status != 0)], dtype=torch.int64,
                           device=dev)
        if world > 1:
            torch.distributed.all_reduce(bad)
        baselines[strategy] = {"value": total * args.steps / float(tb.item()), "unit": "plans/s",
                               "ms_per_step": 1000.0 * float(tb.item()) / args.steps,
                               "failed_plans": int(bad.item())}

    # ---- strategy comparison (cmd_compare's loop, cli.hpp:243-255):
    # every mixture planned by all four strategies and each plan simulated +
    # validated, as ONE staged batch + one k_sim launch per step ----
    compare = None
    if args.compare_mixtures > 0:
        cidx = idx[: max(1, len(idx) * args.compare_mixtures // max(args.mixtures, 1))]
        pc = ws.ProblemSet()
        for i in cidx:
            for strategy in ws.STRATEGIES:
                pc.add_sweep(i, 1, strategy=strategy)
        pc.encode(pinned=True)
        planner.stage(pc, sptr)
        for _ in range(2):
            planner.plan_staged(sptr)
            planner.simulate_staged(sptr)
        barrier()
        cms = []
        with clocks.sampling():
            for _ in range(args.steps):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                planner.plan_staged(sptr)
                planner.simulate_staged(sptr)
                e1.record(stream)
                e1.synchronize()
                cms.append(e0.elapsed_time(e1))
        barrier()
        tc = torch.tensor([sum(cms) / 1000.0, float(len(cidx))], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(tc[:1], op=torch.distributed.ReduceOp.MAX)
            torch.distributed.all_reduce(tc[1:], op=torch.distributed.ReduceOp.SUM)
        n_cmp = int(tc[1].item())
        compare = {"what": "all 4 strategies planned + simulate_plan + validate_plan per mixture "
                           "(one staged batch + one k_sim launch per step)",
                   "mixtures": n_cmp, "value": n_cmp * args.steps / float(tc[0].item()), "unit": "workloads/s",
                   "ms_per_step": 1000.0 * float(tc[0].item()) / args.steps}

    clk = clocks.stop()
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----
    # algorithmic bytes: k_sched reads the compulsory input and
    # writes the schedule (24/MetaOp + 8/level + 24/wave + 24/entry); k_place
    # reads that schedule and writes the compulsory output.
    peak, peak_src = measured_peak()
    kfit_ms = statistics.median(k[0] for k in plan_kernel_ms)
    ksched_ms = statistics.median(k[1] for k in plan_kernel_ms)
    kplace_ms = statistics.median(k[2] for k in plan_kernel_ms)
    sched_bytes = 0
    for i in range(len(ps)):
        r = res.results[i]
        if r.status == 0:
            sched_bytes += 24 * r.n_metaops + 8 * r.n_levels + 24 * r.n_waves + 24 * r.n_entries
    # placement + emission: k_place, then k_emit writes the output records (both
    # inside the "k_place" events); together they move the schedule in and the
    # compulsory output out, as the single k_place of smaller launches does
    if kplace_ms >= ksched_ms:
        dom, dom_ms, dom_bytes = "k_place+k_emit", kplace_ms, sched_bytes + alg_out
    else:
        dom, dom_ms, dom_bytes = "k_sched", ksched_ms, alg_in + sched_bytes
    achieved = dom_bytes / (dom_ms / 1000.0) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"  # dram read+write per launch from the ncu --set full capture
    if tp.exists():
        try:
            tj = json.loads(tp.read_text())
            traffic = sum(tj.get(k) or 0 for k in dom.split("+")) or None
        except Exception:
            traffic = None

    # ---- candidate-plan search of one workload: the 96 planner
    # variants of each BASELINE config planned in one batch, best selected on the
    # device (k_best); latency = host batch in -> best index out ----
    from paper_2409_03365_b200 import candidates as cd
    variants = cd.candidate_variants()
    cand = {"variants": len(variants), "key": "makespan (predicted, planner.hpp:193-194)",
            "what": "stage (H2D) + plan all variants + on-device min-loc + D2H of {key, index}", "configs": {}}
    for name, (fam, tasks, devices) in CONFIGS.items():
        pcs = cd.candidate_set_for_scenario(fam, tasks, devices, 0, variants)
        for _ in range(3):
            cd.best_candidate(planner, pcs, "makespan", sptr)
        samples = []
        for _ in range(max(args.latency_reps // 6, 5)):
            t0 = time.perf_counter()
            bk, bi = cd.best_candidate(planner, pcs, "makespan", sptr)
            samples.append((time.perf_counter() - t0) * 1000.0)
        ms = statistics.median(samples)
        cand["configs"][name] = {"gpu_ms": ms, "candidate_plans_per_s": len(variants) / ms * 1000.0,
                                 "best_index": bi, "best_makespan": bk}
        if not args.no_cpu_baseline:
            try:
                import pyoracle as po
                if po.ref_available():
                    rms, rbi = po.ref_candidates_ms(pcs.dump_workload(0), pcs.dump_topology(0), variants,
                                                    os.cpu_count() or 1)
                    cand["configs"][name].update({"cpu_reference_ms": rms, "cpu_threads": os.cpu_count(),
                                                  "reference_best_index": rbi})
            except Exception:
                pass

    # ---- single-plan latency of the BASELINE configs ----
    latency = {}
    for name, (fam, tasks, devices) in CONFIGS.items():
        one = ws.ProblemSet()
        one.add_scenario(fam, tasks, devices, 0)
        one.encode(pinned=True)
        ro = None
        for _ in range(5):
            ro = planner.plan(one, sptr, out=ro)
        samples = []
        for _ in range(args.latency_reps):
            t0 = time.perf_counter()
            ro = planner.plan(one, sptr, out=ro)
            samples.append((time.perf_counter() - t0) * 1000.0)
        ss = sorted(samples)
        latency[name] = {"gpu_e2e_ms_median": statistics.median(samples), "gpu_e2e_ms_p10": ss[len(ss) // 10],
                         "gpu_e2e_ms_p90": ss[(9 * len(ss)) // 10], "samples": len(ss),
                         "path": ("C-ABI only: ws_plan_batch_host on a pre-encoded plan, pinned host in, "
                                  "binary records out, warm context (no encode/decode; the reference-typed "
                                  "drop-in with both is dropin.latency_ms)")}

    cpu = None
    evaluation = {"what": "simulate_plan + validate_plan of every planned mixture (k_sim, device-resident records)",
                  "value": sim_value, "unit": "evaluations/s", "ms_per_step": 1000.0 * float(ts[0].item()) / args.steps,
                  "plan_and_evaluate_per_s": total / (t_max / args.steps + float(ts[0].item()) / args.steps),
                  "invalid_plans": n_invalid, "best_simulated_makespan": best_sim, "best_index": best_sim_idx}
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_sample, os.cpu_count() or 1)
        try:
            import pyoracle as po
            if po.ref_available():
                n_ev = max(args.cpu_sample // 2, 500)
                evaluation["cpu_reference_plan_and_evaluate_per_s"] = po.ref_sweep_sim_bench(
                    0, n_ev, os.cpu_count() or 1)
                evaluation["cpu_reference_sample"] = (f"sweep mixtures 0..{n_ev - 1}, reference plan_workload + "
                                                      f"simulate_plan + validate_plan, {os.cpu_count()} threads")
        except Exception:
            pass
        try:
            import pyoracle as po
            if po.ref_available():
                for name, (fam, tasks, devices) in CONFIGS.items():
                    latency[name]["cpu_reference_ms_median"] = po.ref_latency_ms(fam, tasks, devices, max(args.latency_reps, 1))
        except Exception:
            pass
        try:
            import pyoracle as po
            if po.ref_available():
                n_b = max(args.cpu_sample // 2, 500)
                for strategy in baselines:
                    baselines[strategy]["cpu_reference_per_s"] = po.ref_sweep_bench_strategy(
                        0, n_b, os.cpu_count() or 1, strategy)
                    baselines[strategy]["cpu_reference_sample"] = (
                        f"sweep mixtures 0..{n_b - 1}, reference plan_for_strategy, {os.cpu_count()} threads")
        except Exception:
            pass

        try:
            import pyoracle as po
            if po.ref_available() and compare is not None:
                n_c = max(args.cpu_sample // 8, 200)
                compare["cpu_reference_per_s"] = po.ref_sweep_compare_bench(0, n_c, os.cpu_count() or 1)
                compare["cpu_reference_sample"] = (f"sweep mixtures 0..{n_c - 1}, reference plan_for_strategy x4 + "
                                                   f"validate_plan + simulate_plan, {os.cpu_count()} threads")
        except Exception:
            pass

    # ---- the drop-in through the reference's own types (wavesched_gpu::plan_workload:
    # reference WorkloadSpec in, reference PlannerResult out, every host step
    # inside the timer) next to the reference planner, same process and host ----
    dropin = None
    exe = ROOT / "oracle" / "_ref" / "dropin_bench"
    if exe.exists() and not args.no_dropin:
        try:
            r = subprocess.run([str(exe), str(args.latency_reps), str(args.dropin_plans), str(os.cpu_count() or 1)],
                               capture_output=True, text=True, timeout=900,
                               env={**os.environ, "CUDA_VISIBLE_DEVICES": str(local)} if world > 1 else None)
            dropin = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-500:]}
            dropin["what"] = ("oracle/ref/dropin_bench.cpp: wavesched_gpu::plan_workload (reference types in, "
                              "PlannerResult out: conversion, encode, H2D, kernels, D2H, decode all timed) vs the "
                              "reference plan_workload in the same process; cold_start_ms = first call of the "
                              "process (CUDA context + module load); throughput = host threads each calling "
                              "the drop-in (one pooled context per thread) vs the reference on the same threads; "
                              "batched = plan_workloads(_each): one device batch, decode on all threads")
        except Exception as e:  # noqa: BLE001
            dropin = {"error": str(e)}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "plans/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * t_max / args.steps,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(args, world),
        "e2e": {"value": e2e_value, "unit": "plans/s", "h2d_bytes_per_step": in_bytes_blob,
                "d2h_bytes_per_step": d2h_step,
                "path": ("ws_plan_batch_host, the C-ABI (pinned host batch in, result headers + plan records "
                         "out); a caller of the reference-typed API also pays encode + decode per plan on "
                         "host threads: see dropin")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": dom,
                     "algorithmic_bytes_per_launch": dom_bytes, "kernel_ms": dom_ms, "peak_source": peak_src,
                     "kernels_ms": {"k_fit": kfit_ms, "k_sched": ksched_ms, "k_place": kplace_ms},
                     "kernels_note": ("k_sched (three phase kernels) is launched programmatic-dependent on "
                                      "k_fit (its graph stage overlaps the fit), so the k_sched time includes "
                                      "k_fit's; the k_place time includes k_emit (output records)"
                                      if kfit_ms < 0.01 else "kernels timed separately"),
                     "planner_alg_bytes": {"in": alg_in, "out": alg_out, "schedule": sched_bytes}},
        "cpu_baseline": cpu,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk,
        "rank_step_ms": rank_step_ms,
        "latency_ms": latency,
        "dropin": dropin,
        "evaluation": evaluation,
        "baselines": baselines,
        "compare": compare,
        "candidates": cand,
        "parity": {"infeasible_plans": int(infeasible.item()), "best_gap": best_key, "best_index": best_idx},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def ctypes_sizeof_result() -> int:
    import ctypes
    from paper_2409_03365_b200 import PlanResult
    return ctypes.sizeof(PlanResult)


if __name__ == "__main__":
    main()
