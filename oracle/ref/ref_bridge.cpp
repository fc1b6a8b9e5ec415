// ref_bridge.cpp — compiled ONLY in the build container against the reference
// headers (/root/reference/proj/include, read in place, never copied) into
// oracle/_ref/libwsref.so.  Test infrastructure: it runs the reference planner
// itself so the oracle restatement and the CUDA planner can be pinned to it,
// and it is the "reference" CPU baseline of bench.py (kind "reference").
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "wavesched/baselines.hpp"
#include "wavesched/cli.hpp"
#include "wavesched/planner.hpp"
#include "wavesched/scenarios.hpp"
#include "wavesched/simulate.hpp"
#include "wavesched/validate.hpp"

// The acceptance suite is compiled in place (not copied) so its fuzz
// generator (acceptance.cpp:284-323) and tiny instances are reused verbatim.
#define main wsref_acceptance_main
#include "tests/acceptance.cpp"
#undef main

using namespace wavesched;

extern "C" {
typedef struct wsref_opts {
    double eps;
    int max_iters;
    double drop_floor;
    int sequential;
    int bt_depth;
    int bt_branching;
    double grad_mult;
    double synth_noise;
    unsigned long long synth_seed;
    int strategy;  // 0 wavefront, 1 decoupled-sequential (plan_for_strategy, cli.hpp:163-171)
} wsref_opts;
typedef struct wsref_sim_opts {
    double backward_ratio;
    int zero_volumes;
    int skip_sync;
} wsref_sim_opts;
}

namespace {

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

PlannerOptions to_opts(const wsref_opts* o) {
    PlannerOptions opt;
    if (!o) return opt;
    opt.alloc.eps = o->eps;
    opt.alloc.max_iters = o->max_iters;
    opt.alloc.drop_floor = o->drop_floor;
    opt.placement.sequential = o->sequential != 0;
    opt.placement.backtrack_depth = o->bt_depth;
    opt.placement.backtrack_branching = o->bt_branching;
    opt.grad_opt_multiplier = o->grad_mult;
    opt.synth_noise = o->synth_noise;
    opt.synth_seed = o->synth_seed;
    return opt;
}

// plan_for_strategy (cli.hpp:163-171) for the strategies built on the device
ExecutionPlan plan_strategy(const WorkloadSpec& spec, const ClusterTopology& topo, const PlannerOptions& opt,
                            int strategy) {
    if (strategy == 1) return plan_decoupled_sequential(prepare_planning_base(spec, topo, opt), topo, opt);
    if (strategy == 2) return plan_distmm_mt(prepare_planning_base(spec, topo, opt), topo, opt);
    if (strategy == 3) return plan_task_level_optimus(prepare_planning_base(spec, topo, opt), topo, opt);
    return plan_workload(spec, topo, opt).plan;
}

// Reference outcome as text: the plan file, or "error <Class>: <what>".
std::string outcome(const WorkloadSpec& spec, const ClusterTopology& topo, const PlannerOptions& opt,
                    int strategy = 0) {
    try {
        return write_plan(plan_strategy(spec, topo, opt, strategy));
    } catch (const CyclicWorkload& e) {
        return std::string("error CyclicWorkload: ") + e.what() + "\n";
    } catch (const UnknownModule& e) {
        return std::string("error UnknownModule: ") + e.what() + "\n";
    } catch (const EmptyWorkload& e) {
        return std::string("error EmptyWorkload: ") + e.what() + "\n";
    } catch (const InsufficientProfile& e) {
        return std::string("error InsufficientProfile: ") + e.what() + "\n";
    } catch (const ParseError& e) {
        return std::string("error ParseError: ") + e.what() + "\n";
    } catch (const DegenerateFit& e) {
        return std::string("error DegenerateFit: ") + e.what() + "\n";
    } catch (const NoValidAllocation& e) {
        return std::string("error NoValidAllocation: ") + e.what() + "\n";
    } catch (const PlacementInfeasible& e) {
        return std::string("error PlacementInfeasible: ") + e.what() + "\n";
    } catch (const OutOfRange& e) {
        return std::string("error OutOfRange: ") + e.what() + "\n";
    } catch (const EmptyLevel& e) {
        return std::string("error EmptyLevel: ") + e.what() + "\n";
    } catch (const InvariantError& e) {
        return std::string("error InvariantError: ") + e.what() + "\n";
    } catch (const Error& e) {
        return std::string("error Error: ") + e.what() + "\n";
    }
}

// Canonical evaluation text of a plan (the parity format shared with the
// oracle and the CUDA evaluator, see paper_2409_03365_b200/csrc/host/sim_text.cpp):
// simulate_plan's report scalars and per-device / per-entity maps, then
// validate_plan's verdict and its first 16 violation messages.
std::string sim_text(const ExecutionPlan& plan, const wsref_sim_opts* so) {
    SimulatorOptions opt;
    if (so) {
        opt.backward_ratio = so->backward_ratio;
        opt.zero_volumes = so->zero_volumes != 0;
        opt.skip_sync = so->skip_sync != 0;
    }
    const SimulationReport r = simulate_plan(plan, opt);
    const ValidationReport v = validate_plan(plan);
    std::string out = "sim makespan=" + fmt_exact(r.makespan) + " fwd_bwd=" + fmt_exact(r.fwd_bwd_seconds) +
                      " param_sync=" + fmt_exact(r.param_sync_seconds) + " send_recv=" +
                      fmt_exact(r.send_recv_seconds) + " fracs=" + fmt_exact(r.fwd_bwd_fraction) + "," +
                      fmt_exact(r.param_sync_fraction) + "," + fmt_exact(r.send_recv_fraction) +
                      " transferred=" + fmt_exact(r.total_transferred_bytes) +
                      " inter=" + fmt_exact(r.total_inter_island_bytes) +
                      " timeline=" + std::to_string(r.timeline.size()) + "\n";
    out += "busy";
    for (const auto& [d, b] : r.per_device_busy) out += " " + std::to_string(d) + "=" + fmt_exact(b);
    out += "\nmem";
    for (const auto& [d, b] : r.per_device_peak_memory) out += " " + std::to_string(d) + "=" + fmt_exact(b);
    out += "\nutil";
    for (const auto& [id, u] : r.per_entity_utilization) out += " " + id + "=" + fmt_exact(u);
    out += "\nvalid " + std::to_string(v.ok ? 1 : 0) + " " + std::to_string(v.violations.size()) + "\n";
    for (std::size_t i = 0; i < v.violations.size() && i < 16; ++i) out += "v " + v.violations[i] + "\n";
    return out;
}

Scenario sweep(long i) {
    static const char* fam[3] = {"clip-like", "ofasys-like", "qwen-val-like"};
    static const int devs[4] = {8, 16, 32, 64};
    return generate_scenario(fam[i % 3], 2 + static_cast<int>((i / 3) % 15), devs[(i / 45) % 4],
                             static_cast<std::uint64_t>(i));
}

}  // namespace

extern "C" {

void wsref_free(char* p) { std::free(p); }

// Reference plan text for workload/topology texts (parsed by the reference).
char* wsref_plan_text(const char* workload, const char* topology, const wsref_opts* o) {
    try {
        WorkloadSpec spec = parse_workload(workload);
        ClusterTopology topo = parse_topology(topology);
        return dup(outcome(spec, topo, to_opts(o), o ? o->strategy : 0));
    } catch (const Error& e) {
        return dup(std::string("error Parse: ") + e.what() + "\n");
    }
}

// generate_scenario texts (scenarios.hpp:292-299).
int wsref_scenario(const char* name, int tasks, int devices, unsigned long long seed, char** workload,
                   char** topology) {
    try {
        Scenario sc = generate_scenario(name, tasks, devices, seed);
        *workload = dup(sc.workload_text);
        *topology = dup(sc.topology_text);
        return 0;
    } catch (const Error& e) {
        *workload = dup(e.what());
        *topology = nullptr;
        return 1;
    }
}

// The acceptance fuzz sequence (Rng(2024), acceptance.cpp:451-456): workload i
// as dump_workload text plus its topology text.
int wsref_fuzz(int count, char*** workloads, char*** topologies) {
    Rng rng(2024);
    *workloads = static_cast<char**>(std::malloc(sizeof(char*) * count));
    *topologies = static_cast<char**>(std::malloc(sizeof(char*) * count));
    for (int i = 0; i < count; ++i) {
        WorkloadSpec spec = fuzz_workload(rng);
        const int devices = 2 << rng.next_int(0, 3);
        ClusterTopology topo = make_topology(devices, std::max(2, devices / 2), 100e9, 20e9, 1ull << 50);
        (*workloads)[i] = dup(dump_workload(spec));
        (*topologies)[i] = dup(dump_topology(topo));
    }
    return 0;
}

void wsref_free_list(char** list, int count) {
    for (int i = 0; i < count; ++i) std::free(list[i]);
    std::free(list);
}

// Reference plan text of sweep mixture i, default options.
char* wsref_sweep_plan(long i) {
    Scenario sc = sweep(i);
    return dup(outcome(parse_workload(sc.workload_text), parse_topology(sc.topology_text), PlannerOptions{}));
}

char* wsref_sweep_workload(long i, char** topology) {
    Scenario sc = sweep(i);
    *topology = dup(sc.topology_text);
    return dup(sc.workload_text);
}

// CPU baseline: reference plan_workload over sweep mixtures [start, start+count)
// (inputs pre-parsed outside the timed region) on `threads` std::threads.
// Returns plans/s; writes the number of infeasible plans.
double wsref_sweep_bench(long start, long count, int threads, long* infeasible) {
    std::vector<WorkloadSpec> specs(count);
    std::vector<ClusterTopology> topos(count);
    for (long i = 0; i < count; ++i) {
        Scenario sc = sweep(start + i);
        specs[i] = parse_workload(sc.workload_text);
        topos[i] = parse_topology(sc.topology_text);
    }
    std::atomic<long> next{0}, bad{0};
    auto worker = [&] {
        for (long i; (i = next.fetch_add(1)) < count;) {
            try {
                PlannerResult r = plan_workload(specs[i], topos[i]);
                (void)r;
            } catch (const Error&) {
                bad.fetch_add(1);
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (infeasible) *infeasible = bad.load();
    return static_cast<double>(count) / sec;
}

// Pre-parsed sweep mixtures [start, start + count) (generation + parse spread
// over `threads`), so the reference arm can plan the identical 100k set every
// step with only plan_workload inside the timed region.
struct wsref_sweep_set {
    std::vector<WorkloadSpec> specs;
    std::vector<ClusterTopology> topos;
};

wsref_sweep_set* wsref_sweep_prepare(long start, long count, int threads) {
    auto* s = new wsref_sweep_set();
    s->specs.resize(count);
    s->topos.resize(count);
    std::atomic<long> next{0};
    auto worker = [&] {
        for (long i; (i = next.fetch_add(1)) < count;) {
            Scenario sc = sweep(start + i);
            s->specs[i] = parse_workload(sc.workload_text);
            s->topos[i] = parse_topology(sc.topology_text);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(threads, 1); ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return s;
}

void wsref_sweep_free(wsref_sweep_set* s) { delete s; }

// plan_workload over plans [first, first + count) of a prepared set on
// `threads` std::threads; returns plans/s, infeasible count in *bad
double wsref_sweep_run(const wsref_sweep_set* s, long first, long count, int threads, long* infeasible) {
    count = std::max(0L, std::min<long>(count, static_cast<long>(s->specs.size()) - first));
    std::atomic<long> next{0}, bad{0};
    auto worker = [&] {
        for (long i; (i = next.fetch_add(1)) < count;) {
            try {
                PlannerResult r = plan_workload(s->specs[first + i], s->topos[first + i]);
                (void)r;
            } catch (const Error&) {
                bad.fetch_add(1);
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (infeasible) *infeasible = bad.load();
    return static_cast<double>(count) / sec;
}

// Reference plan_workload + simulate_plan + validate_plan: the canonical
// evaluation text (or the planner's "error ..." outcome).
char* wsref_sim_text(const char* workload, const char* topology, const wsref_opts* o, const wsref_sim_opts* so) {
    try {
        WorkloadSpec spec = parse_workload(workload);
        ClusterTopology topo = parse_topology(topology);
        const int strategy = o ? o->strategy : 0;
        try {
            return dup(sim_text(plan_strategy(spec, topo, to_opts(o), strategy), so));
        } catch (const Error&) {
            return dup(outcome(spec, topo, to_opts(o), strategy));
        }
    } catch (const Error& e) {
        return dup(std::string("error Parse: ") + e.what() + "\n");
    }
}

// plan_for_strategy (cli.hpp:163-171) for any of the four strategies: plan text or error.
char* wsref_strategy_plan_text(const char* workload, const char* topology, const char* strategy,
                               const wsref_opts* o) {
    try {
        const WorkloadSpec spec = parse_workload(workload);
        const ClusterTopology topo = parse_topology(topology);
        const PlannerOptions opt = to_opts(o);
        const std::string s = strategy;
        try {
            if (s == "wavefront") return dup(write_plan(plan_workload(spec, topo, opt).plan));
            const PlanningBase base = prepare_planning_base(spec, topo, opt);
            if (s == "decoupled-sequential") return dup(write_plan(plan_decoupled_sequential(base, topo, opt)));
            if (s == "task-level-optimus") return dup(write_plan(plan_task_level_optimus(base, topo, opt)));
            if (s == "distmm-mt") return dup(write_plan(plan_distmm_mt(base, topo, opt)));
            return dup("error ParseError: unknown strategy '" + s + "'\n");
        } catch (const Error& e) {
            return dup(std::string("error Error: ") + e.what() + "\n");
        }
    } catch (const Error& e) {
        return dup(std::string("error Parse: ") + e.what() + "\n");
    }
}

// Reference plan text for JSON workload/topology (cli.hpp:46-110 ingestion).
char* wsref_json_plan_text(const char* workload, const char* topology, const wsref_opts* o) {
    try {
        WorkloadSpec spec = workload_from_json(workload);
        ClusterTopology topo = topology_from_json(topology);
        return dup(outcome(spec, topo, to_opts(o), o ? o->strategy : 0));
    } catch (const Error& e) {
        return dup(std::string("error Parse: ") + e.what() + "\n");
    }
}

// simulate_plan + validate_plan of a plan file (parse_plan, plan_io.hpp:112-255).
char* wsref_sim_plan_text(const char* plan_text, const wsref_sim_opts* so) {
    try {
        return dup(sim_text(parse_plan(plan_text), so));
    } catch (const Error& e) {
        return dup(std::string("error Parse: ") + e.what() + "\n");
    }
}

// Evaluation text of sweep mixture i (default planner options).
char* wsref_sweep_sim(long i, const wsref_sim_opts* so) {
    Scenario sc = sweep(i);
    const WorkloadSpec spec = parse_workload(sc.workload_text);
    const ClusterTopology topo = parse_topology(sc.topology_text);
    try {
        return dup(sim_text(plan_workload(spec, topo).plan, so));
    } catch (const Error&) {
        return dup(outcome(spec, topo, PlannerOptions{}));
    }
}

// CPU baseline of the evaluation path: plan_workload + simulate_plan +
// validate_plan over sweep mixtures [start, start+count) on `threads` threads.
double wsref_sweep_sim_bench(long start, long count, int threads) {
    std::vector<WorkloadSpec> specs(count);
    std::vector<ClusterTopology> topos(count);
    for (long i = 0; i < count; ++i) {
        Scenario sc = sweep(start + i);
        specs[i] = parse_workload(sc.workload_text);
        topos[i] = parse_topology(sc.topology_text);
    }
    std::atomic<long> next{0};
    auto worker = [&] {
        for (long i; (i = next.fetch_add(1)) < count;) {
            try {
                PlannerResult r = plan_workload(specs[i], topos[i]);
                SimulationReport sr = simulate_plan(r.plan);
                ValidationReport vr = validate_plan(r.plan);
                (void)sr;
                (void)vr;
            } catch (const Error&) {
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return static_cast<double>(count) /
           std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// CPU baseline of a baseline planner (plan_for_strategy): strategy 1 decoupled-sequential,
// 2 distmm-mt, over sweep mixtures [start, start+count) on `threads` threads.
double wsref_sweep_bench_strategy(long start, long count, int threads, int strategy) {
    std::vector<WorkloadSpec> specs(count);
    std::vector<ClusterTopology> topos(count);
    for (long i = 0; i < count; ++i) {
        Scenario sc = sweep(start + i);
        specs[i] = parse_workload(sc.workload_text);
        topos[i] = parse_topology(sc.topology_text);
    }
    std::atomic<long> next{0};
    auto worker = [&] {
        for (long i; (i = next.fetch_add(1)) < count;) {
            try {
                ExecutionPlan p = plan_strategy(specs[i], topos[i], PlannerOptions{}, strategy);
                (void)p;
            } catch (const Error&) {
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return static_cast<double>(count) /
           std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// The reference's own compare / dynamic commands (cli.hpp:243-327), run as
// the CLI runs them (files under out_dir); returns what they print, or
// "error <Class>: <what>" for the exception run_command would map to an exit code.
char* wsref_cmd(int which, const char* input, const char* topology, const char* out_dir, double eps,
                int backtrack_depth, unsigned long long seed) {
    CliOptions cli;
    (which == 0 ? cli.workload : cli.sequence) = input;
    cli.topology = topology;
    cli.out = out_dir;
    cli.eps = eps;
    cli.backtrack_depth = backtrack_depth;
    cli.seed = seed;
    std::ostringstream captured;
    std::streambuf* old = std::cout.rdbuf(captured.rdbuf());
    std::string result;
    try {
        if (which == 0)
            cmd_compare(cli);
        else
            cmd_dynamic(cli);
        result = captured.str();
    } catch (const std::exception& e) {
        const char* cls = "Error";
        if (dynamic_cast<const CyclicWorkload*>(&e)) cls = "CyclicWorkload";
        else if (dynamic_cast<const UnknownModule*>(&e)) cls = "UnknownModule";
        else if (dynamic_cast<const EmptyWorkload*>(&e)) cls = "EmptyWorkload";
        else if (dynamic_cast<const InsufficientProfile*>(&e)) cls = "InsufficientProfile";
        else if (dynamic_cast<const ParseError*>(&e)) cls = "ParseError";
        else if (dynamic_cast<const DegenerateFit*>(&e)) cls = "DegenerateFit";
        else if (dynamic_cast<const NoValidAllocation*>(&e)) cls = "NoValidAllocation";
        else if (dynamic_cast<const PlacementInfeasible*>(&e)) cls = "PlacementInfeasible";
        else if (dynamic_cast<const OutOfRange*>(&e)) cls = "OutOfRange";
        else if (dynamic_cast<const EmptyLevel*>(&e)) cls = "EmptyLevel";
        else if (dynamic_cast<const InvariantError*>(&e)) cls = "InvariantError";
        else if (dynamic_cast<const InfeasibleError*>(&e)) cls = "InfeasibleError";
        result = std::string("error ") + cls + ": " + e.what() + "\n";
    }
    std::cout.rdbuf(old);
    return dup(result);
}

// CPU baseline of strategy comparison (cmd_compare's loop, cli.hpp:243-255):
// per sweep mixture, every strategy planned, validated and simulated; over
// mixtures [start, start+count) on `threads` threads.  Returns workloads/s.
double wsref_sweep_compare_bench(long start, long count, int threads) {
    std::vector<WorkloadSpec> specs(count);
    std::vector<ClusterTopology> topos(count);
    for (long i = 0; i < count; ++i) {
        Scenario sc = sweep(start + i);
        specs[i] = parse_workload(sc.workload_text);
        topos[i] = parse_topology(sc.topology_text);
    }
    std::atomic<long> next{0};
    auto worker = [&] {
        for (long i; (i = next.fetch_add(1)) < count;) {
            for (const std::string& s : all_strategies()) {
                try {
                    const ExecutionPlan plan = plan_for_strategy(s, specs[i], topos[i], PlannerOptions{});
                    const ValidationReport v = validate_plan(plan);
                    const SimulationReport r = simulate_plan(plan);
                    (void)v;
                    (void)r;
                } catch (const Error&) {
                }
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return static_cast<double>(count) /
           std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// CPU baseline of the candidate search: the reference plan_workload under each
// of n option variants of one workload, on `threads` threads; writes the best
// candidate by predicted makespan (ties -> smaller index, failures skipped).
// Returns the wall time in ms (inputs parsed outside the timed region).
double wsref_candidates_ms(const char* workload, const char* topology, const wsref_opts* opts, int n, int threads,
                           long* best_index) {
    const WorkloadSpec spec = parse_workload(workload);
    const ClusterTopology topo = parse_topology(topology);
    std::vector<double> key(n, -1.0);
    std::atomic<int> next{0};
    auto worker = [&] {
        for (int i; (i = next.fetch_add(1)) < n;) {
            try {
                key[i] = plan_workload(spec, topo, to_opts(opts + i)).predicted_makespan;
            } catch (const Error&) {
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    long best = -1;
    for (int i = 0; i < n; ++i)
        if (key[i] >= 0.0 && (best < 0 || key[i] < key[best])) best = i;
    *best_index = best;
    return ms;
}

// Single-plan latency of the reference planner (median of `reps`, ms).
double wsref_latency_ms(const char* name, int tasks, int devices, int reps) {
    Scenario sc = generate_scenario(name, tasks, devices, 0);
    WorkloadSpec spec = parse_workload(sc.workload_text);
    ClusterTopology topo = parse_topology(sc.topology_text);
    std::vector<double> ms;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        PlannerResult res = plan_workload(spec, topo);
        (void)res;
        ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(ms.begin(), ms.end());
    return ms[ms.size() / 2];
}

}  // extern "C"
