// strategies.cpp — plan_for_strategy, strategy comparison and dynamic
// re-planning (cli.hpp:163-171, 237-327) over the device planner.
//
// The reference runs its commands one plan at a time: for every phase and
// every strategy it plans, (compare only) validates, and simulates on one CPU
// core.  Here every (phase, strategy) pair of a command goes into ONE planning
// batch (k_fit/k_sched/k_place) and ONE evaluation launch (k_sim); the host
// then walks the results in the reference's (phase, strategy) order so the
// first error it meets is the one the reference would have thrown, and the
// tables, plan files and cumulative sums come out byte-identical.
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <sstream>

#include "internal.hpp"
#include "wsgpu/planner.hpp"
#include "wsgpu/wsx.h"

namespace wsgpu {
namespace {

std::string fmt_sec(double v) { return fmt_g(v, 9); }  // common.hpp:109

// read_file / write_file (cli.hpp:25-40)
std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ParseError("cannot open '" + path + "'");
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

void write_file(const std::string& path, const std::string& content) {
    const std::filesystem::path parent = std::filesystem::path(path).parent_path();
    std::filesystem::create_directories(parent.empty() ? "." : parent.string());
    std::ofstream out(path, std::ios::binary);
    if (!out) throw Error("cannot write '" + path + "'");
    out << content;
}

bool has_json_extension(const std::string& path) {
    return path.size() > 5 && path.substr(path.size() - 5) == ".json";
}

// load_workload / load_topology (cli.hpp:121-130)
WorkloadSpec load_workload(const std::string& path) {
    const std::string text = read_file(path);
    return has_json_extension(path) ? workload_from_json(text) : parse_workload(text);
}

ClusterTopology load_topology(const std::string& path) {
    const std::string text = read_file(path);
    return has_json_extension(path) ? topology_from_json(text) : parse_topology(text);
}

// Error codes raised inside prepare_planning_base (graph build, contraction,
// curve fit: baselines.hpp:23-32); anything later is strategy-specific.
bool base_stage_error(int code) {
    return (code >= WS_E_CYCLIC_WORKLOAD && code <= WS_E_FIT_NONPOSITIVE) || code == WS_E_HOST_PRESET ||
           (code >= WS_E_LIMIT_DEVICES && code <= WS_E_LIMIT_FLOWS);
}

// One batch = every (workload, strategy) pair, planned and evaluated on the device.
struct Evaluated {
    std::vector<Problem> probs;
    detail::Planned planned;
    std::vector<ws_sim_result> sims;
    std::vector<std::uint8_t> sim_arena;
};

Evaluated plan_and_simulate(const std::vector<const WorkloadSpec*>& specs, const ClusterTopology& topo,
                            const PlannerOptions& opt) {
    Evaluated ev;
    for (const WorkloadSpec* spec : specs) {
        if (!spec) continue;
        for (const std::string& s : all_strategies()) {
            Problem p{spec, &topo, opt};
            p.opt.strategy = strategy_id(s);
            ev.probs.push_back(p);
        }
    }
    if (ev.probs.empty()) return ev;
    detail::CtxLease lease;
    ws_ctx* ctx = lease.ctx();
    ev.planned = detail::plan_on(lease, ev.probs);
    // evaluate the host records: one staging of batch + records, one k_sim launch
    EncodedBatch eb = encode_batch(ev.probs, true);
    const ws_sim_opts so{2.0, 0, 0};  // SimulatorOptions defaults (simulate.hpp:69-73)
    ev.sims.resize(ev.probs.size());
    const std::uint64_t cap = ws_sim_arena_bound(&eb.view);
    ev.sim_arena.resize(cap);
    std::uint64_t used = 0;
    if (ws_simulate_batch_host(ctx, &eb.view, ev.planned.res.data(), ev.planned.arena.data(),
                               ev.planned.arena.size(), &so, ev.sims.data(), ev.sim_arena.data(), cap, &used,
                               nullptr) != 0)
        throw Error(std::string("CUDA evaluator failed: ") + ws_ctx_last_error(ctx));
    return ev;
}

using PlanSink = std::function<void(std::size_t phase, const std::string& strategy, const ExecutionPlan& plan)>;

DynamicReport dynamic_walk(const std::vector<const WorkloadSpec*>& phases, const std::vector<int>& iters,
                           const ClusterTopology& topo, const PlannerOptions& opt,
                           const std::vector<std::exception_ptr>& load_errors, const PlanSink& sink) {
    if (iters.size() != phases.size()) throw Error("dynamic_replan: phases and iters differ in length");
    Evaluated ev = plan_and_simulate(phases, topo, opt);
    DynamicReport rep;
    std::map<std::string, double> cumulative;
    rep.table = "phase,strategy,iters,iteration_time,cumulative\n";
    std::size_t row = 0;
    for (std::size_t p = 0; p < phases.size(); ++p) {
        if (p < load_errors.size() && load_errors[p]) std::rethrow_exception(load_errors[p]);
        if (!phases[p]) throw Error("dynamic_replan: phase " + std::to_string(p) + " has no workload");
        rep.phases.emplace_back();
        for (const std::string& s : all_strategies()) {
            const Problem& prob = ev.probs[row];
            const ws_plan_result& r = ev.planned.res[row];
            const ws_sim_result& sim = ev.sims[row];
            ++row;
            ExecutionPlan plan = decode_result(prob, r, ev.planned.arena.data(), false).plan;  // throws on failure
            if (sim.status != WS_STATUS_OK) throw Error("CUDA evaluator: simulation arena overflow");
            const double iter_time = sim.makespan;
            cumulative[s] += iter_time * iters[p];
            rep.table += std::to_string(p) + "," + s + "," + std::to_string(iters[p]) + "," + fmt_sec(iter_time) +
                         "," + fmt_sec(cumulative[s]) + "\n";
            if (sink) sink(p, s, plan);
            rep.phases.back().push_back({s, std::move(plan), iter_time});
        }
    }
    rep.summary = "strategy,cumulative_seconds\n";
    for (const std::string& s : all_strategies()) rep.summary += s + "," + fmt_sec(cumulative[s]) + "\n";
    return rep;
}

PlannerOptions cli_options(const ws_options* o) {
    PlannerOptions p;
    if (!o) return p;
    p.alloc.eps = o->eps;
    p.alloc.max_iters = o->max_iters;
    p.alloc.drop_floor = o->drop_floor;
    p.placement.sequential = o->sequential != 0;
    p.placement.backtrack_depth = o->bt_depth;
    p.placement.backtrack_branching = o->bt_branching;
    p.grad_opt_multiplier = o->grad_mult;
    p.synth_noise = o->synth_noise;
    p.synth_seed = o->synth_seed;
    return p;
}

}  // namespace

const std::vector<std::string>& all_strategies() {
    static const std::vector<std::string> strategies = {"wavefront", "decoupled-sequential", "task-level-optimus",
                                                        "distmm-mt"};
    return strategies;
}

int strategy_id(const std::string& strategy) {
    if (strategy == "wavefront") return WS_STRATEGY_WAVEFRONT;
    if (strategy == "decoupled-sequential") return WS_STRATEGY_DECOUPLED_SEQUENTIAL;
    if (strategy == "task-level-optimus") return WS_STRATEGY_TASK_OPTIMUS;
    if (strategy == "distmm-mt") return WS_STRATEGY_DISTMM_MT;
    throw ParseError("unknown strategy '" + strategy + "'");
}

ExecutionPlan plan_for_strategy(const std::string& strategy, const WorkloadSpec& spec, const ClusterTopology& topo,
                                const PlannerOptions& opt) {
    validate_workload(spec);  // build_graph's checks come first on every strategy (graph.hpp:98)
    Problem p{&spec, &topo, opt};
    bool known = true;
    try {
        p.opt.strategy = strategy_id(strategy);
    } catch (const ParseError&) {
        // the reference builds the planning base before it rejects the name
        // (cli.hpp:165-170): its errors win, so plan the base-sharing
        // decoupled strategy and surface only base-stage failures
        known = false;
        p.opt.strategy = WS_STRATEGY_DECOUPLED_SEQUENTIAL;
    }
    detail::CtxLease lease;
    detail::Planned r = detail::plan_on(lease, {p});
    if (!known) {
        if (r.res[0].status != WS_STATUS_OK && base_stage_error(r.res[0].err_code)) throw_result_error(p, r.res[0]);
        throw ParseError("unknown strategy '" + strategy + "'");
    }
    return decode_result(p, r.res[0], r.arena.data(), false).plan;
}

CompareReport compare_strategies(const WorkloadSpec& spec, const ClusterTopology& topo, const PlannerOptions& opt) {
    Evaluated ev = plan_and_simulate({&spec}, topo, opt);
    CompareReport rep;
    std::map<std::string, double> makespan;
    for (std::size_t i = 0; i < all_strategies().size(); ++i) {
        const std::string& s = all_strategies()[i];
        const Problem& prob = ev.probs[i];
        const ws_plan_result& r = ev.planned.res[i];
        const ws_sim_result& sim = ev.sims[i];
        ExecutionPlan plan = decode_result(prob, r, ev.planned.arena.data(), false).plan;  // throws on failure
        if (sim.status != WS_STATUS_OK) throw Error("CUDA evaluator: simulation arena overflow");
        if (!sim.valid) {
            const auto names = record_entity_names(prob, r, ev.planned.arena.data());
            const auto msgs = violation_messages(topo, r, sim, ev.sim_arena.data(), names);
            throw InvariantError("strategy " + s + " produced an invalid plan: " + (msgs.empty() ? "" : msgs.front()));
        }
        makespan[s] = sim.makespan;
        rep.runs.push_back({s, std::move(plan), sim.makespan});
    }
    const double reference = makespan.at("decoupled-sequential");
    rep.table = "strategy,makespan,speedup_vs_decoupled\n";
    for (const std::string& s : all_strategies())
        rep.table += s + "," + fmt_sec(makespan[s]) + "," + fmt_sec(reference / makespan[s]) + "\n";
    return rep;
}

DynamicReport dynamic_replan(const std::vector<const WorkloadSpec*>& phases, const std::vector<int>& iters,
                             const ClusterTopology& topo, const PlannerOptions& opt,
                             const std::vector<std::exception_ptr>& load_errors) {
    return dynamic_walk(phases, iters, topo, opt, load_errors, nullptr);
}

std::string cmd_compare(const std::string& workload_path, const std::string& topology_path,
                        const std::string& out_dir, const PlannerOptions& opt) {
    const WorkloadSpec spec = load_workload(workload_path);
    const ClusterTopology topo = load_topology(topology_path);
    const CompareReport rep = compare_strategies(spec, topo, opt);
    write_file(out_dir + "/compare.csv", rep.table);
    return rep.table;
}

std::string cmd_dynamic(const std::string& sequence_path, const std::string& topology_path,
                        const std::string& out_dir, const PlannerOptions& opt) {
    const ClusterTopology topo = load_topology(topology_path);
    const std::vector<SequencePhase> seq = parse_sequence(read_file(sequence_path));
    // every phase's workload is loaded up front (the reference loads it at the
    // top of the phase); a load failure is re-raised when the walk reaches it
    std::vector<WorkloadSpec> specs(seq.size());
    std::vector<const WorkloadSpec*> ptrs(seq.size(), nullptr);
    std::vector<std::exception_ptr> errors(seq.size());
    std::vector<int> iters;
    for (std::size_t p = 0; p < seq.size(); ++p) {
        iters.push_back(seq[p].iters);
        try {
            specs[p] = load_workload(seq[p].workload);
            ptrs[p] = &specs[p];
        } catch (...) {
            errors[p] = std::current_exception();
            break;  // the reference never reaches later phases
        }
    }
    const DynamicReport rep =
        dynamic_walk(ptrs, iters, topo, opt, errors, [&](std::size_t p, const std::string& s, const ExecutionPlan& pl) {
            write_file(out_dir + "/phase" + std::to_string(p) + "." + s + ".plan.txt", write_plan(pl));
        });
    write_file(out_dir + "/dynamic.csv", rep.table);
    write_file(out_dir + "/cumulative.csv", rep.summary);
    return rep.summary;
}

}  // namespace wsgpu

using namespace wsgpu;

namespace {

template <typename Fn>
char* text_or_error(Fn&& fn) {
    try {
        return detail::dup_c(fn());
    } catch (const std::exception& e) {
        return detail::dup_c(std::string("error ") + detail::error_class(e) + ": " + e.what() + "\n");
    }
}

}  // namespace

extern "C" {

char* wsx_plan_strategy_text(const char* workload, const char* topology, const char* strategy,
                             const ws_options* o) {
    return text_or_error([&] {
        const WorkloadSpec spec = parse_workload(workload);
        const ClusterTopology topo = parse_topology(topology);
        return write_plan(plan_for_strategy(strategy, spec, topo, cli_options(o)));
    });
}

char* wsx_cmd_compare(const char* workload_path, const char* topology_path, const char* out_dir,
                      const ws_options* o) {
    return text_or_error([&] { return cmd_compare(workload_path, topology_path, out_dir, cli_options(o)); });
}

char* wsx_cmd_dynamic(const char* sequence_path, const char* topology_path, const char* out_dir,
                      const ws_options* o) {
    return text_or_error([&] { return cmd_dynamic(sequence_path, topology_path, out_dir, cli_options(o)); });
}

}  // extern "C"
