// decode.cpp — ws_plan_result + arena record -> PlannerResult / ExecutionPlan.
//
// Rebuilds the reference's string-keyed result objects (planner.hpp:29-38,
// 196-210; build_entities :99-122) from the device's index-based output, and
// maps error codes back to the reference exception classes and messages.
#include <algorithm>
#include <cstring>

#include "bounds.h"
#include "wsgpu/decode_impl.hpp"
#include "wsgpu/planner.hpp"

namespace wsgpu {
namespace {

std::size_t al8(std::size_t v) { return (v + 7) & ~std::size_t(7); }

struct Sections {
    const ws_out_metaop* mo;
    const ws_out_level* lv;
    const ws_out_piece* pc;
    const ws_out_edge* ed;
    const ws_out_wave* wv;
    const ws_out_entry* en;
    const ws_out_flow* fl;
    const ws_out_scope* sc;
    const std::uint64_t* ext;  // device words 1..3 per entry (clusters of more than 64 devices)
};

Sections sections_of(const ws_plan_result& r, const std::uint8_t* arena) {
    const std::uint8_t* base = arena + r.offset;
    std::size_t off = 0;
    Sections s{};
    s.mo = reinterpret_cast<const ws_out_metaop*>(base + off);
    off += al8(sizeof(ws_out_metaop) * r.n_metaops);
    s.lv = reinterpret_cast<const ws_out_level*>(base + off);
    off += al8(sizeof(ws_out_level) * r.n_levels);
    s.pc = reinterpret_cast<const ws_out_piece*>(base + off);
    off += al8(sizeof(ws_out_piece) * r.n_pieces);
    s.ed = reinterpret_cast<const ws_out_edge*>(base + off);
    off += al8(sizeof(ws_out_edge) * r.n_edges);
    s.wv = reinterpret_cast<const ws_out_wave*>(base + off);
    off += al8(sizeof(ws_out_wave) * r.n_waves);
    s.en = reinterpret_cast<const ws_out_entry*>(base + off);
    off += al8(sizeof(ws_out_entry) * r.n_entries);
    s.fl = reinterpret_cast<const ws_out_flow*>(base + off);
    off += al8(sizeof(ws_out_flow) * r.n_flows);
    s.sc = reinterpret_cast<const ws_out_scope*>(base + off);
    off += al8(sizeof(ws_out_scope) * r.n_scopes);
    s.ext = reinterpret_cast<const std::uint64_t*>(base + off);
    return s;
}

const char* class_of(int code) {
    switch (code) {
        case WS_E_CYCLIC_WORKLOAD: return "CyclicWorkload";
        case WS_E_TRUTH_RANGE:
        case WS_E_NO_SOURCE:
        case WS_E_FIT_BREAKPOINT: return "ParseError";
        case WS_E_CURVE_START:
        case WS_E_CURVE_CONTIG:
        case WS_E_NO_SCHEDULABLE:
        case WS_E_NO_PROGRESS: return "InvariantError";
        case WS_E_FIT_NO_POINTS:
        case WS_E_FIT_BAD_N:
        case WS_E_FIT_BAD_TIME:
        case WS_E_FIT_PIECE_POINTS:
        case WS_E_FIT_DEGENERATE_X: return "InsufficientProfile";
        case WS_E_FIT_NONPOSITIVE: return "DegenerateFit";
        case WS_E_TP_EXCEEDS:
        case WS_E_TASK_NO_VALID: return "NoValidAllocation";
        case WS_E_EVAL_RANGE: return "OutOfRange";
        case WS_E_BT_BUDGET:
        case WS_E_NO_PLACEMENT_W0: return "PlacementInfeasible";
        default: return code >= 40 && code < 60 ? "LimitExceeded" : "Error";
    }
}

std::string module_kind(const WorkloadSpec& spec, std::int64_t index) {
    auto it = spec.modules.begin();
    std::advance(it, index);
    return it->first;
}

// plan.devices list of an entry: ascending device index starting at `rot`
// with wrap-around (the sequential ablation's rolling cursor order,
// placement.hpp:351-357; rot = 0 for the locality placer's sorted sets)
}  // namespace

[[noreturn]] void throw_result_error(const Problem& prob, const ws_plan_result& r) {
    const int N = static_cast<int>(prob.topo->devices.size());
    switch (r.err_code) {
        case WS_E_CYCLIC_WORKLOAD: throw CyclicWorkload("workload data flows form a cycle");
        case WS_E_TRUTH_RANGE: throw ParseError("truth curve does not cover the device range");
        case WS_E_CURVE_START: throw InvariantError("ScalingCurve: pieces must start at n=1");
        case WS_E_CURVE_CONTIG: throw InvariantError("ScalingCurve: pieces must be contiguous");
        case WS_E_NO_SOURCE:
            throw ParseError("module '" + module_kind(*prob.spec, r.err_a) +
                             "' has neither profile points nor a truth curve");
        case WS_E_FIT_NO_POINTS: throw InsufficientProfile("fit: no profile points");
        case WS_E_FIT_BAD_N: throw InsufficientProfile("fit: device count must be >= 1");
        case WS_E_FIT_BAD_TIME: throw InsufficientProfile("fit: non-positive time sample");
        case WS_E_FIT_BREAKPOINT:
            throw ParseError("fit: breakpoint " + std::to_string(r.err_a) + " outside point span");
        case WS_E_FIT_PIECE_POINTS:
            throw InsufficientProfile("fit: piece [" + std::to_string(r.err_a) + ", " + std::to_string(r.err_b) +
                                      "] needs points at >= 2 distinct n");
        case WS_E_FIT_DEGENERATE_X: throw InsufficientProfile("fit: points do not span distinct n");
        case WS_E_FIT_NONPOSITIVE: throw DegenerateFit("fit: non-positive T(" + std::to_string(r.err_a) + ")");
        case WS_E_TASK_NO_VALID:
            throw NoValidAllocation("task '" + prob.spec->tasks[r.err_a].id +
                                    "' has no allocation valid for all its metaops");
        case WS_E_TP_EXCEEDS:
            throw NoValidAllocation("metaop 'm" + std::to_string(r.err_a) + "': tp degree " +
                                    std::to_string(r.err_b) + " exceeds device count " + std::to_string(N));
        case WS_E_EVAL_RANGE:
            throw OutOfRange("eval_time: n=" + fmt_g(r.err_x) + " outside [1, " + fmt_g(r.err_y) + "]");
        case WS_E_NO_SCHEDULABLE: throw InvariantError("schedule_level: no schedulable tuple");
        case WS_E_NO_PROGRESS: throw InvariantError("schedule_level: wave made no progress");
        case WS_E_BT_BUDGET:
            throw PlacementInfeasible("placement backtrack budget exhausted at wave " + std::to_string(r.err_a));
        case WS_E_NO_PLACEMENT_W0: throw PlacementInfeasible("no feasible placement for wave 0");
        case WS_E_HOST_PRESET: {
            // re-run host validation to raise the original exception
            validate_workload(*prob.spec);
            if (N > WS_MAX_DEVICES) throw LimitExceeded("device count " + std::to_string(N) + " exceeds WS_MAX_DEVICES");
            if (prob.spec->modules.size() > WS_MAX_MODULES) throw LimitExceeded("module count exceeds WS_MAX_MODULES");
            throw LimitExceeded("task count exceeds WS_MAX_TASKS");
        }
        default:
            if (r.err_code >= 40 && r.err_code < 60)
                throw LimitExceeded("plan exceeds device limit (code " + std::to_string(r.err_code) + ")");
            throw Error("planner internal error (code " + std::to_string(r.err_code) + ")");
    }
}

namespace {
// Plan of a task-scoped baseline (distmm-mt): entities "m<k>@<task>" built
// like detail::scoped_entity (baselines.hpp:49-55) from the MetaOp's entity.
PlannerResult decode_scoped(const Problem& prob, const ws_plan_result& r, const Sections& s) {
    const WorkloadSpec& spec = *prob.spec;
    std::vector<const ModuleDecl*> mods;
    for (const auto& kv : spec.modules) mods.push_back(&kv.second);
    std::map<std::string, std::set<std::string>> tasks_of;  // graph.hpp:101-121
    for (const TaskDecl& t : spec.tasks)
        for (const FlowStep& st : t.flow)
            for (const FlowBranch& br : st)
                for (const std::string& m : br) tasks_of[m].insert(t.id);
    std::vector<std::string> ids(r.n_metaops);
    PlannerResult res;
    ExecutionPlan& plan = res.plan;
    plan.strategy = prob.opt.strategy == WS_STRATEGY_TASK_OPTIMUS ? "task-level-optimus" : "distmm-mt";
    plan.topo = *prob.topo;
    for (int e = 0; e < r.n_metaops; ++e) {
        const ws_out_metaop& o = s.mo[e];
        const ModuleDecl& md = *mods[o.module];
        const std::string& task = spec.tasks[s.sc[e].task].id;
        ids[e] = "m" + std::to_string(s.sc[e].metaop) + "@" + task;
        PlanEntity x;
        x.id = ids[e];
        x.kind = md.kind;
        x.length = o.length;
        x.level = o.level;
        x.tp_degree = md.tp_degree;
        x.global_batch = md.input.batch;
        const std::set<std::string>& tk = tasks_of[md.kind];
        x.batch_fraction = tk.empty() ? 1.0 : 1.0 / static_cast<double>(tk.size());  // share_fraction
        x.param_group = o.length == md.layers ? md.param_group : "";
        x.param_bytes = static_cast<std::uint64_t>(static_cast<double>(md.param_bytes) * o.length / md.layers);
        x.act_bytes = md.act_bytes;
        x.out_bytes = md.out_bytes;
        x.w = md.flops_proxy;
        x.c = md.comm_proxy;
        x.task_ids = {task};
        std::vector<CurvePiece> pieces;
        for (int i = 0; i < o.piece_count; ++i) {
            const ws_out_piece& p = s.pc[o.piece_begin + i];
            pieces.push_back({p.n_lo, p.n_hi, p.alpha, p.beta_c, p.beta_w});
        }
        plan.curves[x.id] = ScalingCurve::from_pieces(pieces, md.comm_proxy, md.flops_proxy);
        plan.entities[x.id] = std::move(x);
    }
    for (int e = 0; e < r.n_edges; ++e) plan.deps.insert({ids[s.ed[e].from], ids[s.ed[e].to]});
    plan.lower_bound = 0.0;
    plan.grad_opt_multiplier = prob.opt.grad_opt_multiplier;
    for (int w = 0; w < r.n_waves; ++w) {
        Wave wave;
        wave.index = w;
        wave.level = s.wv[w].level;
        wave.start = s.wv[w].start;
        wave.duration = s.wv[w].duration;
        for (int i = 0; i < s.wv[w].n_entries; ++i) {
            const int ei = s.wv[w].entry_begin + i;
            const ws_out_entry& e = s.en[ei];
            const std::uint64_t* ext = prob.topo->devices.size() > 64 ? s.ext + 3 * ei : nullptr;
            wave.entries.push_back({ids[e.metaop], e.n, e.layers, e.span});
            if (detail::entry_placed(e, ext)) {
                std::vector<int> devs;
                detail::entry_devices(prob.topo->devices, e, ext, devs);
                plan.devices[{w, ids[e.metaop]}] = std::move(devs);
            }
        }
        plan.schedule.waves.push_back(std::move(wave));
    }
    plan.schedule.end_time = r.end_time;
    static const char* kModes[3] = {"copy", "intra-island", "inter-island"};
    for (int f = 0; f < r.n_flows; ++f) {
        const ws_out_flow& x = s.fl[f];
        plan.flows.push_back({x.from_wave, ids[x.from_metaop], x.to_wave, ids[x.to_metaop], x.volume, kModes[x.mode]});
    }
    res.schedule = plan.schedule;
    res.predicted_makespan = r.end_time;
    return res;
}
}  // namespace

PlannerResult decode_result(const Problem& prob, const ws_plan_result& r, const std::uint8_t* arena,
                            bool build_graph) {
    if (r.status != WS_STATUS_OK) throw_result_error(prob, r);
    if (r.n_scopes > 0) return decode_scoped(prob, r, sections_of(r, arena));
    PlannerResult res;
    detail::decode_into(*prob.spec, *prob.topo, prob.opt.strategy, prob.opt.grad_opt_multiplier, r, arena,
                        build_graph, res);
    return res;
}

std::string plan_text_or_error(const Problem& prob, const ws_plan_result& r, const std::uint8_t* arena) {
    if (r.status != WS_STATUS_OK) {
        try {
            throw_result_error(prob, r);
        } catch (const std::exception& e) {
            const char* cls = class_of(r.err_code);
            if (r.err_code == WS_E_HOST_PRESET) {
                if (dynamic_cast<const CyclicWorkload*>(&e)) cls = "CyclicWorkload";
                else if (dynamic_cast<const UnknownModule*>(&e)) cls = "UnknownModule";
                else if (dynamic_cast<const EmptyWorkload*>(&e)) cls = "EmptyWorkload";
                else if (dynamic_cast<const ParseError*>(&e)) cls = "ParseError";
                else cls = "LimitExceeded";
            }
            return std::string("error ") + cls + ": " + e.what() + "\n";
        }
    }
    return write_plan(decode_result(prob, r, arena, false).plan);
}

}  // namespace wsgpu

// Arena bytes for a batch: a per-plan estimate generous for the reference's
// workload families (metaops, 2 tuples and 2 curve pieces per MetaOp, dense
// waves/flows); a plan exceeding its share is reported WS_E_ARENA_OVERFLOW and
// re-planned alone by the host wrapper with ws_arena_bound of that one plan.
// (internal) the same bound summed over plans[0, n): a pipelined chunk's share
extern "C" uint64_t wsi_arena_bound_plans(const ws_plan_rec* plans, int n) {
    uint64_t total = 0;
    for (int p = 0; p < n; ++p) total += wsi_plan_arena_bound(plans + p);
    return total;
}

extern "C" uint64_t ws_arena_bound(const ws_batch* in) { return wsi_arena_bound_plans(in->plans, in->n_plans) + 4096; }
