// wavesched_compat.hpp — drop-in for projects that keep the reference types.
//
// Include AFTER the reference's "wavesched/planner.hpp".  Provides
//   wavesched_gpu::plan_workload(const wavesched::WorkloadSpec&,
//                                const wavesched::ClusterTopology&,
//                                const wavesched::PlannerOptions& = {})
//       -> wavesched::PlannerResult
// with the reference signature (planner.hpp:156-157): reentrant (concurrent
// callers plan in parallel on pooled contexts), the device record decoded
// straight into the reference's types (decode_impl.hpp), and the reference's
// own exception classes (common.hpp:20-60) rethrown with the same what() text.
// plan_workloads / plan_workloads_each plan many problems in one device batch
// with the decode spread over host threads.
// Link with paper_2409_03365_b200/lib/libwsgpu.so.
#pragma once

#include <algorithm>
#include <atomic>
#include <thread>

#include "wsgpu/decode_impl.hpp"
#include "wsgpu/planner.hpp"

namespace wavesched_gpu {

namespace detail {

inline wsgpu::WorkloadSpec to_mirror(const wavesched::WorkloadSpec& s) {
    wsgpu::WorkloadSpec o;
    for (const auto& [kind, m] : s.modules) {
        wsgpu::ModuleDecl d;
        d.kind = m.kind;
        d.layers = m.layers;
        d.input = {m.input.batch, m.input.seq, m.input.hidden};
        d.tp_degree = m.tp_degree;
        d.param_group = m.param_group;
        d.param_bytes = m.param_bytes;
        d.flops_proxy = m.flops_proxy;
        d.comm_proxy = m.comm_proxy;
        d.act_bytes = m.act_bytes;
        d.out_bytes = m.out_bytes;
        o.modules.emplace(kind, d);
    }
    for (const auto& t : s.tasks) o.tasks.push_back({t.id, t.flow, t.flow_text});
    for (const auto& [kind, pieces] : s.truth)
        for (const auto& p : pieces) o.truth[kind].push_back({p.n_lo, p.n_hi, p.alpha, p.beta_c, p.beta_w});
    for (const auto& [kind, pts] : s.profiles)
        for (const auto& p : pts) o.profiles[kind].push_back({p.n, p.time, p.parallel_config});
    o.breakpoints = s.breakpoints;
    return o;
}

inline wsgpu::ClusterTopology to_mirror(const wavesched::ClusterTopology& t) {
    wsgpu::ClusterTopology o;
    o.devices = t.devices;
    o.islands = t.islands;
    o.island_of = t.island_of;
    o.intra_bw = t.intra_bw;
    o.inter_bw = t.inter_bw;
    o.mem_capacity = t.mem_capacity;
    return o;
}

inline wsgpu::PlannerOptions to_mirror(const wavesched::PlannerOptions& p) {
    wsgpu::PlannerOptions o;
    o.alloc.eps = p.alloc.eps;
    o.alloc.max_iters = p.alloc.max_iters;
    o.alloc.drop_floor = p.alloc.drop_floor;
    o.placement.sequential = p.placement.sequential;
    o.placement.backtrack_depth = p.placement.backtrack_depth;
    o.placement.backtrack_branching = p.placement.backtrack_branching;
    o.grad_opt_multiplier = p.grad_opt_multiplier;
    o.synth_noise = p.synth_noise;
    o.synth_seed = p.synth_seed;
    return o;
}

inline wavesched::ScalingCurve to_ref(const wsgpu::ScalingCurve& c) {
    std::vector<wavesched::CurvePiece> pieces;
    for (const auto& p : c.pieces()) pieces.push_back({p.n_lo, p.n_hi, p.alpha, p.beta_c, p.beta_w});
    return wavesched::ScalingCurve::from_pieces(pieces, c.c(), c.w());
}

inline wavesched::InputSize to_ref(const wsgpu::InputSize& i) { return {i.batch, i.seq, i.hidden}; }

inline wavesched::WavefrontSchedule to_ref(const wsgpu::WavefrontSchedule& s) {
    wavesched::WavefrontSchedule o;
    for (const auto& w : s.waves) {
        wavesched::Wave x;
        x.index = w.index;
        x.level = w.level;
        x.start = w.start;
        x.duration = w.duration;
        for (const auto& e : w.entries) x.entries.push_back({e.metaop_id, e.n, e.layers, e.span});
        o.waves.push_back(std::move(x));
    }
    o.end_time = s.end_time;
    o.level_boundaries = s.level_boundaries;
    return o;
}

inline wavesched::PlannerResult to_ref(const wsgpu::PlannerResult& r, const wavesched::ClusterTopology& topo) {
    wavesched::PlannerResult o;
    for (const auto& [id, op] : r.graph.operators) {
        wavesched::Operator x;
        x.id = op.id;
        x.kind = op.kind;
        x.task_ids = op.task_ids;
        x.input = to_ref(op.input);
        x.tp_degree = op.tp_degree;
        x.param_group = op.param_group;
        o.graph.operators.emplace(id, std::move(x));
    }
    o.graph.edges = r.graph.edges;
    for (const auto& [id, m] : r.meta.metaops) {
        wavesched::MetaOp x;
        x.id = m.id;
        x.member_ops = m.member_ops;
        x.length = m.length;
        x.kind = m.kind;
        x.input = to_ref(m.input);
        x.global_batch = m.global_batch;
        x.tp_degree = m.tp_degree;
        x.level = m.level;
        x.param_group = m.param_group;
        x.task_ids = m.task_ids;
        o.meta.metaops.emplace(id, std::move(x));
    }
    o.meta.edges = r.meta.edges;
    o.meta.levels = r.meta.levels;
    for (const auto& [id, c] : r.curves) o.curves.emplace(id, to_ref(c));
    for (const auto& lp : r.level_plans) {
        wavesched::AllocationPlan x;
        x.level = lp.level;
        x.c_star = lp.c_star;
        for (const auto& [id, tp] : lp.tuples) {
            wavesched::TuplePair y;
            y.upper = {tp.upper.metaop_id, tp.upper.n, tp.upper.start, tp.upper.layers};
            if (tp.lower) y.lower = wavesched::AslTuple{tp.lower->metaop_id, tp.lower->n, tp.lower->start, tp.lower->layers};
            x.tuples.emplace(id, y);
        }
        o.level_plans.push_back(std::move(x));
    }
    o.schedule = to_ref(r.schedule);
    wavesched::ExecutionPlan& p = o.plan;
    p.strategy = r.plan.strategy;
    p.topo = topo;
    for (const auto& [id, e] : r.plan.entities) {
        wavesched::PlanEntity x;
        x.id = e.id;
        x.kind = e.kind;
        x.length = e.length;
        x.level = e.level;
        x.tp_degree = e.tp_degree;
        x.global_batch = e.global_batch;
        x.batch_fraction = e.batch_fraction;
        x.param_group = e.param_group;
        x.param_bytes = e.param_bytes;
        x.act_bytes = e.act_bytes;
        x.out_bytes = e.out_bytes;
        x.w = e.w;
        x.c = e.c;
        x.task_ids = e.task_ids;
        p.entities.emplace(id, std::move(x));
    }
    for (const auto& [id, c] : r.plan.curves) p.curves.emplace(id, to_ref(c));
    p.deps = r.plan.deps;
    p.schedule = to_ref(r.plan.schedule);
    p.devices = r.plan.devices;
    for (const auto& f : r.plan.flows) p.flows.push_back({f.from_wave, f.from_id, f.to_wave, f.to_id, f.volume, f.mode});
    p.lower_bound = r.plan.lower_bound;
    p.grad_opt_multiplier = r.plan.grad_opt_multiplier;
    o.lower_bound = r.lower_bound;
    o.predicted_makespan = r.predicted_makespan;
    return o;
}

// rethrow a wsgpu exception as the reference class with the same message
[[noreturn]] inline void rethrow_as_reference(const std::exception& e) {
    const std::string w = e.what();
    if (dynamic_cast<const wsgpu::CyclicWorkload*>(&e)) throw wavesched::CyclicWorkload(w);
    if (dynamic_cast<const wsgpu::UnknownModule*>(&e)) throw wavesched::UnknownModule(w);
    if (dynamic_cast<const wsgpu::EmptyWorkload*>(&e)) throw wavesched::EmptyWorkload(w);
    if (dynamic_cast<const wsgpu::InsufficientProfile*>(&e)) throw wavesched::InsufficientProfile(w);
    if (dynamic_cast<const wsgpu::ParseError*>(&e)) throw wavesched::ParseError(w);
    if (dynamic_cast<const wsgpu::DegenerateFit*>(&e)) throw wavesched::DegenerateFit(w);
    if (dynamic_cast<const wsgpu::NoValidAllocation*>(&e)) throw wavesched::NoValidAllocation(w);
    if (dynamic_cast<const wsgpu::PlacementInfeasible*>(&e)) throw wavesched::PlacementInfeasible(w);
    if (dynamic_cast<const wsgpu::InfeasibleError*>(&e)) throw wavesched::InfeasibleError(w);
    if (dynamic_cast<const wsgpu::OutOfRange*>(&e)) throw wavesched::OutOfRange(w);
    if (dynamic_cast<const wsgpu::EmptyLevel*>(&e)) throw wavesched::EmptyLevel(w);
    if (dynamic_cast<const wsgpu::InvariantError*>(&e)) throw wavesched::InvariantError(w);
    throw wavesched::Error(w);
}

}  // namespace detail

inline wavesched::PlannerResult plan_workload(const wavesched::WorkloadSpec& spec,
                                              const wavesched::ClusterTopology& topo,
                                              const wavesched::PlannerOptions& opt = {}) {
    const wsgpu::WorkloadSpec s = detail::to_mirror(spec);
    const wsgpu::ClusterTopology t = detail::to_mirror(topo);
    const wsgpu::PlannerOptions o = detail::to_mirror(opt);
    wavesched::PlannerResult out;
    try {
        wsgpu::plan_workload_raw(s, t, o, [&](const ws_plan_result& r, const std::uint8_t* arena) {
            if (r.status != WS_STATUS_OK) wsgpu::throw_result_error(wsgpu::Problem{&s, &t, o}, r);
            wsgpu::detail::decode_into(spec, topo, WS_STRATEGY_WAVEFRONT, opt.grad_opt_multiplier, r, arena, true, out);
        });
    } catch (const wsgpu::Error& e) {
        detail::rethrow_as_reference(e);
    }
    return out;
}

// plan_workload over many (spec, topology) pairs in ONE device batch, with the
// conversion and the decode into the reference's types spread over `threads`
// host threads (0 = all cores).  Streaming form: `each(i, result, error)` is
// called on a worker thread for every problem as soon as its result is
// decoded (error: the reference exception plan_workload would have thrown),
// so a consumer that keeps only what it needs never holds every PlannerResult.
template <typename Each>
void plan_workloads_each(
    const std::vector<std::pair<const wavesched::WorkloadSpec*, const wavesched::ClusterTopology*>>& problems,
    const wavesched::PlannerOptions& opt, int threads, Each&& each) {
    const std::size_t P = problems.size();
    if (threads <= 0) threads = std::max(1u, std::thread::hardware_concurrency());
    auto par = [&](auto&& fn) {
        std::atomic<std::size_t> next{0};
        auto work = [&] {
            for (std::size_t i; (i = next.fetch_add(16)) < P;)
                for (std::size_t j = i; j < std::min(P, i + 16); ++j) fn(j);
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < threads && static_cast<std::size_t>(t) * 16 < P; ++t) pool.emplace_back(work);
        work();
        for (auto& th : pool) th.join();
    };
    std::vector<wsgpu::WorkloadSpec> specs(P);
    std::vector<wsgpu::ClusterTopology> topos(P);
    par([&](std::size_t i) {
        specs[i] = detail::to_mirror(*problems[i].first);
        topos[i] = detail::to_mirror(*problems[i].second);
    });
    const wsgpu::PlannerOptions o = detail::to_mirror(opt);
    std::vector<wsgpu::Problem> probs(P);
    for (std::size_t i = 0; i < P; ++i) probs[i] = wsgpu::Problem{&specs[i], &topos[i], o};
    wsgpu::plan_workloads_raw(probs, threads, [&](const ws_plan_result* res, const std::uint8_t* arena) {
        par([&](std::size_t i) {
            wavesched::PlannerResult r;
            std::exception_ptr err;
            try {
                try {
                    if (res[i].status != WS_STATUS_OK) wsgpu::throw_result_error(probs[i], res[i]);
                    wsgpu::detail::decode_into(*problems[i].first, *problems[i].second, WS_STRATEGY_WAVEFRONT,
                                               opt.grad_opt_multiplier, res[i], arena, true, r);
                } catch (const wsgpu::Error& e) {
                    detail::rethrow_as_reference(e);
                }
            } catch (...) {
                err = std::current_exception();
            }
            each(i, std::move(r), err);
            specs[i] = {};  // release the converted inputs on the worker threads too
            topos[i] = {};
        });
    });
}

// The same, collecting every outcome.
struct Outcome {
    wavesched::PlannerResult result;
    std::exception_ptr error;
};

inline std::vector<Outcome> plan_workloads(
    const std::vector<std::pair<const wavesched::WorkloadSpec*, const wavesched::ClusterTopology*>>& problems,
    const wavesched::PlannerOptions& opt = {}, int threads = 0) {
    std::vector<Outcome> out(problems.size());
    plan_workloads_each(problems, opt, threads, [&](std::size_t i, wavesched::PlannerResult&& r, std::exception_ptr e) {
        out[i].result = std::move(r);
        out[i].error = e;
    });
    return out;
}

}  // namespace wavesched_gpu
