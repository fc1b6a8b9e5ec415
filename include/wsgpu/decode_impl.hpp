// decode_impl.hpp — ws_plan_result + arena record -> PlannerResult, as a
// template over the result types (internal; included by the library's
// decode.cpp for the wsgpu mirror types and by wavesched_compat.hpp for the
// reference's own wavesched:: types, so the reference-typed drop-in decodes
// straight into the caller's types with no intermediate copy).
//
// Rebuilds the string-keyed objects of planner.hpp:29-38 / :196-210 and
// build_entities (planner.hpp:99-122) from the device's index-based record.
// The maps are filled in key order with end() hints (one comparison per
// insert instead of a tree search), which is what makes this cheaper than
// building them the way the reference does.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "wsgpu/ws_abi.h"

namespace wsgpu::detail {

inline std::size_t rec_al8(std::size_t v) { return (v + 7) & ~std::size_t(7); }

// Section pointers of one plan record (ws_abi.h "Arena record" order).
struct RecordView {
    const ws_out_metaop* mo;
    const ws_out_level* lv;
    const ws_out_piece* pc;
    const ws_out_edge* ed;
    const ws_out_wave* wv;
    const ws_out_entry* en;
    const ws_out_flow* fl;
    const ws_out_scope* sc;
    const uint64_t* ext;  // device words 1..3 per entry (clusters of more than 64 devices)
};

inline RecordView record_view(const ws_plan_result& r, const std::uint8_t* arena) {
    const std::uint8_t* base = arena + r.offset;
    std::size_t off = 0;
    RecordView s{};
    s.mo = reinterpret_cast<const ws_out_metaop*>(base + off);
    off += rec_al8(sizeof(ws_out_metaop) * r.n_metaops);
    s.lv = reinterpret_cast<const ws_out_level*>(base + off);
    off += rec_al8(sizeof(ws_out_level) * r.n_levels);
    s.pc = reinterpret_cast<const ws_out_piece*>(base + off);
    off += rec_al8(sizeof(ws_out_piece) * r.n_pieces);
    s.ed = reinterpret_cast<const ws_out_edge*>(base + off);
    off += rec_al8(sizeof(ws_out_edge) * r.n_edges);
    s.wv = reinterpret_cast<const ws_out_wave*>(base + off);
    off += rec_al8(sizeof(ws_out_wave) * r.n_waves);
    s.en = reinterpret_cast<const ws_out_entry*>(base + off);
    off += rec_al8(sizeof(ws_out_entry) * r.n_entries);
    s.fl = reinterpret_cast<const ws_out_flow*>(base + off);
    off += rec_al8(sizeof(ws_out_flow) * r.n_flows);
    s.sc = reinterpret_cast<const ws_out_scope*>(base + off);
    off += rec_al8(sizeof(ws_out_scope) * r.n_scopes);
    s.ext = reinterpret_cast<const uint64_t*>(base + off);
    return s;
}

// indices 0..n-1 ordered by keys[i] (std::string order, i.e. std::map order)
inline std::vector<int> key_order(const std::vector<std::string>& keys) {
    std::vector<int> o(keys.size());
    for (std::size_t i = 0; i < o.size(); ++i) o[i] = static_cast<int>(i);
    std::sort(o.begin(), o.end(), [&](int a, int b) { return keys[a] < keys[b]; });
    return o;
}

// plan.devices list of an entry: ascending device index starting at `rot`
// with wrap-around (the sequential ablation's rolling cursor order,
// placement.hpp:351-357; rot = 0 for the locality placer's sorted sets)
// ext: the entry's device words 1..3 (clusters of more than 64 devices), else null
inline void entry_devices(const std::vector<int>& devs, const ws_out_entry& e, const uint64_t* ext,
                          std::vector<int>& out) {
    const int N = static_cast<int>(devs.size());
    out.clear();
    for (int i = 0; i < N; ++i) {
        const int d = (e.rot + i) % N;
        const uint64_t word = d < 64 ? e.devmask : ext[d / 64 - 1];
        if (word >> (d & 63) & 1ull) out.push_back(devs[d]);
    }
}

// any device in the entry's set (0: not placed)
inline bool entry_placed(const ws_out_entry& e, const uint64_t* ext) {
    return e.devmask || (ext && (ext[0] | ext[1] | ext[2]));
}

// Decodes a successful (status OK, not task-scoped) record into `res`.
// Spec/Topo/Result: the wsgpu mirror types or the reference's wavesched:: types.
template <class Spec, class Topo, class Result>
void decode_into(const Spec& spec, const Topo& topo, int strategy, double grad_mult, const ws_plan_result& r,
                 const std::uint8_t* arena, bool build_graph, Result& res) {
    using MetaOpT = typename decltype(res.meta.metaops)::mapped_type;
    using OperatorT = typename decltype(res.graph.operators)::mapped_type;
    using CurveT = typename decltype(res.curves)::mapped_type;
    using PieceT = typename std::decay_t<decltype(std::declval<const CurveT&>().pieces())>::value_type;
    using AllocT = typename decltype(res.level_plans)::value_type;
    using TuplePairT = typename decltype(std::declval<AllocT&>().tuples)::mapped_type;
    using AslT = decltype(std::declval<TuplePairT&>().upper);
    using WaveT = typename decltype(res.schedule.waves)::value_type;
    using EntryT = typename decltype(std::declval<WaveT&>().entries)::value_type;
    using EntityT = typename decltype(res.plan.entities)::mapped_type;
    using FlowT = typename decltype(res.plan.flows)::value_type;
    using ModuleT = typename std::decay_t<decltype(spec.modules)>::mapped_type;
    using StrSet = std::set<std::string>;

    const RecordView s = record_view(r, arena);
    const int K = r.n_metaops;
    const bool wide = topo.devices.size() > 64;
    std::vector<const ModuleT*> mods;
    mods.reserve(spec.modules.size());
    for (const auto& kv : spec.modules) mods.push_back(&kv.second);

    // tasks routing through each module (graph.hpp:101-121), per module index
    std::map<std::string, StrSet> tasks_by_kind;
    for (const auto& t : spec.tasks)
        for (const auto& st : t.flow)
            for (const auto& br : st)
                for (const std::string& m : br) tasks_by_kind[m].insert(t.id);
    std::vector<const StrSet*> tasks_of(mods.size());
    static const StrSet kNone;
    for (std::size_t i = 0; i < mods.size(); ++i) {
        auto it = tasks_by_kind.find(mods[i]->kind);
        tasks_of[i] = it == tasks_by_kind.end() ? &kNone : &it->second;
    }

    std::vector<std::string> ids(K);
    for (int k = 0; k < K; ++k) ids[k] = "m" + std::to_string(k);
    const std::vector<int> by_id = key_order(ids);  // MetaOps in map order

    // MetaOps + curves (map order, hinted inserts)
    std::vector<std::vector<std::string>> members(K);
    for (int k = 0; k < K; ++k) {
        const ws_out_metaop& o = s.mo[k];
        const std::string& kind = mods[o.module]->kind;
        members[k].reserve(o.length);
        for (int l = 0; l < o.length; ++l) members[k].push_back(kind + "." + std::to_string(o.first_layer + l));
    }
    for (int k : by_id) {
        const ws_out_metaop& o = s.mo[k];
        const ModuleT& md = *mods[o.module];
        MetaOpT m;
        m.id = ids[k];
        m.member_ops = members[k];
        m.length = o.length;
        m.kind = md.kind;
        m.input = md.input;
        m.global_batch = md.input.batch;
        m.tp_degree = md.tp_degree;
        m.level = o.level;
        m.param_group = md.param_group;
        m.task_ids = *tasks_of[o.module];
        std::vector<PieceT> pieces(o.piece_count);
        for (int i = 0; i < o.piece_count; ++i) {
            const ws_out_piece& p = s.pc[o.piece_begin + i];
            pieces[i].n_lo = p.n_lo;
            pieces[i].n_hi = p.n_hi;
            pieces[i].alpha = p.alpha;
            pieces[i].beta_c = p.beta_c;
            pieces[i].beta_w = p.beta_w;
        }
        res.curves.emplace_hint(res.curves.end(), ids[k], CurveT::from_pieces(pieces, md.comm_proxy, md.flops_proxy));
        res.meta.metaops.emplace_hint(res.meta.metaops.end(), ids[k], std::move(m));
    }
    {
        std::vector<std::pair<std::string, std::string>> e;
        e.reserve(r.n_edges);
        for (int i = 0; i < r.n_edges; ++i) e.emplace_back(ids[s.ed[i].from], ids[s.ed[i].to]);
        std::sort(e.begin(), e.end());
        for (auto& x : e) res.meta.edges.emplace_hint(res.meta.edges.end(), std::move(x));
    }
    int n_meta_levels = r.n_levels;  // the baselines carry MetaOp levels but no level plans
    for (int k = 0; k < K; ++k) n_meta_levels = std::max(n_meta_levels, s.mo[k].level + 1);
    res.meta.levels.assign(n_meta_levels, {});
    for (int k : by_id) res.meta.levels[s.mo[k].level].push_back(ids[k]);

    if (build_graph) {  // one operator per member layer, shared by the MetaOp's tasks
        std::vector<std::pair<const std::string*, int>> ops;
        for (int k = 0; k < K; ++k)
            for (const std::string& op : members[k]) ops.emplace_back(&op, k);
        std::sort(ops.begin(), ops.end(), [](const auto& a, const auto& b) { return *a.first < *b.first; });
        for (const auto& [op, k] : ops) {
            const ModuleT& md = *mods[s.mo[k].module];
            OperatorT x;
            x.id = *op;
            x.kind = md.kind;
            x.task_ids = *tasks_of[s.mo[k].module];
            x.input = md.input;
            x.tp_degree = md.tp_degree;
            x.param_group = md.param_group;
            res.graph.operators.emplace_hint(res.graph.operators.end(), *op, std::move(x));
        }
        std::vector<std::pair<const std::string*, const std::string*>> e;
        for (int k = 0; k < K; ++k)
            for (std::size_t i = 1; i < members[k].size(); ++i) e.emplace_back(&members[k][i - 1], &members[k][i]);
        for (int i = 0; i < r.n_edges; ++i)
            e.emplace_back(&members[s.ed[i].from].back(), &members[s.ed[i].to].front());
        std::sort(e.begin(), e.end(), [](const auto& a, const auto& b) {
            const int c = a.first->compare(*b.first);
            return c < 0 || (c == 0 && *a.second < *b.second);
        });
        for (const auto& [a, b] : e) res.graph.edges.emplace_hint(res.graph.edges.end(), *a, *b);
    }

    for (int l = 0; l < r.n_levels; ++l) {
        AllocT ap;
        ap.level = l;
        ap.c_star = s.lv[l].c_star;
        for (const std::string& id : res.meta.levels[l]) {
            const ws_out_metaop& o = s.mo[std::stoi(id.substr(1))];
            TuplePairT tp;
            tp.upper.metaop_id = id;
            tp.upper.n = o.upper_n;
            tp.upper.start = -1.0;
            tp.upper.layers = o.upper_l;
            if (o.lower_l > 0) {
                AslT lo;
                lo.metaop_id = id;
                lo.n = o.lower_n;
                lo.start = -1.0;
                lo.layers = o.lower_l;
                tp.lower = lo;
            }
            ap.tuples.emplace_hint(ap.tuples.end(), id, std::move(tp));
        }
        res.level_plans.push_back(std::move(ap));
        res.schedule.level_boundaries.push_back(s.lv[l].first_wave);
    }
    auto& plan = res.plan;
    std::vector<int> devs;
    for (int w = 0; w < r.n_waves; ++w) {
        WaveT wave;
        wave.index = w;
        wave.level = s.wv[w].level;
        wave.start = s.wv[w].start;
        wave.duration = s.wv[w].duration;
        wave.entries.resize(s.wv[w].n_entries);
        std::vector<int> placed;  // entries placed in this wave, in id order for hinted inserts
        for (int i = 0; i < s.wv[w].n_entries; ++i) {
            const ws_out_entry& e = s.en[s.wv[w].entry_begin + i];
            EntryT& x = wave.entries[i];
            x.metaop_id = ids[e.metaop];
            x.n = e.n;
            x.layers = e.layers;
            x.span = e.span;
            if (entry_placed(e, wide ? s.ext + 3 * (s.wv[w].entry_begin + i) : nullptr))  // else: not placed
                placed.push_back(s.wv[w].entry_begin + i);
        }
        std::sort(placed.begin(), placed.end(), [&](int a, int b) { return ids[s.en[a].metaop] < ids[s.en[b].metaop]; });
        for (int i : placed) {
            entry_devices(topo.devices, s.en[i], wide ? s.ext + 3 * i : nullptr, devs);
            plan.devices.emplace_hint(plan.devices.end(), std::make_pair(w, ids[s.en[i].metaop]), devs);
        }
        res.schedule.waves.push_back(std::move(wave));
    }
    res.schedule.end_time = r.end_time;
    res.lower_bound = r.lower_bound;
    res.predicted_makespan = r.end_time;

    plan.strategy = strategy == WS_STRATEGY_DECOUPLED_SEQUENTIAL ? "decoupled-sequential" : "wavefront";
    plan.topo = topo;
    for (int k : by_id) {  // build_entities (planner.hpp:99-122)
        const ws_out_metaop& o = s.mo[k];
        const ModuleT& md = *mods[o.module];
        EntityT e;
        e.id = ids[k];
        e.kind = md.kind;
        e.length = o.length;
        e.level = o.level;
        e.tp_degree = md.tp_degree;
        e.global_batch = md.input.batch;
        e.batch_fraction = 1.0;
        e.param_group = o.length == md.layers ? md.param_group : "";
        e.param_bytes = static_cast<std::uint64_t>(static_cast<double>(md.param_bytes) * o.length / md.layers);
        e.act_bytes = md.act_bytes;
        e.out_bytes = md.out_bytes;
        e.w = md.flops_proxy;
        e.c = md.comm_proxy;
        e.task_ids = *tasks_of[o.module];
        plan.entities.emplace_hint(plan.entities.end(), ids[k], std::move(e));
    }
    plan.curves = res.curves;
    plan.deps = res.meta.edges;
    plan.schedule = res.schedule;
    plan.lower_bound = res.lower_bound;
    plan.grad_opt_multiplier = grad_mult;
    static const char* kModes[3] = {"copy", "intra-island", "inter-island"};
    plan.flows.resize(r.n_flows);
    for (int f = 0; f < r.n_flows; ++f) {
        const ws_out_flow& x = s.fl[f];
        FlowT& y = plan.flows[f];
        y.from_wave = x.from_wave;
        y.from_id = ids[x.from_metaop];
        y.to_wave = x.to_wave;
        y.to_id = ids[x.to_metaop];
        y.volume = x.volume;
        y.mode = kModes[x.mode];
    }
}

}  // namespace wsgpu::detail
