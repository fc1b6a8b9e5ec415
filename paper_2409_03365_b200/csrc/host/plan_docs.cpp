// plan_docs.cpp — plan files of ANY strategy (parse_plan, plan_io.hpp:112-255)
// as input to the device evaluator (k_sim: simulate_plan + validate_plan).
//
// Each ExecutionPlan becomes one batch row plus one planned record in the
// ws_abi.h layout: every PlanEntity is a module row (layers = length, tp,
// param/act bytes, w/c, batch_fraction, a param-group key id) and a MetaOp
// record whose curve pieces are the plan's curve of that entity.  Entities get
// indices whose "m<index>" spelling sorts like their ids, so the evaluator's
// id order (dec_less) is the plan's std::map order; the host keeps the real
// names for the report.  Ids referenced but not declared get indices >= K
// (validate_plan's "unknown entity").
#include <cuda_runtime_api.h>

#include <algorithm>
#include <cstring>
#include <numeric>

#include "wsgpu/planner.hpp"
#include "wsgpu/wsx.h"

namespace wsgpu {
namespace {

std::size_t a16(std::size_t v) { return (v + 15) & ~std::size_t(15); }
std::size_t a8(std::size_t v) { return (v + 7) & ~std::size_t(7); }

bool dec_less_int(int a, int b) { return "m" + std::to_string(a) < "m" + std::to_string(b); }

}  // namespace

struct PlanDocs {
    std::vector<ExecutionPlan> plans;
    std::string err;
    // encoded
    std::shared_ptr<std::uint8_t> blob;
    ws_batch view{};
    std::vector<ws_plan_result> results;
    std::vector<std::uint8_t> arena;
    std::vector<std::vector<std::string>> names;  // per plan: index -> entity id
    std::vector<int> n_known;                     // per plan: declared entities K

    void encode(bool pinned) {
        const std::size_t P = plans.size();
        std::size_t nm = 0, nd = 0;
        for (const ExecutionPlan& p : plans) {
            nm += p.entities.size();
            nd += p.topo.devices.size();
        }
        std::size_t total = a16(sizeof(ws_plan_rec) * P) + a16(4 * nm) * 5 + a16(8 * nm) * 5 + a16(4 * nd) + 64;
        std::uint8_t* raw = nullptr;
        if (pinned && cudaMallocHost(reinterpret_cast<void**>(&raw), total) == cudaSuccess) {
            blob = std::shared_ptr<std::uint8_t>(raw, [](std::uint8_t* q) { cudaFreeHost(q); });
        } else {
            if (pinned) cudaGetLastError();
            raw = static_cast<std::uint8_t*>(std::aligned_alloc(64, a16(total) + 64));
            blob = std::shared_ptr<std::uint8_t>(raw, [](std::uint8_t* q) { std::free(q); });
        }
        std::memset(raw, 0, total);
        std::size_t off = 0;
        auto carve = [&](std::size_t bytes) {
            std::uint8_t* q = raw + off;
            off = a16(off + bytes);
            return q;
        };
        auto* recs = reinterpret_cast<ws_plan_rec*>(carve(sizeof(ws_plan_rec) * P));
        auto* mod_layers = reinterpret_cast<int32_t*>(carve(4 * nm));
        auto* mod_tp = reinterpret_cast<int32_t*>(carve(4 * nm));
        auto* mod_group = reinterpret_cast<int32_t*>(carve(4 * nm));
        auto* mod_alias = reinterpret_cast<int32_t*>(carve(4 * nm));
        auto* mod_plan = reinterpret_cast<int32_t*>(carve(4 * nm));
        auto* mod_param = reinterpret_cast<uint64_t*>(carve(8 * nm));
        auto* mod_act = reinterpret_cast<uint64_t*>(carve(8 * nm));
        auto* mod_w = reinterpret_cast<double*>(carve(8 * nm));
        auto* mod_c = reinterpret_cast<double*>(carve(8 * nm));
        auto* mod_frac = reinterpret_cast<double*>(carve(8 * nm));
        auto* dev_island = reinterpret_cast<int32_t*>(carve(4 * nd));
        view = ws_batch{};
        view.n_plans = static_cast<int32_t>(P);
        view.n_modules = static_cast<int32_t>(nm);
        view.n_devices = static_cast<int32_t>(nd);
        view.blob = raw;
        view.blob_bytes = total;
        view.plans = recs;
        view.mod_layers = mod_layers;
        view.mod_tp = mod_tp;
        view.mod_group = mod_group;
        view.mod_alias = mod_alias;
        view.mod_plan = mod_plan;
        view.mod_param = mod_param;
        view.mod_act = mod_act;
        view.mod_w = mod_w;
        view.mod_c = mod_c;
        view.mod_frac = mod_frac;
        view.dev_island = dev_island;

        results.assign(P, ws_plan_result{});
        arena.clear();
        names.assign(P, {});
        n_known.assign(P, 0);
        std::size_t im = 0, id = 0;
        for (std::size_t pi = 0; pi < P; ++pi) {
            const ExecutionPlan& plan = plans[pi];
            const ClusterTopology& topo = plan.topo;
            const int K = static_cast<int>(plan.entities.size());
            const int N = static_cast<int>(topo.devices.size());
            if (N > WS_MAX_DEVICES) throw LimitExceeded("plan: more than 256 devices");
            // index of the r-th id (std::map order) = the index whose "m<index>" has rank r
            std::vector<int> perm(K);
            std::iota(perm.begin(), perm.end(), 0);
            std::sort(perm.begin(), perm.end(), dec_less_int);
            std::map<std::string, int> index;
            std::vector<std::string>& nm_of = names[pi];
            nm_of.assign(K, "");
            int r = 0;
            for (const auto& [eid, e] : plan.entities) {
                index[eid] = perm[r];
                nm_of[perm[r]] = eid;
                ++r;
            }
            auto idx = [&](const std::string& s) {
                auto it = index.find(s);
                if (it != index.end()) return it->second;
                const int k = static_cast<int>(nm_of.size());  // referenced, not declared
                index[s] = k;
                nm_of.push_back(s);
                return k;
            };
            // param-group keys (placement.hpp:134, simulate.hpp:131): param_group or the entity id
            std::map<std::string, int> keys;
            for (const auto& [eid, e] : plan.entities) keys.emplace(e.param_group.empty() ? eid : e.param_group, 0);
            int g = 0;
            for (auto& kv : keys) kv.second = g++;
            ws_plan_rec& rec = recs[pi];
            rec.mod_begin = static_cast<int32_t>(im);
            rec.n_mod = K;
            rec.dev_begin = static_cast<int32_t>(id);
            rec.n_dev = N;
            rec.n_islands = static_cast<int32_t>(topo.islands.size());
            rec.n_groups = g;
            rec.mem_capacity = topo.mem_capacity;
            rec.grad_mult = plan.grad_opt_multiplier;
            rec.intra_bw = topo.intra_bw;
            rec.inter_bw = topo.inter_bw;
            std::map<int, int> dev_index;
            for (int d = 0; d < N; ++d) {
                dev_index[topo.devices[d]] = d;
                dev_island[id + d] = topo.island_of.at(topo.devices[d]);
            }
            for (const auto& [eid, e] : plan.entities) {
                const std::size_t m = im + index.at(eid);
                const ScalingCurve& cv = plan.curves.at(eid);
                if (cv.w() != e.w || cv.c() != e.c)
                    throw ParseError("plan: entity '" + eid + "' and its curve disagree on w/c (unsupported)");
                if (static_cast<std::uint64_t>(static_cast<double>(e.param_bytes) * e.length / e.length) !=
                    e.param_bytes)
                    throw ParseError("plan: entity '" + eid + "' param_bytes beyond exact double range");
                mod_layers[m] = e.length;
                mod_tp[m] = e.tp_degree;
                mod_group[m] = keys.at(e.param_group.empty() ? eid : e.param_group);
                mod_alias[m] = -1;
                mod_plan[m] = static_cast<int32_t>(pi);
                mod_param[m] = e.param_bytes;
                mod_act[m] = e.act_bytes;
                mod_w[m] = cv.w();
                mod_c[m] = cv.c();
                mod_frac[m] = e.batch_fraction;
            }
            // record sections
            std::vector<ws_out_metaop> mo(K);
            std::vector<ws_out_piece> pc;
            for (const auto& [eid, e] : plan.entities) {
                const int k = index.at(eid);
                ws_out_metaop& o = mo[k];
                o = ws_out_metaop{};
                o.module = k;
                o.level = e.level;
                o.length = e.length;
                o.piece_begin = static_cast<int32_t>(pc.size());
                for (const CurvePiece& q : plan.curves.at(eid).pieces())
                    pc.push_back({q.n_lo, q.n_hi, q.alpha, q.beta_c, q.beta_w});
                o.piece_count = static_cast<int32_t>(pc.size()) - o.piece_begin;
            }
            std::vector<ws_out_edge> ed;
            for (const auto& [a, b] : plan.deps) ed.push_back({idx(a), idx(b)});
            std::vector<ws_out_wave> wv;
            std::vector<ws_out_entry> en;
            std::vector<std::uint64_t> ext;  // device words 1..3 per entry (N > 64, ws_abi.h)
            for (std::size_t w = 0; w < plan.schedule.waves.size(); ++w) {
                const Wave& wave = plan.schedule.waves[w];
                if (wave.index != static_cast<int>(w))
                    throw ParseError("plan: wave indices must follow file order (unsupported)");
                ws_out_wave x{};
                x.start = wave.start;
                x.duration = wave.duration;
                x.level = wave.level;
                x.entry_begin = static_cast<int32_t>(en.size());
                x.n_entries = static_cast<int32_t>(wave.entries.size());
                wv.push_back(x);
                for (const WaveEntry& e : wave.entries) {
                    ws_out_entry y{};
                    std::uint64_t w[4] = {0, 0, 0, 0};
                    y.span = e.span;
                    y.metaop = idx(e.metaop_id);
                    y.n = e.n;
                    y.layers = e.layers;
                    auto it = plan.devices.find({wave.index, e.metaop_id});
                    if (it != plan.devices.end() && !it->second.empty()) {
                        for (std::size_t i = 0; i < it->second.size(); ++i) {
                            auto di = dev_index.find(it->second[i]);
                            if (di == dev_index.end())
                                throw ParseError("plan: device " + std::to_string(it->second[i]) +
                                                 " not in the topology (unsupported)");
                            const int d = di->second;
                            if (w[d / 64] >> (d % 64) & 1ull)
                                throw ParseError("plan: device listed twice in one entry (unsupported)");
                            w[d / 64] |= 1ull << (d % 64);
                            if (i == 0) y.rot = d;  // lists are ascending from their first device
                        }
                    }
                    y.devmask = w[0];
                    en.push_back(y);
                    if (N > 64) ext.insert(ext.end(), w + 1, w + 4);
                }
            }
            std::vector<ws_out_flow> fl;
            for (const Flow& f : plan.flows) {
                ws_out_flow x{};
                x.volume = f.volume;
                x.from_wave = f.from_wave;
                x.from_metaop = idx(f.from_id);
                x.to_wave = f.to_wave;
                x.to_metaop = idx(f.to_id);
                x.mode = f.mode == "copy" ? WS_FLOW_COPY : (f.mode == "inter-island" ? WS_FLOW_INTER : WS_FLOW_INTRA);
                fl.push_back(x);
            }
            if (static_cast<int>(nm_of.size()) > WS_MAX_MODULES)
                throw LimitExceeded("plan: more than 64 entities");
            n_known[pi] = K;
            ws_plan_result& res = results[pi];
            res.status = WS_STATUS_OK;
            res.n_metaops = K;
            res.n_edges = static_cast<int32_t>(ed.size());
            res.n_levels = 0;
            res.n_waves = static_cast<int32_t>(wv.size());
            res.n_entries = static_cast<int32_t>(en.size());
            res.n_flows = static_cast<int32_t>(fl.size());
            res.n_pieces = static_cast<int32_t>(pc.size());
            res.lower_bound = plan.lower_bound;
            res.end_time = plan.schedule.end_time;
            res.offset = arena.size();
            auto put = [&](const void* src, std::size_t bytes) {
                const std::size_t at = arena.size();
                arena.resize(at + a8(bytes), 0);
                if (bytes) std::memcpy(arena.data() + at, src, bytes);
            };
            put(mo.data(), sizeof(ws_out_metaop) * mo.size());
            put(pc.data(), sizeof(ws_out_piece) * pc.size());
            put(ed.data(), sizeof(ws_out_edge) * ed.size());
            put(wv.data(), sizeof(ws_out_wave) * wv.size());
            put(en.data(), sizeof(ws_out_entry) * en.size());
            put(fl.data(), sizeof(ws_out_flow) * fl.size());
            put(ext.data(), sizeof(std::uint64_t) * ext.size());
            res.size = arena.size() - res.offset;
            im += K;
            id += N;
        }
        if (arena.empty()) arena.resize(8, 0);
    }
};

}  // namespace wsgpu

using wsgpu::PlanDocs;

struct wsx_plans : PlanDocs {};

extern "C" {

wsx_plans* wsx_plans_new(void) { return new wsx_plans(); }
void wsx_plans_free(wsx_plans* p) { delete p; }
int32_t wsx_plans_size(const wsx_plans* p) { return static_cast<int32_t>(p->plans.size()); }
const char* wsx_plans_error(const wsx_plans* p) { return p->err.c_str(); }

int32_t wsx_plans_add_text(wsx_plans* p, const char* plan_text) {
    try {
        p->plans.push_back(wsgpu::parse_plan(plan_text));
        return static_cast<int32_t>(p->plans.size()) - 1;
    } catch (const std::exception& e) {
        p->err = e.what();
        return -1;
    }
}

const ws_batch* wsx_plans_encode(wsx_plans* p, int32_t pinned, const ws_plan_result** results,
                                 const uint8_t** arena, uint64_t* arena_bytes) {
    try {
        p->encode(pinned != 0);
    } catch (const std::exception& e) {
        p->err = e.what();
        return nullptr;
    }
    *results = p->results.data();
    *arena = p->arena.data();
    *arena_bytes = p->arena.size();
    return &p->view;
}

char* wsx_plans_write(const wsx_plans* p, int32_t i) {
    const std::string s = wsgpu::write_plan(p->plans[i]);
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}

char* wsx_plans_sim_text(const wsx_plans* p, int32_t i, const ws_sim_result* sims, const uint8_t* sim_arena) {
    std::string s;
    try {
        s = wsgpu::sim_text_named(p->plans[i].topo, p->results[i], sims[i], sim_arena, p->names[i]);
    } catch (const std::exception& e) {
        s = std::string("error DecodeFailure: ") + e.what() + "\n";
    }
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
}

}  // extern "C"
