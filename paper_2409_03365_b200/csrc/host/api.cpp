// api.cpp — the C++ drop-in plan_workload (planner.hpp:156-212) over the
// C-ABI, and the wsx.h helper API used by FFI callers.
#include <cuda_runtime_api.h>

#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>

#include "internal.hpp"
#include "wsgpu/planner.hpp"
#include "wsgpu/wsx.h"

namespace wsgpu {
namespace {

PlannerOptions from_c(const ws_options* o) {
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
    p.strategy = o->strategy;
    return p;
}

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

// Process-wide default context for the drop-in call (one per process,
// serialized; batch users create their own ws_ctx per thread/GPU).
struct DefaultCtx {
    std::mutex mu;
    ws_ctx* ctx = nullptr;
    std::string error;
    ws_ctx* get() {
        if (!ctx) {
            const char* env = std::getenv("WSGPU_DEVICE");
            const int dev = env ? std::atoi(env) : 0;
            if (ws_ctx_create(dev, &ctx) != 0) {
                ctx = nullptr;
                error = "CUDA planner unavailable (ws_ctx_create failed on device " + std::to_string(dev) + ")";
            }
        }
        return ctx;
    }
};

DefaultCtx& default_ctx() {
    static DefaultCtx d;
    return d;
}

}  // namespace

namespace detail {

Planned plan_on(ws_ctx* ctx, const std::vector<Problem>& probs) {
    Planned out;
    EncodedBatch eb = encode_batch(probs, true);
    out.res.resize(probs.size());
    std::uint64_t cap = ws_arena_bound(&eb.view), used = 0;
    out.arena.resize(cap);
    if (ws_plan_batch_host(ctx, &eb.view, out.res.data(), out.arena.data(), cap, &used, nullptr) != 0)
        throw Error(std::string("CUDA planner failed: ") + ws_ctx_last_error(ctx));
    out.arena.resize(used);
    for (std::size_t i = 0; i < probs.size(); ++i) {
        if (out.res[i].err_code != WS_E_ARENA_OVERFLOW) continue;
        EncodedBatch one = encode_batch({probs[i]}, true);
        const std::uint64_t big = std::uint64_t(64) << 20;
        std::vector<std::uint8_t> ar(big);
        ws_plan_result r{};
        std::uint64_t u = 0;
        if (ws_plan_batch_host(ctx, &one.view, &r, ar.data(), big, &u, nullptr) != 0)
            throw Error(std::string("CUDA planner failed: ") + ws_ctx_last_error(ctx));
        r.offset += out.arena.size();
        out.arena.insert(out.arena.end(), ar.begin(), ar.begin() + u);
        out.res[i] = r;
    }
    return out;
}

ws_ctx* default_ctx_locked(std::unique_lock<std::mutex>& lock) {
    DefaultCtx& d = default_ctx();
    lock = std::unique_lock<std::mutex>(d.mu);
    ws_ctx* ctx = d.get();
    if (!ctx) throw Error(d.error);
    return ctx;
}

const char* error_class(const std::exception& e) {
    if (dynamic_cast<const CyclicWorkload*>(&e)) return "CyclicWorkload";
    if (dynamic_cast<const UnknownModule*>(&e)) return "UnknownModule";
    if (dynamic_cast<const EmptyWorkload*>(&e)) return "EmptyWorkload";
    if (dynamic_cast<const InsufficientProfile*>(&e)) return "InsufficientProfile";
    if (dynamic_cast<const ParseError*>(&e)) return "ParseError";
    if (dynamic_cast<const DegenerateFit*>(&e)) return "DegenerateFit";
    if (dynamic_cast<const NoValidAllocation*>(&e)) return "NoValidAllocation";
    if (dynamic_cast<const PlacementInfeasible*>(&e)) return "PlacementInfeasible";
    if (dynamic_cast<const OutOfRange*>(&e)) return "OutOfRange";
    if (dynamic_cast<const EmptyLevel*>(&e)) return "EmptyLevel";
    if (dynamic_cast<const InvariantError*>(&e)) return "InvariantError";
    if (dynamic_cast<const InfeasibleError*>(&e)) return "InfeasibleError";
    if (dynamic_cast<const LimitExceeded*>(&e)) return "LimitExceeded";
    return "Error";
}

char* dup_c(const std::string& s) { return dup(s); }

}  // namespace detail

using detail::Planned;
using detail::plan_on;

PlannerResult plan_workload(const WorkloadSpec& spec, const ClusterTopology& topo, const PlannerOptions& opt) {
    validate_workload(spec);  // host-side checks first, as build_graph does (graph.hpp:98)
    DefaultCtx& d = default_ctx();
    std::lock_guard<std::mutex> lock(d.mu);
    ws_ctx* ctx = d.get();
    if (!ctx) throw Error(d.error);
    Problem p{&spec, &topo, opt};
    Planned r = plan_on(ctx, {p});
    return decode_result(p, r.res[0], r.arena.data(), true);
}

}  // namespace wsgpu

using namespace wsgpu;

struct wsx_set {
    std::deque<WorkloadSpec> specs;
    std::deque<ClusterTopology> topos;
    std::vector<Problem> probs;
    EncodedBatch enc;
    std::string error;
};

extern "C" {

void wsx_default_options(ws_options* o) {
    PlannerOptions p;
    o->eps = p.alloc.eps;
    o->max_iters = p.alloc.max_iters;
    o->sequential = p.placement.sequential;
    o->drop_floor = p.alloc.drop_floor;
    o->bt_depth = p.placement.backtrack_depth;
    o->bt_branching = p.placement.backtrack_branching;
    o->grad_mult = p.grad_opt_multiplier;
    o->synth_noise = p.synth_noise;
    o->synth_seed = p.synth_seed;
    o->strategy = p.strategy;
    o->pad = 0;
}

wsx_set* wsx_set_new(void) { return new wsx_set(); }
void wsx_set_free(wsx_set* s) { delete s; }
int32_t wsx_set_size(const wsx_set* s) { return static_cast<int32_t>(s->probs.size()); }
const char* wsx_set_error(const wsx_set* s) { return s->error.c_str(); }

// JSON workload/topology (cli.hpp:46-110); either may also be the text grammar
// when it does not start with '{'.
int32_t wsx_add_json(wsx_set* s, const char* workload, const char* topology, const ws_options* o) {
    auto is_json = [](const char* t) {
        while (*t == ' ' || *t == '\n' || *t == '\t' || *t == '\r') ++t;
        return *t == '{';
    };
    try {
        WorkloadSpec spec = is_json(workload) ? workload_from_json(workload) : parse_workload(workload);
        ClusterTopology topo = is_json(topology) ? topology_from_json(topology) : parse_topology(topology);
        s->specs.push_back(std::move(spec));
        s->topos.push_back(std::move(topo));
    } catch (const std::exception& e) {
        s->error = e.what();
        return -1;
    }
    s->probs.push_back({&s->specs.back(), &s->topos.back(), from_c(o)});
    return static_cast<int32_t>(s->probs.size() - 1);
}

int32_t wsx_add_text(wsx_set* s, const char* workload, const char* topology, const ws_options* o) {
    try {
        WorkloadSpec spec = parse_workload(workload);
        ClusterTopology topo = parse_topology(topology);
        s->specs.push_back(std::move(spec));
        s->topos.push_back(std::move(topo));
    } catch (const std::exception& e) {
        s->error = e.what();
        return -1;
    }
    s->probs.push_back({&s->specs.back(), &s->topos.back(), from_c(o)});
    return static_cast<int32_t>(s->probs.size() - 1);
}

int32_t wsx_add_scenario(wsx_set* s, const char* name, int32_t tasks, int32_t devices, uint64_t seed,
                         const ws_options* o) {
    try {
        Scenario sc = generate_scenario(name, tasks, devices, seed);
        s->specs.push_back(std::move(sc.spec));
        s->topos.push_back(std::move(sc.topo));
    } catch (const std::exception& e) {
        s->error = e.what();
        return -1;
    }
    s->probs.push_back({&s->specs.back(), &s->topos.back(), from_c(o)});
    return static_cast<int32_t>(s->probs.size() - 1);
}

int32_t wsx_add_sweep(wsx_set* s, int64_t start, int64_t count, const ws_options* o) {
    int32_t first = static_cast<int32_t>(s->probs.size());
    for (int64_t i = start; i < start + count; ++i) {
        Scenario sc = sweep_mixture(i);
        s->specs.push_back(std::move(sc.spec));
        s->topos.push_back(std::move(sc.topo));
        s->probs.push_back({&s->specs.back(), &s->topos.back(), from_c(o)});
    }
    return first;
}

const ws_batch* wsx_encode(wsx_set* s, int32_t pinned) {
    s->enc = encode_batch(s->probs, pinned != 0);
    return &s->enc.view;
}

uint64_t wsx_encoded_bytes(const wsx_set* s) { return s->enc.nbytes; }

char* wsx_result_text(const wsx_set* s, int32_t i, const ws_plan_result* results, const uint8_t* arena) {
    try {
        return dup(plan_text_or_error(s->probs[i], results[i], arena));
    } catch (const std::exception& e) {
        return dup(std::string("error DecodeFailure: ") + e.what() + "\n");
    }
}

char* wsx_sim_text(const wsx_set* s, int32_t i, const ws_plan_result* results, const uint8_t* arena,
                   const ws_sim_result* sims, const uint8_t* sim_arena) {
    try {
        return dup(sim_text(s->probs[i], results[i], arena, sims[i], sim_arena));
    } catch (const std::exception& e) {
        return dup(std::string("error DecodeFailure: ") + e.what() + "\n");
    }
}

char* wsx_dump_workload(const wsx_set* s, int32_t i) { return dup(dump_workload(*s->probs[i].spec)); }
char* wsx_dump_topology(const wsx_set* s, int32_t i) { return dup(dump_topology(*s->probs[i].topo)); }
void wsx_free_str(char* p) { std::free(p); }

// SURVEY §8(d) compulsory bytes per plan: in = 72*modules + 40*truth_pieces +
// 8*flow_tokens + 8*tasks + 4*N + 24; out = 24*MetaOps + 40*curve_pieces +
// 8*levels + 24*waves + 24*entries + 4*sum(n) + 32*flows + 16.
void wsx_algorithmic_bytes(const wsx_set* s, const ws_plan_result* results, const uint8_t* arena,
                           uint64_t* in_bytes, uint64_t* out_bytes) {
    const ws_batch& b = s->enc.view;
    uint64_t in = 0, out = 0;
    for (int p = 0; p < b.n_plans; ++p) {
        const ws_plan_rec& r = b.plans[p];
        uint64_t pieces = 0, toks = 0;
        for (int m = 0; m < r.n_mod; ++m) {
            const int g = r.mod_begin + m;
            pieces += b.mod_truth_n[g] > 0 ? b.mod_truth_n[g] : 0;
        }
        for (int t = 0; t < r.n_tasks; ++t) toks += b.task_tok_n[r.task_begin + t];
        in += 72ull * r.n_mod + 40ull * pieces + 8ull * toks + 8ull * r.n_tasks + 4ull * r.n_dev + 24;
        const ws_plan_result& x = results[p];
        if (x.status != WS_STATUS_OK) {
            out += 16;
            continue;
        }
        uint64_t sum_n = 0;
        std::size_t off = ((sizeof(ws_out_metaop) * x.n_metaops + 7) & ~std::size_t(7)) +
                          ((sizeof(ws_out_level) * x.n_levels + 7) & ~std::size_t(7)) +
                          ((sizeof(ws_out_piece) * x.n_pieces + 7) & ~std::size_t(7)) +
                          ((sizeof(ws_out_edge) * x.n_edges + 7) & ~std::size_t(7)) +
                          ((sizeof(ws_out_wave) * x.n_waves + 7) & ~std::size_t(7));
        const auto* en = reinterpret_cast<const ws_out_entry*>(arena + x.offset + off);
        for (int e = 0; e < x.n_entries; ++e) sum_n += static_cast<uint64_t>(en[e].n);
        out += 24ull * x.n_metaops + 40ull * x.n_pieces + 8ull * x.n_levels + 24ull * x.n_waves +
               24ull * x.n_entries + 4ull * sum_n + 32ull * x.n_flows + 16;
    }
    *in_bytes = in;
    *out_bytes = out;
}

void* wsx_host_alloc(uint64_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes ? bytes : 8) == cudaSuccess) return p;
    cudaGetLastError();
    return std::malloc(bytes ? bytes : 8);
}

void wsx_host_free(void* p) {
    if (!p) return;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost) {
        cudaFreeHost(p);
        return;
    }
    cudaGetLastError();
    std::free(p);
}

char* wsx_plan_workload_text(const char* workload, const char* topology, const ws_options* o) {
    WorkloadSpec spec;
    ClusterTopology topo;
    try {
        spec = parse_workload(workload);
        topo = parse_topology(topology);
    } catch (const std::exception& e) {
        return dup(std::string("error ParseError: ") + e.what() + "\n");
    }
    DefaultCtx& d = default_ctx();
    std::lock_guard<std::mutex> lock(d.mu);
    ws_ctx* ctx = d.get();
    if (!ctx) return dup("error Error: " + d.error + "\n");
    Problem p{&spec, &topo, from_c(o)};
    try {
        Planned r = plan_on(ctx, {p});
        return dup(plan_text_or_error(p, r.res[0], r.arena.data()));
    } catch (const std::exception& e) {
        return dup(std::string("error Error: ") + e.what() + "\n");
    }
}

}  // extern "C"
