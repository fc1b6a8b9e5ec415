// api.cpp — the C++ drop-in plan_workload (planner.hpp:156-212) over the
// C-ABI, and the wsx.h helper API used by FFI callers.
#include <cuda_runtime_api.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

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

int host_threads(int requested) {
    if (requested > 0) return requested;
    const unsigned hc = std::thread::hardware_concurrency();
    return hc ? static_cast<int>(hc) : 1;
}

// fn(i) for i in [0, n) over `threads` host threads (dynamic chunks)
template <typename Fn>
void parallel_for(std::size_t n, int threads, Fn&& fn) {
    if (threads <= 1 || n < 2) {
        for (std::size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<std::size_t> next{0};
    const std::size_t chunk = std::max<std::size_t>(1, std::min<std::size_t>(64, n / (4 * threads)));
    auto work = [&] {
        for (std::size_t i; (i = next.fetch_add(chunk)) < n;)
            for (std::size_t j = i; j < std::min(n, i + chunk); ++j) fn(j);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < std::min<int>(threads, static_cast<int>(n)); ++t) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
}

}  // namespace

namespace detail {

// Pooled per-device contexts (never destroyed: they live until process exit,
// so no CUDA call runs during static destruction).
struct Lease {
    ws_ctx* ctx = nullptr;
    HostBuffer in, results, arena;
};

namespace {
struct DevicePool {
    std::mutex mu;
    std::vector<Lease*> idle;
};

DevicePool& pool_of(int device) {
    static std::mutex mu;
    static std::map<int, DevicePool*>* pools = new std::map<int, DevicePool*>();
    std::lock_guard<std::mutex> g(mu);
    DevicePool*& p = (*pools)[device];
    if (!p) p = new DevicePool();
    return *p;
}

int calling_device() {
    if (const char* env = std::getenv("WSGPU_DEVICE")) return std::atoi(env);
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) {
        cudaGetLastError();
        d = 0;
    }
    return d;
}
}  // namespace

CtxLease::CtxLease() : CtxLease(calling_device()) {}

CtxLease::CtxLease(int device) : device_(device) {
    DevicePool& pool = pool_of(device);
    {
        std::lock_guard<std::mutex> g(pool.mu);
        if (!pool.idle.empty()) {
            l_ = pool.idle.back();
            pool.idle.pop_back();
            return;
        }
    }
    auto* l = new Lease();
    if (ws_ctx_create(device, &l->ctx) != 0) {
        delete l;
        throw Error("CUDA planner unavailable (ws_ctx_create failed on device " + std::to_string(device) + ")");
    }
    l_ = l;
}

CtxLease::~CtxLease() {
    if (!l_) return;
    DevicePool& pool = pool_of(device_);
    std::lock_guard<std::mutex> g(pool.mu);
    pool.idle.push_back(l_);
}

ws_ctx* CtxLease::ctx() const { return l_->ctx; }
HostBuffer& CtxLease::in() const { return l_->in; }
HostBuffer& CtxLease::results() const { return l_->results; }
HostBuffer& CtxLease::arena() const { return l_->arena; }

namespace {
// Plans `probs` on the lease: headers and records land in the lease's
// page-locked buffers; a plan whose record overflowed its arena share is
// re-planned alone and the batch is then copied into `owned`.
struct BatchOut {
    const ws_plan_result* res = nullptr;
    const std::uint8_t* arena = nullptr;
    std::uint64_t used = 0;
    Planned owned;
};

void plan_core(CtxLease& L, const std::vector<Problem>& probs, int threads, BatchOut& out) {
    EncodedBatch eb = encode_batch_with(probs, true, &L.in(), threads);
    const std::size_t P = probs.size();
    const std::uint64_t cap = ws_arena_bound(&eb.view);
    if (!L.results().ensure(sizeof(ws_plan_result) * std::max<std::size_t>(P, 1)) || !L.arena().ensure(cap))
        throw Error("CUDA planner failed: cudaMallocHost of the drop-in buffers");
    auto* res = reinterpret_cast<ws_plan_result*>(L.results().p);
    std::uint64_t used = 0;
    if (ws_plan_batch_host(L.ctx(), &eb.view, res, L.arena().p, cap, &used, nullptr) != 0)
        throw Error(std::string("CUDA planner failed: ") + ws_ctx_last_error(L.ctx()));
    out.res = res;
    out.arena = L.arena().p;
    out.used = used;
    bool overflow = false;
    for (std::size_t i = 0; i < P; ++i) overflow |= res[i].err_code == WS_E_ARENA_OVERFLOW;
    if (!overflow) return;
    Planned& o = out.owned;
    o.res.assign(res, res + P);
    o.arena.assign(L.arena().p, L.arena().p + used);
    for (std::size_t i = 0; i < P; ++i) {
        if (o.res[i].err_code != WS_E_ARENA_OVERFLOW) continue;
        EncodedBatch one = encode_batch({probs[i]}, true);
        const std::uint64_t big = std::uint64_t(64) << 20;
        std::vector<std::uint8_t> ar(big);
        ws_plan_result r{};
        std::uint64_t u = 0;
        if (ws_plan_batch_host(L.ctx(), &one.view, &r, ar.data(), big, &u, nullptr) != 0)
            throw Error(std::string("CUDA planner failed: ") + ws_ctx_last_error(L.ctx()));
        r.offset += o.arena.size();
        o.arena.insert(o.arena.end(), ar.begin(), ar.begin() + u);
        o.res[i] = r;
    }
    out.res = o.res.data();
    out.arena = o.arena.data();
    out.used = o.arena.size();
}
}  // namespace

namespace {
// Coalescing of concurrent drop-in calls (leader/follower): a caller that
// finds no batch in flight (at most kLeaders at a time) takes every pending
// request and plans them as ONE device batch on a leased context; the others
// wait for it.  Each caller then decodes its own record on its own thread,
// while the next batch is already planning on another context.  Results are
// those of planning each problem alone (plans are independent; the batch
// parity tests pin batched == single).  Opt-in ($WSGPU_COALESCE=1): measured
// with 16 host threads (20k sweep plans, reference types in and out) it gives
// 17.9k plans/s against 31.9k for the default, one pooled context per
// concurrent caller on the 7-call small-batch path.
struct SharedBatch {
    explicit SharedBatch(int device) : lease(device) {}
    CtxLease lease;  // released when the last member has decoded its record
    BatchOut out;
};

struct Request {
    const Problem* prob = nullptr;
    std::shared_ptr<SharedBatch> batch;
    std::size_t index = 0;
    std::exception_ptr error;
    bool done = false;
};

class Coalescer {
public:
    static constexpr int kLeaders = 2;  // batches planning at once (host encode overlaps the other's kernels)
    void run(int device, Request& r) {
        std::unique_lock<std::mutex> lk(mu_);
        pending_.push_back(&r);
        while (!r.done) {
            if (leaders_ < kLeaders && !pending_.empty()) {
                std::vector<Request*> batch;
                batch.swap(pending_);
                ++leaders_;
                lk.unlock();
                std::shared_ptr<SharedBatch> sb;
                std::exception_ptr err;
                try {
                    std::vector<Problem> probs;
                    probs.reserve(batch.size());
                    for (Request* q : batch) probs.push_back(*q->prob);
                    sb = std::make_shared<SharedBatch>(device);
                    plan_core(sb->lease, probs, 1, sb->out);
                } catch (...) {
                    err = std::current_exception();
                    sb.reset();
                }
                lk.lock();
                --leaders_;
                for (std::size_t i = 0; i < batch.size(); ++i) {
                    batch[i]->batch = sb;
                    batch[i]->index = i;
                    batch[i]->error = err;
                    batch[i]->done = true;
                }
                cv_.notify_all();
            } else {
                cv_.wait(lk);
            }
        }
    }

private:
    std::mutex mu_;
    std::condition_variable cv_;
    std::vector<Request*> pending_;
    int leaders_ = 0;
};

Coalescer& coalescer_of(int device) {
    static std::mutex mu;
    static std::map<int, Coalescer*>* all = new std::map<int, Coalescer*>();
    std::lock_guard<std::mutex> g(mu);
    Coalescer*& c = (*all)[device];
    if (!c) c = new Coalescer();
    return *c;
}

bool coalescing() {
    static const bool on = [] {
        const char* env = std::getenv("WSGPU_COALESCE");
        return env && std::atoi(env) != 0;
    }();
    return on;
}
}  // namespace

// Plans one problem (coalesced with concurrent callers) and hands its record to `consume`.
void plan_single(const Problem& p, const std::function<void(const ws_plan_result&, const std::uint8_t*)>& consume) {
    if (!coalescing()) {
        CtxLease lease;
        const PlannedOne r = plan_one(lease, p);
        consume(*r.res, r.arena);
        return;
    }
    Request req;
    req.prob = &p;
    coalescer_of(calling_device()).run(calling_device(), req);
    if (req.error) std::rethrow_exception(req.error);
    const BatchOut& b = req.batch->out;
    consume(b.res[req.index], b.arena);
}

Planned plan_on(CtxLease& lease, const std::vector<Problem>& probs, int threads) {
    BatchOut b;
    plan_core(lease, probs, threads, b);
    if (!b.owned.res.empty()) return std::move(b.owned);
    Planned out;
    out.res.assign(b.res, b.res + probs.size());
    out.arena.assign(b.arena, b.arena + b.used);
    return out;
}

PlannedOne plan_one(CtxLease& lease, const Problem& prob) {
    BatchOut b;
    plan_core(lease, {prob}, 1, b);
    PlannedOne o{b.res, b.arena, {}};
    if (!b.owned.res.empty()) {  // rare: keep the re-planned record alive
        o.own = std::move(b.owned.arena);
        static thread_local ws_plan_result r;
        r = b.owned.res[0];
        o.res = &r;
        o.arena = o.own.data();
    }
    return o;
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

void plan_batch_raw(const std::vector<Problem>& probs, int threads,
                    const std::function<void(const ws_plan_result*, const std::uint8_t*)>& consume) {
    CtxLease lease;
    BatchOut b;
    plan_core(lease, probs, host_threads(threads), b);
    consume(b.res, b.arena);
}

}  // namespace detail

PlannerResult plan_workload(const WorkloadSpec& spec, const ClusterTopology& topo, const PlannerOptions& opt) {
    validate_workload(spec);  // host-side checks first, as build_graph does (graph.hpp:98)
    const Problem p{&spec, &topo, opt};
    PlannerResult out;
    detail::plan_single(p, [&](const ws_plan_result& r, const std::uint8_t* arena) {
        out = decode_result(p, r, arena, true);
    });
    return out;
}

void plan_workload_raw(const WorkloadSpec& spec, const ClusterTopology& topo, const PlannerOptions& opt,
                       const std::function<void(const ws_plan_result&, const std::uint8_t*)>& consume) {
    validate_workload(spec);
    detail::plan_single(Problem{&spec, &topo, opt}, consume);
}

void plan_workloads_raw(const std::vector<Problem>& problems, int threads,
                        const std::function<void(const ws_plan_result*, const std::uint8_t*)>& consume) {
    detail::plan_batch_raw(problems, threads, consume);
}

std::vector<PlanOutcome> plan_workloads(const std::vector<Problem>& problems, int threads) {
    std::vector<PlanOutcome> out(problems.size());
    const int T = host_threads(threads);
    detail::plan_batch_raw(problems, T, [&](const ws_plan_result* res, const std::uint8_t* arena) {
        parallel_for(problems.size(), T, [&](std::size_t i) {
            try {
                out[i].result = decode_result(problems[i], res[i], arena, true);
            } catch (...) {
                out[i].error = std::current_exception();
            }
        });
    });
    return out;
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
    Problem p{&spec, &topo, from_c(o)};
    try {
        std::string text;
        detail::plan_single(p, [&](const ws_plan_result& r, const std::uint8_t* arena) {
            text = plan_text_or_error(p, r, arena);
        });
        return dup(text);
    } catch (const std::exception& e) {
        return dup(std::string("error Error: ") + e.what() + "\n");
    }
}

}  // extern "C"
