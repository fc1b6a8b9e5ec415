// encode.cpp — WorkloadSpec/ClusterTopology/PlannerOptions -> ws_batch SoA.
//
// The encoder performs only host-side work the reference also does before the
// planning path proper: validate_workload (workload.hpp:104-127), resolving
// module names to indices, ranking task-id strings, and (synth_noise > 0 only)
// drawing the noisy synthetic profile with glibc math (scaling.hpp:327-339,
// SURVEY P11).  Graph construction, contraction, fitting, allocation,
// scheduling and placement all run on the device.
#include <cuda_runtime_api.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>

#include "internal.hpp"
#include "wsgpu/planner.hpp"

namespace wsgpu {
namespace {

std::size_t align16(std::size_t v) { return (v + 15) & ~std::size_t(15); }

// "m<k>" with canonical decimal k names the same placement group key as the
// entity m<k> (placement.hpp:134: group = param_group or entity id).
int entity_alias(const std::string& g) {
    if (g.size() < 2 || g.size() > 4 || g[0] != 'm') return -1;
    for (std::size_t i = 1; i < g.size(); ++i)
        if (g[i] < '0' || g[i] > '9') return -1;
    if (g.size() > 2 && g[1] == '0') return -1;
    return std::stoi(g.substr(1));
}

// Box-Muller normal (common.hpp:86-92) on a splitmix64 stream.
struct NoiseRng {
    std::uint64_t s;
    std::uint64_t u64() {
        std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double unit() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
    double normal() {
        double u1 = unit();
        double u2 = unit();
        if (u1 < 1e-300) u1 = 1e-300;
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    }
};

struct PlanScratch {
    bool ok = true;
    std::string err_class, err_msg;
    std::vector<const ModuleDecl*> mods;
    std::vector<std::string> kinds;
    // per module curve source
    std::vector<std::vector<CurvePiece>> truth;  // declared
    std::vector<int> has_truth;
    std::vector<std::vector<std::pair<int, double>>> points;
    std::vector<int> has_points;
    std::vector<std::vector<int>> bps;
    std::vector<int> has_bps;
    std::vector<int> pre_err;
    std::vector<int> group, alias;
    int n_groups = 0;
    std::vector<std::vector<int>> task_tokens;
    std::vector<int> task_rank;
    std::vector<int> island_of;
    int n_islands = 0;
};

// planner.hpp:43-53 restated for the host-synthesized noisy profile only.
bool host_truth(const std::vector<CurvePiece>& declared, int n_max, std::vector<CurvePiece>& out, int& err) {
    out.clear();
    for (CurvePiece p : declared) {
        if (p.n_lo >= n_max) continue;
        p.n_hi = std::min(p.n_hi, static_cast<double>(n_max));
        out.push_back(p);
    }
    if (out.empty()) {
        err = WS_E_TRUTH_RANGE;
        return false;
    }
    out.back().n_hi = static_cast<double>(n_max);
    try {
        ScalingCurve::from_pieces(out, 0.0, 1.0);
    } catch (const InvariantError& e) {
        err = std::string(e.what()).find("start") != std::string::npos ? WS_E_CURVE_START : WS_E_CURVE_CONTIG;
        return false;
    }
    std::sort(out.begin(), out.end(), [](const CurvePiece& a, const CurvePiece& b) { return a.n_lo < b.n_lo; });
    return true;
}

void prepare(const Problem& pr, PlanScratch& ps) {
    const WorkloadSpec& spec = *pr.spec;
    const ClusterTopology& topo = *pr.topo;
    validate_workload(spec);
    const int N = static_cast<int>(topo.devices.size());
    if (N > WS_MAX_DEVICES) throw LimitExceeded("device count " + std::to_string(N) + " exceeds WS_MAX_DEVICES");
    if (spec.modules.size() > WS_MAX_MODULES) throw LimitExceeded("module count exceeds WS_MAX_MODULES");
    if (spec.tasks.size() > WS_MAX_TASKS) throw LimitExceeded("task count exceeds WS_MAX_TASKS");

    std::map<std::string, int> index;
    std::map<std::string, int> group_ids;
    for (const auto& [kind, m] : spec.modules) {
        index[kind] = static_cast<int>(ps.mods.size());
        ps.mods.push_back(&m);
        ps.kinds.push_back(kind);
        int gid = -1, al = -1;
        if (!m.param_group.empty()) {
            auto it = group_ids.emplace(m.param_group, static_cast<int>(group_ids.size())).first;
            gid = it->second;
            al = entity_alias(m.param_group);
        }
        ps.group.push_back(gid);
        ps.alias.push_back(al);
    }
    ps.n_groups = static_cast<int>(group_ids.size());
    const std::size_t M = ps.mods.size();
    ps.truth.assign(M, {});
    ps.has_truth.assign(M, 0);
    ps.points.assign(M, {});
    ps.has_points.assign(M, 0);
    ps.bps.assign(M, {});
    ps.has_bps.assign(M, 0);
    ps.pre_err.assign(M, 0);
    for (std::size_t i = 0; i < M; ++i) {
        const std::string& kind = ps.kinds[i];
        if (auto it = spec.breakpoints.find(kind); it != spec.breakpoints.end()) {
            ps.has_bps[i] = 1;
            ps.bps[i] = it->second;
        }
        if (auto it = spec.profiles.find(kind); it != spec.profiles.end()) {
            ps.has_points[i] = 1;
            for (const ProfilePoint& p : it->second) ps.points[i].push_back({p.n, p.time});
        } else if (auto tt = spec.truth.find(kind); tt != spec.truth.end()) {
            if (pr.opt.synth_noise > 0.0) {
                // planner.hpp:79-87 with noise: points drawn here (glibc log/cos/sqrt),
                // breakpoints resolved here, fit on the device.
                std::vector<CurvePiece> pieces;
                int err = 0;
                if (!host_truth(tt->second, N, pieces, err)) {
                    ps.pre_err[i] = err;
                    ps.has_points[i] = 1;
                    continue;
                }
                const ModuleDecl& m = *ps.mods[i];
                NoiseRng rng{pr.opt.synth_seed};
                ps.has_points[i] = 1;
                for (int n = 1; n <= N; ++n) {
                    const CurvePiece* p = &pieces.back();
                    for (const CurvePiece& q : pieces)
                        if (n <= q.n_hi + 1e-9) {
                            p = &q;
                            break;
                        }
                    double t = p->alpha + p->beta_c * m.comm_proxy + p->beta_w * m.flops_proxy / n;
                    t *= std::max(1e-6, 1.0 + pr.opt.synth_noise * rng.normal());
                    ps.points[i].push_back({n, t});
                }
                std::vector<int> breaks;
                for (int b : ps.bps[i])
                    if (b > 1 && b < N) breaks.push_back(b);
                if (breaks.empty())
                    for (std::size_t k = 0; k + 1 < pieces.size(); ++k) {
                        const int b = static_cast<int>(std::llround(pieces[k].n_hi));
                        if (b > 1 && b < N) breaks.push_back(b);
                    }
                ps.has_bps[i] = 1;
                ps.bps[i] = breaks;
            } else {
                ps.has_truth[i] = 1;
                ps.truth[i] = tt->second;
            }
        }
    }
    // tasks: tokens and id ranks (std::set<std::string> order, graph.hpp:16)
    std::vector<std::string> ids;
    for (const TaskDecl& t : spec.tasks) ids.push_back(t.id);
    std::vector<std::string> sorted_ids = ids;
    std::sort(sorted_ids.begin(), sorted_ids.end());
    for (const TaskDecl& t : spec.tasks) {
        ps.task_rank.push_back(static_cast<int>(std::lower_bound(sorted_ids.begin(), sorted_ids.end(), t.id) -
                                                sorted_ids.begin()));
        std::vector<int> toks;
        for (std::size_t s = 0; s < t.flow.size(); ++s) {
            if (s) toks.push_back(WS_TOK_STEP);
            for (std::size_t b = 0; b < t.flow[s].size(); ++b) {
                if (b) toks.push_back(WS_TOK_BRANCH);
                for (const std::string& mod : t.flow[s][b]) toks.push_back(index.at(mod));
            }
        }
        ps.task_tokens.push_back(std::move(toks));
    }
    // topology: device index order = ascending id; island index = declaration order
    ps.n_islands = static_cast<int>(topo.islands.size());
    for (int d : topo.devices) ps.island_of.push_back(topo.island_of.at(d));
}

template <typename T>
T* carve(std::uint8_t* base, std::size_t& off, std::size_t count) {
    T* p = reinterpret_cast<T*>(base + off);
    off = align16(off + sizeof(T) * count);
    return p;
}

}  // namespace

namespace {
// per-problem host preparation (validation, name resolution, ranks); spread
// over host threads for large batches (problems are independent)
void prepare_all(const std::vector<Problem>& problems, std::vector<PlanScratch>& ps, EncodedBatch& eb, int threads) {
    const std::size_t P = problems.size();
    auto one = [&](std::size_t i) {
        try {
            prepare(problems[i], ps[i]);
        } catch (const CyclicWorkload& e) {
            eb.host_error_class[i] = "CyclicWorkload", eb.host_error_msg[i] = e.what();
        } catch (const UnknownModule& e) {
            eb.host_error_class[i] = "UnknownModule", eb.host_error_msg[i] = e.what();
        } catch (const EmptyWorkload& e) {
            eb.host_error_class[i] = "EmptyWorkload", eb.host_error_msg[i] = e.what();
        } catch (const ParseError& e) {
            eb.host_error_class[i] = "ParseError", eb.host_error_msg[i] = e.what();
        } catch (const LimitExceeded& e) {
            eb.host_error_class[i] = "LimitExceeded", eb.host_error_msg[i] = e.what();
        }
        if (!eb.host_error_class[i].empty()) {
            ps[i] = PlanScratch{};
            ps[i].ok = false;
        }
    };
    if (threads <= 1 || P < 2048) {
        for (std::size_t i = 0; i < P; ++i) one(i);
        return;
    }
    std::atomic<std::size_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&] {
            for (std::size_t i; (i = next.fetch_add(256)) < P;)
                for (std::size_t j = i; j < std::min(P, i + 256); ++j) one(j);
        });
    for (auto& th : pool) th.join();
}
}  // namespace

namespace detail {
bool HostBuffer::ensure(std::size_t bytes) {
    if (bytes <= cap && p) return true;
    if (p) retired.push_back(p);  // cudaFreeHost would synchronize the device: freed with the buffer
    p = nullptr;
    const std::size_t want = std::max<std::size_t>({bytes, 2 * cap, std::size_t(64) << 10});
    cap = 0;
    if (cudaMallocHost(reinterpret_cast<void**>(&p), want) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        return false;
    }
    cap = want;
    return true;
}

HostBuffer::~HostBuffer() {
    if (p) cudaFreeHost(p);
    for (std::uint8_t* q : retired) cudaFreeHost(q);
}
}  // namespace detail

EncodedBatch encode_batch(const std::vector<Problem>& problems, bool pinned) {
    return detail::encode_batch_with(problems, pinned, nullptr, 1);
}

namespace detail {

EncodedBatch encode_batch_with(const std::vector<Problem>& problems, bool pinned, HostBuffer* reuse, int threads) {
    EncodedBatch eb;
    const std::size_t P = problems.size();
    std::vector<PlanScratch> ps(P);
    eb.host_error_class.assign(P, "");
    eb.host_error_msg.assign(P, "");
    prepare_all(problems, ps, eb, threads);
    std::size_t nm = 0, nt = 0, ntok = 0, nd = 0, npc = 0, npt = 0, nbp = 0, nname = 0;
    for (std::size_t i = 0; i < P; ++i) {
        if (!ps[i].ok) continue;
        const PlanScratch& s = ps[i];
        nm += s.mods.size();
        nt += s.task_tokens.size();
        for (const auto& t : s.task_tokens) ntok += t.size();
        nd += s.island_of.size();
        for (std::size_t m = 0; m < s.mods.size(); ++m) {
            npc += s.truth[m].size();
            npt += s.points[m].size();
            nbp += s.bps[m].size();
            nname += s.kinds[m].size();
        }
    }
    std::size_t total = 0;
    total += align16(sizeof(ws_plan_rec) * P);
    total += align16(4 * nm) * 15 + align16(8 * nm) * 6;
    total += align16(4 * nt) * 3 + align16(4 * ntok) + align16(4 * nd) + align16(40 * npc);
    total += align16(4 * npt) + align16(8 * npt) + align16(4 * nbp) + align16(nname) + 64;

    std::uint8_t* raw = nullptr;
    if (reuse && reuse->ensure(total)) {  // caller-owned page-locked buffer, reused across calls
        raw = reuse->p;
        eb.pinned = true;
        eb.buffer = std::shared_ptr<std::uint8_t>(raw, [](std::uint8_t*) {});
    } else if (pinned && cudaMallocHost(reinterpret_cast<void**>(&raw), total) == cudaSuccess) {
        eb.pinned = true;
        eb.buffer = std::shared_ptr<std::uint8_t>(raw, [](std::uint8_t* p) { cudaFreeHost(p); });
    } else {
        if (pinned) cudaGetLastError();
        raw = static_cast<std::uint8_t*>(std::aligned_alloc(64, align16(total) + 64));
        eb.buffer = std::shared_ptr<std::uint8_t>(raw, [](std::uint8_t* p) { std::free(p); });
    }
    std::memset(raw, 0, total);
    eb.nbytes = total;
    std::size_t off = 0;
    ws_batch& v = eb.view;
    v.n_plans = static_cast<int32_t>(P);
    v.n_modules = static_cast<int32_t>(nm);
    v.n_task_total = static_cast<int32_t>(nt);
    v.n_tokens = static_cast<int32_t>(ntok);
    v.n_devices = static_cast<int32_t>(nd);
    v.n_pieces = static_cast<int32_t>(npc);
    v.n_points = static_cast<int32_t>(npt);
    v.n_bps = static_cast<int32_t>(nbp);
    v.n_name_bytes = static_cast<int32_t>(nname);
    v.blob = raw;
    v.blob_bytes = total;
    auto* plans = carve<ws_plan_rec>(raw, off, P);
    auto* mod_plan = carve<int32_t>(raw, off, nm);
    auto* mod_layers = carve<int32_t>(raw, off, nm);
    auto* mod_tp = carve<int32_t>(raw, off, nm);
    auto* mod_group = carve<int32_t>(raw, off, nm);
    auto* mod_alias = carve<int32_t>(raw, off, nm);
    auto* mod_batch = carve<int64_t>(raw, off, nm);
    auto* mod_param = carve<uint64_t>(raw, off, nm);
    auto* mod_act = carve<uint64_t>(raw, off, nm);
    auto* mod_out = carve<uint64_t>(raw, off, nm);
    auto* mod_w = carve<double>(raw, off, nm);
    auto* mod_c = carve<double>(raw, off, nm);
    auto* mod_name_off = carve<int32_t>(raw, off, nm);
    auto* mod_name_len = carve<int32_t>(raw, off, nm);
    auto* mod_truth_off = carve<int32_t>(raw, off, nm);
    auto* mod_truth_n = carve<int32_t>(raw, off, nm);
    auto* mod_prof_off = carve<int32_t>(raw, off, nm);
    auto* mod_prof_n = carve<int32_t>(raw, off, nm);
    auto* mod_bp_off = carve<int32_t>(raw, off, nm);
    auto* mod_bp_n = carve<int32_t>(raw, off, nm);
    auto* mod_pre_err = carve<int32_t>(raw, off, nm);
    auto* task_tok_off = carve<int32_t>(raw, off, nt);
    auto* task_tok_n = carve<int32_t>(raw, off, nt);
    auto* task_rank = carve<int32_t>(raw, off, nt);
    auto* tokens = carve<int32_t>(raw, off, ntok);
    auto* dev_island = carve<int32_t>(raw, off, nd);
    auto* truth = carve<double>(raw, off, 5 * npc);
    auto* prof_n = carve<int32_t>(raw, off, npt);
    auto* prof_t = carve<double>(raw, off, npt);
    auto* bps = carve<int32_t>(raw, off, nbp);
    auto* names = carve<uint8_t>(raw, off, nname);
    v.plans = plans;
    v.mod_plan = mod_plan;
    v.mod_layers = mod_layers;
    v.mod_tp = mod_tp;
    v.mod_group = mod_group;
    v.mod_alias = mod_alias;
    v.mod_batch = mod_batch;
    v.mod_param = mod_param;
    v.mod_act = mod_act;
    v.mod_out = mod_out;
    v.mod_w = mod_w;
    v.mod_c = mod_c;
    v.mod_name_off = mod_name_off;
    v.mod_name_len = mod_name_len;
    v.mod_truth_off = mod_truth_off;
    v.mod_truth_n = mod_truth_n;
    v.mod_prof_off = mod_prof_off;
    v.mod_prof_n = mod_prof_n;
    v.mod_bp_off = mod_bp_off;
    v.mod_bp_n = mod_bp_n;
    v.mod_pre_err = mod_pre_err;
    v.task_tok_off = task_tok_off;
    v.task_tok_n = task_tok_n;
    v.task_rank = task_rank;
    v.tokens = tokens;
    v.dev_island = dev_island;
    v.truth = truth;
    v.prof_n = prof_n;
    v.prof_t = prof_t;
    v.bps = bps;
    v.names = names;

    std::size_t im = 0, it = 0, itok = 0, id = 0, ipc = 0, ipt = 0, ibp = 0, iname = 0;
    for (std::size_t i = 0; i < P; ++i) {
        const PlanScratch& s = ps[i];
        const Problem& pr = problems[i];
        ws_plan_rec& r = plans[i];
        r.mod_begin = static_cast<int32_t>(im);
        r.n_mod = static_cast<int32_t>(s.mods.size());
        r.task_begin = static_cast<int32_t>(it);
        r.n_tasks = static_cast<int32_t>(s.task_tokens.size());
        r.dev_begin = static_cast<int32_t>(id);
        r.n_dev = static_cast<int32_t>(s.island_of.size());
        r.n_islands = s.n_islands;
        r.n_groups = s.n_groups;
        r.max_iters = pr.opt.alloc.max_iters;
        r.sequential = pr.opt.placement.sequential ? 1 : 0;
        r.bt_depth = pr.opt.placement.backtrack_depth;
        r.bt_branching = pr.opt.placement.backtrack_branching;
        r.mem_capacity = pr.topo ? pr.topo->mem_capacity : 0;
        r.eps = pr.opt.alloc.eps;
        r.drop_floor = pr.opt.alloc.drop_floor;
        r.grad_mult = pr.opt.grad_opt_multiplier;
        r.intra_bw = pr.topo ? pr.topo->intra_bw : 1.0;
        r.inter_bw = pr.topo ? pr.topo->inter_bw : 1.0;
        r.strategy = pr.opt.strategy;
        if (!s.ok) continue;
        for (std::size_t m = 0; m < s.mods.size(); ++m, ++im) {
            const ModuleDecl& md = *s.mods[m];
            mod_plan[im] = static_cast<int32_t>(i);
            mod_layers[im] = md.layers;
            mod_tp[im] = md.tp_degree;
            mod_group[im] = s.group[m];
            mod_alias[im] = s.alias[m];
            mod_batch[im] = md.input.batch;
            mod_param[im] = md.param_bytes;
            mod_act[im] = md.act_bytes;
            mod_out[im] = md.out_bytes;
            mod_w[im] = md.flops_proxy;
            mod_c[im] = md.comm_proxy;
            mod_name_off[im] = static_cast<int32_t>(iname);
            mod_name_len[im] = static_cast<int32_t>(s.kinds[m].size());
            std::memcpy(names + iname, s.kinds[m].data(), s.kinds[m].size());
            iname += s.kinds[m].size();
            mod_truth_off[im] = static_cast<int32_t>(ipc);
            mod_truth_n[im] = s.has_truth[m] ? static_cast<int32_t>(s.truth[m].size()) : -1;
            for (const CurvePiece& p : s.truth[m]) {
                truth[5 * ipc + 0] = p.n_lo;
                truth[5 * ipc + 1] = p.n_hi;
                truth[5 * ipc + 2] = p.alpha;
                truth[5 * ipc + 3] = p.beta_c;
                truth[5 * ipc + 4] = p.beta_w;
                ++ipc;
            }
            mod_prof_off[im] = static_cast<int32_t>(ipt);
            mod_prof_n[im] = s.has_points[m] ? static_cast<int32_t>(s.points[m].size()) : -1;
            for (const auto& [n, t] : s.points[m]) {
                prof_n[ipt] = n;
                prof_t[ipt] = t;
                ++ipt;
            }
            mod_bp_off[im] = static_cast<int32_t>(ibp);
            mod_bp_n[im] = s.has_bps[m] ? static_cast<int32_t>(s.bps[m].size()) : -1;
            for (int b : s.bps[m]) bps[ibp++] = b;
            mod_pre_err[im] = s.pre_err[m];
        }
        for (std::size_t t = 0; t < s.task_tokens.size(); ++t, ++it) {
            task_tok_off[it] = static_cast<int32_t>(itok);
            task_tok_n[it] = static_cast<int32_t>(s.task_tokens[t].size());
            task_rank[it] = s.task_rank[t];
            for (int tok : s.task_tokens[t]) tokens[itok++] = tok;
        }
        for (int isl : s.island_of) dev_island[id++] = isl;
    }
    return eb;
}

}  // namespace detail
}  // namespace wsgpu
