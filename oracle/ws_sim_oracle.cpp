// ws_sim_oracle.cpp — CPU ORACLE (test infrastructure only) for the plan
// evaluation path: a serial restatement of
//   simulate_plan  (/root/reference/proj/include/wavesched/simulate.hpp:74-324)
//   validate_plan  (/root/reference/proj/include/wavesched/validate.hpp:27-188)
// over planned records (ws_plan_result + arena, ws_abi.h).  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline leg may call it.
//
// Parity pin: its canonical evaluation text (host formatter sim_text.cpp) is
// compared with the reference simulate/validate run on the reference planner's
// plans (oracle/_ref/libwsref.so, tests/golden/sim_cases.json.gz).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "wsgpu/ws_abi.h"

namespace {

std::size_t al8(std::size_t v) { return (v + 7) & ~std::size_t(7); }

struct Rec {  // sections of one plan record (ws_abi.h arena layout)
    const ws_out_metaop* mo;
    const ws_out_level* lv;
    const ws_out_piece* pc;
    const ws_out_edge* ed;
    const ws_out_wave* wv;
    const ws_out_entry* en;
    const ws_out_flow* fl;
    const ws_out_scope* sc;  // task-scoped entities (n_scopes > 0)
};

Rec view(const ws_plan_result& r, const uint8_t* arena) {
    const uint8_t* b = arena + r.offset;
    Rec v;
    std::size_t o = 0;
    v.mo = reinterpret_cast<const ws_out_metaop*>(b + o);
    o += al8(sizeof(ws_out_metaop) * r.n_metaops);
    v.lv = reinterpret_cast<const ws_out_level*>(b + o);
    o += al8(sizeof(ws_out_level) * r.n_levels);
    v.pc = reinterpret_cast<const ws_out_piece*>(b + o);
    o += al8(sizeof(ws_out_piece) * r.n_pieces);
    v.ed = reinterpret_cast<const ws_out_edge*>(b + o);
    o += al8(sizeof(ws_out_edge) * r.n_edges);
    v.wv = reinterpret_cast<const ws_out_wave*>(b + o);
    o += al8(sizeof(ws_out_wave) * r.n_waves);
    v.en = reinterpret_cast<const ws_out_entry*>(b + o);
    o += al8(sizeof(ws_out_entry) * r.n_entries);
    v.fl = reinterpret_cast<const ws_out_flow*>(b + o);
    o += al8(sizeof(ws_out_flow) * r.n_flows);
    v.sc = reinterpret_cast<const ws_out_scope*>(b + o);
    return v;
}

bool id_less(int a, int b) { return "m" + std::to_string(a) < "m" + std::to_string(b); }

// "m<a>@<task a>" < "m<b>@<task b>" (task-scoped entity ids), tasks by id rank
bool wsdev_scoped_less(int a, int ta, int b, int tb) {
    if (a == b) return ta < tb;
    const std::string sa = std::to_string(a), sb = std::to_string(b);
    if (sb.size() > sa.size() && sb.compare(0, sa.size(), sa) == 0) return false;
    if (sa.size() > sb.size() && sa.compare(0, sb.size(), sb) == 0) return true;
    return sa < sb;
}

struct Entity {  // PlanEntity fields used by the evaluator (planner.hpp:99-122)
    int length = 0, tp = 1;
    std::uint64_t param_bytes = 0, act_bytes = 0;
    double w = 1.0, c = 0.0, frac = 1.0;  // frac: batch_fraction
    std::string group;  // param_group, or the entity id when empty
    std::vector<ws_out_piece> pieces;
    // ScalingCurve::eval_batch_fraction (scaling.hpp:83-86)
    double eval_bf(double n, double frac) const {
        const double nmax = pieces.back().n_hi;
        const ws_out_piece* p = &pieces.front();
        if (!(n < 1.0)) {
            const double x = std::min(n, nmax);
            p = &pieces.back();
            for (const ws_out_piece& q : pieces)  // locate (scaling.hpp:149-154)
                if (x <= q.n_hi + 1e-9) {
                    p = &q;
                    break;
                }
        }
        return p->alpha + p->beta_c * c + p->beta_w * w * frac / n;
    }
};

// plan.devices order: ascending, starting at device index rot (the sequential
// ablation's rolling cursor, placement.hpp:351-357; rot = 0 otherwise)
std::vector<int> dev_list(const ws_out_entry& e) {
    std::vector<int> out;
    for (int d = e.rot; d < 64; ++d)
        if (e.devmask >> d & 1ull) out.push_back(d);
    for (int d = 0; d < e.rot && d < 64; ++d)
        if (e.devmask >> d & 1ull) out.push_back(d);
    return out;
}

struct Viol {
    int code, wave, a, b;
    double x, y;
};

struct Eval {
    const ws_batch& B;
    const ws_plan_rec& P;
    const ws_plan_result& R;
    Rec V;
    ws_sim_opts opt;
    int N, K;
    std::vector<Entity> ent;
    std::map<std::pair<int, int>, const ws_out_entry*> devices;  // (wave, metaop) -> entry

    Eval(const ws_batch& b, int p, const ws_plan_result& r, const uint8_t* arena, const ws_sim_opts& o)
        : B(b), P(b.plans[p]), R(r), V(view(r, arena)), opt(o), N(b.plans[p].n_dev), K(r.n_metaops) {
        ent.resize(K);
        for (int k = 0; k < K; ++k) {
            const ws_out_metaop& m = V.mo[k];
            const int gm = P.mod_begin + m.module;
            Entity& e = ent[k];
            e.length = m.length;
            e.tp = B.mod_tp[gm];
            e.param_bytes = static_cast<std::uint64_t>(static_cast<double>(B.mod_param[gm]) * m.length /
                                                       B.mod_layers[gm]);
            e.act_bytes = B.mod_act[gm];
            e.w = B.mod_w[gm];
            e.c = B.mod_c[gm];
            e.frac = B.mod_frac ? B.mod_frac[gm] : 1.0;
            const int grp = m.length == B.mod_layers[gm] ? B.mod_group[gm] : -1;
            if (R.n_scopes > 0) {  // entities "m<metaop>@<task>" (baselines.hpp:49-55)
                int users = 0;     // share_fraction: tasks routing through the module
                for (int t = 0; t < P.n_tasks; ++t) {
                    const int tg = P.task_begin + t;
                    bool in = false;
                    for (int i = 0; i < B.task_tok_n[tg]; ++i) in |= B.tokens[B.task_tok_off[tg] + i] == m.module;
                    users += in;
                }
                e.frac = users ? 1.0 / users : 1.0;
            }
            if (grp < 0)
                e.group = "m" + std::to_string(k);
            else if (B.mod_alias[gm] >= 0 && R.n_scopes == 0)
                e.group = "m" + std::to_string(B.mod_alias[gm]);  // param_group spelled "m<j>"
            else
                e.group = "g" + std::to_string(grp);  // no entity id starts with "g"
            e.pieces.assign(V.pc + m.piece_begin, V.pc + m.piece_begin + m.piece_count);
        }
        for (int w = 0; w < R.n_waves; ++w)
            for (int i = 0; i < V.wv[w].n_entries; ++i) {
                const ws_out_entry& e = V.en[V.wv[w].entry_begin + i];
                if (e.devmask) devices[{w, e.metaop}] = &e;  // later entries overwrite (std::map assignment)
            }
    }

    const ws_out_entry* find(int w, int k) const {
        auto it = devices.find({w, k});
        return it == devices.end() ? nullptr : it->second;
    }

    // compute_device_memory (validate.hpp:27-50)
    std::vector<double> device_memory() const {
        std::vector<double> mem(N, 0.0);
        std::map<int, std::set<std::string>> charged;
        for (int w = 0; w < R.n_waves; ++w)
            for (int i = 0; i < V.wv[w].n_entries; ++i) {
                const ws_out_entry& e = V.en[V.wv[w].entry_begin + i];
                const ws_out_entry* pl = find(w, e.metaop);
                if (!pl || e.metaop < 0 || e.metaop >= K) continue;
                const Entity& x = ent[e.metaop];
                for (int d : dev_list(*pl)) {
                    if (d >= N) continue;
                    if (!charged[d].count(x.group)) {
                        mem[d] += (1.0 + P.grad_mult) * static_cast<double>(x.param_bytes) / x.tp;
                        charged[d].insert(x.group);
                    }
                    mem[d] += e.layers * (static_cast<double>(x.act_bytes) * x.frac / e.n);
                }
            }
        return mem;
    }

    // simulate (simulate.hpp:171-320) with build_param_groups (:127-165)
    void simulate(ws_sim_result& out, std::vector<double>& busy_v, uint64_t& busy_mask, std::vector<double>& util,
                  uint64_t& util_mask) const {
        std::vector<double> avail(N, 0.0);
        std::map<int, double> busy_c;
        double frontier = 0.0;
        int timeline = 0;
        auto frontier_of = [&] {
            double f = 0.0;
            for (double t : avail) f = std::max(f, t);
            return f;
        };
        auto attribute = [&](double* bucket) {
            const double f = frontier_of();
            *bucket += f - frontier;
            frontier = f;
        };
        auto busy = [&](int d, double from, double dur) {
            if (dur <= 0.0) {
                avail[d] = std::max(avail[d], from);
                return;
            }
            ++timeline;
            avail[d] = from + dur;
        };
        std::vector<int> order(R.n_waves);
        for (int w = 0; w < R.n_waves; ++w) order[w] = w;
        std::sort(order.begin(), order.end(), [&](int a, int b) {
            if (V.wv[a].start != V.wv[b].start) return V.wv[a].start < V.wv[b].start;
            return a < b;
        });
        std::map<int, std::vector<int>> into, out_of;
        for (int f = 0; f < R.n_flows; ++f) {
            into[V.fl[f].to_wave].push_back(f);
            out_of[V.fl[f].from_wave].push_back(f);
        }
        auto flow_duration = [&](const ws_out_flow& f) {
            if (f.volume == 0 || f.mode == WS_FLOW_COPY) return 0.0;
            const double bw = f.mode == WS_FLOW_INTER ? P.inter_bw : P.intra_bw;
            return static_cast<double>(f.volume) / bw;
        };
        auto run_flow = [&](const ws_out_flow& f) {
            const double dur = opt.zero_volumes ? 0.0 : flow_duration(f);
            const ws_out_entry* a = find(f.from_wave, f.from_metaop);
            const ws_out_entry* b = find(f.to_wave, f.to_metaop);
            if (!a || !b) return;
            std::set<int> parties;
            for (int d : dev_list(*a)) parties.insert(d);
            for (int d : dev_list(*b)) parties.insert(d);
            double t0 = 0.0;
            for (int d : parties) t0 = std::max(t0, avail[d]);
            for (int d : parties) busy(d, t0, dur);
            if (!opt.zero_volumes) {
                out.total_transferred_bytes += static_cast<double>(f.volume);
                if (f.mode == WS_FLOW_INTER) out.total_inter_island_bytes += static_cast<double>(f.volume);
            }
        };
        auto run_wave = [&](int w, bool backward) {
            const double scale = backward ? opt.backward_ratio : 1.0;
            const ws_out_wave& wave = V.wv[w];
            std::set<int> participants;
            for (int i = 0; i < wave.n_entries; ++i) {
                const ws_out_entry* pl = find(w, V.en[wave.entry_begin + i].metaop);
                if (!pl) continue;
                for (int d : dev_list(*pl)) participants.insert(d);
            }
            double t0 = 0.0;
            for (int d : participants) t0 = std::max(t0, avail[d]);
            for (int i = 0; i < wave.n_entries; ++i) {
                const ws_out_entry& e = V.en[wave.entry_begin + i];
                const ws_out_entry* pl = find(w, e.metaop);
                if (!pl) continue;
                for (int d : dev_list(*pl)) {
                    busy(d, t0, e.span * scale);
                    busy_c[d] += e.span * scale;
                }
            }
            for (int d : participants) avail[d] = std::max(avail[d], t0 + wave.duration * scale);
        };
        for (int w : order) {
            for (int f : into[w]) run_flow(V.fl[f]);
            attribute(&out.send_recv_seconds);
            run_wave(w, false);
            attribute(&out.fwd_bwd_seconds);
        }
        for (auto it = order.rbegin(); it != order.rend(); ++it) {
            run_wave(*it, true);
            attribute(&out.fwd_bwd_seconds);
            for (int f : out_of[*it]) run_flow(V.fl[f]);
            attribute(&out.send_recv_seconds);
        }
        if (!opt.skip_sync) {
            std::map<std::string, std::set<int>> group_devices;
            std::map<std::string, std::uint64_t> group_bytes;
            for (int w = 0; w < R.n_waves; ++w)
                for (int i = 0; i < V.wv[w].n_entries; ++i) {
                    const ws_out_entry& e = V.en[V.wv[w].entry_begin + i];
                    const ws_out_entry* pl = find(w, e.metaop);
                    if (!pl || e.metaop < 0 || e.metaop >= K) continue;
                    const Entity& x = ent[e.metaop];
                    for (int d : dev_list(*pl)) group_devices[x.group].insert(d);
                    const std::uint64_t g = 2ull * x.param_bytes / static_cast<std::uint64_t>(x.tp);
                    group_bytes[x.group] = std::max(group_bytes[x.group], g);
                }
            std::map<std::vector<int>, std::uint64_t> pooled;
            for (const auto& [g, devs] : group_devices)
                pooled[std::vector<int>(devs.begin(), devs.end())] += group_bytes[g];
            for (const auto& [devs, bytes_u] : pooled) {
                double dur = 0.0;
                if (devs.size() >= 2) {
                    std::map<int, int> per_island;
                    for (int d : devs) per_island[B.dev_island[P.dev_begin + d]]++;
                    const double bytes = static_cast<double>(bytes_u);
                    std::size_t widest = 0;
                    for (const auto& [isl, cnt] : per_island) widest = std::max(widest, static_cast<std::size_t>(cnt));
                    if (widest >= 2)
                        dur += 2.0 * (static_cast<double>(widest) - 1.0) / static_cast<double>(widest) * bytes /
                               P.intra_bw;
                    const std::size_t islands = per_island.size();
                    if (islands >= 2)
                        dur += 2.0 * (static_cast<double>(islands) - 1.0) / static_cast<double>(islands) * bytes /
                               P.inter_bw;
                }
                if (dur <= 0.0) continue;
                double t0 = 0.0;
                for (int d : devs) t0 = std::max(t0, avail[d]);
                for (int d : devs) busy(d, t0, dur);
            }
            attribute(&out.param_sync_seconds);
        }
        out.makespan = frontier_of();
        const double span = std::max(out.makespan, 1e-300);
        out.fwd_bwd_fraction = out.fwd_bwd_seconds / span;
        out.param_sync_fraction = out.param_sync_seconds / span;
        out.send_recv_fraction = out.send_recv_seconds / span;
        out.timeline_items = timeline;
        busy_v.assign(N, 0.0);
        busy_mask = 0;
        for (const auto& [d, b] : busy_c) {
            busy_v[d] = b;
            busy_mask |= 1ull << d;
        }
        // utilization proxy (simulate.hpp:283-300)
        double peak_rate = 0.0;
        std::map<int, double> layer_s, device_s;
        for (int w = 0; w < R.n_waves; ++w)
            for (int i = 0; i < V.wv[w].n_entries; ++i) {
                const ws_out_entry& e = V.en[V.wv[w].entry_begin + i];
                if (e.metaop < 0 || e.metaop >= K) continue;
                const Entity& x = ent[e.metaop];
                layer_s[e.metaop] += x.w * x.frac * e.layers;
                device_s[e.metaop] += e.span * e.n;
            }
        for (int k = 0; k < K; ++k) {
            const double t1 = ent[k].eval_bf(1.0, ent[k].frac);
            if (t1 > 0.0) peak_rate = std::max(peak_rate, ent[k].w * ent[k].frac / t1);
        }
        util.assign(K, 0.0);
        util_mask = 0;
        for (const auto& [k, ls] : layer_s) {
            const double ds = device_s[k];
            util[k] = (ds > 0.0 && peak_rate > 0.0) ? (ls / ds) / peak_rate : 0.0;
            util_mask |= 1ull << k;
        }
    }

    // validate_plan (validate.hpp:58-188)
    std::vector<Viol> validate(const std::vector<double>& mem) const {
        std::vector<Viol> v;
        auto fail = [&](int code, int wave, int a, int b, double x, double y) { v.push_back({code, wave, a, b, x, y}); };
        const double horizon = std::max(1.0, R.end_time);
        const double tol = 1e-6 * horizon;
        struct Iv {
            int id;
            double start, end;
            int n, layers;
        };
        std::vector<Iv> ivs;
        std::map<int, int> executed;
        for (int w = 0; w < R.n_waves; ++w) {
            const ws_out_wave& wave = V.wv[w];
            std::set<int> seen;
            int used = 0;
            for (int i = 0; i < wave.n_entries; ++i) {
                const ws_out_entry& e = V.en[wave.entry_begin + i];
                if (e.metaop < 0 || e.metaop >= K) {
                    fail(WS_V_UNKNOWN_ENTITY, w, e.metaop, 0, 0, 0);
                    continue;
                }
                if (!seen.insert(e.metaop).second) fail(WS_V_DUPLICATE, w, e.metaop, 0, 0, 0);
                const double per_layer = ent[e.metaop].eval_bf(e.n, ent[e.metaop].frac);
                const double span = e.layers * per_layer;
                if (std::abs(span - e.span) > tol + 1e-9 * std::abs(span))
                    fail(WS_V_SPAN, w, e.metaop, 0, e.span, span);
                if (e.span > wave.duration + tol) fail(WS_V_SPAN_DURATION, w, 0, 0, 0, 0);
                ivs.push_back({e.metaop, wave.start, wave.start + span, e.n, e.layers});
                executed[e.metaop] += e.layers;
                used += e.n;
            }
            if (used > N) fail(WS_V_WAVE_DEVICES, w, 0, 0, 0, 0);
        }
        std::vector<int> ids(K);
        for (int k = 0; k < K; ++k) ids[k] = k;
        if (R.n_scopes > 0) {
            auto tr = [&](int k) { return B.task_rank[P.task_begin + V.sc[k].task]; };
            std::sort(ids.begin(), ids.end(), [&](int a, int b) {
                return wsdev_scoped_less(V.sc[a].metaop, tr(a), V.sc[b].metaop, tr(b));
            });
        } else {
            std::sort(ids.begin(), ids.end(), id_less);
        }
        for (int k : ids) {
            auto it = executed.find(k);
            const int done = it == executed.end() ? 0 : it->second;
            if (done != ent[k].length) fail(WS_V_WORK, -1, k, done, ent[k].length, 0);
        }
        std::vector<std::pair<double, int>> events;
        for (const Iv& iv : ivs) {
            events.push_back({iv.start, iv.n});
            events.push_back({std::max(iv.start, iv.end - tol), -iv.n});
        }
        std::sort(events.begin(), events.end(), [](const auto& a, const auto& b) {
            if (a.first != b.first) return a.first < b.first;
            return a.second < b.second;
        });
        int active = 0;
        for (const auto& [t, delta] : events) {
            active += delta;
            if (active > N) {
                fail(WS_V_CAPACITY, -1, active, 0, t, 0);
                break;
            }
        }
        std::map<int, std::vector<Iv>> by_entity;  // int keys: iterate in id string order below
        for (const Iv& iv : ivs) by_entity[iv.id].push_back(iv);
        for (int k : ids) {
            auto it = by_entity.find(k);
            if (it == by_entity.end()) continue;
            auto& list = it->second;
            std::sort(list.begin(), list.end(), [](const Iv& a, const Iv& b) { return a.start < b.start; });
            for (std::size_t i = 0; i + 1 < list.size(); ++i)
                if (list[i].end > list[i + 1].start + tol) {
                    fail(WS_V_OVERLAP, -1, k, 0, 0, 0);
                    break;
                }
        }
        for (int e = 0; e < R.n_edges; ++e) {
            const int from = V.ed[e].from, to = V.ed[e].to;
            auto fi = by_entity.find(from), ti = by_entity.find(to);
            if (fi == by_entity.end() || ti == by_entity.end()) continue;
            double from_end = 0.0;
            for (const Iv& iv : fi->second) from_end = std::max(from_end, iv.end);
            double to_start = horizon * 2;
            for (const Iv& iv : ti->second) to_start = std::min(to_start, iv.start);
            if (to_start + tol < from_end) fail(WS_V_DEPENDENCY, -1, from, to, to_start, from_end);
        }
        if (!devices.empty()) {
            for (int w = 0; w < R.n_waves; ++w) {
                const ws_out_wave& wave = V.wv[w];
                std::set<int> taken;
                for (int i = 0; i < wave.n_entries; ++i) {
                    const ws_out_entry& e = V.en[wave.entry_begin + i];
                    const ws_out_entry* pl = find(w, e.metaop);
                    if (!pl) {
                        fail(WS_V_UNPLACED, w, e.metaop, 0, 0, 0);
                        continue;
                    }
                    const std::vector<int> dl = dev_list(*pl);
                    if (static_cast<int>(dl.size()) != e.n)
                        fail(WS_V_DEVICE_COUNT, w, e.metaop, static_cast<int>(dl.size()), e.n, 0);
                    for (int d : dl) {
                        if (d >= N)
                            fail(WS_V_UNKNOWN_DEVICE, -1, d, 0, 0, 0);
                        else if (!taken.insert(d).second)
                            fail(WS_V_DEVICE_TWICE, w, d, 0, 0, 0);
                    }
                }
            }
            for (int d = 0; d < N; ++d)
                if (mem[d] > static_cast<double>(P.mem_capacity) * (1.0 + 1e-9))
                    {
                    double capbits;  // the capacity's u64 bits travel in y
                    std::memcpy(&capbits, &P.mem_capacity, 8);
                    fail(WS_V_MEMORY, -1, d, 0, mem[d], capbits);
                }
        }
        return v;
    }
};

}  // namespace

extern "C" {

// Simulates + validates every planned record serially; same output contract
// as ws_simulate_batch_host.  Returns 0, or 1 if the arena was too small.
int wso_simulate_batch(const ws_batch* in, const ws_plan_result* plans, const uint8_t* plan_arena,
                       const ws_sim_opts* opts, ws_sim_result* out, uint8_t* arena, uint64_t arena_cap,
                       uint64_t* arena_used) {
    ws_sim_opts o{2.0, 0, 0};
    if (opts) o = *opts;
    uint64_t top = 0;
    int rc = 0;
    for (int p = 0; p < in->n_plans; ++p) {
        ws_sim_result& r = out[p];
        std::memset(&r, 0, sizeof(r));
        if (plans[p].status != WS_STATUS_OK) {
            r.status = plans[p].status;
            continue;
        }
        Eval ev(*in, p, plans[p], plan_arena, o);
        std::vector<double> busy, util;
        uint64_t busy_mask = 0, util_mask = 0;
        ev.simulate(r, busy, busy_mask, util, util_mask);
        const std::vector<double> mem = ev.device_memory();
        const std::vector<Viol> v = ev.validate(mem);
        r.valid = v.empty() ? 1 : 0;
        r.n_violations = static_cast<int>(v.size());
        const int N = ev.N, K = ev.K;
        const int nv = std::min<int>(r.n_violations, WS_SIM_MAX_VIOLATIONS);
        const uint64_t sz = 8ull * N + 8 + 8ull * N + 8ull * K + 8 + sizeof(ws_out_violation) * nv;
        if (top + sz > arena_cap) {
            r.status = WS_STATUS_INTERNAL;
            rc = 1;
            continue;
        }
        r.offset = top;
        r.size = sz;
        uint8_t* b = arena + top;
        top += sz;
        std::memcpy(b, busy.data(), 8ull * N);
        std::memcpy(b + 8ull * N, &busy_mask, 8);
        std::memcpy(b + 8ull * N + 8, mem.data(), 8ull * N);
        std::memcpy(b + 16ull * N + 8, util.data(), 8ull * K);
        std::memcpy(b + 16ull * N + 8 + 8ull * K, &util_mask, 8);
        auto* vo = reinterpret_cast<ws_out_violation*>(b + 16ull * N + 16 + 8ull * K);
        for (int i = 0; i < nv; ++i) vo[i] = {v[i].code, v[i].wave, v[i].a, v[i].b, v[i].x, v[i].y};
    }
    *arena_used = top;
    return rc;
}

}  // extern "C"
