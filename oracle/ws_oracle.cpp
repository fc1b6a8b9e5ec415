// ws_oracle.cpp — CPU ORACLE (test infrastructure only).
//
// A serial, obviously-sequential restatement of the reference planning path
// (/root/reference/proj/include/wavesched/planner.hpp:156-212 and the L2
// headers it calls) over the ws_abi.h batch format.  It exists to check the
// CUDA planner: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
// leg may call it; the product path never does.
//
// Parity pin: decoded through the host decoder, its write_plan() text is
// compared byte-for-byte with the reference planner compiled from the
// reference headers (oracle/_ref, see oracle/Makefile) over the bundled
// suite, the acceptance fuzz workloads and thousands of sweep mixtures
// (tests/test_oracle.py against the fixtures tests/golden/make_golden.py
// generates from the reference; oracle/ref/pin.cpp for direct runs against it).
//
// Sorting uses std::sort with the reference comparators, i.e. the same
// libstdc++ algorithm the reference runs.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "wsgpu/ws_abi.h"

namespace {

// the restatement keeps device sets in one u64: clusters of up to 64 devices
// (wider clusters are pinned to the reference directly, tests/golden/wide_cases)
constexpr int kOracleMaxDevices = 64;

struct Fail {
    int code;
    int64_t a = 0, b = 0;
    double x = 0, y = 0;
};

int popc(uint64_t m) { return __builtin_popcountll(m); }
int nth_bit(uint64_t m, int k) {  // index of the k-th set bit (k from 0)
    for (int i = 0; i < 64; ++i)
        if (m >> i & 1ull) {
            if (k == 0) return i;
            --k;
        }
    return -1;
}

struct Piece {
    double lo, hi, alpha, bc, bw;
};

// ScalingCurve (scaling.hpp:35-164)
struct Curve {
    std::vector<Piece> p;
    double c = 0, w = 1, nmax = 1;
    double value(const Piece& q, double n) const { return q.alpha + q.bc * c + q.bw * w / n; }
    const Piece& locate(double n) const {  // scaling.hpp:149-154
        for (const Piece& q : p)
            if (n <= q.hi + 1e-9) return q;
        return p.back();
    }
    double eval(double n) const {  // scaling.hpp:66-70
        if (n < 1.0 - 1e-9 || n > nmax + 1e-9) throw Fail{WS_E_EVAL_RANGE, 0, 0, n, nmax};
        return value(locate(n), n);
    }
    double inverse_exact(double target) const {  // scaling.hpp:118-137
        if (target <= value(p.back(), nmax)) return nmax;
        for (const Piece& q : p) {
            const double hi_val = value(q, q.lo);
            const double lo_val = value(q, q.hi);
            const double b = q.bw * w;
            const double base = q.alpha + q.bc * c;
            if (target > hi_val + 1e-15 * std::abs(hi_val)) {
                if (b <= 0.0) return 0.0;
                return b / (target - base);
            }
            if (target >= lo_val) {
                if (b <= 0.0) return q.lo;
                if (target <= base) return q.hi;
                return std::clamp(b / (target - base), q.lo, q.hi);
            }
        }
        return nmax;
    }
};

// ScalingCurve::from_pieces (scaling.hpp:39-57)
Curve make_curve(std::vector<Piece> pieces, double c, double w) {
    std::sort(pieces.begin(), pieces.end(), [](const Piece& a, const Piece& b) { return a.lo < b.lo; });
    if (std::abs(pieces.front().lo - 1.0) > 1e-9) throw Fail{WS_E_CURVE_START};
    for (std::size_t i = 0; i + 1 < pieces.size(); ++i)
        if (std::abs(pieces[i].hi - pieces[i + 1].lo) > 1e-9) throw Fail{WS_E_CURVE_CONTIG};
    Curve cv;
    cv.p = std::move(pieces);
    cv.c = c;
    cv.w = w;
    cv.nmax = cv.p.back().hi;
    return cv;
}

struct Pt {
    int n;
    double t;
};

// fit_curve (scaling.hpp:229-322)
Curve fit_curve(const std::vector<Pt>& pts, const std::vector<int>& breaks, double c, double w) {
    if (pts.empty()) throw Fail{WS_E_FIT_NO_POINTS};
    int nmax = 1;
    for (const Pt& q : pts) {
        if (q.n < 1) throw Fail{WS_E_FIT_BAD_N};
        if (q.t <= 0.0) throw Fail{WS_E_FIT_BAD_TIME};
        nmax = std::max(nmax, q.n);
    }
    std::vector<int> bounds{1};
    for (int b : breaks) {
        if (b <= bounds.back() || b >= nmax) throw Fail{WS_E_FIT_BREAKPOINT, b};
        bounds.push_back(b);
    }
    bounds.push_back(nmax);
    std::vector<Piece> pieces;
    for (std::size_t i = 0; i + 1 < bounds.size(); ++i) {
        const int lo = bounds[i], hi = bounds[i + 1];
        std::vector<Pt> seg;
        for (const Pt& q : pts) {
            const bool in = i == 0 ? (q.n >= lo && q.n <= hi) : (q.n > lo && q.n <= hi);
            if (in) seg.push_back(q);
        }
        std::set<int> distinct;
        for (const Pt& q : seg) distinct.insert(q.n);
        if (distinct.size() < 2) throw Fail{WS_E_FIT_PIECE_POINTS, lo, hi};
        // fit_inverse_linear (scaling.hpp:175-190): sums in point order
        double sx = 0, sy = 0, sxy = 0, sxx = 0;
        const double m = static_cast<double>(seg.size());
        for (const Pt& q : seg) {
            const double x = 1.0 / static_cast<double>(q.n);
            sx += x;
            sy += q.t;
            sxy += x * q.t;
            sxx += x * x;
        }
        const double denom = m * sxx - sx * sx;
        if (std::abs(denom) < 1e-18) throw Fail{WS_E_FIT_DEGENERATE_X};
        const double slope = (m * sxy - sx * sy) / denom;
        const double intercept = (sy - slope * sx) / m;
        pieces.push_back({static_cast<double>(lo), static_cast<double>(hi), intercept, 0.0, slope / w});
    }
    for (std::size_t i = 1; i < pieces.size(); ++i) {  // continuity join (:282-287)
        const double bound = pieces[i].lo;
        const double left = pieces[i - 1].alpha + pieces[i - 1].bw * w / bound;
        const double right = pieces[i].alpha + pieces[i].bw * w / bound;
        pieces[i].alpha += left - right;
    }
    Curve cv = make_curve(pieces, c, w);
    // isotonic correction over integer anchors (:293-316, PAV :193-220)
    std::vector<double> v(static_cast<std::size_t>(nmax));
    for (int k = 1; k <= nmax; ++k) v[k - 1] = cv.eval(k);
    struct Block {
        double sum;
        int count;
    };
    std::vector<Block> blocks;
    bool changed = false;
    for (double x : v) {
        blocks.push_back({x, 1});
        while (blocks.size() >= 2) {
            Block& prev = blocks[blocks.size() - 2];
            Block& last = blocks.back();
            if (prev.sum / prev.count >= last.sum / last.count - 1e-15) break;
            prev.sum += last.sum;
            prev.count += last.count;
            blocks.pop_back();
            changed = true;
        }
    }
    if (changed) {
        std::size_t i = 0;
        for (const Block& bl : blocks) {
            const double mean = bl.sum / bl.count;
            for (int k = 0; k < bl.count; ++k) v[i++] = mean;
        }
        std::vector<Piece> fixed;
        for (int k = 1; k < nmax; ++k) {
            const double v0 = v[k - 1], v1 = v[k];
            const double b = (v0 - v1) / (1.0 / k - 1.0 / (k + 1.0));
            Piece q;
            q.lo = k;
            q.hi = k + 1;
            q.bw = b / w;
            q.alpha = v0 - b / k;
            q.bc = 0.0;
            fixed.push_back(q);
        }
        cv = make_curve(fixed, c, w);
    }
    for (int k = 1; k <= nmax; ++k)
        if (cv.eval(k) <= 0.0) throw Fail{WS_E_FIT_NONPOSITIVE, k};
    return cv;
}

bool dec_less(int a, int b) {  // "m<a>" < "m<b>" as std::string
    const std::string sa = std::to_string(a), sb = std::to_string(b);
    return sa < sb;
}

struct Tuple {
    int k;  // metaop number
    int n;
    int layers;
};

struct EntryRec {
    int k, n, layers;
    double span;
    uint64_t mask = 0;
    int rot = 0;
};

struct WaveRec {
    int level;
    double start, dur;
    std::vector<int> entries;  // global entry indices
};

struct FlowRec {
    int from_wave, from_k, to_wave, to_k;
    uint64_t vol;
    int mode;
};

struct PlanOut {
    // metaop k -> module
    std::vector<int> mod_of, level, upper_n, upper_l, lower_n, lower_l;
    std::vector<std::vector<Piece>> curve_of;  // per metaop
    std::vector<std::pair<int, int>> edges;
    std::vector<double> c_star;
    std::vector<int> level_first_wave, level_nwaves;
    std::vector<WaveRec> waves;
    std::vector<EntryRec> entries;
    std::vector<FlowRec> flows;
    std::vector<std::pair<int, int>> scope;  // per entity (metaop, task) for task-scoped strategies
    double lower_bound = 0, end_time = 0;
};

class Planner {
public:
    Planner(const ws_batch& b, int plan) : B(b), R(b.plans[plan]) {}

    void run(PlanOut& out) {
        N = R.n_dev;
        M = R.n_mod;
        if (N > kOracleMaxDevices) throw Fail{WS_E_LIMIT_DEVICES};  // u64 device masks
        if (M > WS_MAX_MODULES) throw Fail{WS_E_LIMIT_MODULES};
        build_graph();          // graph.hpp:97-147 + topo order/contract/levels :66-226
        fit_modules();          // planner.hpp:66-94
        if (R.strategy == WS_STRATEGY_DECOUPLED_SEQUENTIAL)
            decoupled();        // baselines.hpp:104-131
        else if (R.strategy == WS_STRATEGY_DISTMM_MT)
            distmm();           // baselines.hpp:323-413
        else if (R.strategy == WS_STRATEGY_TASK_OPTIMUS)
            optimus();          // baselines.hpp:133-321
        else
            allocate_and_schedule(out);
        if (!scoped) {          // entities are the MetaOps (planner.hpp:99-122)
            KE = K;
            e_mod.resize(K);
            for (int k = 0; k < K; ++k) e_mod[k] = k;
            e_task.assign(K, -1);
            e_frac.assign(K, 1.0);
            e_by_rank = by_rank;
            e_idrank = idrank;
            e_edges = edges;
        }
        place(out);
        fill(out);
    }

private:
    const ws_batch& B;
    const ws_plan_rec& R;
    int N = 0, M = 0;

    // module level (index = local module, std::map<kind> order)
    std::vector<uint64_t> adj, taskmask;
    uint64_t used = 0;
    // metaops
    int K = 0;
    std::vector<int> mod_of, k_of_mod, idrank, level;
    std::vector<int> by_rank;  // metaop numbers in id-string order
    std::vector<std::vector<int>> levels;
    std::vector<std::pair<int, int>> edges;
    std::vector<Curve> mcurve;  // per module
    std::vector<uint64_t> valid;  // per metaop, bit n-1
    // schedule
    std::vector<int> upper_n, upper_l, lower_n, lower_l;
    std::vector<double> cstar;
    // placement entities: the MetaOps, or (MetaOp, task) pairs for the task-scoped baselines
    bool scoped = false;
    struct PGroup {  // one place() call: waves (record order) on devices [off, off+cnt)
        std::vector<int> waves;
        int off = 0, cnt = 0;
    };
    std::vector<PGroup> pgroups;  // empty: a single call over everything
    int KE = 0;
    std::vector<int> e_mod, e_task, e_by_rank, e_idrank;
    std::vector<double> e_frac;
    std::vector<std::pair<int, int>> e_edges;  // deps between entities, std::set<pair<string,string>> order
    const std::vector<Curve>* curve_override = nullptr;  // per MetaOp, while a scaled level runs
    std::vector<WaveRec> waves;
    std::vector<EntryRec> entries;
    std::vector<FlowRec> flows;
    std::vector<int> level_first_wave, level_nwaves;
    double lower_bound = 0, end_time = 0;

    int mg(int m) const { return R.mod_begin + m; }
    std::string kind(int m) const {
        return std::string(reinterpret_cast<const char*>(B.names) + B.mod_name_off[mg(m)], B.mod_name_len[mg(m)]);
    }
    std::string op_id(int m, int layer) const { return kind(m) + "." + std::to_string(layer); }
    int layers(int m) const { return B.mod_layers[mg(m)]; }

    // ---- subsystem (1): graph, lexicographic Kahn, contraction, levels ----
    void build_graph() {
        adj.assign(M, 0);
        taskmask.assign(M, 0);
        for (int t = 0; t < R.n_tasks; ++t) {
            const int tg = R.task_begin + t;
            const int* tok = B.tokens + B.task_tok_off[tg];
            const int ntok = B.task_tok_n[tg];
            const uint64_t tbit = 1ull << B.task_rank[tg];
            uint64_t prev_tails = 0, heads = 0, tails = 0;
            int last = -1;
            bool branch_start = true;
            auto end_branch = [&] {
                if (last >= 0) tails |= 1ull << last;
                last = -1;
                branch_start = true;
            };
            for (int i = 0; i <= ntok; ++i) {
                const int v = i < ntok ? tok[i] : WS_TOK_STEP;
                if (v >= 0) {
                    used |= 1ull << v;
                    taskmask[v] |= tbit;
                    if (branch_start) heads |= 1ull << v;      // graph.hpp:130
                    else adj[last] |= 1ull << v;               // chained module (:131)
                    branch_start = false;
                    last = v;
                } else if (v == WS_TOK_BRANCH) {
                    end_branch();
                } else {
                    end_branch();
                    for (int f = 0; f < M; ++f)                // step edges (:137-139)
                        if (prev_tails >> f & 1ull) adj[f] |= heads;
                    prev_tails = tails;
                    heads = tails = 0;
                }
            }
        }
        // topo order with lexicographic tie-break over operator ids (graph.hpp:66-90)
        std::vector<int> indeg(M, 0), cursor(M, 0);
        for (int a = 0; a < M; ++a)
            for (int b = 0; b < M; ++b)
                if (adj[a] >> b & 1ull) indeg[b]++;
        k_of_mod.assign(M, -1);
        long total_ops = 0, popped = 0;
        for (int m = 0; m < M; ++m)
            if (used >> m & 1ull) total_ops += layers(m);
        while (true) {
            int best = -1;
            std::string best_key;
            for (int m = 0; m < M; ++m) {
                if (!(used >> m & 1ull) || cursor[m] >= layers(m)) continue;
                if (cursor[m] == 0 && indeg[m] != 0) continue;
                std::string key = op_id(m, cursor[m]);
                if (best < 0 || key < best_key) {
                    best = m;
                    best_key = key;
                }
            }
            if (best < 0) break;
            ++popped;
            if (cursor[best] == 0) {  // contract(): the chain head opens MetaOp m<K> (:172-176)
                k_of_mod[best] = K++;
                mod_of.push_back(best);
            }
            if (++cursor[best] == layers(best))
                for (int s = 0; s < M; ++s)
                    if (adj[best] >> s & 1ull) indeg[s]--;
        }
        if (popped != total_ops) throw Fail{WS_E_CYCLIC_WORKLOAD};
        // MetaOp ids "m<k>" in std::map order
        by_rank.resize(K);
        for (int k = 0; k < K; ++k) by_rank[k] = k;
        std::sort(by_rank.begin(), by_rank.end(), dec_less);
        idrank.assign(K, 0);
        for (int r = 0; r < K; ++r) idrank[by_rank[r]] = r;
        // metagraph edges (:196-200), std::set order
        for (int a = 0; a < M; ++a)
            for (int b = 0; b < M; ++b)
                if ((adj[a] >> b & 1ull) && a != b) edges.push_back({k_of_mod[a], k_of_mod[b]});
        std::sort(edges.begin(), edges.end(), [&](const auto& x, const auto& y) {
            if (idrank[x.first] != idrank[y.first]) return idrank[x.first] < idrank[y.first];
            return idrank[x.second] < idrank[y.second];
        });
        // longest-path levels (:207-226); numbering order is topological
        level.assign(K, 0);
        int maxl = 0;
        for (int k = 0; k < K; ++k) {
            int lv = 0;
            for (const auto& e : edges)
                if (e.second == k) lv = std::max(lv, level[e.first] + 1);
            level[k] = lv;
            maxl = std::max(maxl, lv);
        }
        levels.assign(maxl + 1, {});
        for (int r = 0; r < K; ++r) levels[level[by_rank[r]]].push_back(by_rank[r]);
    }

    // ---- subsystem (2): curve fit per module kind (planner.hpp:66-94) ----
    void fit_modules() {
        mcurve.assign(M, Curve{});
        for (int m = 0; m < M; ++m) {
            const int g = mg(m);
            const double c = B.mod_c[g], w = B.mod_w[g];
            if (B.mod_pre_err[g]) throw Fail{B.mod_pre_err[g]};
            std::vector<int> breaks;
            if (B.mod_bp_n[g] >= 0)
                for (int i = 0; i < B.mod_bp_n[g]; ++i) {
                    const int b = B.bps[B.mod_bp_off[g] + i];
                    if (b > 1 && b < N) breaks.push_back(b);
                }
            std::vector<Pt> pts;
            if (B.mod_prof_n[g] >= 0) {
                for (int i = 0; i < B.mod_prof_n[g]; ++i)
                    pts.push_back({B.prof_n[B.mod_prof_off[g] + i], B.prof_t[B.mod_prof_off[g] + i]});
            } else if (B.mod_truth_n[g] >= 0) {
                // materialize_truth (planner.hpp:43-53)
                std::vector<Piece> pieces;
                for (int i = 0; i < B.mod_truth_n[g]; ++i) {
                    const double* q = B.truth + 5 * (B.mod_truth_off[g] + i);
                    Piece p{q[0], q[1], q[2], q[3], q[4]};
                    if (p.lo >= N) continue;
                    p.hi = std::min(p.hi, static_cast<double>(N));
                    pieces.push_back(p);
                }
                if (pieces.empty()) throw Fail{WS_E_TRUTH_RANGE};
                pieces.back().hi = N;
                const Curve truth = make_curve(pieces, c, w);
                for (int n = 1; n <= N; ++n) pts.push_back({n, truth.eval(n)});  // synth_profile, noise 0
                if (breaks.empty())
                    for (std::size_t i = 0; i + 1 < truth.p.size(); ++i) {
                        const int b = static_cast<int>(std::llround(truth.p[i].hi));
                        if (b > 1 && b < N) breaks.push_back(b);
                    }
            } else {
                throw Fail{WS_E_NO_SOURCE, m};
            }
            mcurve[m] = fit_curve(pts, breaks, c, w);
            if (static_cast<int>(mcurve[m].p.size()) > WS_MAX_PIECES) throw Fail{WS_E_LIMIT_PIECES};
        }
    }

    const Curve& curve(int k) const { return curve_override ? (*curve_override)[k] : mcurve[mod_of[k]]; }
    double T(int k, int n) const { return curve(k).eval(n); }

    // ---- subsystem (3)+(4a): allocation and wave scheduling per level ----
    void allocate_and_schedule(PlanOut&) {
        valid.assign(K, 0);
        for (int r = 0; r < K; ++r) {  // valid_allocations in id order (allocation.hpp:51-63)
            const int k = by_rank[r];
            const int g = mg(mod_of[k]);
            const int tp = B.mod_tp[g];
            if (tp > N) throw Fail{WS_E_TP_EXCEEDS, k, tp};
            for (int n = 1; n <= N; ++n) {
                if (n % tp != 0) continue;
                if (B.mod_batch[g] % (n / tp) != 0) continue;
                valid[k] |= 1ull << (n - 1);
            }
        }
        upper_n.assign(K, 0);
        upper_l.assign(K, 0);
        lower_n.assign(K, 0);
        lower_l.assign(K, 0);
        double offset = 0.0;
        for (std::size_t L = 0; L < levels.size(); ++L) {
            const std::vector<int>& lv = levels[L];
            const double cs = solve_and_discretize(lv);
            cstar.push_back(cs);
            lower_bound += cs;
            // schedule_level + merge_levels (schedule.hpp:233-309)
            level_first_wave.push_back(static_cast<int>(waves.size()));
            const std::size_t w0 = waves.size();
            schedule_level(lv, static_cast<int>(L));
            double level_end = offset;
            for (std::size_t w = w0; w < waves.size(); ++w) {
                waves[w].start += offset;
                level_end = std::max(level_end, waves[w].start + waves[w].dur);
            }
            offset = level_end;
            level_nwaves.push_back(static_cast<int>(waves.size() - w0));
        }
        end_time = offset;
    }

    // plan_decoupled_sequential (baselines.hpp:104-131): MetaOps in
    // detail::topo_order (ready set ordered by id string, graph.hpp:67-90),
    // each alone on valid_allocations(m).back() for m.length * eval(n).
    void decoupled() {
        std::vector<int> indeg(K, 0);
        std::vector<std::vector<int>> succ(K);
        for (const auto& [a, b] : edges) {
            succ[a].push_back(b);
            ++indeg[b];
        }
        std::set<std::string> ready;
        for (int k = 0; k < K; ++k)
            if (!indeg[k]) ready.insert("m" + std::to_string(k));
        upper_n.assign(K, 0);
        upper_l.assign(K, 0);
        lower_n.assign(K, 0);
        lower_l.assign(K, 0);
        valid.assign(K, 0);
        double now = 0.0;
        while (!ready.empty()) {
            const int k = std::stoi(ready.begin()->substr(1));
            ready.erase(ready.begin());
            const int g = mg(mod_of[k]);
            const int tp = B.mod_tp[g];
            if (tp > N) throw Fail{WS_E_TP_EXCEEDS, k, tp};
            int n = 0;
            for (int x = 1; x <= N; ++x)
                if (x % tp == 0 && B.mod_batch[g] % (x / tp) == 0) n = x;
            const int L = layers(mod_of[k]);
            const double span = L * curve(k).eval(n);
            WaveRec wv;
            wv.level = level[k];
            wv.start = now;
            wv.dur = span;
            wv.entries.push_back(static_cast<int>(entries.size()));
            EntryRec e;
            e.k = k;
            e.n = n;
            e.layers = L;
            e.span = span;
            entries.push_back(e);
            waves.push_back(wv);
            upper_n[k] = n;
            upper_l[k] = L;
            now += span;
            for (int q : succ[k])
                if (--indeg[q] == 0) ready.insert("m" + std::to_string(q));
        }
        end_time = now;
    }

    // "m<a>@<task a>" < "m<b>@<task b>" as std::string; tasks by id rank
    static bool scoped_less(int a, int ta, int b, int tb) {
        if (a == b) return ta < tb;
        const std::string sa = std::to_string(a), sb = std::to_string(b);
        if (sb.size() > sa.size() && sb.compare(0, sa.size(), sa) == 0) return false;  // '@' > digit
        if (sa.size() > sb.size() && sa.compare(0, sb.size(), sb) == 0) return true;
        return sa < sb;
    }

    // plan_distmm_mt (baselines.hpp:323-413): tasks in declaration order; in a
    // task, same-level MetaOps (task_view levels) split the cluster through
    // solve_continuous/discretize/schedule_level on curves whose per-device
    // term is scaled by the share fraction, dependent stages run alone on
    // their largest valid allocation.  Entities are (MetaOp, task) pairs.
    void distmm() {
        scoped = true;
        valid.assign(K, 0);
        for (int k = 0; k < K; ++k) {
            const int g = mg(mod_of[k]);
            const int tp = B.mod_tp[g];
            for (int n = 1; n <= N; ++n)
                if (n % tp == 0 && B.mod_batch[g] % (n / tp) == 0) valid[k] |= 1ull << (n - 1);
        }
        upper_n.assign(K, 0);
        upper_l.assign(K, 0);
        lower_n.assign(K, 0);
        lower_l.assign(K, 0);
        std::map<std::pair<int, int>, int> ent_of;
        std::vector<int> task_rank_of;
        auto entity = [&](int k, int t) {
            auto it = ent_of.find({k, t});
            if (it != ent_of.end()) return it->second;
            const int e = KE++;
            e_mod.push_back(k);
            e_task.push_back(t);
            e_frac.push_back(1.0 / static_cast<double>(popc(taskmask[mod_of[k]])));  // share_fraction
            ent_of[{k, t}] = e;
            return e;
        };
        std::vector<std::pair<int, int>> sdeps;  // (entity, entity)
        double now = 0.0;
        for (int t = 0; t < R.n_tasks; ++t) {
            const int tr = B.task_rank[R.task_begin + t];
            task_rank_of.push_back(tr);
            std::vector<char> mem(K, 0);
            for (int k = 0; k < K; ++k) mem[k] = (taskmask[mod_of[k]] >> tr & 1ull) ? 1 : 0;
            std::vector<std::pair<int, int>> tedges;  // task_view edges, set order
            for (const auto& e : edges)
                if (mem[e.first] && mem[e.second]) tedges.push_back(e);
            // detail::topo_order over the members (ready set by id string)
            std::vector<int> indeg(K, 0), order;
            for (const auto& e : tedges) ++indeg[e.second];
            std::set<int> ready;
            for (int k = 0; k < K; ++k)
                if (mem[k] && !indeg[k]) ready.insert(idrank[k]);
            while (!ready.empty()) {
                const int k = by_rank[*ready.begin()];
                ready.erase(ready.begin());
                order.push_back(k);
                for (const auto& e : tedges)
                    if (e.first == k && --indeg[e.second] == 0) ready.insert(idrank[e.second]);
            }
            std::vector<int> lvl(K, 0);
            int max_level = 0;
            for (int k : order) {
                int lv = 0;
                for (const auto& e : tedges)
                    if (e.second == k) lv = std::max(lv, lvl[e.first] + 1);
                lvl[k] = lv;
                max_level = std::max(max_level, lv);
            }
            for (int l = 0; l <= max_level; ++l) {
                std::vector<int> ids;
                for (int k : order)
                    if (lvl[k] == l) ids.push_back(k);
                if (ids.empty()) continue;
                std::vector<Curve> scaled(K);
                for (int k : ids) {
                    const int e = entity(k, t);
                    std::vector<Piece> pcs = mcurve[mod_of[k]].p;  // detail::scale_curve
                    for (Piece& q : pcs) q.bw *= e_frac[e];
                    scaled[k] = make_curve(pcs, mcurve[mod_of[k]].c, mcurve[mod_of[k]].w);
                    const int tp = B.mod_tp[mg(mod_of[k])];
                    if (tp > N) throw Fail{WS_E_TP_EXCEEDS, k, tp};  // valid_allocations
                }
                if (ids.size() == 1) {
                    const int k = ids[0];
                    const int n = 64 - __builtin_clzll(valid[k]);  // valid.back()
                    const int L = layers(mod_of[k]);
                    const double span = L * scaled[k].eval(n);
                    WaveRec wv;
                    wv.level = l;
                    wv.start = now;
                    wv.dur = span;
                    wv.entries.push_back(static_cast<int>(entries.size()));
                    EntryRec en;
                    en.k = entity(k, t);
                    en.n = n;
                    en.layers = L;
                    en.span = span;
                    entries.push_back(en);
                    waves.push_back(wv);
                    now += span;
                } else {
                    curve_override = &scaled;
                    solve_and_discretize(ids);  // sums in task order
                    std::vector<int> ids_id(ids);
                    std::sort(ids_id.begin(), ids_id.end(), [&](int a, int b) { return idrank[a] < idrank[b]; });
                    const std::size_t w0 = waves.size(), e0 = entries.size();
                    schedule_level(ids_id, l);
                    curve_override = nullptr;
                    double t_end = 0.0;
                    for (std::size_t w = w0; w < waves.size(); ++w) t_end += waves[w].dur;
                    for (std::size_t w = w0; w < waves.size(); ++w) waves[w].start += now;
                    now += t_end;
                    for (std::size_t x = e0; x < entries.size(); ++x) entries[x].k = entity(entries[x].k, t);
                }
            }
            for (const auto& e : tedges) sdeps.push_back({entity(e.first, t), entity(e.second, t)});
        }
        auto eless = [&](int a, int b) {
            return scoped_less(e_mod[a], task_rank_of[e_task[a]], e_mod[b], task_rank_of[e_task[b]]);
        };
        e_by_rank.resize(KE);
        for (int e = 0; e < KE; ++e) e_by_rank[e] = e;
        std::sort(e_by_rank.begin(), e_by_rank.end(), eless);
        e_idrank.assign(KE, 0);
        for (int r = 0; r < KE; ++r) e_idrank[e_by_rank[r]] = r;
        std::sort(sdeps.begin(), sdeps.end(), [&](const auto& x, const auto& y) {
            if (x.first != y.first) return e_idrank[x.first] < e_idrank[y.first];
            return e_idrank[x.second] < e_idrank[y.second];
        });
        sdeps.erase(std::unique(sdeps.begin(), sdeps.end()), sdeps.end());
        e_edges = sdeps;
        end_time = now;
    }

    // ScalingCurve::eval_batch_fraction (scaling.hpp:83-86)
    double eval_bf(const Curve& cv, double n, double frac) const {
        const Piece& q = n < 1.0 ? cv.p.front() : cv.locate(std::min(n, cv.nmax));
        return q.alpha + q.bc * cv.c + q.bw * cv.w * frac / n;
    }

    // plan_task_level_optimus (baselines.hpp:133-321): every task gets a
    // device block sized by marginal gain of its critical-path time, runs its
    // MetaOps one after another on the whole block, and is placed on its own
    // sub-topology; waves take global indices by (start, id).
    void optimus() {
        scoped = true;
        valid.assign(K, 0);
        for (int k = 0; k < K; ++k) {
            const int g = mg(mod_of[k]);
            const int tp = B.mod_tp[g];
            for (int n = 1; n <= N; ++n)
                if (n % tp == 0 && B.mod_batch[g] % (n / tp) == 0) valid[k] |= 1ull << (n - 1);
        }
        upper_n.assign(K, 0);
        upper_l.assign(K, 0);
        lower_n.assign(K, 0);
        lower_l.assign(K, 0);
        struct Task {
            int t = 0;
            std::vector<int> order;
            std::vector<std::pair<int, int>> tedges;
            uint64_t valid = 0;
            int alloc = 0;
        };
        std::vector<Task> tasks;
        std::vector<int> task_rank_of;
        for (int t = 0; t < R.n_tasks; ++t) {
            Task task;
            task.t = t;
            const int tr = B.task_rank[R.task_begin + t];
            task_rank_of.push_back(tr);
            std::vector<char> mem(K, 0);
            for (int k = 0; k < K; ++k) mem[k] = (taskmask[mod_of[k]] >> tr & 1ull) ? 1 : 0;
            for (const auto& e : edges)
                if (mem[e.first] && mem[e.second]) task.tedges.push_back(e);
            std::vector<int> indeg(K, 0);
            for (const auto& e : task.tedges) ++indeg[e.second];
            std::set<int> ready;
            for (int k = 0; k < K; ++k)
                if (mem[k] && !indeg[k]) ready.insert(idrank[k]);
            while (!ready.empty()) {
                const int k = by_rank[*ready.begin()];
                ready.erase(ready.begin());
                task.order.push_back(k);
                for (const auto& e : task.tedges)
                    if (e.first == k && --indeg[e.second] == 0) ready.insert(idrank[e.second]);
            }
            for (int n = 1; n <= N; ++n) {  // valid for every member (valid_allocations per n, in order)
                bool ok = true;
                for (int k : task.order) {
                    const int tp = B.mod_tp[mg(mod_of[k])];
                    if (tp > N) throw Fail{WS_E_TP_EXCEEDS, k, tp};
                    if (!(valid[k] >> (n - 1) & 1ull)) {
                        ok = false;
                        break;
                    }
                }
                if (ok) task.valid |= 1ull << (n - 1);
            }
            if (!task.valid) throw Fail{WS_E_TASK_NO_VALID, t};
            tasks.push_back(task);
        }
        auto frac_of = [&](int k) { return 1.0 / static_cast<double>(popc(taskmask[mod_of[k]])); };
        auto task_time = [&](const Task& task, int n) {  // critical path at allocation n
            std::vector<double> finish(K, 0.0);
            double total = 0.0;
            for (int k : task.order) {
                const double weight = layers(mod_of[k]) * eval_bf(mcurve[mod_of[k]], n, frac_of(k));
                double start = 0.0;
                for (const auto& e : task.tedges)
                    if (e.second == k) start = std::max(start, finish[e.first]);
                finish[k] = start + weight;
                total = std::max(total, finish[k]);
            }
            return total;
        };
        auto lowest = [](uint64_t v) { return __builtin_ctzll(v) + 1; };
        std::vector<std::vector<std::size_t>> batches;
        {
            std::vector<std::size_t> current;
            int used = 0;
            for (std::size_t i = 0; i < tasks.size(); ++i) {
                const int need = lowest(tasks[i].valid);
                if (used + need > N && !current.empty()) {
                    batches.push_back(current);
                    current.clear();
                    used = 0;
                }
                current.push_back(i);
                used += need;
            }
            if (!current.empty()) batches.push_back(current);
        }
        std::map<std::pair<int, int>, int> ent_of;
        auto entity = [&](int k, int t) {
            auto it = ent_of.find({k, t});
            if (it != ent_of.end()) return it->second;
            const int e = KE++;
            e_mod.push_back(k);
            e_task.push_back(t);
            e_frac.push_back(frac_of(k));
            ent_of[{k, t}] = e;
            return e;
        };
        struct Placement {
            std::vector<int> wave_ids;  // creation order
            int off = 0, cnt = 0;
        };
        std::vector<Placement> placements;
        std::vector<WaveRec> ws;
        std::vector<EntryRec> es;
        std::vector<std::pair<int, int>> sdeps;
        double batch_offset = 0.0;
        for (const auto& batch : batches) {
            for (std::size_t ti : batch) tasks[ti].alloc = lowest(tasks[ti].valid);
            while (true) {
                int usedn = 0;
                for (std::size_t ti : batch) usedn += tasks[ti].alloc;
                const int free = N - usedn;
                if (free <= 0) break;
                std::size_t best = tasks.size();
                double best_gain = -1.0;
                int best_next = 0;
                for (std::size_t ti : batch) {
                    const Task& task = tasks[ti];
                    const uint64_t above = task.valid & ~((task.alloc >= 64) ? ~0ull : ((1ull << task.alloc) - 1));
                    if (!above) continue;  // std::upper_bound at the end
                    const int nx = lowest(above);
                    if (nx - task.alloc > free) continue;
                    const double gain = (task_time(task, task.alloc) - task_time(task, nx)) / (nx - task.alloc);
                    if (gain > best_gain) {
                        best_gain = gain;
                        best = ti;
                        best_next = nx;
                    }
                }
                if (best == tasks.size()) break;
                tasks[best].alloc = best_next;
            }
            double batch_end = batch_offset;
            int cursor = 0;
            for (std::size_t ti : batch) {
                Task& task = tasks[ti];
                Placement pl;
                pl.off = cursor;
                pl.cnt = task.alloc;
                cursor += task.alloc;
                double now = batch_offset;
                for (int k : task.order) {
                    const int e = entity(k, task.t);
                    const int L = layers(mod_of[k]);
                    const double span = L * eval_bf(mcurve[mod_of[k]], task.alloc, e_frac[e]);
                    WaveRec wv;
                    wv.level = level[k];
                    wv.start = now;
                    wv.dur = span;
                    wv.entries.push_back(static_cast<int>(es.size()));
                    EntryRec en;
                    en.k = e;
                    en.n = task.alloc;
                    en.layers = L;
                    en.span = span;
                    es.push_back(en);
                    pl.wave_ids.push_back(static_cast<int>(ws.size()));
                    ws.push_back(wv);
                    now += span;
                }
                for (const auto& ed : task.tedges) sdeps.push_back({entity(ed.first, task.t), entity(ed.second, task.t)});
                batch_end = std::max(batch_end, now);
                placements.push_back(pl);
            }
            batch_offset = batch_end;
        }
        // global indices by (start, id of the first entry)
        std::vector<int> order(ws.size());
        for (std::size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
        auto eless = [&](int a, int b) {
            return scoped_less(e_mod[a], task_rank_of[e_task[a]], e_mod[b], task_rank_of[e_task[b]]);
        };
        std::sort(order.begin(), order.end(), [&](int a, int b) {
            if (ws[a].start != ws[b].start) return ws[a].start < ws[b].start;
            return eless(es[ws[a].entries.front()].k, es[ws[b].entries.front()].k);
        });
        std::vector<int> gidx(ws.size());
        for (std::size_t i = 0; i < order.size(); ++i) gidx[order[i]] = static_cast<int>(i);
        waves.clear();
        entries.clear();
        for (int wi : order) {
            WaveRec wv = ws[wi];
            wv.entries.clear();
            for (int x : ws[wi].entries) {
                wv.entries.push_back(static_cast<int>(entries.size()));
                entries.push_back(es[x]);
            }
            waves.push_back(wv);
            end_time = std::max(end_time, wv.start + wv.dur);
        }
        if (static_cast<int>(waves.size()) > WS_MAX_WAVES) throw Fail{WS_E_LIMIT_WAVES};
        for (const Placement& pl : placements) {
            PGroup g;
            for (int wi : pl.wave_ids) g.waves.push_back(gidx[wi]);
            g.off = pl.off;
            g.cnt = pl.cnt;
            pgroups.push_back(g);
        }
        e_by_rank.resize(KE);
        for (int e = 0; e < KE; ++e) e_by_rank[e] = e;
        std::sort(e_by_rank.begin(), e_by_rank.end(), eless);
        e_idrank.assign(KE, 0);
        for (int r = 0; r < KE; ++r) e_idrank[e_by_rank[r]] = r;
        std::sort(sdeps.begin(), sdeps.end(), [&](const auto& x, const auto& y) {
            if (x.first != y.first) return e_idrank[x.first] < e_idrank[y.first];
            return e_idrank[x.second] < e_idrank[y.second];
        });
        sdeps.erase(std::unique(sdeps.begin(), sdeps.end()), sdeps.end());
        e_edges = sdeps;
    }

    std::vector<int> valid_list(int k) const {
        std::vector<int> v;
        for (int n = 1; n <= N; ++n)
            if (valid[k] >> (n - 1) & 1ull) v.push_back(n);
        return v;
    }

    double solve_and_discretize(const std::vector<int>& lv) {
        // solve_continuous (allocation.hpp:71-99)
        const double nd = N;
        double c_lo = 0.0, c_hi = 0.0;
        for (int k : lv) {
            const Curve& cv = curve(k);
            const double ncap = std::min(nd, cv.nmax);
            const int L = layers(mod_of[k]);
            c_lo = std::max(c_lo, cv.eval(ncap) * L);
            c_hi += cv.eval(1.0) * L;
        }
        auto probe = [&](double c) {
            double total = 0.0;
            for (int k : lv) total += std::min(curve(k).inverse_exact(c / layers(mod_of[k])), nd);
            return total;
        };
        for (int it = 0; it < R.max_iters && (c_hi - c_lo) > R.eps * c_hi; ++it) {
            const double mid = 0.5 * (c_lo + c_hi);
            if (probe(mid) < nd)
                c_hi = mid;
            else
                c_lo = mid;
        }
        const double cs = 0.5 * (c_lo + c_hi);
        // discretize (allocation.hpp:149-214), MetaOps in id order (the sums above
        // run in LevelInput order, which the distmm baseline sets to task order)
        std::vector<int> lv_id(lv);
        std::sort(lv_id.begin(), lv_id.end(), [&](int a, int b) { return idrank[a] < idrank[b]; });
        for (int k : lv_id) {
            const double nstar = std::min(curve(k).inverse_exact(cs / layers(mod_of[k])), nd);
            const std::vector<int> v = valid_list(k);
            const int L = layers(mod_of[k]);
            int exact = -1;
            for (int x : v)
                if (std::abs(x - nstar) < 1e-9) {
                    exact = x;
                    break;
                }
            int n_over = -1, n_under = -1;
            if (exact < 0)
                for (int x : v) {
                    if (x < nstar) n_under = x;
                    if (x > nstar) {
                        n_over = x;
                        break;
                    }
                }
            lower_l[k] = 0;
            lower_n[k] = 0;
            upper_l[k] = L;
            if (exact >= 0) {
                upper_n[k] = exact;
            } else if (n_over == -1) {
                upper_n[k] = v.back();
            } else if (n_under == -1) {
                upper_n[k] = v.front();
            } else {
                const double t_over = T(k, n_over);
                const double t_under = T(k, n_under);
                if (t_under - t_over <= 0.0) {
                    upper_n[k] = n_under;
                } else {
                    double lr = (cs - t_under * L) / (t_over - t_under);
                    lr = std::clamp(lr, 0.0, static_cast<double>(L));
                    int l_over = static_cast<int>(std::floor(lr + 0.5));
                    int l_under = L - l_over;
                    if (R.drop_floor > 0.0 && l_over > 0 && l_under > 0) {
                        if (l_over * t_over < R.drop_floor * cs) {
                            l_under += l_over;
                            l_over = 0;
                        } else if (l_under * t_under < R.drop_floor * cs) {
                            l_over += l_under;
                            l_under = 0;
                        }
                    }
                    if (l_over == 0) {
                        upper_n[k] = n_under;
                    } else if (l_under == 0) {
                        upper_n[k] = n_over;
                    } else {
                        upper_n[k] = n_over;
                        upper_l[k] = l_over;
                        lower_n[k] = n_under;
                        lower_l[k] = l_under;
                    }
                }
            }
        }
        // repair_capacity (allocation.hpp:107-139)
        while (true) {
            int widest = 0;
            for (int k : lv_id) widest += std::max(upper_n[k], lower_l[k] ? lower_n[k] : 0);
            if (widest <= N) break;
            int best = -1, best_target = 0;
            double best_pen = 0.0;
            for (int k : lv_id) {
                const std::vector<int> v = valid_list(k);
                auto it = std::lower_bound(v.begin(), v.end(), upper_n[k]);
                if (it == v.begin()) continue;
                const int target = *(it - 1);
                if (lower_l[k] && target <= lower_n[k]) continue;
                const double pen = upper_l[k] * (T(k, target) - T(k, upper_n[k]));
                if (best < 0 || pen < best_pen) {  // ties keep the smaller id (iteration order)
                    best = k;
                    best_pen = pen;
                    best_target = target;
                }
            }
            if (best < 0) break;
            upper_n[best] = best_target;
        }
        return cs;
    }

    // schedule.hpp:49-61
    double remaining_time(const std::vector<Tuple>& rem, int k, int at_n) const {
        int l = 0;
        for (const Tuple& t : rem)
            if (t.k == k) l += t.layers;
        return l * T(k, at_n);
    }

    int next_valid(int k, int n) const {  // std::upper_bound over the valid set
        for (int x = n + 1; x <= N; ++x)
            if (valid[k] >> (x - 1) & 1ull) return x;
        return -1;
    }

    // extend_resources_if_needed (schedule.hpp:144-173)
    void extend(std::vector<Tuple>& rem, const std::vector<std::size_t>& sel) const {
        while (true) {
            int usedn = 0;
            for (std::size_t i : sel) usedn += rem[i].n;
            const int idle = N - usedn;
            if (idle <= 0) break;
            std::size_t best = rem.size();
            double best_time = -1.0;
            int best_next = 0;
            for (std::size_t i : sel) {
                const Tuple& t = rem[i];
                const int nx = next_valid(t.k, t.n);
                if (nx < 0 || nx - t.n > idle) continue;
                const double r = remaining_time(rem, t.k, t.n);
                if (r > best_time || (r == best_time && best < rem.size() && idrank[t.k] < idrank[rem[best].k])) {
                    best = i;
                    best_time = r;
                    best_next = nx;
                }
            }
            if (best == rem.size()) break;
            rem[best].n = best_next;
        }
    }

    // propose_candidate_set (schedule.hpp:76-139)
    std::vector<std::size_t> propose(const std::vector<Tuple>& rem) const {
        auto greedy = [&](const std::vector<std::size_t>& order) {
            std::vector<std::size_t> sel;
            std::vector<int> taken;
            int cap = N;
            for (std::size_t i : order) {
                const Tuple& t = rem[i];
                if (t.n > cap) continue;
                if (std::find(taken.begin(), taken.end(), t.k) != taken.end()) continue;
                sel.push_back(i);
                taken.push_back(t.k);
                cap -= t.n;
            }
            return sel;
        };
        auto tt = [&](const Tuple& t) { return t.layers * T(t.k, t.n); };
        auto rt = [&](const Tuple& t) { return remaining_time(rem, t.k, t.n); };
        std::vector<std::size_t> by_n(rem.size()), by_time(rem.size()), by_cheap(rem.size());
        for (std::size_t i = 0; i < rem.size(); ++i) by_n[i] = by_time[i] = by_cheap[i] = i;
        std::sort(by_n.begin(), by_n.end(), [&](std::size_t a, std::size_t b) {
            if (rem[a].n != rem[b].n) return rem[a].n > rem[b].n;
            const double ra = tt(rem[a]), rb = tt(rem[b]);
            if (ra != rb) return ra > rb;
            return idrank[rem[a].k] < idrank[rem[b].k];
        });
        std::sort(by_time.begin(), by_time.end(), [&](std::size_t a, std::size_t b) {
            const double ra = rt(rem[a]), rb = rt(rem[b]);
            if (ra != rb) return ra > rb;
            if (rem[a].n != rem[b].n) return rem[a].n > rem[b].n;
            return idrank[rem[a].k] < idrank[rem[b].k];
        });
        std::sort(by_cheap.begin(), by_cheap.end(), [&](std::size_t a, std::size_t b) {
            if (rem[a].n != rem[b].n) return rem[a].n < rem[b].n;
            const double ra = rt(rem[a]), rb = rt(rem[b]);
            if (ra != rb) return ra > rb;
            return idrank[rem[a].k] < idrank[rem[b].k];
        });
        std::vector<std::size_t> best;
        long best_key = -1;
        for (const auto* order : {&by_n, &by_time, &by_cheap}) {
            std::vector<std::size_t> sel = greedy(*order);
            std::vector<Tuple> scratch = rem;
            extend(scratch, sel);
            int usedn = 0;
            for (std::size_t i : sel) usedn += scratch[i].n;
            const long key = static_cast<long>(usedn) * 1000 + static_cast<long>(sel.size());
            if (key > best_key) {
                best_key = key;
                best = sel;
            }
        }
        return best;
    }

    void schedule_level(const std::vector<int>& lv, int lvl) {
        std::vector<Tuple> rem;
        for (int k : lv) {
            rem.push_back({k, upper_n[k], upper_l[k]});
            if (lower_l[k]) rem.push_back({k, lower_n[k], lower_l[k]});
        }
        if (static_cast<int>(rem.size()) > WS_MAX_TUPLES) throw Fail{WS_E_LIMIT_TUPLES};
        std::vector<double> credit(K, 0.0);
        double now = 0.0;
        while (!rem.empty()) {
            std::vector<std::size_t> sel = propose(rem);
            if (sel.empty()) throw Fail{WS_E_NO_SCHEDULABLE};
            extend(rem, sel);
            // align_time_span (schedule.hpp:190-227)
            std::vector<int> pool(sel.size()), klay(sel.size()), absorbed(sel.size());
            for (std::size_t i = 0; i < sel.size(); ++i) {
                int l = 0;
                for (const Tuple& o : rem)
                    if (o.k == rem[sel[i]].k) l += o.layers;
                pool[i] = l;
            }
            double t_wave = 0.0;
            for (std::size_t i = 0; i < sel.size(); ++i) {
                const double span = pool[i] * T(rem[sel[i]].k, rem[sel[i]].n);
                if (i == 0 || span < t_wave) t_wave = span;
            }
            for (std::size_t i = 0; i < sel.size(); ++i) {
                const Tuple& t = rem[sel[i]];
                const double per = T(t.k, t.n);
                int kk;
                if (pool[i] * per <= t_wave * (1.0 + 1e-12)) {
                    kk = pool[i];
                    credit[t.k] = 0.0;
                } else {
                    const double budget = t_wave + std::min(credit[t.k], per);
                    kk = std::max(1, static_cast<int>(std::floor(budget / per * (1.0 + 1e-12))));
                    kk = std::min(kk, pool[i]);
                    credit[t.k] = std::max(0.0, budget - kk * per);
                }
                klay[i] = kk;
                absorbed[i] = std::max(0, kk - t.layers);
            }
            WaveRec wv;
            wv.level = lvl;
            wv.start = now;
            double dur = 0.0;
            for (std::size_t i = 0; i < sel.size(); ++i) {
                const Tuple& t = rem[sel[i]];
                EntryRec e;
                e.k = t.k;
                e.n = t.n;
                e.layers = klay[i];
                e.span = e.layers * T(t.k, t.n);
                dur = std::max(dur, e.span);
                wv.entries.push_back(static_cast<int>(entries.size()));
                entries.push_back(e);
            }
            wv.dur = dur;
            waves.push_back(wv);
            if (static_cast<int>(waves.size()) > WS_MAX_WAVES) throw Fail{WS_E_LIMIT_WAVES};
            if (static_cast<int>(entries.size()) > WS_MAX_ENTRIES) throw Fail{WS_E_LIMIT_ENTRIES};
            now += dur;
            for (std::size_t i = 0; i < sel.size(); ++i) {
                Tuple& t = rem[sel[i]];
                int ab = absorbed[i];
                t.layers -= klay[i] - ab;
                for (Tuple& o : rem) {
                    if (ab == 0) break;
                    if (&o == &t || o.k != t.k) continue;
                    const int take = std::min(ab, o.layers);
                    o.layers -= take;
                    ab -= take;
                }
            }
            std::vector<Tuple> next;
            for (const Tuple& t : rem)
                if (t.layers > 0) next.push_back(t);
            if (next.size() == rem.size()) throw Fail{WS_E_NO_PROGRESS};
            rem = std::move(next);
        }
    }

    // ---- subsystem (4b): placement (placement.hpp:168-447) ----
    struct Incoming {
        int src;  // global entry index of the producer placement
        uint64_t bytes;
    };

    int latest_entry_before(int k, int wave) const {  // last_wave_of (:152-156)
        for (int w = wave - 1; w >= 0; --w)
            for (int e : waves[w].entries)
                if (entries[e].k == k) return e;
        return -1;
    }
    int wave_of_entry(int e) const {
        for (std::size_t w = 0; w < waves.size(); ++w)
            for (int x : waves[w].entries)
                if (x == e) return static_cast<int>(w);
        return -1;
    }

    // entity tables (planner.hpp:99-151)
    std::vector<uint64_t> cont_bytes, edge_bytes, mem_act, ent_param;
    std::vector<int> gkey;

    std::vector<Incoming> incoming(int wave, int k) const {  // :188-206
        std::vector<Incoming> in;
        const int cont = latest_entry_before(k, wave);
        if (cont >= 0) {
            in.push_back({cont, cont_bytes[k]});
            return in;
        }
        for (const auto& e : e_edges) {  // preds in dep-set order
            if (e.second != k) continue;
            const int pe = latest_entry_before(e.first, wave);
            if (pe < 0) continue;
            in.push_back({pe, edge_bytes[e.first]});
        }
        return in;
    }

    std::vector<uint64_t> island_mask;
    std::vector<int> isl;

    void shard_moves(uint64_t from, uint64_t to, uint64_t full, uint64_t& intra, uint64_t& inter) const {
        intra = inter = 0;  // :74-103
        if (!from || !to) return;
        const uint64_t shared = from & to;
        uint64_t src = from & ~shared, dst = to & ~shared;
        const int units = std::max(popc(from), popc(to));
        const int moving = units - popc(shared);
        if (moving == 0) return;
        if (!src) src = from;
        if (!dst) dst = to;
        const double unit_bytes = static_cast<double>(full) / static_cast<double>(units);
        const uint64_t bytes = static_cast<uint64_t>(std::llround(unit_bytes));
        const int ns = popc(src), nt = popc(dst);
        for (int i = 0; i < moving; ++i) {
            const int s = nth_bit(src, i % ns), t = nth_bit(dst, i % nt);
            if (isl[s] == isl[t])
                intra += bytes;
            else
                inter += bytes;
        }
    }

    struct Score {
        bool feasible;
        int islands;
        double inter, intra, displaced, peak;
        uint64_t devs;
        bool operator<(const Score& o) const {  // :274-282
            if (feasible != o.feasible) return feasible;
            if (inter != o.inter) return inter < o.inter;
            if (intra != o.intra) return intra < o.intra;
            if (displaced != o.displaced) return displaced < o.displaced;
            if (islands != o.islands) return islands < o.islands;
            if (peak != o.peak) return peak < o.peak;
            // std::vector<int> compare of the sorted device lists
            const uint64_t diff = devs ^ o.devs;
            if (!diff) return false;
            return (devs & (diff & (~diff + 1))) != 0;
        }
    };

    struct State {
        double mem[WS_MAX_DEVICES];
        std::vector<uint64_t> charged;  // per group key: device mask
    };

    double delta(const State& st, int k, int d, int lay, int n) const {  // memory_delta :132-140
        double dl = lay * (static_cast<double>(mem_act[k]) / n);
        if (!(st.charged[gkey[k]] >> d & 1ull)) {
            const int tp = B.mod_tp[mg(mod_of[e_mod[k]])];
            dl += (1.0 + R.grad_mult) * static_cast<double>(ent_param[k]) / tp;
        }
        return dl;
    }

    void place(PlanOut&) {
        isl.assign(N, 0);
        island_mask.assign(R.n_islands, 0);
        for (int d = 0; d < N; ++d) {
            isl[d] = B.dev_island[R.dev_begin + d];
            island_mask[isl[d]] |= 1ull << d;
        }
        cont_bytes.assign(KE, 0);
        edge_bytes.assign(KE, 0);
        mem_act.assign(KE, 0);
        ent_param.assign(KE, 0);
        gkey.assign(KE, 0);
        for (int k = 0; k < KE; ++k) {  // build_memory_model / build_flow_inputs (planner.hpp:124-151)
            const int g = mg(mod_of[e_mod[k]]);
            const int L = layers(mod_of[e_mod[k]]);  // one MetaOp per module: length == layers
            const double frac = e_frac[k];            // batch_fraction
            ent_param[k] = static_cast<uint64_t>(static_cast<double>(B.mod_param[g]) * L / B.mod_layers[g]);
            const uint64_t act = B.mod_act[g];
            mem_act[k] = static_cast<uint64_t>(static_cast<double>(act) * frac);
            cont_bytes[k] = static_cast<uint64_t>(static_cast<double>(act) * frac);
            const uint64_t edge = B.mod_out[g] == 0 ? act : B.mod_out[g];
            edge_bytes[k] = static_cast<uint64_t>(static_cast<double>(edge) * frac);
            const bool whole = L == B.mod_layers[g];
            const int grp = whole ? B.mod_group[g] : -1;
            if (grp < 0)
                gkey[k] = R.n_groups + k;
            else if (!scoped && B.mod_alias[g] >= 0 && B.mod_alias[g] < K)
                gkey[k] = R.n_groups + B.mod_alias[g];  // param_group spelled like an entity id "m<j>"
            else
                gkey[k] = grp;
        }
        std::vector<int> last_wave(KE, -1);
        for (std::size_t w = 0; w < waves.size(); ++w)
            for (int e : waves[w].entries) last_wave[entries[e].k] = static_cast<int>(w);
        if (pgroups.empty()) {  // one place() call over every wave and device
            PGroup g;
            for (std::size_t w = 0; w < waves.size(); ++w) g.waves.push_back(static_cast<int>(w));
            g.off = 0;
            g.cnt = N;
            pgroups.push_back(g);
        }
        const std::vector<uint64_t> full_islands = island_mask;
        for (const PGroup& pg : pgroups) place_group(pg, last_wave, full_islands);
    }

    // one place() call (placement.hpp:168-447) over the waves of `pg` on the
    // device block [off, off+cnt) (detail::sub_topology: islands cut to the block)
    void place_group(const PGroup& pg, const std::vector<int>& last_wave, const std::vector<uint64_t>& full_islands) {
        const int gN = pg.cnt;
        const uint64_t all = (gN == 64 ? ~0ull : ((1ull << gN) - 1)) << pg.off;
        island_mask.clear();
        for (uint64_t m : full_islands)
            if (m & all) island_mask.push_back(m & all);
        const int n_isl = static_cast<int>(island_mask.size());
        const int nW = static_cast<int>(pg.waves.size());
        std::vector<int> seq_cursor(nW, 0);
        {
            int cur = 0;
            for (int j = 0; j < nW; ++j) {
                seq_cursor[j] = cur;
                for (int e : waves[pg.waves[j]].entries) cur = (cur + entries[e].n) % gN;
            }
        }
        std::vector<char> in_group(KE, 0);  // entities this place() call knows
        for (int w : pg.waves)
            for (int e : waves[w].entries) in_group[entries[e].k] = 1;
        State st;
        std::fill(st.mem, st.mem + WS_MAX_DEVICES, 0.0);
        st.charged.assign(R.n_groups + KE, 0);

        auto place_wave = [&](int j, int variant) -> bool {  // :340-406
            const int w = pg.waves[j];
            uint64_t free = all;
            std::vector<int> order(waves[w].entries);
            std::vector<std::vector<Incoming>> fin(order.size());
            for (std::size_t i = 0; i < order.size(); ++i) fin[i] = incoming(w, entries[order[i]].k);
            std::vector<std::size_t> idx(order.size());
            for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = i;
            if (!R.sequential)
                std::sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) {  // entry_order :208-221
                    uint64_t va = 0, vb = 0;
                    for (const Incoming& f : fin[a]) va += f.bytes;
                    for (const Incoming& f : fin[b]) vb += f.bytes;
                    if (va != vb) return va > vb;
                    return e_idrank[entries[order[a]].k] < e_idrank[entries[order[b]].k];
                });
            bool first = true;
            std::vector<char> placed_now(KE, 0);
            int cursor = R.sequential ? seq_cursor[j] : 0;
            for (std::size_t oi : idx) {
                EntryRec& e = entries[order[oi]];
                const std::vector<Incoming>& flows_in = fin[oi];
                std::vector<uint64_t> cands;
                std::vector<int> rots;
                if (R.sequential) {
                    if (popc(free) >= e.n) {
                        uint64_t m = 0;
                        for (int i = 0; i < e.n; ++i) m |= 1ull << (pg.off + (cursor + i) % gN);
                        cands.push_back(m);
                        rots.push_back(pg.off + cursor);
                        cursor = (cursor + e.n) % gN;
                    }
                } else {  // candidate_sets :223-263
                    std::set<uint64_t> seen;
                    auto push = [&](uint64_t m) {
                        if (popc(m) != e.n) return;
                        if (seen.insert(m).second) {
                            cands.push_back(m);
                            rots.push_back(0);
                        }
                    };
                    for (const Incoming& f : flows_in) {
                        const uint64_t m = entries[f.src].mask;
                        if (popc(m) == e.n && (m & ~free) == 0) push(m);
                    }
                    auto windows = [&](uint64_t pool) {
                        const int cnt = popc(pool);
                        for (int s = 0; s + e.n <= cnt; ++s) {
                            uint64_t m = 0;
                            for (int j = s; j < s + e.n; ++j) m |= 1ull << nth_bit(pool, j);
                            push(m);
                        }
                    };
                    for (int i = 0; i < n_isl; ++i) windows(free & island_mask[i]);
                    windows(free);
                }
                if (cands.empty()) return false;
                std::vector<Score> scores;
                for (uint64_t devs : cands) {  // score_candidate :285-325
                    Score s{};
                    s.devs = devs;
                    for (int i = 0; i < n_isl; ++i)
                        if (devs & island_mask[i]) s.islands++;
                    for (int r = 0; r < KE; ++r) {
                        const int e2 = e_by_rank[r];
                        if (e2 == e.k || !in_group[e2] || last_wave[e2] < w || placed_now[e2]) continue;
                        const int home = latest_entry_before(e2, w);
                        if (home < 0) continue;
                        const uint64_t hm = entries[home].mask;
                        const int overlap = popc(devs & hm);
                        if (overlap == 0) continue;
                        const double bytes = static_cast<double>(cont_bytes[e2]);
                        s.displaced += bytes * static_cast<double>(overlap) / static_cast<double>(popc(hm));
                    }
                    s.feasible = true;
                    double peak = 0.0;
                    for (int d = 0; d < N; ++d) {
                        if (!(devs >> d & 1ull)) continue;
                        const double usedm = st.mem[d] + delta(st, e.k, d, e.layers, e.n);
                        peak = std::max(peak, usedm);
                        if (usedm > static_cast<double>(R.mem_capacity)) s.feasible = false;
                    }
                    s.peak = peak;
                    for (const Incoming& f : flows_in) {
                        uint64_t a, b;
                        shard_moves(entries[f.src].mask, devs, f.bytes, a, b);
                        s.inter += static_cast<double>(b);
                        s.intra += static_cast<double>(a);
                    }
                    scores.push_back(s);
                }
                std::vector<std::size_t> sidx(scores.size());
                for (std::size_t i = 0; i < sidx.size(); ++i) sidx[i] = i;
                std::sort(sidx.begin(), sidx.end(), [&](std::size_t a, std::size_t b) { return scores[a] < scores[b]; });
                std::size_t pick = 0;
                if (!R.sequential && first) pick = std::min(static_cast<std::size_t>(variant), scores.size() - 1);
                const Score& ch = scores[sidx[pick]];
                if (!ch.feasible) return false;
                // commit_memory :142-149
                for (int d = 0; d < N; ++d) {
                    if (!(ch.devs >> d & 1ull)) continue;
                    st.mem[d] += delta(st, e.k, d, e.layers, e.n);
                    st.charged[gkey[e.k]] |= 1ull << d;
                }
                e.mask = ch.devs;
                e.rot = rots[sidx[pick]];
                for (const Incoming& f : flows_in) {  // flow records :376-400
                    uint64_t a, b;
                    shard_moves(entries[f.src].mask, ch.devs, f.bytes, a, b);
                    const int fw = wave_of_entry(f.src);
                    const int fk = entries[f.src].k;
                    if (a + b == 0) {
                        flows.push_back({fw, fk, w, e.k, 0, WS_FLOW_COPY});
                    } else {
                        if (a > 0) flows.push_back({fw, fk, w, e.k, a, WS_FLOW_INTRA});
                        if (b > 0) flows.push_back({fw, fk, w, e.k, b, WS_FLOW_INTER});
                    }
                }
                free &= ~ch.devs;
                placed_now[e.k] = 1;
                first = false;
            }
            return true;
        };

        // bounded DFS over wave variants (:409-441)
        std::vector<int> variant(nW, 0);
        long attempts = 0, budget = nW;
        for (int d = 0; d < R.bt_depth; ++d) budget *= std::max(1, R.bt_branching);
        std::vector<State> saved{st};
        std::vector<std::size_t> saved_flows{flows.size()};
        int k = 0;
        while (k < nW) {
            if (++attempts > budget) throw Fail{WS_E_BT_BUDGET, k};
            st = saved.back();
            flows.resize(saved_flows.back());
            for (int j = k; j < nW; ++j)
                for (int e : waves[pg.waves[j]].entries) entries[e].mask = 0, entries[e].rot = 0;
            const int branching = R.sequential ? 1 : R.bt_branching;
            if (variant[k] >= branching) {
                variant[k] = 0;
                if (k == 0) throw Fail{WS_E_NO_PLACEMENT_W0};
                saved.pop_back();
                saved_flows.pop_back();
                --k;
                ++variant[k];
                continue;
            }
            if (place_wave(k, variant[k])) {
                saved.push_back(st);
                saved_flows.push_back(flows.size());
                ++k;
            } else {
                ++variant[k];
            }
        }
        if (static_cast<int>(flows.size()) > WS_MAX_FLOWS) throw Fail{WS_E_LIMIT_FLOWS};
    }

    void fill(PlanOut& out) {
        if (scoped) {  // one record per (MetaOp, task) entity; curves are the unscaled base curves
            for (int e = 0; e < KE; ++e) {
                const int k = e_mod[e];
                out.mod_of.push_back(mod_of[k]);
                out.level.push_back(level[k]);
                out.upper_n.push_back(0);
                out.upper_l.push_back(0);
                out.lower_n.push_back(0);
                out.lower_l.push_back(0);
                out.curve_of.push_back(mcurve[mod_of[k]].p);
                out.scope.push_back({k, e_task[e]});
            }
            out.edges = e_edges;
            out.waves = waves;
            out.entries = entries;
            out.flows = flows;
            out.lower_bound = 0.0;
            out.end_time = end_time;
            return;
        }
        out.mod_of = mod_of;
        out.level = level;
        out.upper_n = upper_n;
        out.upper_l = upper_l;
        out.lower_n = lower_n;
        out.lower_l = lower_l;
        for (int k = 0; k < K; ++k) out.curve_of.push_back(curve(k).p);
        out.edges = edges;
        out.c_star = cstar;
        out.level_first_wave = level_first_wave;
        out.level_nwaves = level_nwaves;
        out.waves = waves;
        out.entries = entries;
        out.flows = flows;
        out.lower_bound = lower_bound;
        out.end_time = end_time;
    }
};

int status_of(int code) {
    switch (code) {
        case WS_E_CYCLIC_WORKLOAD:
        case WS_E_TRUTH_RANGE:
        case WS_E_NO_SOURCE:
        case WS_E_FIT_NO_POINTS:
        case WS_E_FIT_BAD_N:
        case WS_E_FIT_BAD_TIME:
        case WS_E_FIT_BREAKPOINT:
        case WS_E_FIT_PIECE_POINTS:
        case WS_E_FIT_DEGENERATE_X:
            return WS_STATUS_PARSE;
        case WS_E_FIT_NONPOSITIVE:
        case WS_E_TP_EXCEEDS:
        case WS_E_TASK_NO_VALID:
        case WS_E_BT_BUDGET:
        case WS_E_NO_PLACEMENT_W0:
            return WS_STATUS_INFEASIBLE;
        case WS_E_CURVE_START:
        case WS_E_CURVE_CONTIG:
        case WS_E_EVAL_RANGE:
        case WS_E_NO_SCHEDULABLE:
        case WS_E_NO_PROGRESS:
            return WS_STATUS_INVARIANT;
        default:
            return code >= 40 && code < 60 ? WS_STATUS_LIMIT : WS_STATUS_INTERNAL;
    }
}

std::size_t al8(std::size_t v) { return (v + 7) & ~std::size_t(7); }

}  // namespace

extern "C" {

// Plans every problem of `in` (host memory) serially; same output contract as
// ws_plan_batch_host.  Returns 0, or 1 if the arena was too small.
int wso_plan_batch(const ws_batch* in, ws_plan_result* results, uint8_t* arena, uint64_t arena_cap,
                   uint64_t* arena_used) {
    uint64_t top = 0;
    int rc = 0;
    for (int p = 0; p < in->n_plans; ++p) {
        ws_plan_result& r = results[p];
        std::memset(&r, 0, sizeof(r));
        PlanOut out;
        try {
            if (in->plans[p].n_mod == 0 && in->plans[p].n_tasks == 0) throw Fail{WS_E_HOST_PRESET};
            Planner(*in, p).run(out);
        } catch (const Fail& f) {
            r.status = status_of(f.code);
            r.err_code = f.code;
            r.err_a = f.a;
            r.err_b = f.b;
            r.err_x = f.x;
            r.err_y = f.y;
            if (f.code == WS_E_TP_EXCEEDS || f.code == WS_E_EVAL_RANGE || f.code == WS_E_HOST_PRESET)
                ;  // message arguments already set
            continue;
        }
        const int K = static_cast<int>(out.mod_of.size());
        int npieces = 0;
        for (const auto& c : out.curve_of) npieces += static_cast<int>(c.size());
        r.n_metaops = K;
        r.n_edges = static_cast<int>(out.edges.size());
        r.n_levels = static_cast<int>(out.c_star.size());
        r.n_waves = static_cast<int>(out.waves.size());
        r.n_entries = static_cast<int>(out.entries.size());
        r.n_flows = static_cast<int>(out.flows.size());
        r.n_pieces = npieces;
        r.lower_bound = out.lower_bound;
        r.end_time = out.end_time;
        r.n_scopes = static_cast<int>(out.scope.size());
        std::size_t sz = al8(sizeof(ws_out_metaop) * K) + al8(sizeof(ws_out_level) * r.n_levels) +
                         al8(sizeof(ws_out_piece) * npieces) + al8(sizeof(ws_out_edge) * r.n_edges) +
                         al8(sizeof(ws_out_wave) * r.n_waves) + al8(sizeof(ws_out_entry) * r.n_entries) +
                         al8(sizeof(ws_out_flow) * r.n_flows) + al8(sizeof(ws_out_scope) * r.n_scopes);
        if (top + sz > arena_cap) {
            r.status = WS_STATUS_INTERNAL;
            r.err_code = WS_E_ARENA_OVERFLOW;
            rc = 1;
            continue;
        }
        r.offset = top;
        r.size = sz;
        uint8_t* base = arena + top;
        top += sz;
        std::size_t off = 0;
        auto* mo = reinterpret_cast<ws_out_metaop*>(base + off);
        off += al8(sizeof(ws_out_metaop) * K);
        auto* lv = reinterpret_cast<ws_out_level*>(base + off);
        off += al8(sizeof(ws_out_level) * r.n_levels);
        auto* pc = reinterpret_cast<ws_out_piece*>(base + off);
        off += al8(sizeof(ws_out_piece) * npieces);
        auto* ed = reinterpret_cast<ws_out_edge*>(base + off);
        off += al8(sizeof(ws_out_edge) * r.n_edges);
        auto* wv = reinterpret_cast<ws_out_wave*>(base + off);
        off += al8(sizeof(ws_out_wave) * r.n_waves);
        auto* en = reinterpret_cast<ws_out_entry*>(base + off);
        off += al8(sizeof(ws_out_entry) * r.n_entries);
        auto* fl = reinterpret_cast<ws_out_flow*>(base + off);
        int pi = 0;
        for (int k = 0; k < K; ++k) {
            ws_out_metaop& m = mo[k];
            std::memset(&m, 0, sizeof(m));
            m.module = out.mod_of[k];
            m.level = out.level[k];
            m.first_layer = 0;
            m.length = in->mod_layers[in->plans[p].mod_begin + out.mod_of[k]];
            m.piece_begin = pi;
            m.piece_count = static_cast<int>(out.curve_of[k].size());
            for (const Piece& q : out.curve_of[k]) pc[pi++] = {q.lo, q.hi, q.alpha, q.bc, q.bw};
            m.upper_n = out.upper_n[k];
            m.upper_l = out.upper_l[k];
            m.lower_n = out.lower_n[k];
            m.lower_l = out.lower_l[k];
        }
        for (int l = 0; l < r.n_levels; ++l) {
            std::memset(&lv[l], 0, sizeof(lv[l]));
            lv[l].c_star = out.c_star[l];
            lv[l].first_wave = out.level_first_wave[l];
            lv[l].n_waves = out.level_nwaves[l];
        }
        for (int e = 0; e < r.n_edges; ++e) ed[e] = {out.edges[e].first, out.edges[e].second};
        for (int w = 0; w < r.n_waves; ++w) {
            std::memset(&wv[w], 0, sizeof(wv[w]));
            wv[w].start = out.waves[w].start;
            wv[w].duration = out.waves[w].dur;
            wv[w].level = out.waves[w].level;
            wv[w].entry_begin = out.waves[w].entries.empty() ? 0 : out.waves[w].entries.front();
            wv[w].n_entries = static_cast<int>(out.waves[w].entries.size());
        }
        for (int e = 0; e < r.n_entries; ++e) {
            std::memset(&en[e], 0, sizeof(en[e]));
            en[e].span = out.entries[e].span;
            en[e].devmask = out.entries[e].mask;
            en[e].metaop = out.entries[e].k;
            en[e].n = out.entries[e].n;
            en[e].layers = out.entries[e].layers;
            en[e].rot = out.entries[e].rot;
        }
        for (int f = 0; f < r.n_flows; ++f) {
            std::memset(&fl[f], 0, sizeof(fl[f]));
            fl[f].volume = out.flows[f].vol;
            fl[f].from_wave = out.flows[f].from_wave;
            fl[f].from_metaop = out.flows[f].from_k;
            fl[f].to_wave = out.flows[f].to_wave;
            fl[f].to_metaop = out.flows[f].to_k;
            fl[f].mode = out.flows[f].mode;
        }
        auto* sc = reinterpret_cast<ws_out_scope*>(base + off + al8(sizeof(ws_out_flow) * r.n_flows));
        for (int e = 0; e < r.n_scopes; ++e) sc[e] = {out.scope[e].first, out.scope[e].second};
    }
    *arena_used = top;
    return rc;
}

}  // extern "C"
