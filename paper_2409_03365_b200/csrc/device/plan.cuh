// plan.cuh — the warp-per-plan planning kernel (subsystems 1, 3, 4a, 4b).
//
// One 32-lane warp owns one planning problem.  Lanes split the parallel
// dimension of each step (tasks while building the module DAG, MetaOps in
// bisection probes and discretization, candidate device sets in placement
// scoring, devices in memory commits); the strictly sequential parts
// (lexicographic Kahn, the wave loop, the DFS over wave variants) run on lane
// 0 or warp-uniformly.  Every floating-point expression follows the
// reference's evaluation order; the file is compiled with -fmad=false.
#pragma once
#include "common.cuh"
#include "fit.cuh"
#include "layout.cuh"

namespace wsdev {

struct PlanArgs {
    ws_batch B;
    FitOut fit;            // read side of K2 output
    Caps caps;
    Layout L;
    char* scratch;         // [n_plans_in_launch * L.bytes]
    const int32_t* plan_ids;  // optional plan index list (retry pass)
    const int32_t* n_ids;     // device count of plan_ids (retry pass)
    int plan_base;            // first plan of this launch (no plan_ids)
    int n_launch;
    ws_plan_result* results;
    uint8_t* arena;
    unsigned long long* arena_top;
    unsigned long long arena_cap;
};

struct Ctl {  // per-warp control block in shared memory
    int err;
    int pad;
    long long a, b;
    double x, y;
    double level_offset;  // merge_levels running offset (lane 0 -> warp)
    int i0, i1, i2, i3;
};

// error-capturing T(n) lookup (ScalingCurve::eval at integer n, scaling.hpp:66-70)
struct TLookup {
    const double* ttab;
    const int32_t* nmax;  // per module (global index)
    int tstride;
    int mbase;            // plan's first module
    const int* mod_of;    // metaop -> local module
    Ctl* ctl;
    __device__ double operator()(int k, int n) const {
        const int m = mbase + mod_of[k];
        if (n > nmax[m]) {
            if (!ctl->err) {
                ctl->err = WS_E_EVAL_RANGE;
                ctl->x = n;
                ctl->y = nmax[m];
            }
            return 1.0;
        }
        return ttab[static_cast<int64_t>(m) * tstride + (n - 1)];
    }
};

struct PlanCtx {
    const ws_batch* B;
    const ws_plan_rec* R;
    const FitOut* fit;
    const Layout* L;
    char* base;
    Ctl* ctl;
    int lane, N, M, K, mbase;
    template <typename T>
    __device__ __forceinline__ T* at(int off) const {
        return reinterpret_cast<T*>(base + off);
    }
};

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool set_err(Ctl* ctl, int code, long long a = 0, long long b = 0) {
    if (!ctl->err) {
        ctl->err = code;
        ctl->a = a;
        ctl->b = b;
    }
    return false;
}

// kind byte i of module m followed by `suffix` (used for op ids "kind.layer")
struct OpKey {
    const uint8_t* name;
    int len;
    char tail[12];
    int tlen;
    __device__ int size() const { return len + tlen; }
    __device__ char at(int i) const { return i < len ? static_cast<char>(name[i]) : tail[i - len]; }
};

__device__ __forceinline__ OpKey op_key(const ws_batch& B, int gm, int layer, bool with_layer) {
    OpKey k;
    k.name = B.names + B.mod_name_off[gm];
    k.len = B.mod_name_len[gm];
    k.tail[0] = '.';
    k.tlen = 1;
    if (with_layer) {
        char t[11];
        int n = 0, v = layer;
        do { t[n++] = static_cast<char>('0' + v % 10); v /= 10; } while (v);
        while (n) k.tail[k.tlen++] = t[--n];
    }
    return k;
}

__device__ __forceinline__ bool key_less(const OpKey& a, const OpKey& b) {  // std::string operator<
    const int la = a.size(), lb = b.size();
    const int l = la < lb ? la : lb;
    for (int i = 0; i < l; ++i) {
        const unsigned char ca = static_cast<unsigned char>(a.at(i)), cb = static_cast<unsigned char>(b.at(i));
        if (ca != cb) return ca < cb;
    }
    return la < lb;
}

// ScalingCurve::inverse_exact (scaling.hpp:118-137) over the fitted pieces
__device__ double inverse_exact(const double* pc, int np, double c, double w, double nmax, double target) {
    auto val = [&](int i, double n) { return pc[5 * i + 2] + pc[5 * i + 3] * c + pc[5 * i + 4] * w / n; };
    if (target <= val(np - 1, nmax)) return nmax;
    for (int i = 0; i < np; ++i) {
        const double lo = pc[5 * i + 0], hi = pc[5 * i + 1];
        const double hi_val = val(i, lo);
        const double lo_val = val(i, hi);
        const double b = pc[5 * i + 4] * w;
        const double base = pc[5 * i + 2] + pc[5 * i + 3] * c;
        if (target > hi_val + 1e-15 * fabs(hi_val)) {
            if (b <= 0.0) return 0.0;
            return b / (target - base);
        }
        if (target >= lo_val) {
            if (b <= 0.0) return lo;
            if (target <= base) return hi;
            const double v = b / (target - base);
            return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
        }
    }
    return nmax;
}

// shard_moves (placement.hpp:74-103) on device-index bitmasks
__device__ __forceinline__ void shard_moves(uint64_t from, uint64_t to, uint64_t full, const int* isl,
                                            uint64_t& intra, uint64_t& inter) {
    intra = inter = 0;
    if (!from || !to) return;
    const uint64_t shared = from & to;
    uint64_t src = from & ~shared, dst = to & ~shared;
    const int pf = popc64(from), pt = popc64(to);
    const int units = pf > pt ? pf : pt;
    const int moving = units - popc64(shared);
    if (moving == 0) return;
    if (!src) src = from;
    if (!dst) dst = to;
    const double unit_bytes = static_cast<double>(full) / static_cast<double>(units);
    const uint64_t bytes = static_cast<uint64_t>(llround(unit_bytes));
    uint64_t rs = src, rt = dst;
    int same = 0;
    for (int i = 0; i < moving; ++i) {
        const int s = low_bit(rs);
        rs &= rs - 1;
        if (!rs) rs = src;
        const int t = low_bit(rt);
        rt &= rt - 1;
        if (!rt) rt = dst;
        same += isl[s] == isl[t];
    }
    intra = static_cast<uint64_t>(same) * bytes;
    inter = static_cast<uint64_t>(moving - same) * bytes;
}

// Score (placement.hpp:265-283)
struct Score {
    int valid;
    int feasible;
    int islands;
    double inter, intra, displaced, peak;
    uint64_t devs;
    int rot;
};

__device__ __forceinline__ bool score_less(const Score& a, const Score& b) {
    if (a.feasible != b.feasible) return a.feasible;
    if (a.inter != b.inter) return a.inter < b.inter;
    if (a.intra != b.intra) return a.intra < b.intra;
    if (a.displaced != b.displaced) return a.displaced < b.displaced;
    if (a.islands != b.islands) return a.islands < b.islands;
    if (a.peak != b.peak) return a.peak < b.peak;
    const uint64_t diff = a.devs ^ b.devs;  // sorted device-list lexicographic order
    if (!diff) return false;
    return (a.devs & (diff & (~diff + 1))) != 0;
}

__device__ __forceinline__ Score shfl_score(const Score& s, int src) {
    Score o;
    o.valid = __shfl_sync(kFull, s.valid, src);
    o.feasible = __shfl_sync(kFull, s.feasible, src);
    o.islands = __shfl_sync(kFull, s.islands, src);
    o.inter = __shfl_sync(kFull, s.inter, src);
    o.intra = __shfl_sync(kFull, s.intra, src);
    o.displaced = __shfl_sync(kFull, s.displaced, src);
    o.peak = __shfl_sync(kFull, s.peak, src);
    o.devs = __shfl_sync(kFull, s.devs, src);
    o.rot = __shfl_sync(kFull, s.rot, src);
    return o;
}

__device__ __forceinline__ Score warp_min_score(Score s) {
    for (int off = 16; off; off >>= 1) {
        Score o = shfl_score(s, (threadIdx.x & 31) ^ off);
        if (o.valid && (!s.valid || score_less(o, s))) s = o;
    }
    return s;
}

// ---------------------------------------------------------------------------
// subsystem (1): module DAG from the flows, lexicographic Kahn, contraction
// numbering, MetaGraph edges and longest-path levels (graph.hpp:66-226)
// ---------------------------------------------------------------------------
__device__ bool stage_graph(PlanCtx& C) {
    const ws_batch& B = *C.B;
    const ws_plan_rec& R = *C.R;
    const int M = C.M, lane = C.lane;
    uint64_t* adj = C.at<uint64_t>(C.L->adj);
    uint64_t* tmask = C.at<uint64_t>(C.L->tmask);
    int* kofm = C.at<int>(C.L->kofm);
    int* indeg = C.at<int>(C.L->indeg);
    int* keyrank = C.at<int>(C.L->keyrank);
    int* modat = C.at<int>(C.L->modat);
    for (int m = lane; m < M; m += 32) {
        adj[m] = 0;
        tmask[m] = 0;
        kofm[m] = -1;
    }
    __syncwarp();
    // tasks in parallel (graph.hpp:124-145): lane t walks the flow of task t
    for (int t = lane; t < R.n_tasks; t += 32) {
        const int tg = R.task_begin + t;
        const int* tok = B.tokens + B.task_tok_off[tg];
        const int ntok = B.task_tok_n[tg];
        const uint64_t tbit = 1ull << B.task_rank[tg];
        uint64_t prev_tails = 0, heads = 0, tails = 0;
        int last = -1;
        bool start = true;
        for (int i = 0; i <= ntok; ++i) {
            const int v = i < ntok ? tok[i] : WS_TOK_STEP;
            if (v >= 0) {
                atomicOr(reinterpret_cast<unsigned long long*>(&tmask[v]), tbit);
                if (start)
                    heads |= 1ull << v;
                else
                    atomicOr(reinterpret_cast<unsigned long long*>(&adj[last]), 1ull << v);
                start = false;
                last = v;
            } else {
                if (last >= 0) tails |= 1ull << last;
                last = -1;
                start = true;
                if (v == WS_TOK_STEP) {
                    for (uint64_t f = prev_tails; f; f &= f - 1)
                        atomicOr(reinterpret_cast<unsigned long long*>(&adj[low_bit(f)]), heads);
                    prev_tails = tails;
                    heads = tails = 0;
                }
            }
        }
    }
    __syncwarp();
    // used modules, in-degrees, rank of kind+"." and prefix conflicts
    uint64_t used = 0;
    for (int base = 0; base < M; base += 32) {
        const int m = base + lane;
        const bool u = m < M && tmask[m] != 0;
        const unsigned b = __ballot_sync(kFull, u);
        used |= static_cast<uint64_t>(b) << base;
    }
    int conflict = 0;
    for (int m = lane; m < M; m += 32) {
        int d = 0;
        for (int a = 0; a < M; ++a) d += (adj[a] >> m) & 1ull;
        indeg[m] = d;
        if (!(used >> m & 1ull)) {
            keyrank[m] = -1;
            continue;
        }
        const OpKey km = op_key(B, C.mbase + m, 0, false);
        int r = 0;
        for (uint64_t o = used; o; o &= o - 1) {
            const int q = low_bit(o);
            if (q == m) continue;
            const OpKey kq = op_key(B, C.mbase + q, 0, false);
            if (key_less(kq, km)) ++r;
            // kind(q) starts with kind(m)+"." : op-id order can depend on layers
            if (kq.len > km.len + 0) {
                bool pre = true;
                for (int i = 0; i <= km.len && pre; ++i) pre = kq.at(i) == km.at(i);
                if (pre) conflict = 1;
            }
        }
        keyrank[m] = r;
        modat[r] = m;
    }
    conflict = __any_sync(kFull, conflict);
    __syncwarp();
    const int nused = popc64(used);
    if (lane == 0) {
        int K = 0;
        int* mod_of = C.at<int>(C.L->mod_of);
        if (!conflict) {
            // Kahn over modules: once kind.0 pops, its layers pop consecutively
            // (SURVEY P1b), so the op-level lexicographic order is the module
            // order by key kind+"."
            uint64_t ready = 0;
            for (uint64_t u = used; u; u &= u - 1) {
                const int m = low_bit(u);
                if (indeg[m] == 0) ready |= 1ull << keyrank[m];
            }
            while (ready) {
                const int r = low_bit(ready);
                ready &= ready - 1;
                const int m = modat[r];
                kofm[m] = K;
                mod_of[K] = m;
                ++K;
                for (uint64_t s = adj[m]; s; s &= s - 1) {
                    const int q = low_bit(s);
                    if (--indeg[q] == 0) ready |= 1ull << keyrank[q];
                }
            }
        } else {
            // general operator-level lexicographic Kahn with layer cursors
            int* cursor = C.at<int>(C.L->lastent);  // reuse as cursor scratch
            for (int m = 0; m < M; ++m) cursor[m] = 0;
            while (true) {
                int best = -1;
                OpKey bk;
                for (uint64_t u = used; u; u &= u - 1) {
                    const int m = low_bit(u);
                    const int L = B.mod_layers[C.mbase + m];
                    if (cursor[m] >= L || (cursor[m] == 0 && indeg[m] != 0)) continue;
                    const OpKey k = op_key(B, C.mbase + m, cursor[m], true);
                    if (best < 0 || key_less(k, bk)) {
                        best = m;
                        bk = k;
                    }
                }
                if (best < 0) break;
                if (cursor[best] == 0) {
                    kofm[best] = K;
                    mod_of[K] = best;
                    ++K;
                }
                if (++cursor[best] == B.mod_layers[C.mbase + best])
                    for (uint64_t s = adj[best]; s; s &= s - 1)
                        --indeg[low_bit(s)];
            }
        }
        C.ctl->i0 = K;
        if (K != nused) set_err(C.ctl, WS_E_CYCLIC_WORKLOAD);
    }
    __syncwarp();
    if (C.ctl->err) return false;
    const int K = C.ctl->i0;
    C.K = K;
    int* mod_of = C.at<int>(C.L->mod_of);
    int* idrank = C.at<int>(C.L->idrank);
    int* by_rank = C.at<int>(C.L->by_rank);
    // MetaOp id ranks ("m<k>" in std::map order)
    for (int k = lane; k < K; k += 32) {
        int r = 0;
        for (int j = 0; j < K; ++j) r += dec_less(j, k);
        idrank[k] = r;
        by_rank[r] = k;
    }
    __syncwarp();
    uint64_t* predk = C.at<uint64_t>(C.L->predk);
    uint64_t* pred_r = C.at<uint64_t>(C.L->pred_r);
    uint64_t* succ_r = C.at<uint64_t>(C.L->succ_r);
    for (int k = lane; k < K; k += 32) {
        const int m = mod_of[k];
        uint64_t pk = 0, pr = 0, sr = 0;
        for (int j = 0; j < K; ++j) {
            if (j == k) continue;
            const int q = mod_of[j];
            if (adj[q] >> m & 1ull) pk |= 1ull << j, pr |= 1ull << idrank[j];
            if (adj[m] >> q & 1ull) sr |= 1ull << idrank[j];
        }
        predk[k] = pk;
        pred_r[k] = pr;
        succ_r[k] = sr;
    }
    __syncwarp();
    if (lane == 0) {  // longest-path levels; numbering order is topological
        int* level = C.at<int>(C.L->level);
        int maxl = 0;
        for (int k = 0; k < K; ++k) {
            int lv = 0;
            for (uint64_t p = predk[k]; p; p &= p - 1) {
                const int q = level[low_bit(p)] + 1;
                lv = q > lv ? q : lv;
            }
            level[k] = lv;
            maxl = lv > maxl ? lv : maxl;
        }
        int* lb = C.at<int>(C.L->lvl_begin);
        int* lm = C.at<int>(C.L->lvl_mem);
        for (int l = 0; l <= maxl + 1; ++l) lb[l] = 0;
        for (int k = 0; k < K; ++k) lb[level[k] + 1]++;
        for (int l = 0; l <= maxl; ++l) lb[l + 1] += lb[l];
        int fill[WS_MAX_MODULES];
        for (int l = 0; l <= maxl; ++l) fill[l] = lb[l];
        for (int r = 0; r < K; ++r) {
            const int k = by_rank[r];
            lm[fill[level[k]]++] = k;
        }
        C.ctl->i1 = maxl + 1;
    }
    __syncwarp();
    return true;
}

// ---------------------------------------------------------------------------
// subsystem (2) results: first module (kind order) whose fit failed
// ---------------------------------------------------------------------------
__device__ bool stage_fit_status(PlanCtx& C) {
    const int M = C.M;
    for (int base = 0; base < M; base += 32) {
        const int m = base + C.lane;
        const int e = m < M ? C.fit->err[C.mbase + m] : 0;
        const unsigned b = __ballot_sync(kFull, e != 0);
        if (b) {
            const int first = base + __ffs(b) - 1;
            if (C.lane == 0) {
                const int gm = C.mbase + first;
                const int code = C.fit->err[gm];
                set_err(C.ctl, code, code == WS_E_NO_SOURCE ? first : C.fit->err_a[gm], C.fit->err_b[gm]);
            }
            __syncwarp();
            return false;
        }
    }
    return true;
}

// ---------------------------------------------------------------------------
// subsystem (3): valid sets, bisection, discretization, repair
// (allocation.hpp:51-214); one level at a time, lane per MetaOp
// ---------------------------------------------------------------------------
__device__ bool stage_valid(PlanCtx& C) {
    const ws_batch& B = *C.B;
    const int K = C.K, N = C.N, lane = C.lane;
    const int* mod_of = C.at<int>(C.L->mod_of);
    const int* by_rank = C.at<int>(C.L->by_rank);
    uint64_t* valid = C.at<uint64_t>(C.L->valid);
    // tp > N check in id order (planner.hpp:168-171)
    for (int base = 0; base < K; base += 32) {
        const int r = base + lane;
        bool bad = false;
        if (r < K) bad = B.mod_tp[C.mbase + mod_of[by_rank[r]]] > N;
        const unsigned b = __ballot_sync(kFull, bad);
        if (b) {
            if (lane == 0) {
                const int k = by_rank[base + __ffs(b) - 1];
                set_err(C.ctl, WS_E_TP_EXCEEDS, k, B.mod_tp[C.mbase + mod_of[k]]);
            }
            __syncwarp();
            return false;
        }
    }
    for (int k = 0; k < K; ++k) {  // ballot over lanes = device counts n
        const int gm = C.mbase + mod_of[k];
        const int tp = B.mod_tp[gm];
        const long long batch = B.mod_batch[gm];
        uint64_t v = 0;
        for (int base = 0; base < N; base += 32) {
            const int n = base + lane + 1;
            bool ok = n <= N && n % tp == 0;
            if (ok) ok = batch % (n / tp) == 0;
            v |= static_cast<uint64_t>(__ballot_sync(kFull, ok)) << base;
        }
        if (lane == 0) valid[k] = v;
    }
    __syncwarp();
    return true;
}

// ordered (reference order) sum of one value per member, members striped on lanes
__device__ __forceinline__ double ordered_sum(double v0, double v1, int w) {
    double total = 0.0;
    for (int j = 0; j < 32 && j < w; ++j) total += shfl_d(v0, j);
    for (int j = 0; j + 32 < w; ++j) total += shfl_d(v1, j);
    return total;
}

__device__ bool stage_level_alloc(PlanCtx& C, const TLookup& T, int lvl, double& c_star_out) {
    const ws_batch& B = *C.B;
    const ws_plan_rec& R = *C.R;
    const int N = C.N, lane = C.lane;
    const int* lb = C.at<int>(C.L->lvl_begin);
    const int* lm = C.at<int>(C.L->lvl_mem) + lb[lvl];
    const int w = lb[lvl + 1] - lb[lvl];
    const int* mod_of = C.at<int>(C.L->mod_of);
    const uint64_t* valid = C.at<uint64_t>(C.L->valid);
    int* up_n = C.at<int>(C.L->up_n);
    int* up_l = C.at<int>(C.L->up_l);
    int* lo_n = C.at<int>(C.L->lo_n);
    int* lo_l = C.at<int>(C.L->lo_l);
    const double nd = static_cast<double>(N);
    // per-lane member data (members lane and lane+32)
    struct Mem {
        int k, gm, L, np;
        const double* pc;
        double c, w, nmax;
    } mem[2];
    for (int s = 0; s < 2; ++s) {
        const int i = lane + 32 * s;
        Mem& q = mem[s];
        q.k = -1;
        if (i < w) {
            q.k = lm[i];
            q.gm = C.mbase + mod_of[q.k];
            q.L = B.mod_layers[q.gm];
            q.np = C.fit->npieces[q.gm];
            q.pc = C.fit->pieces + 5 * C.fit->piece_off[q.gm];
            q.c = B.mod_c[q.gm];
            q.w = B.mod_w[q.gm];
            q.nmax = C.fit->nmax[q.gm];
        }
    }
    // bracket [max T(min(N,nmax))*L, sum T(1)*L] (allocation.hpp:75-80)
    double lo0 = 0.0, hi0[2] = {0.0, 0.0};
    for (int s = 0; s < 2; ++s) {
        const Mem& q = mem[s];
        if (q.k < 0) continue;
        const double ncap = (q.nmax < nd) ? q.nmax : nd;
        const double v = T(q.k, static_cast<int>(ncap)) * q.L;
        lo0 = (lo0 < v) ? v : lo0;
        hi0[s] = T(q.k, 1) * q.L;
    }
    for (int off = 16; off; off >>= 1) {
        const double o = __shfl_xor_sync(kFull, lo0, off);
        lo0 = (lo0 < o) ? o : lo0;
    }
    double c_lo = lo0;
    double c_hi = ordered_sum(hi0[0], hi0[1], w);
    auto probe_term = [&](const Mem& q, double cc) {
        const double v = inverse_exact(q.pc, q.np, q.c, q.w, q.nmax, cc / q.L);
        return (nd < v) ? nd : v;  // std::min(v, N)
    };
    for (int it = 0; it < R.max_iters && (c_hi - c_lo) > R.eps * c_hi; ++it) {
        const double mid = 0.5 * (c_lo + c_hi);
        const double t0 = mem[0].k >= 0 ? probe_term(mem[0], mid) : 0.0;
        const double t1 = mem[1].k >= 0 ? probe_term(mem[1], mid) : 0.0;
        if (ordered_sum(t0, t1, w) < nd)
            c_hi = mid;
        else
            c_lo = mid;
    }
    const double cs = 0.5 * (c_lo + c_hi);
    c_star_out = cs;
    // discretize (allocation.hpp:149-214), lane per MetaOp
    int eidx0 = 0x7fffffff;
    double ex0 = 0, ey0 = 0;
    for (int s = 0; s < 2; ++s) {
        const Mem& q = mem[s];
        if (q.k < 0) continue;
        const double nstar = probe_term(q, cs);
        const uint64_t v = valid[q.k];
        const int L = q.L;
        int exact = -1, n_over = -1, n_under = -1;
        for (uint64_t b = v; b; b &= b - 1) {
            const int x = low_bit(b) + 1;
            if (fabs(x - nstar) < 1e-9) {
                exact = x;
                break;
            }
        }
        if (exact < 0)
            for (uint64_t b = v; b; b &= b - 1) {
                const int x = low_bit(b) + 1;
                if (x < nstar) n_under = x;
                if (x > nstar) {
                    n_over = x;
                    break;
                }
            }
        int un = 0, ul = L, ln = 0, ll = 0;
        if (exact >= 0) {
            un = exact;
        } else if (n_over == -1) {
            un = 64 - __clzll(static_cast<long long>(v));
        } else if (n_under == -1) {
            un = low_bit(v) + 1;
        } else {
            Ctl local{};
            TLookup Tl = T;
            Tl.ctl = &local;
            const double t_over = Tl(q.k, n_over);
            const double t_under = local.err ? 0.0 : Tl(q.k, n_under);
            if (local.err) {
                const int idx = lane + 32 * s;
                if (idx < eidx0) eidx0 = idx, ex0 = local.x, ey0 = local.y;
                continue;
            }
            if (t_under - t_over <= 0.0) {
                un = n_under;
            } else {
                double lr = (cs - t_under * L) / (t_over - t_under);
                lr = lr < 0.0 ? 0.0 : (static_cast<double>(L) < lr ? static_cast<double>(L) : lr);
                int l_over = static_cast<int>(floor(lr + 0.5));
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
                    un = n_under;
                } else if (l_under == 0) {
                    un = n_over;
                } else {
                    un = n_over;
                    ul = l_over;
                    ln = n_under;
                    ll = l_under;
                }
            }
        }
        up_n[q.k] = un;
        up_l[q.k] = ul;
        lo_n[q.k] = ln;
        lo_l[q.k] = ll;
    }
    // first member (id order) whose discretization hit OutOfRange
    {
        int emin = eidx0;
        for (int off = 16; off; off >>= 1) {
            const int o = __shfl_xor_sync(kFull, emin, off);
            emin = o < emin ? o : emin;
        }
        if (emin != 0x7fffffff) {
            const int src = emin & 31;
            const double xx = shfl_d(ex0, src), yy = shfl_d(ey0, src);
            if (lane == 0) {
                C.ctl->err = WS_E_EVAL_RANGE;
                C.ctl->x = xx;
                C.ctl->y = yy;
            }
            __syncwarp();
            return false;
        }
    }
    __syncwarp();
    // repair_capacity (allocation.hpp:107-139)
    while (true) {
        int wid = 0;
        for (int s = 0; s < 2; ++s) {
            const Mem& q = mem[s];
            if (q.k < 0) continue;
            const int a = up_n[q.k], b = lo_l[q.k] ? lo_n[q.k] : 0;
            wid += a > b ? a : b;
        }
        for (int off = 16; off; off >>= 1) wid += __shfl_xor_sync(kFull, wid, off);
        if (wid <= N) break;
        double best_pen = 0.0;
        int best_i = 0x7fffffff, best_t = 0, eidx = 0x7fffffff;
        double ex = 0, ey = 0;
        for (int s = 0; s < 2; ++s) {
            const Mem& q = mem[s];
            if (q.k < 0) continue;
            const int un = up_n[q.k];
            const uint64_t below = valid[q.k] & ((1ull << (un - 1)) - 1ull);  // valid values < un
            if (!below) continue;
            const int target = 63 - __clzll(static_cast<long long>(below)) + 1;
            if (lo_l[q.k] && target <= lo_n[q.k]) continue;
            Ctl local{};
            TLookup Tl = T;
            Tl.ctl = &local;
            const double a = Tl(q.k, target);
            const double b = local.err ? 0.0 : Tl(q.k, un);
            if (local.err) {
                const int idx = lane + 32 * s;
                if (idx < eidx) eidx = idx, ex = local.x, ey = local.y;
                continue;
            }
            const double pen = up_l[q.k] * (a - b);
            const int idx = lane + 32 * s;
            if (best_i == 0x7fffffff || pen < best_pen) best_pen = pen, best_i = idx, best_t = target;
        }
        // errors: the lowest member index that threw precedes any choice
        int emin = eidx;
        for (int off = 16; off; off >>= 1) {
            const int o = __shfl_xor_sync(kFull, emin, off);
            emin = o < emin ? o : emin;
        }
        if (emin != 0x7fffffff) {
            const int src = emin & 31;
            const double xx = shfl_d(ex, src), yy = shfl_d(ey, src);
            if (lane == 0) {
                C.ctl->err = WS_E_EVAL_RANGE;
                C.ctl->x = xx;
                C.ctl->y = yy;
            }
            __syncwarp();
            return false;
        }
        // argmin over (penalty, member index)
        for (int off = 16; off; off >>= 1) {
            const double op = __shfl_xor_sync(kFull, best_pen, off);
            const int oi = __shfl_xor_sync(kFull, best_i, off);
            const int ot = __shfl_xor_sync(kFull, best_t, off);
            if (oi != 0x7fffffff && (best_i == 0x7fffffff || op < best_pen || (op == best_pen && oi < best_i)))
                best_pen = op, best_i = oi, best_t = ot;
        }
        if (best_i == 0x7fffffff) break;
        if (lane == 0) up_n[lm[best_i]] = best_t;
        __syncwarp();
    }
    return true;
}

// ---------------------------------------------------------------------------
// subsystem (4a): wave scheduling of one level (schedule.hpp:49-309), lane 0
// ---------------------------------------------------------------------------
struct SchedState {
    int* tk;
    int* tn;
    int* tl;
    int R;
    const int* sumlay;
    const int* idrank;
    const uint64_t* valid;
    int N;
    TLookup T;
};

struct CmpByN {  // schedule.hpp:98-104
    const SchedState* s;
    __device__ bool operator()(int a, int b) const {
        if (s->tn[a] != s->tn[b]) return s->tn[a] > s->tn[b];
        const double ra = s->tl[a] * s->T(s->tk[a], s->tn[a]);
        const double rb = s->tl[b] * s->T(s->tk[b], s->tn[b]);
        if (ra != rb) return ra > rb;
        return s->idrank[s->tk[a]] < s->idrank[s->tk[b]];
    }
};
struct CmpByTime {  // schedule.hpp:105-111
    const SchedState* s;
    __device__ bool operator()(int a, int b) const {
        const double ra = s->sumlay[s->tk[a]] * s->T(s->tk[a], s->tn[a]);
        const double rb = s->sumlay[s->tk[b]] * s->T(s->tk[b], s->tn[b]);
        if (ra != rb) return ra > rb;
        if (s->tn[a] != s->tn[b]) return s->tn[a] > s->tn[b];
        return s->idrank[s->tk[a]] < s->idrank[s->tk[b]];
    }
};
struct CmpByCheap {  // schedule.hpp:112-118
    const SchedState* s;
    __device__ bool operator()(int a, int b) const {
        if (s->tn[a] != s->tn[b]) return s->tn[a] < s->tn[b];
        const double ra = s->sumlay[s->tk[a]] * s->T(s->tk[a], s->tn[a]);
        const double rb = s->sumlay[s->tk[b]] * s->T(s->tk[b], s->tn[b]);
        if (ra != rb) return ra > rb;
        return s->idrank[s->tk[a]] < s->idrank[s->tk[b]];
    }
};

// extend_resources_if_needed (schedule.hpp:144-173) on allocation array n[]
__device__ void sched_extend(const SchedState& S, int* n, const int* sel, int nsel) {
    while (true) {
        int usedn = 0;
        for (int i = 0; i < nsel; ++i) usedn += n[sel[i]];
        const int idle = S.N - usedn;
        if (idle <= 0) break;
        int best = -1, best_next = 0;
        double best_time = -1.0;
        for (int i = 0; i < nsel; ++i) {
            const int t = sel[i];
            const int k = S.tk[t];
            const uint64_t above = S.valid[k] & ~bits_upto(n[t] - 1);  // valid values > n
            if (!above) continue;
            const int nx = low_bit(above) + 1;
            if (nx - n[t] > idle) continue;
            const double rem = S.sumlay[k] * S.T(k, n[t]);
            if (S.T.ctl->err) return;
            if (rem > best_time || (rem == best_time && best >= 0 && S.idrank[k] < S.idrank[S.tk[best]])) {
                best = t;
                best_time = rem;
                best_next = nx;
            }
        }
        if (best < 0) break;
        n[best] = best_next;
    }
}

__device__ int sched_greedy(const SchedState& S, const int* order, int* sel) {
    int ns = 0, cap = S.N;
    uint64_t taken = 0;
    for (int i = 0; i < S.R; ++i) {
        const int t = order[i];
        if (S.tn[t] > cap) continue;
        if (taken >> S.tk[t] & 1ull) continue;
        sel[ns++] = t;
        taken |= 1ull << S.tk[t];
        cap -= S.tn[t];
    }
    return ns;
}

// Returns false on error (ctl->err set).  Appends waves/entries.
__device__ bool stage_schedule_level(PlanCtx& C, const TLookup& T, int lvl, int& nW, int& nE, double& level_end) {
    const Layout& L = *C.L;
    const int* lb = C.at<int>(L.lvl_begin);
    const int* lm = C.at<int>(L.lvl_mem) + lb[lvl];
    const int w = lb[lvl + 1] - lb[lvl];
    const int* up_n = C.at<int>(L.up_n);
    const int* up_l = C.at<int>(L.up_l);
    const int* lo_n = C.at<int>(L.lo_n);
    const int* lo_l = C.at<int>(L.lo_l);
    int* sumlay = C.at<int>(L.sumlay);
    double* credit = C.at<double>(L.credit);
    SchedState S;
    S.tk = C.at<int>(L.tk);
    S.tn = C.at<int>(L.tn);
    S.tl = C.at<int>(L.tl);
    S.sumlay = sumlay;
    S.idrank = C.at<int>(L.idrank);
    S.valid = C.at<uint64_t>(L.valid);
    S.N = C.N;
    S.T = T;
    int* n2 = C.at<int>(L.tn2);
    int* ord = C.at<int>(L.ord);
    int R = 0;
    for (int i = 0; i < w; ++i) {
        const int k = lm[i];
        S.tk[R] = k, S.tn[R] = up_n[k], S.tl[R] = up_l[k], ++R;
        if (lo_l[k]) S.tk[R] = k, S.tn[R] = lo_n[k], S.tl[R] = lo_l[k], ++R;
        credit[k] = 0.0;
    }
    const int cap2 = 2 * C.M;
    int* o0 = ord;
    int* o1 = ord + cap2;
    int* o2 = ord + 2 * cap2;
    int* w_level = C.at<int>(L.w_level);
    double* w_start = C.at<double>(L.w_start);
    double* w_dur = C.at<double>(L.w_dur);
    int* w_eb = C.at<int>(L.w_eb);
    int* w_ec = C.at<int>(L.w_ec);
    int* e_k = C.at<int>(L.e_k);
    int* e_n = C.at<int>(L.e_n);
    int* e_l = C.at<int>(L.e_l);
    double* e_span = C.at<double>(L.e_span);
    double now = 0.0;
    int sel[2 * WS_MAX_MODULES], best[2 * WS_MAX_MODULES], pool[2 * WS_MAX_MODULES];
    while (R > 0) {
        S.R = R;
        for (int i = 0; i < R; ++i) sumlay[S.tk[i]] = 0;
        for (int i = 0; i < R; ++i) sumlay[S.tk[i]] += S.tl[i];
        // propose_candidate_set (schedule.hpp:76-139)
        for (int i = 0; i < R; ++i) o0[i] = o1[i] = o2[i] = i;
        {
            CmpByN c0{&S};
            ls_sort(o0, R, c0);
            CmpByTime c1{&S};
            ls_sort(o1, R, c1);
            CmpByCheap c2{&S};
            ls_sort(o2, R, c2);
        }
        if (C.ctl->err) return false;
        int nbest = 0;
        long long best_key = -1;
        for (int o = 0; o < 3; ++o) {
            const int* order = o == 0 ? o0 : (o == 1 ? o1 : o2);
            const int ns = sched_greedy(S, order, sel);
            for (int i = 0; i < R; ++i) n2[i] = S.tn[i];
            sched_extend(S, n2, sel, ns);
            if (C.ctl->err) return false;
            int usedn = 0;
            for (int i = 0; i < ns; ++i) usedn += n2[sel[i]];
            const long long key = static_cast<long long>(usedn) * 1000 + ns;
            if (key > best_key) {
                best_key = key;
                nbest = ns;
                for (int i = 0; i < ns; ++i) best[i] = sel[i];
            }
        }
        if (nbest == 0) return set_err(C.ctl, WS_E_NO_SCHEDULABLE);
        sched_extend(S, S.tn, best, nbest);
        if (C.ctl->err) return false;
        // align_time_span (schedule.hpp:190-227)
        double t_wave = 0.0;
        for (int i = 0; i < nbest; ++i) {
            const int t = best[i];
            pool[i] = sumlay[S.tk[t]];
            const double span = pool[i] * T(S.tk[t], S.tn[t]);
            if (i == 0 || span < t_wave) t_wave = span;
        }
        if (C.ctl->err) return false;
        const int W_CAP = C.ctl->i2, E_CAP = C.ctl->i3;
        if (nW + 1 > W_CAP) return set_err(C.ctl, WS_E_LIMIT_WAVES);
        if (nE + nbest > E_CAP) return set_err(C.ctl, WS_E_LIMIT_ENTRIES);
        double dur = 0.0;
        const int eb = nE;
        int klay[2 * WS_MAX_MODULES];
        for (int i = 0; i < nbest; ++i) {
            const int t = best[i];
            const int k = S.tk[t];
            const double per = T(k, S.tn[t]);
            int kk;
            if (pool[i] * per <= t_wave * (1.0 + 1e-12)) {
                kk = pool[i];
                credit[k] = 0.0;
            } else {
                const double carried = credit[k];
                const double budget = t_wave + ((per < carried) ? per : carried);
                kk = static_cast<int>(floor(budget / per * (1.0 + 1e-12)));
                kk = kk < 1 ? 1 : kk;
                kk = kk < pool[i] ? kk : pool[i];
                const double rest = budget - kk * per;
                credit[k] = (0.0 < rest) ? rest : 0.0;
            }
            klay[i] = kk;
            e_k[nE] = k;
            e_n[nE] = S.tn[t];
            e_l[nE] = kk;
            const double span = kk * T(k, S.tn[t]);
            e_span[nE] = span;
            dur = (dur < span) ? span : dur;
            ++nE;
        }
        if (C.ctl->err) return false;
        w_level[nW] = lvl;
        w_start[nW] = now;
        w_dur[nW] = dur;
        w_eb[nW] = eb;
        w_ec[nW] = nbest;
        ++nW;
        now += dur;
        for (int i = 0; i < nbest; ++i) {  // layer bookkeeping (schedule.hpp:268-279)
            const int t = best[i];
            int ab = klay[i] - S.tl[t];
            ab = ab > 0 ? ab : 0;
            S.tl[t] -= klay[i] - ab;
            for (int j = 0; j < R && ab; ++j) {
                if (j == t || S.tk[j] != S.tk[t]) continue;
                const int take = ab < S.tl[j] ? ab : S.tl[j];
                S.tl[j] -= take;
                ab -= take;
            }
        }
        int R2 = 0;
        for (int i = 0; i < R; ++i)
            if (S.tl[i] > 0) S.tk[R2] = S.tk[i], S.tn[R2] = S.tn[i], S.tl[R2] = S.tl[i], ++R2;
        if (R2 == R) return set_err(C.ctl, WS_E_NO_PROGRESS);
        R = R2;
    }
    level_end = now;  // relative to the level start
    return true;
}

// ---------------------------------------------------------------------------
// subsystem (4b): placement (placement.hpp:168-447, planner.hpp:99-151)
// ---------------------------------------------------------------------------
struct PlaceState {
    int nW, nE, nF, Fcap;
    int K, N, G, n_isl;
    uint64_t all;
};

// One wave: returns 1 placed, 0 infeasible (caller tries the next variant),
// -1 hard error (ctl->err).
__device__ int place_wave(PlanCtx& C, PlaceState& P, int w, int variant) {
    const Layout& L = *C.L;
    const ws_plan_rec& R = *C.R;
    const int lane = C.lane, N = P.N;
    const int* w_eb = C.at<int>(L.w_eb);
    const int* w_ec = C.at<int>(L.w_ec);
    const int* e_k = C.at<int>(L.e_k);
    const int* e_n = C.at<int>(L.e_n);
    const int* e_l = C.at<int>(L.e_l);
    uint64_t* e_mask = C.at<uint64_t>(L.e_mask);
    int* e_rot = C.at<int>(L.e_rot);
    const int* e_wave = C.at<int>(L.e_wave);
    const int* home = C.at<int>(L.home);
    const int* lastw = C.at<int>(L.lastw);
    const int* by_rank = C.at<int>(L.by_rank);
    const int* idrank = C.at<int>(L.idrank);
    const uint64_t* pred_r = C.at<uint64_t>(L.pred_r);
    const uint64_t* contb = C.at<uint64_t>(L.contb);
    const uint64_t* edgeb = C.at<uint64_t>(L.edgeb);
    const uint64_t* memact = C.at<uint64_t>(L.memact);
    const uint64_t* parb = C.at<uint64_t>(L.parb);
    const int* gkey = C.at<int>(L.gkey);
    double* mem = C.at<double>(L.mem);
    uint64_t* chg = C.at<uint64_t>(L.chg);
    const int* isl = C.at<int>(L.isl);
    const uint64_t* islmask = C.at<uint64_t>(L.islmask);
    int* fin_src = C.at<int>(L.fin_src);
    uint64_t* fin_bytes = C.at<uint64_t>(L.fin_bytes);
    uint64_t* disp_mask = C.at<uint64_t>(L.disp_mask);
    double* disp_bytes = C.at<double>(L.disp_bytes);
    int* disp_cnt = C.at<int>(L.disp_cnt);
    int* eorder = C.at<int>(L.eorder);
    uint64_t* va = C.at<uint64_t>(L.va);
    uint64_t* f_vol = C.at<uint64_t>(L.f_vol);
    int* f_meta = C.at<int>(L.f_meta);
    const int* w_cursor = C.at<int>(L.w_cursor);
    const int eb = w_eb[w], ec = w_ec[w];

    // incoming volume per entry (placement.hpp:188-206), entry order (:208-221)
    for (int i = lane; i < ec; i += 32) {
        const int k = e_k[eb + i];
        uint64_t v = 0;
        if (home[k] >= 0) {
            v = contb[k];
        } else {
            for (uint64_t pr = pred_r[k]; pr; pr &= pr - 1) {
                const int p = by_rank[low_bit(pr)];
                if (home[p] >= 0) v += edgeb[p];
            }
        }
        va[i] = v;
    }
    __syncwarp();
    for (int i = lane; i < ec; i += 32) {
        int pos = i;
        if (!R.sequential) {
            pos = 0;
            const int ki = e_k[eb + i];
            for (int j = 0; j < ec; ++j) {
                if (j == i) continue;
                const int kj = e_k[eb + j];
                if (va[j] > va[i] || (va[j] == va[i] && idrank[kj] < idrank[ki])) ++pos;
            }
        }
        eorder[pos] = i;
    }
    __syncwarp();
    uint64_t free = P.all;
    uint64_t placed_now = 0;
    int cursor = R.sequential ? w_cursor[w] : 0;
    for (int oi = 0; oi < ec; ++oi) {
        const int e = eb + eorder[oi];
        const int k = e_k[e], n = e_n[e], lay = e_l[e];
        // flows_in: continuation of k, else producers in dep order
        int nfin = 0;
        if (home[k] >= 0) {
            if (lane == 0) fin_src[0] = home[k], fin_bytes[0] = contb[k];
            nfin = 1;
        } else {
            for (uint64_t pr = pred_r[k]; pr; pr &= pr - 1) {
                const int p = by_rank[low_bit(pr)];
                if (home[p] < 0) continue;
                if (lane == 0) fin_src[nfin] = home[p], fin_bytes[nfin] = edgeb[p];
                ++nfin;
            }
        }
        // entities whose home this entry could displace (score_candidate :293-305)
        int ndisp = 0;
        for (int base = 0; base < P.K; base += 32) {
            const int r = base + lane;
            bool ok = false;
            int e2 = -1;
            if (r < P.K) {
                e2 = by_rank[r];
                ok = e2 != k && lastw[e2] >= w && !(placed_now >> e2 & 1ull) && home[e2] >= 0;
            }
            const unsigned b = __ballot_sync(kFull, ok);
            if (ok) {
                const int slot = ndisp + __popc(b & ((1u << lane) - 1u));
                const uint64_t hm = e_mask[home[e2]];
                disp_mask[slot] = hm;
                disp_bytes[slot] = static_cast<double>(contb[e2]);
                disp_cnt[slot] = popc64(hm);
            }
            ndisp += __popc(b);
        }
        __syncwarp();
        // memory delta constants (memory_delta :132-140)
        const double A = lay * (static_cast<double>(memact[k]) / n);
        const int tp = C.B->mod_tp[C.mbase + C.at<int>(L.mod_of)[k]];
        const double Pm = (1.0 + R.grad_mult) * static_cast<double>(parb[k]) / tp;
        const uint64_t charged = chg[gkey[k]];
        const double cap = static_cast<double>(R.mem_capacity);

        auto score_of = [&](uint64_t devs, int rot) {
            Score s;
            s.valid = 1;
            s.devs = devs;
            s.rot = rot;
            s.islands = 0;
            for (int i = 0; i < P.n_isl; ++i) s.islands += (devs & islmask[i]) != 0;
            s.displaced = 0.0;
            for (int j = 0; j < ndisp; ++j) {
                const int ov = popc64(devs & disp_mask[j]);
                if (ov == 0) continue;
                s.displaced += disp_bytes[j] * static_cast<double>(ov) / static_cast<double>(disp_cnt[j]);
            }
            s.feasible = 1;
            double peak = 0.0;
            for (uint64_t d = devs; d; d &= d - 1) {
                const int dv = low_bit(d);
                double delta = A;
                if (!(charged >> dv & 1ull)) delta += Pm;
                const double used = mem[dv] + delta;
                peak = (peak < used) ? used : peak;
                if (used > cap) s.feasible = 0;
            }
            s.peak = peak;
            s.inter = 0.0;
            s.intra = 0.0;
            for (int f = 0; f < nfin; ++f) {
                uint64_t a, b;
                shard_moves(e_mask[fin_src[f]], devs, fin_bytes[f], isl, a, b);
                s.inter += static_cast<double>(b);
                s.intra += static_cast<double>(a);
            }
            return s;
        };

        Score chosen;
        chosen.valid = 0;
        if (R.sequential) {
            if (popc64(free) >= n) {  // rolling cursor block (placement.hpp:350-358)
                uint64_t m = 0;
                for (int i = 0; i < n; ++i) m |= 1ull << ((cursor + i) % N);
                chosen = score_of(m, cursor);
                cursor = (cursor + n) % N;
            }
        } else {
            // candidate sets (placement.hpp:223-263): reuse, island windows, global windows
            const int nfree = popc64(free);
            if (nfree >= n) {
                int nwin_isl[WS_MAX_DEVICES];
                int total = nfin;
                for (int i = 0; i < P.n_isl; ++i) {
                    const int c = popc64(free & islmask[i]);
                    nwin_isl[i] = c >= n ? c - n + 1 : 0;
                    total += nwin_isl[i];
                }
                total += nfree - n + 1;
                const int rounds = (!R.sequential && oi == 0) ? variant + 1 : 1;
                Score prev;
                prev.valid = 0;
                for (int rd = 0; rd < rounds; ++rd) {
                    Score best;
                    best.valid = 0;
                    for (int j = lane; j < total; j += 32) {
                        uint64_t m = 0;
                        if (j < nfin) {
                            m = e_mask[fin_src[j]];
                            if (popc64(m) != n || (m & ~free)) continue;
                        } else {
                            int r = j - nfin;
                            int i = 0;
                            for (; i < P.n_isl && r >= nwin_isl[i]; ++i) r -= nwin_isl[i];
                            m = i < P.n_isl ? window_mask(free & islmask[i], r, n) : window_mask(free, r, n);
                        }
                        const Score s = score_of(m, 0);
                        if (prev.valid && !score_less(prev, s)) continue;  // next distinct rank
                        if (!best.valid || score_less(s, best)) best = s;
                    }
                    best = warp_min_score(best);
                    if (!best.valid) break;  // fewer distinct candidates than variant+1
                    prev = best;
                    chosen = best;
                }
            }
        }
        if (!chosen.valid) return 0;    // no candidate
        if (!chosen.feasible) return 0;
        // commit_memory (placement.hpp:142-149), lane per device
        for (int dv = lane; dv < N; dv += 32) {
            if (!(chosen.devs >> dv & 1ull)) continue;
            double delta = A;
            if (!(charged >> dv & 1ull)) delta += Pm;
            mem[dv] += delta;
        }
        if (lane == 0) {
            chg[gkey[k]] = charged | chosen.devs;
            e_mask[e] = chosen.devs;
            e_rot[e] = chosen.rot;
        }
        // flow records (placement.hpp:376-400)
        for (int f = 0; f < nfin; ++f) {
            uint64_t a, b;
            const int src = fin_src[f];
            shard_moves(e_mask[src], chosen.devs, fin_bytes[f], isl, a, b);
            const int need = (a + b == 0) ? 1 : (a > 0) + (b > 0);
            if (P.nF + need > P.Fcap) {  // flow cap
                if (lane == 0) set_err(C.ctl, WS_E_LIMIT_FLOWS);
                __syncwarp();
                return -1;
            }
            if (lane == 0) {
                auto put = [&](uint64_t vol, int mode) {
                    f_vol[P.nF] = vol;
                    int* fm = f_meta + 6 * P.nF;
                    fm[0] = e_wave[src];
                    fm[1] = e_k[src];
                    fm[2] = w;
                    fm[3] = k;
                    fm[4] = mode;
                    fm[5] = 0;
                };
                if (a + b == 0) {
                    put(0, WS_FLOW_COPY);
                    P.nF++;
                } else {
                    if (a > 0) put(a, WS_FLOW_INTRA), P.nF++;
                    if (b > 0) put(b, WS_FLOW_INTER), P.nF++;
                }
            } else {
                P.nF += need;
            }
        }
        free &= ~chosen.devs;
        placed_now |= 1ull << k;
        __syncwarp();
    }
    return 1;
}

__device__ bool stage_place(PlanCtx& C, PlaceState& P) {
    const Layout& L = *C.L;
    const ws_batch& B = *C.B;
    const ws_plan_rec& R = *C.R;
    const int lane = C.lane, K = C.K, N = C.N;
    const int* mod_of = C.at<int>(L.mod_of);
    const int* e_k = C.at<int>(L.e_k);
    const int* e_n = C.at<int>(L.e_n);
    const int* w_eb = C.at<int>(L.w_eb);
    const int* w_ec = C.at<int>(L.w_ec);
    int* e_prev = C.at<int>(L.e_prev);
    int* e_wave = C.at<int>(L.e_wave);
    int* home = C.at<int>(L.home);
    int* lastw = C.at<int>(L.lastw);
    int* lastent = C.at<int>(L.lastent);
    int* gkey = C.at<int>(L.gkey);
    uint64_t* contb = C.at<uint64_t>(L.contb);
    uint64_t* edgeb = C.at<uint64_t>(L.edgeb);
    uint64_t* memact = C.at<uint64_t>(L.memact);
    uint64_t* parb = C.at<uint64_t>(L.parb);
    double* mem = C.at<double>(L.mem);
    uint64_t* chg = C.at<uint64_t>(L.chg);
    double* snap_mem = C.at<double>(L.snap_mem);
    uint64_t* snap_chg = C.at<uint64_t>(L.snap_chg);
    int* snap_nf = C.at<int>(L.snap_nf);
    int* variant = C.at<int>(L.variant);
    int* isl = C.at<int>(L.isl);
    uint64_t* islmask = C.at<uint64_t>(L.islmask);
    int* w_cursor = C.at<int>(L.w_cursor);
    const int nW = P.nW;
    // entity tables (planner.hpp:99-151); one MetaOp per module: length == layers
    for (int k = lane; k < K; k += 32) {
        const int gm = C.mbase + mod_of[k];
        const int Lk = B.mod_layers[gm];
        parb[k] = static_cast<uint64_t>(static_cast<double>(B.mod_param[gm]) * Lk / B.mod_layers[gm]);
        const uint64_t act = B.mod_act[gm];
        memact[k] = static_cast<uint64_t>(static_cast<double>(act) * 1.0);
        contb[k] = static_cast<uint64_t>(static_cast<double>(act) * 1.0);
        const uint64_t edge = B.mod_out[gm] == 0 ? act : B.mod_out[gm];
        edgeb[k] = static_cast<uint64_t>(static_cast<double>(edge) * 1.0);
        const int grp = (Lk == B.mod_layers[gm]) ? B.mod_group[gm] : -1;
        const int al = B.mod_alias[gm];
        gkey[k] = grp < 0 ? R.n_groups + k : ((al >= 0 && al < K) ? R.n_groups + al : grp);
        home[k] = -1;
        lastw[k] = -1;
        lastent[k] = -1;
    }
    for (int d = lane; d < N; d += 32) {
        isl[d] = B.dev_island[R.dev_begin + d];
        mem[d] = 0.0;
    }
    for (int g = lane; g < P.G; g += 32) chg[g] = 0;
    for (int i = lane; i < P.n_isl; i += 32) islmask[i] = 0;
    for (int w = lane; w < nW; w += 32) variant[w] = 0;
    __syncwarp();
    if (lane == 0) {
        for (int d = 0; d < N; ++d) islmask[isl[d]] |= 1ull << d;
        int cur = 0;
        for (int w = 0; w < nW; ++w) {
            w_cursor[w] = cur;
            for (int i = 0; i < w_ec[w]; ++i) {
                const int e = w_eb[w] + i;
                e_wave[e] = w;
                e_prev[e] = lastent[e_k[e]];
                lastent[e_k[e]] = e;
                lastw[e_k[e]] = w;
                cur = (cur + e_n[e]) % N;
            }
        }
    }
    __syncwarp();
    // snapshot 0 = empty state
    for (int d = lane; d < N; d += 32) snap_mem[d] = 0.0;
    for (int g = lane; g < P.G; g += 32) snap_chg[g] = 0;
    if (lane == 0) snap_nf[0] = 0;
    __syncwarp();
    // depth-first search over per-wave variants (placement.hpp:409-441)
    long long attempts = 0, budget = nW;
    for (int d = 0; d < R.bt_depth; ++d) budget *= (R.bt_branching > 1 ? R.bt_branching : 1);
    const int branching = R.sequential ? 1 : R.bt_branching;
    int k = 0;
    bool dirty = false;
    P.nF = 0;
    while (k < nW) {
        if (++attempts > budget) {
            if (lane == 0) set_err(C.ctl, WS_E_BT_BUDGET, k);
            __syncwarp();
            return false;
        }
        if (dirty) {  // restore the state saved before wave k
            for (int d = lane; d < N; d += 32) mem[d] = snap_mem[k * N + d];
            for (int g = lane; g < P.G; g += 32) chg[g] = snap_chg[k * P.G + g];
            P.nF = snap_nf[k];
            dirty = false;
            __syncwarp();
        }
        if (variant[k] >= branching) {
            __syncwarp();
            if (lane == 0) variant[k] = 0;
            if (k == 0) {
                if (lane == 0) set_err(C.ctl, WS_E_NO_PLACEMENT_W0);
                __syncwarp();
                return false;
            }
            --k;
            // home[] back to "latest entry before wave k"
            for (int i = lane; i < w_ec[k]; i += 32) {
                const int e = w_eb[k] + i;
                home[e_k[e]] = e_prev[e];
            }
            if (lane == 0) variant[k]++;
            dirty = true;
            __syncwarp();
            continue;
        }
        const int r = place_wave(C, P, k, variant[k]);
        __syncwarp();
        if (r < 0) return false;
        if (r > 0) {
            for (int d = lane; d < N; d += 32) snap_mem[(k + 1) * N + d] = mem[d];
            for (int g = lane; g < P.G; g += 32) snap_chg[(k + 1) * P.G + g] = chg[g];
            if (lane == 0) snap_nf[k + 1] = P.nF;
            for (int i = lane; i < w_ec[k]; i += 32) {
                const int e = w_eb[k] + i;
                home[e_k[e]] = e;
            }
            ++k;
        } else {
            if (lane == 0) variant[k]++;
            dirty = true;
        }
        __syncwarp();
    }
    return true;
}

// ---------------------------------------------------------------------------
// output: one compact record per plan in the arena (ws_abi.h layout)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t al8(uint64_t v) { return (v + 7) & ~7ull; }

__device__ void emit(PlanCtx& C, int p, const PlaceState& P, int n_levels, double lower_bound, double end_time,
                     const PlanArgs& A) {
    const Layout& L = *C.L;
    const ws_batch& B = *C.B;
    const int lane = C.lane, K = C.K;
    const int* mod_of = C.at<int>(L.mod_of);
    const int* level = C.at<int>(L.level);
    const int* by_rank = C.at<int>(L.by_rank);
    const uint64_t* succ_r = C.at<uint64_t>(L.succ_r);
    int npieces = 0, nedges = 0;
    for (int k = 0; k < K; ++k) npieces += C.fit->npieces[C.mbase + mod_of[k]];
    for (int k = lane; k < K; k += 32) nedges += popc64(succ_r[k]);
    for (int off = 16; off; off >>= 1) nedges += __shfl_xor_sync(kFull, nedges, off);
    const uint64_t sz = al8(sizeof(ws_out_metaop) * K) + al8(sizeof(ws_out_level) * n_levels) +
                        al8(sizeof(ws_out_piece) * npieces) + al8(sizeof(ws_out_edge) * nedges) +
                        al8(sizeof(ws_out_wave) * P.nW) + al8(sizeof(ws_out_entry) * P.nE) +
                        al8(sizeof(ws_out_flow) * P.nF);
    unsigned long long off = 0;
    if (lane == 0) off = atomicAdd(A.arena_top, static_cast<unsigned long long>(sz));
    off = __shfl_sync(kFull, off, 0);
    ws_plan_result* res = A.results + p;
    if (off + sz > A.arena_cap) {
        if (lane == 0) {
            res->status = WS_STATUS_INTERNAL;
            res->err_code = WS_E_ARENA_OVERFLOW;
        }
        return;
    }
    uint8_t* base = A.arena + off;
    uint64_t o = 0;
    auto* mo = reinterpret_cast<ws_out_metaop*>(base + o);
    o += al8(sizeof(ws_out_metaop) * K);
    auto* lv = reinterpret_cast<ws_out_level*>(base + o);
    o += al8(sizeof(ws_out_level) * n_levels);
    auto* pc = reinterpret_cast<ws_out_piece*>(base + o);
    o += al8(sizeof(ws_out_piece) * npieces);
    auto* ed = reinterpret_cast<ws_out_edge*>(base + o);
    o += al8(sizeof(ws_out_edge) * nedges);
    auto* wv = reinterpret_cast<ws_out_wave*>(base + o);
    o += al8(sizeof(ws_out_wave) * P.nW);
    auto* en = reinterpret_cast<ws_out_entry*>(base + o);
    o += al8(sizeof(ws_out_entry) * P.nE);
    auto* fl = reinterpret_cast<ws_out_flow*>(base + o);
    // metaops + curve pieces (prefix over k, computed uniformly)
    {
        int pb = 0;
        for (int k = 0; k < K; ++k) {
            const int gm = C.mbase + mod_of[k];
            const int np = C.fit->npieces[gm];
            if ((k & 31) == lane) {
                ws_out_metaop x;
                x.module = mod_of[k];
                x.level = level[k];
                x.first_layer = 0;
                x.length = B.mod_layers[gm];
                x.piece_begin = pb;
                x.piece_count = np;
                x.upper_n = C.at<int>(L.up_n)[k];
                x.upper_l = C.at<int>(L.up_l)[k];
                x.lower_n = C.at<int>(L.lo_n)[k];
                x.lower_l = C.at<int>(L.lo_l)[k];
                mo[k] = x;
            }
            const double* src = C.fit->pieces + 5 * C.fit->piece_off[gm];
            for (int i = lane; i < np; i += 32)
                pc[pb + i] = ws_out_piece{src[5 * i], src[5 * i + 1], src[5 * i + 2], src[5 * i + 3], src[5 * i + 4]};
            pb += np;
        }
    }
    const double* cstar = C.at<double>(L.cstar);
    const int* lfw = C.at<int>(L.lvl_fw);
    const int* lnw = C.at<int>(L.lvl_nw);
    for (int l = lane; l < n_levels; l += 32) {
        ws_out_level x;
        x.c_star = cstar[l];
        x.first_wave = lfw[l];
        x.n_waves = lnw[l];
        lv[l] = x;
    }
    if (lane == 0) {  // MetaGraph edges in std::set<pair<string,string>> order
        int ne = 0;
        for (int ra = 0; ra < K; ++ra) {
            const int a = by_rank[ra];
            for (uint64_t s = succ_r[a]; s; s &= s - 1) ed[ne++] = ws_out_edge{a, by_rank[low_bit(s)]};
        }
    }
    const double* w_start = C.at<double>(L.w_start);
    const double* w_dur = C.at<double>(L.w_dur);
    const int* w_level = C.at<int>(L.w_level);
    const int* w_eb = C.at<int>(L.w_eb);
    const int* w_ec = C.at<int>(L.w_ec);
    for (int w = lane; w < P.nW; w += 32) {
        ws_out_wave x;
        x.start = w_start[w];
        x.duration = w_dur[w];
        x.level = w_level[w];
        x.entry_begin = w_eb[w];
        x.n_entries = w_ec[w];
        x.pad = 0;
        wv[w] = x;
    }
    const int* e_k = C.at<int>(L.e_k);
    const int* e_n = C.at<int>(L.e_n);
    const int* e_l = C.at<int>(L.e_l);
    const double* e_span = C.at<double>(L.e_span);
    const uint64_t* e_mask = C.at<uint64_t>(L.e_mask);
    const int* e_rot = C.at<int>(L.e_rot);
    for (int e = lane; e < P.nE; e += 32) {
        ws_out_entry x;
        x.span = e_span[e];
        x.devmask = e_mask[e];
        x.metaop = e_k[e];
        x.n = e_n[e];
        x.layers = e_l[e];
        x.rot = e_rot[e];
        en[e] = x;
    }
    const uint64_t* f_vol = C.at<uint64_t>(L.f_vol);
    const int* f_meta = C.at<int>(L.f_meta);
    for (int f = lane; f < P.nF; f += 32) {
        ws_out_flow x;
        x.volume = f_vol[f];
        x.from_wave = f_meta[6 * f];
        x.from_metaop = f_meta[6 * f + 1];
        x.to_wave = f_meta[6 * f + 2];
        x.to_metaop = f_meta[6 * f + 3];
        x.mode = f_meta[6 * f + 4];
        x.pad = 0;
        fl[f] = x;
    }
    if (lane == 0) {
        ws_plan_result r{};
        r.status = WS_STATUS_OK;
        r.n_metaops = K;
        r.n_edges = nedges;
        r.n_levels = n_levels;
        r.n_waves = P.nW;
        r.n_entries = P.nE;
        r.n_flows = P.nF;
        r.n_pieces = npieces;
        r.lower_bound = lower_bound;
        r.end_time = end_time;
        r.offset = off;
        r.size = sz;
        *res = r;
    }
}

__device__ int status_of(int code) {
    switch (code) {
        case WS_E_FIT_NONPOSITIVE:
        case WS_E_TP_EXCEEDS:
        case WS_E_BT_BUDGET:
        case WS_E_NO_PLACEMENT_W0: return WS_STATUS_INFEASIBLE;
        case WS_E_CURVE_START:
        case WS_E_CURVE_CONTIG:
        case WS_E_EVAL_RANGE:
        case WS_E_NO_SCHEDULABLE:
        case WS_E_NO_PROGRESS: return WS_STATUS_INVARIANT;
        default:
            if (code >= 40 && code < 60) return WS_STATUS_LIMIT;
            if (code >= 60) return WS_STATUS_INTERNAL;
            return WS_STATUS_PARSE;
    }
}

// ---------------------------------------------------------------------------
// K1+K3+K4+K5 driver: one warp per plan
// ---------------------------------------------------------------------------
constexpr int kPlanWarps = 4;  // warps per block

__global__ void __launch_bounds__(32 * kPlanWarps) k_plan(PlanArgs A) {
    __shared__ Ctl ctl_s[kPlanWarps];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = blockIdx.x * kPlanWarps + wid;
    if (slot >= A.n_launch) return;
    if (A.n_ids && slot >= *A.n_ids) return;
    const int p = A.plan_ids ? A.plan_ids[slot] : A.plan_base + slot;
    Ctl* ctl = &ctl_s[wid];
    if (lane == 0) *ctl = Ctl{};
    __syncwarp();
    const ws_plan_rec& R = A.B.plans[p];
    PlanCtx C;
    C.B = &A.B;
    C.R = &R;
    C.fit = &A.fit;
    C.L = &A.L;
    C.base = A.scratch + static_cast<int64_t>(slot) * A.L.bytes;
    C.ctl = ctl;
    C.lane = lane;
    C.N = R.n_dev;
    C.M = R.n_mod;
    C.K = 0;
    C.mbase = R.mod_begin;
    int n_levels = 0;
    double lower_bound = 0.0, end_time = 0.0;
    PlaceState P{};
    bool ok = true;
    if (R.n_mod == 0 && R.n_tasks == 0) {
        ok = false;
        if (lane == 0) ctl->err = WS_E_HOST_PRESET;
    } else if (R.n_dev > A.caps.N || R.n_dev > WS_MAX_DEVICES) {
        ok = false;
        if (lane == 0) ctl->err = WS_E_LIMIT_DEVICES;
    } else if (R.n_mod > A.caps.M) {
        ok = false;
        if (lane == 0) ctl->err = WS_E_LIMIT_MODULES;
    }
    __syncwarp();
    if (ok) ok = stage_graph(C);
    if (ok) ok = stage_fit_status(C);
    if (ok) ok = stage_valid(C);
    if (ok) {
        n_levels = ctl->i1;
        TLookup T{A.fit.ttab, A.fit.nmax, A.fit.tstride, C.mbase, C.at<int>(A.L.mod_of), ctl};
        double* cstar = C.at<double>(A.L.cstar);
        int* lfw = C.at<int>(A.L.lvl_fw);
        int* lnw = C.at<int>(A.L.lvl_nw);
        double* w_start = C.at<double>(A.L.w_start);
        double* w_dur = C.at<double>(A.L.w_dur);
        double offset = 0.0;
        int nW = 0, nE = 0;
        if (lane == 0) ctl->i2 = A.caps.W, ctl->i3 = A.caps.E;
        __syncwarp();
        for (int l = 0; l < n_levels && ok; ++l) {
            double cs = 0.0;
            ok = stage_level_alloc(C, T, l, cs);
            if (!ok) break;
            lower_bound += cs;
            if (lane == 0) {
                cstar[l] = cs;
                lfw[l] = nW;
                double rel_end = 0.0;
                const int w0 = nW;
                if (stage_schedule_level(C, T, l, nW, nE, rel_end)) {
                    // merge_levels (schedule.hpp:292-309)
                    double level_end = offset;
                    for (int w = w0; w < nW; ++w) {
                        w_start[w] += offset;
                        const double e = w_start[w] + w_dur[w];
                        level_end = (level_end < e) ? e : level_end;
                    }
                    offset = level_end;
                    lnw[l] = nW - w0;
                }
                ctl->i0 = nW;
                ctl->i1 = nE;
                ctl->level_offset = offset;
            }
            __syncwarp();
            if (ctl->err) {
                ok = false;
                break;
            }
            nW = ctl->i0;
            nE = ctl->i1;
            offset = ctl->level_offset;
        }
        end_time = offset;
        P.nW = nW;
        P.nE = nE;
    }
    if (ok) {
        P.K = C.K;
        P.N = C.N;
        P.G = R.n_groups + C.K;
        P.n_isl = R.n_islands;
        P.all = C.N == 64 ? ~0ull : ((1ull << C.N) - 1ull);
        if (P.G > A.caps.G || P.n_isl > A.caps.IS) {
            ok = false;
            if (lane == 0) set_err(ctl, WS_E_LIMIT_MODULES);
            __syncwarp();
        }
        P.Fcap = A.caps.F;
        if (ok) ok = stage_place(C, P);
    }
    __syncwarp();
    if (ok) {
        emit(C, p, P, n_levels, lower_bound, end_time, A);
    } else if (lane == 0) {
        ws_plan_result r{};
        r.err_code = ctl->err;
        r.status = status_of(ctl->err);
        r.err_a = ctl->a;
        r.err_b = ctl->b;
        r.err_x = ctl->x;
        r.err_y = ctl->y;
        A.results[p] = r;
    }
}

}  // namespace wsdev
