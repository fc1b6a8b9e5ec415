// sched.cuh — k_sched: subsystems (1) graph/contraction/levels, (3) allocation
// and (4a) wavefront scheduling.  One warp per plan; the per-plan working set
// lives in dynamic shared memory; the schedule is handed to k_place through a
// per-plan record in global memory.
#pragma once
#include "kcommon.cuh"
#include "mask.cuh"

namespace wsdev {

constexpr int kSchedWarps = 4;

// ---- per-plan schedule record (global), written by k_sched, read by k_place
struct SchedHdr {
    int ok, K, n_levels, nW;
    int nE, scoped, n_pg, pad2;  // scoped: entities are (MetaOp, task) pairs (e_met/e_task);
                                 // n_pg > 0: placement groups (one place() call each, pg_*)
    double lower_bound, end_time;
};

struct RecCaps {
    int M, W, E;
};

struct RecLayout {
    int hdr, mod_of, level, up_n, up_l, lo_n, lo_l, by_rank, idrank, pred_r, succ_r, cstar, lvl_fw, lvl_nw;
    int e_frac, e_met, e_task;  // per entity: batch_fraction, MetaOp, task (-1: the MetaOp itself)
    int pg_off, pg_cnt, pg_wbeg, pg_wn, pg_list;  // placement groups: device block, waves (task-level-optimus)
    int w_level, w_eb, w_ec, w_start, w_dur, e_k, e_n, e_l, e_span;
    int bytes;
};

__host__ __device__ inline int al16(int v) { return (v + 15) & ~15; }

__host__ __device__ inline RecLayout make_rec_layout(const RecCaps& c) {
    RecLayout L{};
    int o = 0;
    auto take = [&](int b) {
        const int at = o;
        o = al16(o + b);
        return at;
    };
    L.hdr = take(sizeof(SchedHdr));
    L.mod_of = take(4 * c.M);
    L.level = take(4 * c.M);
    L.up_n = take(4 * c.M);
    L.up_l = take(4 * c.M);
    L.lo_n = take(4 * c.M);
    L.lo_l = take(4 * c.M);
    L.by_rank = take(4 * c.M);
    L.idrank = take(4 * c.M);
    L.pred_r = take(8 * c.M);
    L.succ_r = take(8 * c.M);
    L.cstar = take(8 * c.M);
    L.lvl_fw = take(4 * c.M);
    L.lvl_nw = take(4 * c.M);
    L.e_frac = take(8 * c.M);
    L.e_met = take(4 * c.M);
    L.e_task = take(4 * c.M);
    L.pg_off = take(4 * c.M);
    L.pg_cnt = take(4 * c.M);
    L.pg_wbeg = take(4 * c.M);
    L.pg_wn = take(4 * c.M);
    L.pg_list = take(4 * c.W);
    L.w_level = take(4 * c.W);
    L.w_eb = take(4 * c.W);
    L.w_ec = take(4 * c.W);
    L.w_start = take(8 * c.W);
    L.w_dur = take(8 * c.W);
    L.e_k = take(4 * c.E);
    L.e_n = take(4 * c.E);
    L.e_l = take(4 * c.E);
    L.e_span = take(8 * c.E);
    L.bytes = o;
    return L;
}

// ---- k_sched shared working set (per warp)
struct SmLayout {
    int adj, tmask, predk, pred_r, succ_r, valid, credit;                   // [M] 8 B
    int indeg, keyrank, modat, kofm, mod_of, idrank, by_rank, level;         // [M] 4 B
    int up_n, up_l, lo_n, lo_l, sumlay, lvl_mem, gm_of, nmax_of, Lk, absorb;  // [M] 4 B
    int lvl_begin;                                                           // [M+1]
    int cstar_sm, aerr_x, aerr_y, aerr;                                      // [M] per level
    int tk, tn, tl, tn2, sel, best, pool, klay;                              // [2M]
    int ord;                                                                 // [3*2M]
    // task-scoped baselines only (sizes 0 otherwise)
    int ent_met, ent_task, ent_frac, epred;                                  // [64] entities
    int ent_of, kscale, tlvl, vord;                                          // [M] per task
    int tvalid, talloc, cw_start, cw_dur, cw_level, cw_ent, cw_n, cw_L;     // [64] optimus tasks / waves
    int pl_off, pl_cnt, pl_wbeg, pl_wn, perm, tfin;                         // [64] placements, [M] finish
    int tcur, tnext, tnxn;                                                  // [64] optimus task-time cache
    int bytes;
};

// M: MetaOps per plan; scoped: the batch has task-scoped baseline plans;
// tasks: the batch's largest task count (task-indexed optimus arrays)
// mb: bytes of one valid-allocation set (8: n <= 64; 32: DevMask<4>, n <= 256)
__host__ __device__ inline SmLayout make_sm_layout(int M, bool scoped = false, int tasks = WS_MAX_TASKS, int mb = 8) {
    SmLayout L{};
    int o = 0;
    auto take = [&](int b) {
        const int at = o;
        o = (o + b + 7) & ~7;
        return at;
    };
    const int T = 2 * M;
    // the part phases 2 and 3 read (phase-split launches carry it between
    // the phase kernels: sched_state_bytes) ...
    L.pred_r = take(8 * M);
    L.succ_r = take(8 * M);
    L.valid = take(mb * M);
    L.credit = take(8 * M);
    L.mod_of = take(4 * M);
    L.idrank = take(4 * M);
    L.by_rank = take(4 * M);
    L.level = take(4 * M);
    L.up_n = take(4 * M);
    L.up_l = take(4 * M);
    L.lo_n = take(4 * M);
    L.lo_l = take(4 * M);
    L.sumlay = take(4 * M);
    L.lvl_mem = take(4 * M);
    L.gm_of = take(4 * M);
    L.nmax_of = take(4 * M);
    L.Lk = take(4 * M);
    L.absorb = take(4 * M);
    L.lvl_begin = take(4 * (M + 1));
    L.cstar_sm = take(8 * M);
    L.aerr_x = take(8 * M);
    L.aerr_y = take(8 * M);
    L.aerr = take(4 * M);
    // ... graph construction scratch and the task masks, read after phase 1
    // only by the task-scoped baselines (which run unsplit) ...
    L.adj = take(8 * M);
    L.tmask = take(8 * M);
    L.predk = take(8 * M);
    L.indeg = take(4 * M);
    L.keyrank = take(4 * M);
    L.modat = take(4 * M);
    L.kofm = take(4 * M);
    // ... and the wave-scheduling scratch (written by phase 3 before it is read)
    L.tk = take(4 * T);
    L.tn = take(4 * T);
    L.tl = take(4 * T);
    L.tn2 = take(4 * T);
    L.sel = take(4 * T);
    L.best = take(4 * T);
    L.pool = take(4 * T);
    L.klay = take(4 * T);
    L.ord = take(4 * 3 * T);
    const int EM = scoped ? WS_MAX_MODULES : 0, MS = scoped ? M : 0, TT = scoped ? tasks : 0;
    L.ent_met = take(4 * EM);
    L.ent_task = take(4 * EM);
    L.ent_frac = take(8 * EM);
    L.epred = take(8 * EM);
    L.ent_of = take(4 * MS);
    L.kscale = take(8 * MS);
    L.tlvl = take(4 * MS);
    L.vord = take(4 * MS);
    L.tvalid = take(mb * TT);
    L.talloc = take(4 * TT);
    L.cw_start = take(8 * EM);
    L.cw_dur = take(8 * EM);
    L.cw_level = take(4 * EM);
    L.cw_ent = take(4 * EM);
    L.cw_n = take(4 * EM);
    L.cw_L = take(4 * EM);
    L.pl_off = take(4 * TT);
    L.pl_cnt = take(4 * TT);
    L.pl_wbeg = take(4 * TT);
    L.pl_wn = take(4 * TT);
    L.perm = take(4 * EM);
    L.tfin = take(8 * MS);
    L.tcur = take(8 * TT);
    L.tnext = take(8 * TT);
    L.tnxn = take(4 * TT);
    L.bytes = (o + 15) & ~15;
    return L;
}

struct SchedArgs {
    ws_batch B;
    FitOut fit;
    RecCaps caps;
    RecLayout RL;
    SmLayout SL;
    char* recs;              // [n_plans * RL.bytes]
    const int32_t* plan_ids; // launch order (cost-sorted) or retry list
    const int32_t* n_ids;    // device count of plan_ids (retry pass) or null
    int n_launch;
    int rec_by_slot;         // retry pass: records indexed by launch slot
    int M_cap;               // modules per plan this launch supports
    int scoped_ok;           // SL carries the task-scoped working set (distmm-mt plans)
    ws_plan_result* results;
    // phase-split launches (k_sched<DM, 1..3>): per launch slot the warp's
    // shared working set, control block and flags between the phases
    char* state;
    long long state_stride;  // bytes per slot: SL.bytes + kSchedStateHdr
    int warp_smem;           // dynamic shared bytes per warp of this launch (a phase kernel
                             // gets only the layout prefix it touches: sched_phase_bytes)
};

// bytes before the saved shared working set of a phase-split slot: Ctl + flags
constexpr int kSchedStateHdr = 128;

struct SCtx {
    const ws_batch* B;
    const ws_plan_rec* R;
    const FitOut* F;
    const SmLayout* L;
    char* sm;
    Ctl* ctl;
    int lane, N, M, K, mbase;
    const double* kscale = nullptr;  // per-MetaOp beta_w scale while a scaled level runs (distmm-mt)
    template <typename T>
    __device__ __forceinline__ T* at(int off) const {
        return reinterpret_cast<T*>(sm + off);
    }
};

// T_k(n): the T-table, or the scaled curve of a task-scoped baseline level
__device__ __forceinline__ double T_of(const SCtx& C, int k, int n) {
    const int gm = C.at<int>(C.L->gm_of)[k];
#ifdef WS_NO_SCALE
    return t_at(*C.F, gm, n);
#else
    return C.kscale ? t_scaled(*C.F, *C.B, gm, n, C.kscale[k]) : t_at(*C.F, gm, n);
#endif
}

// ---------------------------------------------------------------------------
// (1) module DAG from the flows (graph.hpp:97-147), lexicographic Kahn and
// contraction numbering (:66-90, :153-202), MetaGraph edges, levels (:207-226)
// ---------------------------------------------------------------------------
__device__ bool s_graph(SCtx& C) {
    const ws_batch& B = *C.B;
    const ws_plan_rec& R = *C.R;
    const int M = C.M, lane = C.lane;
    uint64_t* adj = C.at<uint64_t>(C.L->adj);
    uint64_t* tmask = C.at<uint64_t>(C.L->tmask);
    int* kofm = C.at<int>(C.L->kofm);
    int* indeg = C.at<int>(C.L->indeg);
    int* keyrank = C.at<int>(C.L->keyrank);
    int* modat = C.at<int>(C.L->modat);
    int* mod_of = C.at<int>(C.L->mod_of);
    #pragma unroll 1
    for (int m = lane; m < M; m += 32) {
        adj[m] = 0;
        tmask[m] = 0;
        kofm[m] = -1;
    }
    __syncwarp();
    // tasks in parallel: lane t walks the flow of task t
    #pragma unroll 1
    for (int t = lane; t < R.n_tasks; t += 32) {
        const int tg = R.task_begin + t;
        const int* tok = B.tokens + B.task_tok_off[tg];
        const int ntok = B.task_tok_n[tg];
        const uint64_t tbit = 1ull << B.task_rank[tg];
        uint64_t prev_tails = 0, heads = 0, tails = 0;
        int last = -1;
        bool start = true;
        #pragma unroll 1
        for (int i = 0; i <= ntok; ++i) {
            const int v = i < ntok ? __ldg(tok + i) : WS_TOK_STEP;
            if (v >= 0) {
                atomicOr(reinterpret_cast<unsigned long long*>(&tmask[v]), tbit);
                if (start)
                    heads |= 1ull << v;  // branch head (graph.hpp:130)
                else
                    atomicOr(reinterpret_cast<unsigned long long*>(&adj[last]), 1ull << v);  // chained (:131)
                start = false;
                last = v;
            } else {
                if (last >= 0) tails |= 1ull << last;
                last = -1;
                start = true;
                if (v == WS_TOK_STEP) {  // every tail of step k feeds every head of step k+1 (:137-139)
                    #pragma unroll 1
                    for (uint64_t f = prev_tails; f; f &= f - 1)
                        atomicOr(reinterpret_cast<unsigned long long*>(&adj[low_bit(f)]), heads);
                    prev_tails = tails;
                    heads = tails = 0;
                }
            }
        }
    }
    __syncwarp();
    uint64_t used = 0;
    #pragma unroll 1
    for (int base = 0; base < M; base += 32) {
        const int m = base + lane;
        used |= static_cast<uint64_t>(__ballot_sync(kFull, m < M && tmask[m] != 0)) << base;
    }
    // keys kind+"." packed big-endian into their first 8 bytes (zero padded);
    // `valid` is scratch here, s_valid fills it later
    uint64_t* key8 = C.at<uint64_t>(C.L->valid);
    #pragma unroll 1
    for (int m = lane; m < M; m += 32) {
        const uint8_t* nm = B.names + B.mod_name_off[C.mbase + m];
        const int len = B.mod_name_len[C.mbase + m];
        uint64_t k = 0;
        #pragma unroll 1
        for (int i = 0; i < 8 && i <= len; ++i)
            k |= static_cast<uint64_t>(i < len ? nm[i] : static_cast<uint8_t>('.')) << (56 - 8 * i);
        key8[m] = k;
    }
    __syncwarp();
    // in-degrees, rank of the key kind+"." and kinds prefixed by another kind+"."
    int conflict = 0;
    #pragma unroll 1
    for (int m = lane; m < M; m += 32) {
        int d = 0;
        #pragma unroll 1
        for (int a = 0; a < M; ++a) d += (adj[a] >> m) & 1ull;
        indeg[m] = d;
        if (!(used >> m & 1ull)) {
            keyrank[m] = -1;
            continue;
        }
        const uint64_t k8 = key8[m];
        const int lm_ = B.mod_name_len[C.mbase + m];
        const uint64_t pmask = lm_ < 7 ? ~0ull << (56 - 8 * lm_) : ~0ull;  // bytes 0..len
        int r = 0;
        #pragma unroll 1
        for (uint64_t o = used; o; o &= o - 1) {
            const int q = low_bit(o);
            if (q == m) continue;
            const uint64_t q8 = key8[q];
            const int lq = B.mod_name_len[C.mbase + q];
            if (q8 != k8) {
                r += q8 < k8;  // the first differing byte lies in the packed prefix
            } else if (key_less(op_key(B, C.mbase + q, 0, false), op_key(B, C.mbase + m, 0, false))) {
                ++r;
            }
            if (lq > lm_) {  // kq starts with km + "."
                bool pre;
                if (lm_ < 8) {
                    pre = ((q8 ^ k8) & pmask) == 0;
                } else {
                    const OpKey km = op_key(B, C.mbase + m, 0, false), kq = op_key(B, C.mbase + q, 0, false);
                    pre = true;
                    #pragma unroll 1
                    for (int i = 0; i <= km.len && pre; ++i) pre = kq.at(i) == km.at(i);
                }
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
        if (!conflict) {
            // once kind.0 pops, its remaining layers pop consecutively,
            // so the operator-level lexicographic Kahn is the module Kahn by kind+"."
            uint64_t ready = 0;
            #pragma unroll 1
            for (uint64_t u = used; u; u &= u - 1) {
                const int m = low_bit(u);
                if (indeg[m] == 0) ready |= 1ull << keyrank[m];
            }
            while (ready) {
                const int r = low_bit(ready);
                ready &= ready - 1;
                const int m = modat[r];
                kofm[m] = K;
                mod_of[K++] = m;
                #pragma unroll 1
                for (uint64_t s = adj[m]; s; s &= s - 1) {
                    const int q = low_bit(s);
                    if (--indeg[q] == 0) ready |= 1ull << keyrank[q];
                }
            }
        } else {
            // general operator-level lexicographic Kahn with per-module layer cursors
            int* cursor = C.at<int>(C.L->sumlay);
            #pragma unroll 1
            for (int m = 0; m < M; ++m) cursor[m] = 0;
            while (true) {
                int best = -1;
                OpKey bk;
                #pragma unroll 1
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
                    mod_of[K++] = best;
                }
                if (++cursor[best] == B.mod_layers[C.mbase + best])
                    #pragma unroll 1
                    for (uint64_t s = adj[best]; s; s &= s - 1) --indeg[low_bit(s)];
            }
        }
        C.ctl->i0 = K;
        if (K != nused) set_err(C.ctl, WS_E_CYCLIC_WORKLOAD);
    }
    __syncwarp();
    if (C.ctl->err) return false;
    const int K = C.ctl->i0;
    C.K = K;
    int* idrank = C.at<int>(C.L->idrank);
    int* by_rank = C.at<int>(C.L->by_rank);
    int* gm_of = C.at<int>(C.L->gm_of);
    int* Lk = C.at<int>(C.L->Lk);
    #pragma unroll 1
    for (int k = lane; k < K; k += 32) {  // MetaOp ids "m<k>" in std::map order
        int r = 0;
        #pragma unroll 1
        for (int j = 0; j < K; ++j) r += dec_less(j, k);
        idrank[k] = r;
        by_rank[r] = k;
        const int gm = C.mbase + mod_of[k];
        gm_of[k] = gm;
        Lk[k] = B.mod_layers[gm];  // nmax_of (a k_fit output) is read after griddepcontrol.wait
    }
    __syncwarp();
    uint64_t* predk = C.at<uint64_t>(C.L->predk);
    uint64_t* pred_r = C.at<uint64_t>(C.L->pred_r);
    uint64_t* succ_r = C.at<uint64_t>(C.L->succ_r);
    #pragma unroll 1
    for (int k = lane; k < K; k += 32) {
        const int m = mod_of[k];
        uint64_t pk = 0, pr = 0, sr = 0;
        #pragma unroll 1
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
        #pragma unroll 1
        for (int k = 0; k < K; ++k) {
            int lv = 0;
            #pragma unroll 1
            for (uint64_t p = predk[k]; p; p &= p - 1) {
                const int q = level[low_bit(p)] + 1;
                lv = q > lv ? q : lv;
            }
            level[k] = lv;
            maxl = lv > maxl ? lv : maxl;
        }
        int* lb = C.at<int>(C.L->lvl_begin);
        int* lm = C.at<int>(C.L->lvl_mem);
        int* fill = C.at<int>(C.L->absorb);
        #pragma unroll 1
        for (int l = 0; l <= maxl + 1; ++l) lb[l] = 0;
        #pragma unroll 1
        for (int k = 0; k < K; ++k) lb[level[k] + 1]++;
        #pragma unroll 1
        for (int l = 0; l <= maxl; ++l) lb[l + 1] += lb[l];
        #pragma unroll 1
        for (int l = 0; l <= maxl; ++l) fill[l] = lb[l];
        #pragma unroll 1
        for (int r = 0; r < K; ++r) {
            const int k = by_rank[r];
            lm[fill[level[k]]++] = k;
        }
        C.ctl->i1 = maxl + 1;
    }
    __syncwarp();
    return true;
}

// (2) results of k_fit: the first module in kind order whose fit failed
__device__ bool s_fit_status(SCtx& C) {
    const int M = C.M;
    #pragma unroll 1
    for (int base = 0; base < M; base += 32) {
        const int m = base + C.lane;
        const int e = m < M ? C.F->err[C.mbase + m] : 0;
        const unsigned b = __ballot_sync(kFull, e != 0);
        if (b) {
            const int first = base + __ffs(b) - 1;
            if (C.lane == 0) {
                const int gm = C.mbase + first;
                const int code = C.F->err[gm];
                set_err(C.ctl, code, code == WS_E_NO_SOURCE ? first : C.F->err_a[gm], C.F->err_b[gm]);
            }
            __syncwarp();
            return false;
        }
    }
    return true;
}

// (3a) valid allocation sets n = tp*r with r | B (allocation.hpp:51-63)
// check_tp: the planner's NoValidAllocation in id order; the baselines check
// each MetaOp when they reach it (an over-wide tp leaves an empty set).
template <class DM>
__device__ bool s_valid(SCtx& C, bool check_tp) {
    const ws_batch& B = *C.B;
    const int K = C.K, N = C.N, lane = C.lane;
    const int* gm_of = C.at<int>(C.L->gm_of);
    const int* by_rank = C.at<int>(C.L->by_rank);
    DM* valid = C.at<DM>(C.L->valid);
    #pragma unroll 1
    for (int base = 0; base < K && check_tp; base += 32) {  // tp > N in id order (planner.hpp:168-171)
        const int r = base + lane;
        const bool bad = r < K && B.mod_tp[gm_of[by_rank[r]]] > N;
        const unsigned b = __ballot_sync(kFull, bad);
        if (b) {
            if (lane == 0) {
                const int k = by_rank[base + __ffs(b) - 1];
                set_err(C.ctl, WS_E_TP_EXCEEDS, k, B.mod_tp[gm_of[k]]);
            }
            __syncwarp();
            return false;
        }
    }
    #pragma unroll 1
    for (int k = 0; k < K; ++k) {  // lanes = device counts n, one ballot per 32 n
        const int gm = gm_of[k];
        const int tp = B.mod_tp[gm];
        const long long batch = B.mod_batch[gm];
        DM v = dm_zero<DM>();
        #pragma unroll 1
        for (int base = 0; base < N; base += 32) {
            const int n = base + lane + 1;
            bool ok = n <= N && n % tp == 0;
            if (ok)  // 32-bit remainder when the batch fits (same result, fewer instructions)
                ok = batch <= 0xffffffffll ? (static_cast<unsigned>(batch) % static_cast<unsigned>(n / tp)) == 0u
                                           : batch % (n / tp) == 0;
            dm_or_bits32(v, base, __ballot_sync(kFull, ok));
        }
        if (lane == 0) valid[k] = v;
    }
    __syncwarp();
    return true;
}

__device__ __forceinline__ double ordered_sum(double v0, double v1, int w) {
    double total = 0.0;  // reference order: ((0 + v_0) + v_1) + ...
    #pragma unroll 1
    for (int j = 0; j < 32 && j < w; ++j) total += shfl_d(v0, j);
    #pragma unroll 1
    for (int j = 0; j + 32 < w; ++j) total += shfl_d(v1, j);
    return total;
}

// repair_capacity (allocation.hpp:107-139) for one level; lane i holds members
// i, i+32.  Ties and the first error go by MetaOp id (plan.tuples is an id map).
template <class DM>
__device__ bool s_level_repair(SCtx& C, int lvl) {
    const int N = C.N, lane = C.lane;
    const int* idrank = C.at<int>(C.L->idrank);
    const int* lb = C.at<int>(C.L->lvl_begin);
    const int* lm = C.at<int>(C.L->lvl_mem) + lb[lvl];
    const int w = lb[lvl + 1] - lb[lvl];
    const int* gm_of = C.at<int>(C.L->gm_of);
    const int* nmax_of = C.at<int>(C.L->nmax_of);
    const DM* valid = C.at<DM>(C.L->valid);
    int* up_n = C.at<int>(C.L->up_n);
    const int* up_l = C.at<int>(C.L->up_l);
    const int* lo_n = C.at<int>(C.L->lo_n);
    const int* lo_l = C.at<int>(C.L->lo_l);
    const FitOut& F = *C.F;
    while (true) {
        int wid = 0;
        #pragma unroll 1
        for (int i = lane; i < w; i += 32) {
            const int k = lm[i];
            const int a = up_n[k], b = lo_l[k] ? lo_n[k] : 0;
            wid += a > b ? a : b;
        }
        if (warp_sum(wid) <= N) break;
        double best_pen = 0.0;
        int best_i = 0x7fffffff, best_key = 0x7fffffff, best_t = 0, eidx = 0x7fffffff;
        double ex = 0, ey = 0;
        #pragma unroll 1
        for (int i = lane; i < w; i += 32) {
            const int k = lm[i];
            const int key = idrank[k];
            const int un = up_n[k];
            const DM below = valid[k] & dm_first<DM>(un - 1);  // valid values < un
            if (!dm_any(below)) continue;
            const int target = dm_high(below) + 1;
            if (lo_l[k] && target <= lo_n[k]) continue;
            const int nmax = nmax_of[k];
            if (target > nmax || un > nmax) {  // eval(target) first, then eval(t.n)
                if (key < eidx) eidx = key, ex = target > nmax ? target : un, ey = nmax;
                continue;
            }
            const double pen = up_l[k] * (T_of(C, k, target) - T_of(C, k, un));
            if (best_i == 0x7fffffff || pen < best_pen || (pen == best_pen && key < best_key))
                best_pen = pen, best_i = i, best_key = key, best_t = target;
        }
        const int emin = warp_min_i(eidx);
        if (emin != 0x7fffffff) {
            const int src = __ffs(__ballot_sync(kFull, eidx == emin)) - 1;
            const double xx = shfl_d(ex, src), yy = shfl_d(ey, src);
            if (lane == 0) {
                C.ctl->err = WS_E_EVAL_RANGE;
                C.ctl->x = xx;
                C.ctl->y = yy;
            }
            __syncwarp();
            return false;
        }
        #pragma unroll 1
        for (int off = 16; off; off >>= 1) {  // argmin over (penalty, MetaOp id)
            const double op = __shfl_xor_sync(kFull, best_pen, off);
            const int oi = __shfl_xor_sync(kFull, best_i, off);
            const int okey = __shfl_xor_sync(kFull, best_key, off);
            const int ot = __shfl_xor_sync(kFull, best_t, off);
            if (oi != 0x7fffffff && (best_i == 0x7fffffff || op < best_pen || (op == best_pen && okey < best_key)))
                best_pen = op, best_i = oi, best_key = okey, best_t = ot;
        }
        if (best_i == 0x7fffffff) break;
        if (lane == 0) up_n[lm[best_i]] = best_t;
        __syncwarp();
    }
    return true;
}

// bi-point discretization of one MetaOp (allocation.hpp:149-214).  Returns
// false on OutOfRange (x = n, y = n_max; eval(n_over) is evaluated first).
// scale: non-null for a scaled curve (T evaluated from the pieces, not the T-table)
template <class DM>
__device__ __forceinline__ bool discretize_one(const FitOut& F, const ws_plan_rec& R, int gm, int L, double nmax,
                                               const DM& v, double nstar, double cs, int& un, int& ul, int& ln,
                                               int& ll, double& ex, const ws_batch* B = nullptr,
                                               double scale = 1.0) {
    int exact = -1, n_over = -1, n_under = -1;
    #pragma unroll 1
    for (DM b = v; dm_any(b); b = dm_drop_low(b)) {
        const int x = dm_low(b) + 1;
        if (fabs(x - nstar) < 1e-9) {
            exact = x;
            break;
        }
    }
    if (exact < 0)
        #pragma unroll 1
        for (DM b = v; dm_any(b); b = dm_drop_low(b)) {
            const int x = dm_low(b) + 1;
            if (x < nstar) n_under = x;
            if (x > nstar) {
                n_over = x;
                break;
            }
        }
    un = 0, ul = L, ln = 0, ll = 0;
    if (exact >= 0) {
        un = exact;
    } else if (n_over == -1) {
        un = dm_high(v) + 1;
    } else if (n_under == -1) {
        un = dm_low(v) + 1;
    } else {
        if (n_over > nmax || n_under > nmax) {
            ex = n_over > nmax ? n_over : n_under;
            return false;
        }
        const double t_over = B ? t_scaled(F, *B, gm, n_over, scale) : t_at(F, gm, n_over);
        const double t_under = B ? t_scaled(F, *B, gm, n_under, scale) : t_at(F, gm, n_under);
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
    return true;
}

// (3b) bisection on the capacity equation, bi-point discretization and
// capacity repair for one level; lane i holds members i and i+32
template <class DM>
__device__ bool s_level_alloc(SCtx& C, int lvl, double& c_star_out) {
    const ws_batch& B = *C.B;
    const ws_plan_rec& R = *C.R;
    const int N = C.N, lane = C.lane;
    const int* lb = C.at<int>(C.L->lvl_begin);
    const int* lm = C.at<int>(C.L->lvl_mem) + lb[lvl];
    const int w = lb[lvl + 1] - lb[lvl];
    const int* gm_of = C.at<int>(C.L->gm_of);
    const int* nmax_of = C.at<int>(C.L->nmax_of);
    const int* Lk = C.at<int>(C.L->Lk);
    const DM* valid = C.at<DM>(C.L->valid);
    int* up_n = C.at<int>(C.L->up_n);
    int* up_l = C.at<int>(C.L->up_l);
    int* lo_n = C.at<int>(C.L->lo_n);
    int* lo_l = C.at<int>(C.L->lo_l);
    const double nd = static_cast<double>(N);
    const FitOut& F = *C.F;
    struct Mem {
        int k, gm, L;
        double nmax;
        InvPre inv;
    } mem[2];
    for (int s = 0; s < 2; ++s) {
        const int i = lane + 32 * s;
        Mem& q = mem[s];
        q.k = -1;
        if (i < w) {
            q.k = lm[i];
            q.gm = gm_of[q.k];
            q.L = Lk[q.k];
            q.nmax = nmax_of[q.k];
            q.inv.init(F.pieces + 5 * F.piece_off[q.gm], F.npieces[q.gm], B.mod_c[q.gm], B.mod_w[q.gm], q.nmax,
                       C.kscale ? C.kscale[q.k] : 1.0);
        }
    }
    // bracket [max T(min(N,nmax))*L, sum T(1)*L] (allocation.hpp:75-80)
    double lo0 = 0.0, hi0[2] = {0.0, 0.0};
    for (int s = 0; s < 2; ++s) {
        const Mem& q = mem[s];
        if (q.k < 0) continue;
        const double ncap = (q.nmax < nd) ? q.nmax : nd;
        const double v = T_of(C, q.k, static_cast<int>(ncap)) * q.L;
        lo0 = (lo0 < v) ? v : lo0;
        hi0[s] = T_of(C, q.k, 1) * q.L;
    }
    double c_lo = warp_max_nonneg(lo0);
    double c_hi = ordered_sum(hi0[0], hi0[1], w);
    auto probe_term = [&](const Mem& q, double cc) {
        const double v = q.inv(cc / q.L);
        return (nd < v) ? nd : v;  // std::min(v, N)
    };
    #pragma unroll 1
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
    // discretize (allocation.hpp:149-214)
    int eidx0 = 0x7fffffff;
    double ex0 = 0, ey0 = 0;
    for (int s = 0; s < 2; ++s) {
        const Mem& q = mem[s];
        if (q.k < 0) continue;
        int un, ul, ln, ll;
        double ex;
        if (!discretize_one(F, R, q.gm, q.L, q.nmax, valid[q.k], probe_term(q, cs), cs, un, ul, ln, ll, ex,
                            C.kscale ? &B : nullptr, C.kscale ? C.kscale[q.k] : 1.0)) {
            const int idx = C.at<int>(C.L->idrank)[q.k];  // first failure in MetaOp id order
            if (idx < eidx0) eidx0 = idx, ex0 = ex, ey0 = q.nmax;
            continue;
        }
        up_n[q.k] = un;
        up_l[q.k] = ul;
        lo_n[q.k] = ln;
        lo_l[q.k] = ll;
    }
    {
        const int emin = warp_min_i(eidx0);
        if (emin != 0x7fffffff) {
            const int src = __ffs(__ballot_sync(kFull, eidx0 == emin)) - 1;
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
    return s_level_repair<DM>(C, lvl);
}


// (3b) all levels at once (K <= 32): levels are independent, so lane i holds
// the i-th MetaOp in level-major order and each level's bisection runs in its
// own lane segment; segment-local ordered sums reproduce each level's
// reference summation order exactly.  Per level: c* (cstar_sm) and the first
// discretization OutOfRange (aerr_*), reported in level order by the caller.
template <class DM>
__device__ void s_alloc_concurrent(SCtx& C, int n_levels) {
    const ws_batch& B = *C.B;
    const ws_plan_rec& R = *C.R;
    const int N = C.N, lane = C.lane, K = C.K;
    const int* lb = C.at<int>(C.L->lvl_begin);
    const int* lm = C.at<int>(C.L->lvl_mem);
    const int* level = C.at<int>(C.L->level);
    const int* gm_of = C.at<int>(C.L->gm_of);
    const int* nmax_of = C.at<int>(C.L->nmax_of);
    const int* Lk = C.at<int>(C.L->Lk);
    const DM* valid = C.at<DM>(C.L->valid);
    double* cstar_sm = C.at<double>(C.L->cstar_sm);
    double* aerr_x = C.at<double>(C.L->aerr_x);
    double* aerr_y = C.at<double>(C.L->aerr_y);
    int* aerr = C.at<int>(C.L->aerr);
    const double nd = static_cast<double>(N);
    const FitOut& F = *C.F;
    const bool has = lane < K;
    const int k = has ? lm[lane] : 0;
    const int lv = has ? level[k] : 0;
    const int s0 = has ? lb[lv] : lane;
    const int sw = has ? lb[lv + 1] - lb[lv] : 0;
    int maxw = 0;
    #pragma unroll 1
    for (int l = 0; l < n_levels; ++l) maxw = lb[l + 1] - lb[l] > maxw ? lb[l + 1] - lb[l] : maxw;
    const int gm = has ? gm_of[k] : 0;
    const int L = has ? Lk[k] : 1;
    const double nmax = has ? nmax_of[k] : 1.0;
    InvPre inv;
    if (has) inv.init(F.pieces + 5 * F.piece_off[gm], F.npieces[gm], B.mod_c[gm], B.mod_w[gm], nmax);
    auto seg_sum = [&](double v) {  // ((0 + v_s) + v_s+1) + ... over this lane's segment
        double total = 0.0;
        #pragma unroll 1
        for (int j = 0; j < maxw; ++j) {
            const double x = __shfl_sync(kFull, v, s0 + (j < sw ? j : (sw ? sw - 1 : 0)));
            if (j < sw) total += x;
        }
        return total;
    };
    auto seg_max = [&](double v) {
        double m = 0.0;
        #pragma unroll 1
        for (int j = 0; j < maxw; ++j) {
            const double x = __shfl_sync(kFull, v, s0 + (j < sw ? j : (sw ? sw - 1 : 0)));
            if (j < sw) m = (m < x) ? x : m;
        }
        return m;
    };
    auto probe_term = [&](double cc) {
        const double v = inv(cc / L);
        return (nd < v) ? nd : v;  // std::min(v, N)
    };
    // bracket [max T(min(N,nmax))*L, sum T(1)*L] (allocation.hpp:75-80)
    double lo_t = 0.0, hi_t = 0.0;
    if (has) {
        const double ncap = (nmax < nd) ? nmax : nd;
        lo_t = t_at(F, gm, static_cast<int>(ncap)) * L;
        hi_t = t_at(F, gm, 1) * L;
    }
    double c_lo = seg_max(lo_t);
    double c_hi = seg_sum(hi_t);
    int it = 0;
    bool active = has && it < R.max_iters && (c_hi - c_lo) > R.eps * c_hi;
    while (__any_sync(kFull, active)) {  // allocation.hpp:87-93, every level in its segment
        const double mid = 0.5 * (c_lo + c_hi);
        const double total = seg_sum(has ? probe_term(mid) : 0.0);
        if (active) {
            if (total < nd)
                c_hi = mid;
            else
                c_lo = mid;
            ++it;
        }
        active = has && it < R.max_iters && (c_hi - c_lo) > R.eps * c_hi;
    }
    const double cs = 0.5 * (c_lo + c_hi);
    bool bad = false;
    double ex = 0.0;
    if (has) {
        int un, ul, ln, ll;
        bad = !discretize_one(F, R, gm, L, nmax, valid[k], probe_term(cs), cs, un, ul, ln, ll, ex);
        if (!bad) {
            C.at<int>(C.L->up_n)[k] = un;
            C.at<int>(C.L->up_l)[k] = ul;
            C.at<int>(C.L->lo_n)[k] = ln;
            C.at<int>(C.L->lo_l)[k] = ll;
        }
    }
    // first failing member of each level (segment), recorded by the segment head
    const unsigned eb = __ballot_sync(kFull, bad);
    const unsigned segm = sw ? ((sw >= 32 ? 0xffffffffu : ((1u << sw) - 1u)) << s0) : 0u;
    const unsigned mine = eb & segm;
    const int src = mine ? __ffs(mine) - 1 : lane;
    const double xx = __shfl_sync(kFull, ex, src);
    const double yy = __shfl_sync(kFull, nmax, src);
    if (has && lane == s0) {
        cstar_sm[lv] = cs;
        aerr[lv] = mine ? WS_E_EVAL_RANGE : 0;
        aerr_x[lv] = xx;
        aerr_y[lv] = yy;
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// (4a) wave scheduling of one level (schedule.hpp:49-288)
// ---------------------------------------------------------------------------
template <class DM>
struct SchedViewT {
    int* tk;
    int* tn;
    int* tl;
    int R;
    const int* sumlay;
    const int* idrank;
    const DM* valid;
    int N;
    TErr T;
};
using SchedView = SchedViewT<uint64_t>;

template <class SV>
struct CmpByN {  // schedule.hpp:98-104
    const SV* s;
    __device__ bool operator()(int a, int b) const {
        if (s->tn[a] != s->tn[b]) return s->tn[a] > s->tn[b];
        const double ra = s->tl[a] * s->T(s->tk[a], s->tn[a]);
        const double rb = s->tl[b] * s->T(s->tk[b], s->tn[b]);
        if (ra != rb) return ra > rb;
        return s->idrank[s->tk[a]] < s->idrank[s->tk[b]];
    }
};
template <class SV>
struct CmpByTime {  // schedule.hpp:105-111
    const SV* s;
    __device__ bool operator()(int a, int b) const {
        const double ra = s->sumlay[s->tk[a]] * s->T(s->tk[a], s->tn[a]);
        const double rb = s->sumlay[s->tk[b]] * s->T(s->tk[b], s->tn[b]);
        if (ra != rb) return ra > rb;
        if (s->tn[a] != s->tn[b]) return s->tn[a] > s->tn[b];
        return s->idrank[s->tk[a]] < s->idrank[s->tk[b]];
    }
};
template <class SV>
struct CmpByCheap {  // schedule.hpp:112-118
    const SV* s;
    __device__ bool operator()(int a, int b) const {
        if (s->tn[a] != s->tn[b]) return s->tn[a] < s->tn[b];
        const double ra = s->sumlay[s->tk[a]] * s->T(s->tk[a], s->tn[a]);
        const double rb = s->sumlay[s->tk[b]] * s->T(s->tk[b], s->tn[b]);
        if (ra != rb) return ra > rb;
        return s->idrank[s->tk[a]] < s->idrank[s->tk[b]];
    }
};

// serial path (lane 0): any tuple count, out-of-range-capable curves
template <class DM>
__device__ void ser_extend(const SchedViewT<DM>& S, int* n, const int* sel, int nsel) {  // schedule.hpp:144-173
    while (true) {
        int usedn = 0;
        #pragma unroll 1
        for (int i = 0; i < nsel; ++i) usedn += n[sel[i]];
        const int idle = S.N - usedn;
        if (idle <= 0) break;
        int best = -1, best_next = 0;
        double best_time = -1.0;
        #pragma unroll 1
        for (int i = 0; i < nsel; ++i) {
            const int t = sel[i];
            const int k = S.tk[t];
            const DM above = S.valid[k] & ~dm_first<DM>(n[t]);
            if (!dm_any(above)) continue;
            const int nx = dm_low(above) + 1;
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

template <class DM>
__device__ int ser_greedy(const SchedViewT<DM>& S, const int* order, int* sel) {
    int ns = 0, cap = S.N;
    uint64_t taken = 0;
    #pragma unroll 1
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

// One wave on lane 0: propose (3 exact std::sort emulations), extend, align.
// Fills best[0..nbest) (selection order) and klay[]; returns nbest or -1.
template <class DM>
__device__ int ser_wave(SCtx& C, SchedViewT<DM>& S) {
    int* n2 = C.at<int>(C.L->tn2);
    int* sel = C.at<int>(C.L->sel);
    int* best = C.at<int>(C.L->best);
    int* pool = C.at<int>(C.L->pool);
    int* klay = C.at<int>(C.L->klay);
    double* credit = C.at<double>(C.L->credit);
    const int cap2 = 2 * C.M;
    int* o0 = C.at<int>(C.L->ord);
    int* o1 = o0 + cap2;
    int* o2 = o0 + 2 * cap2;
    const int R = S.R;
    #pragma unroll 1
    for (int i = 0; i < R; ++i) o0[i] = o1[i] = o2[i] = i;
    CmpByN<SchedViewT<DM>> c0{&S};
    ls_sort(o0, R, c0);
    CmpByTime<SchedViewT<DM>> c1{&S};
    ls_sort(o1, R, c1);
    CmpByCheap<SchedViewT<DM>> c2{&S};
    ls_sort(o2, R, c2);
    if (C.ctl->err) return -1;
    int nbest = 0;
    long long best_key = -1;
    for (int o = 0; o < 3; ++o) {
        const int* order = o == 0 ? o0 : (o == 1 ? o1 : o2);
        const int ns = ser_greedy(S, order, sel);
        #pragma unroll 1
        for (int i = 0; i < R; ++i) n2[i] = S.tn[i];
        ser_extend(S, n2, sel, ns);
        if (C.ctl->err) return -1;
        int usedn = 0;
        #pragma unroll 1
        for (int i = 0; i < ns; ++i) usedn += n2[sel[i]];
        const long long key = static_cast<long long>(usedn) * 1000 + ns;
        if (key > best_key) {  // strict: earlier orders win ties
            best_key = key;
            nbest = ns;
            #pragma unroll 1
            for (int i = 0; i < ns; ++i) best[i] = sel[i];
        }
    }
    if (nbest == 0) {
        set_err(C.ctl, WS_E_NO_SCHEDULABLE);
        return -1;
    }
    ser_extend(S, S.tn, best, nbest);
    if (C.ctl->err) return -1;
    // align_time_span (schedule.hpp:190-227)
    double t_wave = 0.0;
    #pragma unroll 1
    for (int i = 0; i < nbest; ++i) {
        const int t = best[i];
        pool[i] = S.sumlay[S.tk[t]];
        const double span = pool[i] * S.T(S.tk[t], S.tn[t]);
        if (i == 0 || span < t_wave) t_wave = span;
    }
    if (C.ctl->err) return -1;
    #pragma unroll 1
    for (int i = 0; i < nbest; ++i) {
        const int t = best[i];
        const int k = S.tk[t];
        const double per = S.T(k, S.tn[t]);
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
    }
    return C.ctl->err ? -1 : nbest;
}

// argmax over candidate lanes of (rem desc, id asc) with single-instruction
// warp reductions: rem > 0, so its IEEE bits order like its value.
__device__ __forceinline__ int warp_argmax_rem(bool cand, double rem, int idr) {
    if (!__any_sync(kFull, cand)) return -1;
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(rem));
    const unsigned hi = cand ? static_cast<unsigned>(bits >> 32) : 0u;
    const unsigned mh = __reduce_max_sync(kFull, hi);
    const bool e1 = cand && hi == mh;
    const unsigned lo = static_cast<unsigned>(bits);
    const unsigned ml = __reduce_max_sync(kFull, e1 ? lo : 0u);
    const bool e2 = e1 && lo == ml;
    const unsigned mi = __reduce_min_sync(kFull, e2 ? static_cast<unsigned>(idr) : 0xffffffffu);
    return __ffs(__ballot_sync(kFull, e2 && static_cast<unsigned>(idr) == mi)) - 1;
}

// extend_resources_if_needed (schedule.hpp:144-173), lanes = selected tuples:
// grow the tuple whose MetaOp has the most remaining time to its next valid
// allocation while idle devices remain.
template <class DM>
__device__ __forceinline__ int ext_lanes(bool in, int n, int N, const DM& vmask, int sl, int idr, const SCtx& C,
                                         int k) {
    const int lane = threadIdx.x & 31;
    while (true) {
        const int idle = N - static_cast<int>(__reduce_add_sync(kFull, in ? static_cast<unsigned>(n) : 0u));
        if (idle <= 0) break;
        bool cand = false;
        int nx = 0;
        double rem = 0.0;
        if (in) {
            const DM above = vmask & ~dm_first<DM>(n);
            if (dm_any(above)) {
                nx = dm_low(above) + 1;
                if (nx - n <= idle) {
                    cand = true;
                    rem = sl * T_of(C, k, n);
                }
            }
        }
        const int win = warp_argmax_rem(cand, rem, idr);
        if (win < 0) break;
        if (lane == win) n = nx;
    }
    return n;
}

// Fast path (R <= 16 tuples, every curve defined up to N): lanes = tuples.
// Stable ranks reproduce std::sort exactly for <= 16 elements (insertion
// sort); greedy runs warp-uniformly; extension/alignment are lane-parallel.
template <class DM>
__device__ int fast_wave(SCtx& C, SchedViewT<DM>& S) {
    const int lane = C.lane, R = S.R, N = S.N;
    const FitOut& F = *C.F;
    const int* gm_of = C.at<int>(C.L->gm_of);
    int* best = C.at<int>(C.L->best);
    int* klay = C.at<int>(C.L->klay);
    double* credit = C.at<double>(C.L->credit);
    int* o0 = C.at<int>(C.L->ord);
    const int cap2 = 2 * C.M;
    const bool mine = lane < R;
    const int k = mine ? S.tk[lane] : 0;
    const int n0 = mine ? S.tn[lane] : 0;
    const int tl = mine ? S.tl[lane] : 0;
    const int sl = mine ? S.sumlay[k] : 0;
    const int idr = mine ? S.idrank[k] : 0;
    const DM vmask = mine ? S.valid[k] : dm_zero<DM>();
    const int gm = mine ? gm_of[k] : 0;
    const double T0 = mine ? T_of(C, k, n0) : 0.0;
    const double tt = tl * T0;  // tuple_time
    const double rt = sl * T0;  // metaop_remaining_time at own n
    // stable ranks under the three comparators
    int p0 = 0, p1 = 0, p2 = 0;
    #pragma unroll 1
    for (int j = 0; j < R; ++j) {
        const int nj = __shfl_sync(kFull, n0, j);
        const double ttj = __shfl_sync(kFull, tt, j);
        const double rtj = __shfl_sync(kFull, rt, j);
        const int idj = __shfl_sync(kFull, idr, j);
        if (!mine || j == lane) continue;
        // comp(j, i) or (j < i and equivalent)
        bool lt0, eq0, lt1, eq1, lt2, eq2;
        if (nj != n0) lt0 = nj > n0, eq0 = false;
        else if (ttj != tt) lt0 = ttj > tt, eq0 = false;
        else lt0 = idj < idr, eq0 = idj == idr;
        if (rtj != rt) lt1 = rtj > rt, eq1 = false;
        else if (nj != n0) lt1 = nj > n0, eq1 = false;
        else lt1 = idj < idr, eq1 = idj == idr;
        if (nj != n0) lt2 = nj < n0, eq2 = false;
        else if (rtj != rt) lt2 = rtj > rt, eq2 = false;
        else lt2 = idj < idr, eq2 = idj == idr;
        p0 += lt0 || (eq0 && j < lane);
        p1 += lt1 || (eq1 && j < lane);
        p2 += lt2 || (eq2 && j < lane);
    }
    if (mine) {
        o0[p0] = lane;
        o0[cap2 + p1] = lane;
        o0[2 * cap2 + p2] = lane;
    }
    __syncwarp();
    // three greedy selections (warp-uniform), scratch extension, keys
    unsigned best_sel = 0;
    int best_cnt = 0;
    long long best_key = -1;
    int my_best_pos = -1;
    for (int o = 0; o < 3; ++o) {
        const int* order = o0 + o * cap2;
        unsigned sel = 0;
        int cap = N, ns = 0, mypos = -1;
        uint64_t taken = 0;
        #pragma unroll 1
        for (int i = 0; i < R; ++i) {
            const int t = order[i];
            const int nt = S.tn[t], kt = S.tk[t];
            if (nt > cap || (taken >> kt & 1ull)) continue;
            sel |= 1u << t;
            taken |= 1ull << kt;
            cap -= nt;
            if (t == lane) mypos = ns;
            ++ns;
        }
        // scratch extension (schedule.hpp:126-131)
        const bool in = (sel >> lane) & 1u;
        const int n = ext_lanes(in, n0, N, vmask, sl, idr, C, k);
        const int usedn = static_cast<int>(__reduce_add_sync(kFull, in ? static_cast<unsigned>(n) : 0u));
        const long long key = static_cast<long long>(usedn) * 1000 + ns;
        if (key > best_key) {
            best_key = key;
            best_sel = sel;
            best_cnt = ns;
            my_best_pos = mypos;
        }
    }
    if (best_cnt == 0) {
        if (lane == 0) set_err(C.ctl, WS_E_NO_SCHEDULABLE);
        __syncwarp();
        return -1;
    }
    // real extension on the chosen set
    const bool in = (best_sel >> lane) & 1u;
    const int n = ext_lanes(in, n0, N, vmask, sl, idr, C, k);
    if (mine) S.tn[lane] = n;
    // align_time_span: t_wave = min span over the chosen set
    const double per = in ? T_of(C, k, n) : 0.0;
    const double span = in ? sl * per : 0.0;
    const double t_wave = warp_min_nonneg(in ? span : __longlong_as_double(0x7ff0000000000000ll));
    if (in) {
        int kk;
        if (sl * per <= t_wave * (1.0 + 1e-12)) {
            kk = sl;
            credit[k] = 0.0;
        } else {
            const double carried = credit[k];
            const double budget = t_wave + ((per < carried) ? per : carried);
            kk = static_cast<int>(floor(budget / per * (1.0 + 1e-12)));
            kk = kk < 1 ? 1 : kk;
            kk = kk < sl ? kk : sl;
            const double rest = budget - kk * per;
            credit[k] = (0.0 < rest) ? rest : 0.0;
        }
        best[my_best_pos] = lane;
        klay[my_best_pos] = kk;
    }
    __syncwarp();
    return best_cnt;
}

// plan_decoupled_sequential (baselines.hpp:104-131): every MetaOp alone on
// its largest valid allocation, one wave each, in lexicographic topological
// order (detail::topo_order, graph.hpp:67-90); lane 0, K <= 64 steps.
template <class DM>
__device__ bool s_decoupled(SCtx& C, char* rec, const RecLayout& RL, int& nW, int& nE, double& end_time, int W_CAP,
                            int E_CAP) {
    const int K = C.K, lane = C.lane;
    const int* by_rank = C.at<int>(C.L->by_rank);
    const int* idrank = C.at<int>(C.L->idrank);
    const int* gm_of = C.at<int>(C.L->gm_of);
    const int* nmax_of = C.at<int>(C.L->nmax_of);
    const int* Lk = C.at<int>(C.L->Lk);
    const int* level = C.at<int>(C.L->level);
    const uint64_t* pred_r = C.at<uint64_t>(C.L->pred_r);
    const uint64_t* succ_r = C.at<uint64_t>(C.L->succ_r);
    const DM* valid = C.at<DM>(C.L->valid);
    int* indeg = C.at<int>(C.L->absorb);
    int* up_n = C.at<int>(C.L->up_n);
    int* up_l = C.at<int>(C.L->up_l);
    int* lo_n = C.at<int>(C.L->lo_n);
    int* lo_l = C.at<int>(C.L->lo_l);
    if (lane == 0) {
        int* w_level = reinterpret_cast<int*>(rec + RL.w_level);
        int* w_eb = reinterpret_cast<int*>(rec + RL.w_eb);
        int* w_ec = reinterpret_cast<int*>(rec + RL.w_ec);
        double* w_start = reinterpret_cast<double*>(rec + RL.w_start);
        double* w_dur = reinterpret_cast<double*>(rec + RL.w_dur);
        int* e_k = reinterpret_cast<int*>(rec + RL.e_k);
        int* e_n = reinterpret_cast<int*>(rec + RL.e_n);
        int* e_l = reinterpret_cast<int*>(rec + RL.e_l);
        double* e_span = reinterpret_cast<double*>(rec + RL.e_span);
        uint64_t ready = 0;
        #pragma unroll 1
        for (int k = 0; k < K; ++k) {
            indeg[k] = popc64(pred_r[k]);
            if (!indeg[k]) ready |= 1ull << idrank[k];
            up_n[k] = up_l[k] = lo_n[k] = lo_l[k] = 0;
        }
        double now = 0.0;
        while (ready) {
            const int r = low_bit(ready);
            ready &= ready - 1;
            const int k = by_rank[r];
            const int gm = gm_of[k];
            const int tp = C.B->mod_tp[gm];
            if (tp > C.N) {  // valid_allocations (allocation.hpp:51-54)
                set_err(C.ctl, WS_E_TP_EXCEEDS, k, tp);
                break;
            }
            const int n = dm_high(valid[k]) + 1;  // valid.back()
            if (n > nmax_of[k]) {  // ScalingCurve::eval OutOfRange (scaling.hpp:66-68)
                C.ctl->err = WS_E_EVAL_RANGE;
                C.ctl->x = n;
                C.ctl->y = nmax_of[k];
                break;
            }
            if (nW + 1 > W_CAP || nE + 1 > E_CAP) {
                set_err(C.ctl, nW + 1 > W_CAP ? WS_E_LIMIT_WAVES : WS_E_LIMIT_ENTRIES);
                break;
            }
            const double span = Lk[k] * t_at(*C.F, gm, n);
            w_level[nW] = level[k];
            w_eb[nW] = nE;
            w_ec[nW] = 1;
            w_start[nW] = now;
            w_dur[nW] = span;
            e_k[nE] = k;
            e_n[nE] = n;
            e_l[nE] = Lk[k];
            e_span[nE] = span;
            up_n[k] = n;
            up_l[k] = Lk[k];
            ++nW;
            ++nE;
            now += span;
            #pragma unroll 1
            for (uint64_t sr = succ_r[k]; sr; sr &= sr - 1) {
                const int q = by_rank[low_bit(sr)];
                if (--indeg[q] == 0) ready |= 1ull << idrank[q];
            }
        }
        end_time = now;
        C.ctl->i2 = nW;
        C.ctl->i3 = nE;
    }
    __syncwarp();
    nW = C.ctl->i2;
    nE = C.ctl->i3;
    end_time = __shfl_sync(kFull, end_time, 0);
    return C.ctl->err == 0;
}

// (4a) schedule_level + merge_levels offsets; appends waves/entries to the record
template <class DM>
__device__ bool s_schedule_level(SCtx& C, char* rec, const RecLayout& RL, int lvl, int& nW, int& nE,
                                 double offset, double& level_end, int W_CAP, int E_CAP) {
    const int lane = C.lane;
    const int* lb = C.at<int>(C.L->lvl_begin);
    const int* lm = C.at<int>(C.L->lvl_mem) + lb[lvl];
    const int w = lb[lvl + 1] - lb[lvl];
    const int* up_n = C.at<int>(C.L->up_n);
    const int* up_l = C.at<int>(C.L->up_l);
    const int* lo_n = C.at<int>(C.L->lo_n);
    const int* lo_l = C.at<int>(C.L->lo_l);
    const int* nmax_of = C.at<int>(C.L->nmax_of);
    int* sumlay = C.at<int>(C.L->sumlay);
    double* credit = C.at<double>(C.L->credit);
    int* best = C.at<int>(C.L->best);
    int* klay = C.at<int>(C.L->klay);
    int* absorb = C.at<int>(C.L->absorb);
    SchedViewT<DM> S;
    S.tk = C.at<int>(C.L->tk);
    S.tn = C.at<int>(C.L->tn);
    S.tl = C.at<int>(C.L->tl);
    S.sumlay = sumlay;
    S.idrank = C.at<int>(C.L->idrank);
    S.valid = C.at<DM>(C.L->valid);
    S.N = C.N;
    S.T = TErr{C.F, C.at<int>(C.L->gm_of), nmax_of, C.ctl, C.kscale, C.B};
    int* w_level = reinterpret_cast<int*>(rec + RL.w_level);
    int* w_eb = reinterpret_cast<int*>(rec + RL.w_eb);
    int* w_ec = reinterpret_cast<int*>(rec + RL.w_ec);
    double* w_start = reinterpret_cast<double*>(rec + RL.w_start);
    double* w_dur = reinterpret_cast<double*>(rec + RL.w_dur);
    int* e_k = reinterpret_cast<int*>(rec + RL.e_k);
    int* e_n = reinterpret_cast<int*>(rec + RL.e_n);
    int* e_l = reinterpret_cast<int*>(rec + RL.e_l);
    double* e_span = reinterpret_cast<double*>(rec + RL.e_span);
    // remaining tuples in id order: upper then lower (schedule.hpp:236-240)
    int R = 0;
    bool all_defined = true;
    if (lane == 0) {
        #pragma unroll 1
        for (int i = 0; i < w; ++i) {
            const int k = lm[i];
            S.tk[R] = k, S.tn[R] = up_n[k], S.tl[R] = up_l[k], ++R;
            if (lo_l[k]) S.tk[R] = k, S.tn[R] = lo_n[k], S.tl[R] = lo_l[k], ++R;
            credit[k] = 0.0;
            absorb[k] = 0;
        }
        C.ctl->i2 = R;
    }
    #pragma unroll 1
    for (int i = lane; i < w; i += 32) all_defined &= nmax_of[lm[i]] >= C.N;
    all_defined = __all_sync(kFull, all_defined);
    __syncwarp();
    R = C.ctl->i2;
    double now = 0.0;
    while (R > 0) {
        S.R = R;
        // layers each MetaOp still owes (schedule.hpp:49-61)
        if (lane == 0) {
            #pragma unroll 1
            for (int i = 0; i < R; ++i) sumlay[S.tk[i]] = 0;
            #pragma unroll 1
            for (int i = 0; i < R; ++i) sumlay[S.tk[i]] += S.tl[i];
        }
        __syncwarp();
        int nbest;
        if (all_defined && R <= 16) {
            nbest = fast_wave(C, S);
        } else {
            if (lane == 0) C.ctl->i3 = ser_wave(C, S);
            __syncwarp();
            nbest = C.ctl->i3;
        }
        if (nbest < 0 || C.ctl->err) return false;
        if (nW + 1 > W_CAP || nE + nbest > E_CAP) {
            if (lane == 0) set_err(C.ctl, nW + 1 > W_CAP ? WS_E_LIMIT_WAVES : WS_E_LIMIT_ENTRIES);
            __syncwarp();
            return false;
        }
        // wave entries in selection order; duration = max span
        double span = 0.0;
        if (lane < nbest) {
            const int t = best[lane];
            const int k = S.tk[t];
            const int kk = klay[lane];
            span = kk * T_of(C, k, S.tn[t]);
            e_k[nE + lane] = k;
            e_n[nE + lane] = S.tn[t];
            e_l[nE + lane] = kk;
            e_span[nE + lane] = span;
            // bookkeeping: own tuple pays its layers, the sibling covers the absorbed rest
            int ab = kk - S.tl[t];
            ab = ab > 0 ? ab : 0;
            S.tl[t] -= kk - ab;
            absorb[k] = ab;
        }
        const double dur = warp_max_nonneg(span);
        if (lane == 0) {
            w_level[nW] = lvl;
            w_eb[nW] = nE;
            w_ec[nW] = nbest;
            w_start[nW] = now + offset;  // merge_levels offset (schedule.hpp:292-309)
            w_dur[nW] = dur;
        }
        ++nW;
        nE += nbest;
        now += dur;
        __syncwarp();
        // the sibling tuple (same MetaOp, not selected) gives up the absorbed layers
        #pragma unroll 1
        for (int j = lane; j < R; j += 32) {
            const int kj = S.tk[j];
            const int ab = absorb[kj];
            bool selected = false;
            #pragma unroll 1
            for (int i = 0; i < nbest; ++i) selected |= best[i] == j;
            if (ab > 0 && !selected) {
                const int take = ab < S.tl[j] ? ab : S.tl[j];
                S.tl[j] -= take;
            }
        }
        __syncwarp();
        #pragma unroll 1
        for (int i = lane; i < nbest; i += 32) absorb[S.tk[best[i]]] = 0;
        __syncwarp();
        // compact the remaining tuples (order kept)
        if (lane == 0) {
            int R2 = 0;
            #pragma unroll 1
            for (int i = 0; i < R; ++i)
                if (S.tl[i] > 0) S.tk[R2] = S.tk[i], S.tn[R2] = S.tn[i], S.tl[R2] = S.tl[i], ++R2;
            if (R2 == R) set_err(C.ctl, WS_E_NO_PROGRESS);
            C.ctl->i2 = R2;
        }
        __syncwarp();
        if (C.ctl->err) return false;
        R = C.ctl->i2;
    }
    // merge_levels: level end = max over its waves of start + duration
    double le = offset;
    #pragma unroll 1
    for (int i = lane; i < nW; i += 32)
        if (w_level[i] == lvl) {
            const double e = w_start[i] + w_dur[i];
            le = (le < e) ? e : le;
        }
    level_end = warp_max_nonneg(le);
    return true;
}

// WS_SCHED_MINB: optional resident-blocks target for register tuning builds
// ScalingCurve::eval_batch_fraction (scaling.hpp:83-86) of a fitted module curve
__device__ __forceinline__ double eval_bf_fit(const FitOut& F, const ws_batch& B, int gm, double n, double frac) {
    const double* pc = F.pieces + 5 * F.piece_off[gm];
    const int np = F.npieces[gm];
    int i = 0;
    if (!(n < 1.0)) {
        const double nmax = __ldg(pc + 5 * (np - 1) + 1);
        const double x = n < nmax ? n : nmax;  // locate(std::min(n, n_max_))
        while (i < np - 1 && !(x <= __ldg(pc + 5 * i + 1) + 1e-9)) ++i;
    }
    return __ldg(pc + 5 * i + 2) + __ldg(pc + 5 * i + 3) * B.mod_c[gm] + __ldg(pc + 5 * i + 4) * B.mod_w[gm] * frac / n;
}

// plan_task_level_optimus (baselines.hpp:133-321), on lane 0: per task the
// valid allocations common to its MetaOps, tasks packed into batches by their
// smallest allocation, marginal-gain growth of each task's block (critical
// path of the task's sub-DAG at eval_batch_fraction), every MetaOp one wave on
// the whole block, waves indexed by (start, entity id), one placement group
// (device block + waves) per task.
template <class DM>
__device__ bool s_optimus(SCtx& C, char* rec, const RecLayout& RL, int& nW, int& nE, double& end_time, int W_CAP,
                          int E_CAP, int& KE_out, int& npg_out) {
    const ws_batch& B = *C.B;
    const ws_plan_rec& R = *C.R;
    const FitOut& F = *C.F;
    const int K = C.K, N = C.N, lane = C.lane, T = R.n_tasks;
    const int* by_rank = C.at<int>(C.L->by_rank);
    const int* idrank = C.at<int>(C.L->idrank);
    const int* gm_of = C.at<int>(C.L->gm_of);
    const int* Lk = C.at<int>(C.L->Lk);
    const int* level = C.at<int>(C.L->level);
    const int* mod_of = C.at<int>(C.L->mod_of);
    const uint64_t* pred_r = C.at<uint64_t>(C.L->pred_r);
    const uint64_t* succ_r = C.at<uint64_t>(C.L->succ_r);
    const DM* valid = C.at<DM>(C.L->valid);
    const uint64_t* tmask = C.at<uint64_t>(C.L->tmask);
    int* ent_met = C.at<int>(C.L->ent_met);
    int* ent_task = C.at<int>(C.L->ent_task);
    double* ent_frac = C.at<double>(C.L->ent_frac);
    uint64_t* epred = C.at<uint64_t>(C.L->epred);
    int* ent_of = C.at<int>(C.L->ent_of);
    int* vord = C.at<int>(C.L->vord);
    int* indeg = C.at<int>(C.L->absorb);
    DM* tvalid = C.at<DM>(C.L->tvalid);
    int* talloc = C.at<int>(C.L->talloc);
    double* cw_start = C.at<double>(C.L->cw_start);
    double* cw_dur = C.at<double>(C.L->cw_dur);
    int* cw_level = C.at<int>(C.L->cw_level);
    int* cw_ent = C.at<int>(C.L->cw_ent);
    int* cw_n = C.at<int>(C.L->cw_n);
    int* cw_L = C.at<int>(C.L->cw_L);
    int* pl_off = C.at<int>(C.L->pl_off);
    int* pl_cnt = C.at<int>(C.L->pl_cnt);
    int* pl_wbeg = C.at<int>(C.L->pl_wbeg);
    int* pl_wn = C.at<int>(C.L->pl_wn);
    int* perm = C.at<int>(C.L->perm);
    double* tfin = C.at<double>(C.L->tfin);
    double* tcur = C.at<double>(C.L->tcur);
    double* tnext = C.at<double>(C.L->tnext);
    int* tnxn = C.at<int>(C.L->tnxn);
    int KE = 0, ncw = 0, npl = 0;
    #pragma unroll 1
    for (int e = lane; e < WS_MAX_MODULES; e += 32) epred[e] = 0;
    __syncwarp();
    if (lane == 0) {
        auto members = [&](int t) {  // id-rank mask of the task's MetaOps
            const int tr = B.task_rank[R.task_begin + t];
            uint64_t m = 0;
            #pragma unroll 1
            for (int k = 0; k < K; ++k)
                if (tmask[mod_of[k]] >> tr & 1ull) m |= 1ull << idrank[k];
            return m;
        };
        auto task_order = [&](uint64_t memr) {  // detail::topo_order over the task view -> vord
            int n = 0;
            uint64_t ready = 0;
            #pragma unroll 1
            for (uint64_t b = memr; b; b &= b - 1) {
                const int k = by_rank[low_bit(b)];
                indeg[k] = popc64(pred_r[k] & memr);
                if (!indeg[k]) ready |= 1ull << idrank[k];
            }
            while (ready) {
                const int r = low_bit(ready);
                ready &= ready - 1;
                const int k = by_rank[r];
                vord[n++] = k;
                #pragma unroll 1
                for (uint64_t sr = succ_r[k] & memr; sr; sr &= sr - 1) {
                    const int q = by_rank[low_bit(sr)];
                    if (--indeg[q] == 0) ready |= 1ull << idrank[q];
                }
            }
            return n;
        };
        auto frac_of = [&](int k) { return 1.0 / static_cast<double>(popc64(tmask[mod_of[k]])); };
        auto task_time = [&](int t, int n) {  // critical path of the task at allocation n
            const uint64_t memr = members(t);
            const int nm = task_order(memr);
            double total = 0.0;
            #pragma unroll 1
            for (int i = 0; i < nm; ++i) {
                const int k = vord[i];
                const double weight = Lk[k] * eval_bf_fit(F, B, gm_of[k], static_cast<double>(n), frac_of(k));
                double start = 0.0;
                #pragma unroll 1
                for (uint64_t p = pred_r[k] & memr; p; p &= p - 1) {
                    const double f = tfin[by_rank[low_bit(p)]];
                    start = start < f ? f : start;
                }
                tfin[k] = start + weight;
                total = total < tfin[k] ? tfin[k] : total;
            }
            return total;
        };
        #pragma unroll 1
        for (int t = 0; t < T && !C.ctl->err; ++t) {  // common valid allocations (valid_allocations per n)
            const int nm = task_order(members(t));
            DM tv = dm_zero<DM>();
            #pragma unroll 1
            for (int n = 1; n <= N && !C.ctl->err; ++n) {
                bool ok = true;
                #pragma unroll 1
                for (int i = 0; i < nm; ++i) {
                    const int k = vord[i];
                    const int tp = B.mod_tp[gm_of[k]];
                    if (tp > N) {
                        set_err(C.ctl, WS_E_TP_EXCEEDS, k, tp);
                        break;
                    }
                    if (!dm_test(valid[k], n - 1)) {
                        ok = false;
                        break;
                    }
                }
                if (ok && !C.ctl->err) tv |= dm_bit<DM>(n - 1);
            }
            if (!C.ctl->err && !dm_any(tv)) set_err(C.ctl, WS_E_TASK_NO_VALID, t);
            tvalid[t] = tv;
        }
        double batch_offset = 0.0;
        #pragma unroll 1
        for (int b0 = 0; b0 < T && !C.ctl->err;) {  // batches whose minimum allocations fit
            int b1 = b0, used = 0;
            while (b1 < T) {
                const int need = dm_low(tvalid[b1]) + 1;
                if (used + need > N && b1 > b0) break;
                used += need;
                ++b1;
            }
            // task_time(t, n) is a pure function of (t, n): each task's time at its
            // current and at its next allocation is cached and only the grown
            // task's entries are recomputed (the reference re-evaluates both for
            // every task at every step; the values, hence the gains, are identical)
            #pragma unroll 1
            for (int t = b0; t < b1; ++t) {
                talloc[t] = dm_low(tvalid[t]) + 1;
                tcur[t] = -1.0;
                tnxn[t] = -1;
            }
            while (true) {  // marginal gain per added device
                int usedn = 0;
                #pragma unroll 1
                for (int t = b0; t < b1; ++t) usedn += talloc[t];
                const int free = N - usedn;
                if (free <= 0) break;
                int best = -1, best_next = 0;
                double best_gain = -1.0;
                #pragma unroll 1
                for (int t = b0; t < b1; ++t) {
                    const DM above = tvalid[t] & ~dm_first<DM>(talloc[t]);  // std::upper_bound
                    if (!dm_any(above)) continue;
                    const int nx = dm_low(above) + 1;
                    if (nx - talloc[t] > free) continue;
                    if (tcur[t] < 0.0) tcur[t] = task_time(t, talloc[t]);
                    if (tnxn[t] != nx) {
                        tnext[t] = task_time(t, nx);
                        tnxn[t] = nx;
                    }
                    const double gain = (tcur[t] - tnext[t]) / (nx - talloc[t]);
                    if (gain > best_gain) {
                        best_gain = gain;
                        best = t;
                        best_next = nx;
                    }
                }
                if (best < 0) break;
                talloc[best] = best_next;
                tcur[best] = tnext[best];  // == task_time(best, best_next)
                tnxn[best] = -1;
            }
            double batch_end = batch_offset;
            int cursor = 0;
            #pragma unroll 1
            for (int t = b0; t < b1 && !C.ctl->err; ++t) {
                const uint64_t memr = members(t);
                const int nm = task_order(memr);
                pl_off[npl] = cursor;
                pl_cnt[npl] = talloc[t];
                pl_wbeg[npl] = ncw;
                cursor += talloc[t];
                double now = batch_offset;
                #pragma unroll 1
                for (int i = 0; i < nm; ++i) {
                    const int k = vord[i];
                    if (KE >= WS_MAX_MODULES || ncw >= WS_MAX_MODULES) {
                        set_err(C.ctl, WS_E_LIMIT_MODULES);
                        break;
                    }
                    ent_met[KE] = k;
                    ent_task[KE] = t;
                    ent_frac[KE] = frac_of(k);  // share_fraction
                    ent_of[k] = KE;
                    const double span = Lk[k] * eval_bf_fit(F, B, gm_of[k], talloc[t], ent_frac[KE]);
                    cw_start[ncw] = now;
                    cw_dur[ncw] = span;
                    cw_level[ncw] = level[k];
                    cw_ent[ncw] = KE;
                    cw_n[ncw] = talloc[t];
                    cw_L[ncw] = Lk[k];
                    ++ncw;
                    ++KE;
                    now += span;
                }
                pl_wn[npl] = ncw - pl_wbeg[npl];
                ++npl;
                #pragma unroll 1
                for (int i = 0; i < nm; ++i) {  // the task's edges between its entities (deps, scoped)
                    const int k = vord[i];
                    #pragma unroll 1
                    for (uint64_t pr = pred_r[k] & memr; pr; pr &= pr - 1)
                        epred[ent_of[k]] |= 1ull << ent_of[by_rank[low_bit(pr)]];
                }
                batch_end = batch_end < now ? now : batch_end;
            }
            batch_offset = batch_end;
            b0 = b1;
        }
        if (!C.ctl->err && (ncw > W_CAP || ncw > E_CAP))
            set_err(C.ctl, ncw > W_CAP ? WS_E_LIMIT_WAVES : WS_E_LIMIT_ENTRIES);
        if (!C.ctl->err) {
            auto wless = [&](int a, int b) {  // (start, id of the wave's entry)
                if (cw_start[a] != cw_start[b]) return cw_start[a] < cw_start[b];
                const int ea = cw_ent[a], eb = cw_ent[b];
                return scoped_less(ent_met[ea], B.task_rank[R.task_begin + ent_task[ea]], ent_met[eb],
                                   B.task_rank[R.task_begin + ent_task[eb]]);
            };
            #pragma unroll 1
            for (int i = 0; i < ncw; ++i) {  // insertion sort (a strict total order: stable or not alike)
                const int v = i;
                int j = i;
                while (j > 0 && wless(v, perm[j - 1])) perm[j] = perm[j - 1], --j;
                perm[j] = v;
            }
            int* w_level = reinterpret_cast<int*>(rec + RL.w_level);
            int* w_eb = reinterpret_cast<int*>(rec + RL.w_eb);
            int* w_ec = reinterpret_cast<int*>(rec + RL.w_ec);
            double* w_start = reinterpret_cast<double*>(rec + RL.w_start);
            double* w_dur = reinterpret_cast<double*>(rec + RL.w_dur);
            int* e_k = reinterpret_cast<int*>(rec + RL.e_k);
            int* e_n = reinterpret_cast<int*>(rec + RL.e_n);
            int* e_l = reinterpret_cast<int*>(rec + RL.e_l);
            double* e_span = reinterpret_cast<double*>(rec + RL.e_span);
            double end = 0.0;
            #pragma unroll 1
            for (int i = 0; i < ncw; ++i) {
                const int c = perm[i];
                w_level[i] = cw_level[c];
                w_eb[i] = i;
                w_ec[i] = 1;
                w_start[i] = cw_start[c];
                w_dur[i] = cw_dur[c];
                e_k[i] = cw_ent[c];
                e_n[i] = cw_n[c];
                e_l[i] = cw_L[c];
                e_span[i] = cw_dur[c];
                const double fin = cw_start[c] + cw_dur[c];
                end = end < fin ? fin : end;
            }
            end_time = end;
            int* pg_off = reinterpret_cast<int*>(rec + RL.pg_off);
            int* pg_cnt = reinterpret_cast<int*>(rec + RL.pg_cnt);
            int* pg_wbeg = reinterpret_cast<int*>(rec + RL.pg_wbeg);
            int* pg_wn = reinterpret_cast<int*>(rec + RL.pg_wn);
            int* pg_list = reinterpret_cast<int*>(rec + RL.pg_list);
            #pragma unroll 1
            for (int i = 0; i < ncw; ++i) pg_list[perm[i]] = i;  // created wave -> global index
            #pragma unroll 1
            for (int q = 0; q < npl; ++q) {  // pg_list[created wave] = its global index
                pg_off[q] = pl_off[q];
                pg_cnt[q] = pl_cnt[q];
                pg_wbeg[q] = pl_wbeg[q];
                pg_wn[q] = pl_wn[q];
            }
        }
    }
    __syncwarp();
    if (C.ctl->err) return false;
    nW = nE = __shfl_sync(kFull, ncw, 0);
    KE_out = __shfl_sync(kFull, KE, 0);
    npg_out = __shfl_sync(kFull, npl, 0);
    end_time = __shfl_sync(kFull, end_time, 0);
    return true;
}

// plan_distmm_mt (baselines.hpp:323-413): tasks in declaration order; inside
// a task (task_view: members, in-task edges, lexicographic topological order,
// longest-path task levels), a level of one MetaOp runs alone on its largest
// valid allocation, a wider level splits the cluster through the level
// machinery (s_level_alloc + s_schedule_level) on curves whose per-device term
// is scaled by the share fraction 1/|tasks|; entities are (MetaOp, task) pairs.
template <class DM>
__device__ bool s_distmm(SCtx& C, char* rec, const RecLayout& RL, int& nW, int& nE, double& end_time, int W_CAP,
                         int E_CAP, int& KE_out) {
    const ws_batch& B = *C.B;
    const ws_plan_rec& R = *C.R;
    const int K = C.K, N = C.N, lane = C.lane;
    const int* by_rank = C.at<int>(C.L->by_rank);
    const int* idrank = C.at<int>(C.L->idrank);
    const int* gm_of = C.at<int>(C.L->gm_of);
    const int* nmax_of = C.at<int>(C.L->nmax_of);
    const int* Lk = C.at<int>(C.L->Lk);
    const int* mod_of = C.at<int>(C.L->mod_of);
    const uint64_t* pred_r = C.at<uint64_t>(C.L->pred_r);
    const DM* valid = C.at<DM>(C.L->valid);
    const uint64_t* tmask = C.at<uint64_t>(C.L->tmask);
    int* ent_met = C.at<int>(C.L->ent_met);
    int* ent_task = C.at<int>(C.L->ent_task);
    double* ent_frac = C.at<double>(C.L->ent_frac);
    uint64_t* epred = C.at<uint64_t>(C.L->epred);
    int* ent_of = C.at<int>(C.L->ent_of);
    double* kscale = C.at<double>(C.L->kscale);
    int* tlvl = C.at<int>(C.L->tlvl);
    int* vord = C.at<int>(C.L->vord);
    int* lb = C.at<int>(C.L->lvl_begin);
    int* lm = C.at<int>(C.L->lvl_mem);
    int* w_level = reinterpret_cast<int*>(rec + RL.w_level);
    int* w_eb = reinterpret_cast<int*>(rec + RL.w_eb);
    int* w_ec = reinterpret_cast<int*>(rec + RL.w_ec);
    double* w_start = reinterpret_cast<double*>(rec + RL.w_start);
    double* w_dur = reinterpret_cast<double*>(rec + RL.w_dur);
    int* e_k = reinterpret_cast<int*>(rec + RL.e_k);
    int* e_n = reinterpret_cast<int*>(rec + RL.e_n);
    int* e_l = reinterpret_cast<int*>(rec + RL.e_l);
    double* e_span = reinterpret_cast<double*>(rec + RL.e_span);
    int KE = 0;
    double now = 0.0;
    #pragma unroll 1
    for (int e = lane; e < WS_MAX_MODULES; e += 32) epred[e] = 0;
    #pragma unroll 1
    for (int t = 0; t < R.n_tasks; ++t) {
        const int tr = B.task_rank[R.task_begin + t];
        int nm = 0, maxl = 0;
        if (lane == 0) {  // task_view (baselines.hpp:62-73): members in topological order, task levels
            uint64_t memr = 0;  // members as id-rank bits
            #pragma unroll 1
            for (int k = 0; k < K; ++k) {
                ent_of[k] = -1;
                if (tmask[mod_of[k]] >> tr & 1ull) memr |= 1ull << idrank[k];
            }
            int* indeg = C.at<int>(C.L->absorb);
            uint64_t ready = 0;
            #pragma unroll 1
            for (uint64_t b = memr; b; b &= b - 1) {
                const int k = by_rank[low_bit(b)];
                indeg[k] = popc64(pred_r[k] & memr);
                if (!indeg[k]) ready |= 1ull << idrank[k];
            }
            const uint64_t* succ_r = C.at<uint64_t>(C.L->succ_r);
            while (ready) {
                const int r = low_bit(ready);
                ready &= ready - 1;
                const int k = by_rank[r];
                vord[nm++] = k;
                int lv = 0;
                #pragma unroll 1
                for (uint64_t p = pred_r[k] & memr; p; p &= p - 1) {
                    const int q = tlvl[by_rank[low_bit(p)]] + 1;
                    lv = q > lv ? q : lv;
                }
                tlvl[k] = lv;
                maxl = lv > maxl ? lv : maxl;
                #pragma unroll 1
                for (uint64_t sr = succ_r[k] & memr; sr; sr &= sr - 1) {
                    const int q = by_rank[low_bit(sr)];
                    if (--indeg[q] == 0) ready |= 1ull << idrank[q];
                }
            }
        }
        nm = __shfl_sync(kFull, nm, 0);
        maxl = __shfl_sync(kFull, maxl, 0);
        __syncwarp();
        #pragma unroll 1
        for (int l = 0; l <= maxl; ++l) {
            int w = 0;
            if (lane == 0) {  // the level's MetaOps in task order; their entities and scaled curves
                #pragma unroll 1
                for (int i = 0; i < nm; ++i) {
                    const int k = vord[i];
                    if (tlvl[k] != l) continue;
                    lm[w++] = k;
                    if (ent_of[k] < 0) {
                        if (KE >= WS_MAX_MODULES) {
                            set_err(C.ctl, WS_E_LIMIT_MODULES);
                            break;
                        }
                        ent_met[KE] = k;
                        ent_task[KE] = t;
                        ent_frac[KE] = 1.0 / static_cast<double>(popc64(tmask[mod_of[k]]));  // share_fraction
                        ent_of[k] = KE++;
                    }
                    kscale[k] = ent_frac[ent_of[k]];
                    const int tp = B.mod_tp[gm_of[k]];
                    if (tp > N) {  // valid_allocations (allocation.hpp:51-54)
                        set_err(C.ctl, WS_E_TP_EXCEEDS, k, tp);
                        break;
                    }
                }
                lb[0] = 0;
                lb[1] = w;
            }
            w = __shfl_sync(kFull, w, 0);
            KE = __shfl_sync(kFull, KE, 0);
            __syncwarp();
            if (C.ctl->err) return false;
            if (w == 0) continue;
            if (w == 1) {
                if (lane == 0) {
                    const int k = lm[0];
                    const int n = dm_high(valid[k]) + 1;  // valid.back()
                    if (n > nmax_of[k]) {  // scaled.eval(n) OutOfRange (scaling.hpp:66-68)
                        C.ctl->err = WS_E_EVAL_RANGE;
                        C.ctl->x = n;
                        C.ctl->y = nmax_of[k];
                    } else if (nW + 1 > W_CAP || nE + 1 > E_CAP) {
                        set_err(C.ctl, nW + 1 > W_CAP ? WS_E_LIMIT_WAVES : WS_E_LIMIT_ENTRIES);
                    } else {
                        const double span = Lk[k] * t_scaled(*C.F, B, gm_of[k], n, kscale[k]);
                        w_level[nW] = l;
                        w_eb[nW] = nE;
                        w_ec[nW] = 1;
                        w_start[nW] = now;
                        w_dur[nW] = span;
                        e_k[nE] = ent_of[k];
                        e_n[nE] = n;
                        e_l[nE] = Lk[k];
                        e_span[nE] = span;
                        now += span;
                    }
                }
                __syncwarp();
                if (C.ctl->err) return false;
                ++nW;
                ++nE;
                continue;
            }
            C.kscale = kscale;
            double cs = 0.0;
            bool ok = s_level_alloc<DM>(C, 0, cs);  // sums in task order (LevelInput order)
            if (ok) {
                if (lane == 0)  // discretized tuples / schedule_level go by MetaOp id
                    #pragma unroll 1
                    for (int i = 1; i < w; ++i) {
                        const int v = lm[i];
                        int j = i;
                        while (j > 0 && idrank[lm[j - 1]] > idrank[v]) lm[j] = lm[j - 1], --j;
                        lm[j] = v;
                    }
                __syncwarp();
                const int w0 = nW, e0 = nE;
                double level_end = now;
                ok = s_schedule_level<DM>(C, rec, RL, 0, nW, nE, now, level_end, W_CAP, E_CAP);
                if (ok && lane == 0) {
                    double t_end = 0.0;  // schedule_level's own clock, from 0
                    #pragma unroll 1
                    for (int x = w0; x < nW; ++x) {
                        w_level[x] = l;
                        t_end += w_dur[x];
                    }
                    #pragma unroll 1
                    for (int x = e0; x < nE; ++x) e_k[x] = ent_of[e_k[x]];
                    now += t_end;
                }
            }
            C.kscale = nullptr;
            now = __shfl_sync(kFull, now, 0);
            __syncwarp();
            if (!ok) return false;
        }
        if (lane == 0)  // the task's edges between its entities (deps, scoped)
            #pragma unroll 1
            for (int i = 0; i < nm; ++i) {
                const int k = vord[i];
                const uint64_t* succ_r = C.at<uint64_t>(C.L->succ_r);
                #pragma unroll 1
                for (uint64_t sr = succ_r[k]; sr; sr &= sr - 1) {
                    const int q = by_rank[low_bit(sr)];
                    if (ent_of[q] >= 0) epred[ent_of[q]] |= 1ull << ent_of[k];
                }
            }
        __syncwarp();
    }
    end_time = now;
    KE_out = KE;
    return true;
}

// One warp per plan.  SCOPED: the kernel instance for the task-scoped
// baselines (distmm-mt); the planner's instance carries none of that code, so
// its register allocation and instruction stream stay those of the planner.
// Warp copy of a slot's shared working set to / from its global state slot
// (16-byte words; SL.bytes is a multiple of 16) plus the control block and
// the flags that live in registers between the phases.
// Bytes of the working set that travel from phase 1 to phase 3: the layout's
// leading part, up to the phase-1 scratch (make_sm_layout).
__host__ __device__ inline int sched_state_bytes(const SmLayout& L) { return (L.adj + 15) & ~15; }

// Shared bytes per warp a k_sched kernel needs: phase 1 works below the
// wave-scheduling scratch, phase 2 inside the persistent part, phase 3 (and
// the unsplit kernel) on the whole layout.  Smaller phase kernels fit more
// blocks per SM where shared memory is their occupancy limit.
__host__ __device__ inline int sched_phase_bytes(const SmLayout& L, int phase) {
    return phase == 1 ? ((L.tk + 15) & ~15) : phase == 2 ? sched_state_bytes(L) : L.bytes;
}

// The state slot's header: the warp's Ctl, the plan's ok flag and MetaOp count.
__device__ __forceinline__ void sched_state_hdr(bool save, char* g, Ctl* ctl, int& ok, int& K, int lane) {
    int* flags = reinterpret_cast<int*>(g + sizeof(Ctl));
    if (save) {
        if (lane == 0) {
            *reinterpret_cast<Ctl*>(g) = *ctl;
            flags[0] = ok;
            flags[1] = K;
        }
    } else {
        if (lane == 0) *ctl = *reinterpret_cast<const Ctl*>(g);
        ok = flags[0];
        K = flags[1];
    }
    __syncwarp();
}

__device__ __forceinline__ void sched_state_io(bool save, char* g, char* sm, int bytes, Ctl* ctl, int& ok, int& K,
                                               int lane) {
    int4* gs = reinterpret_cast<int4*>(g + kSchedStateHdr);
    int4* ss = reinterpret_cast<int4*>(sm);
    if (save) {
        #pragma unroll 1
        for (int i = lane; i < bytes / 16; i += 32) gs[i] = ss[i];
    } else {
        // restore with cp.async: every 16-byte chunk in flight at once instead
        // of one global-load round trip per loop iteration
        #pragma unroll 1
        for (int i = lane; i < bytes / 16; i += 32) {
            const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(ss + i));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gs + i) : "memory");
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    }
    sched_state_hdr(save, g, ctl, ok, K, lane);
}

// Bytes [lo, hi) of the working set (8-byte aligned layout offsets) to / from
// the plan's state slot; restores are cp.async, waited for by sched_span_wait.
__device__ __forceinline__ void sched_span_io(bool save, char* g, char* sm, int lo, int hi, int lane) {
    uint64_t* gs = reinterpret_cast<uint64_t*>(g + kSchedStateHdr + lo);
    uint64_t* ss = reinterpret_cast<uint64_t*>(sm + lo);
    const int n = (hi - lo) / 8;
    if (save) {
        #pragma unroll 1
        for (int i = lane; i < n; i += 32) gs[i] = ss[i];
    } else {
        #pragma unroll 1
        for (int i = lane; i < n; i += 32) {
            const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(ss + i));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(gs + i) : "memory");
        }
    }
}
__device__ __forceinline__ void sched_span_wait() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncwarp();
}

// PHASE 0: the whole k_sched in one kernel.  Phase-split launches (large
// batches): 1 = graph, contraction, levels, fit status, valid sets; 2 = the
// concurrent bisection + discretization of every level; 3 = repair, wave
// scheduling, the baselines and the hand-off record.  Each phase kernel
// carries only its own code, so the warps resident on an SM share a much
// smaller hot instruction footprint (the monolithic kernel's executed code is
// ~70 KB against a 32 KB L1.5 instruction cache: ncu showed "no instruction"
// as the largest stall).
template <bool SCOPED, class DM = uint64_t, int PHASE = 0>
__device__ __forceinline__ void sched_body(const SchedArgs& A, char* smem_dyn, Ctl* ctl_s) {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = blockIdx.x * kSchedWarps + wid;
    if (slot >= A.n_launch) return;
    if (A.n_ids && slot >= *A.n_ids) return;
    const int p = A.plan_ids[slot];
    const int strat = A.B.plans[p].strategy;
    if ((strat == WS_STRATEGY_DISTMM_MT || strat == WS_STRATEGY_TASK_OPTIMUS) != SCOPED) return;  // the other instance's
    Ctl* ctl = &ctl_s[wid];
    if (PHASE <= 1 && lane == 0) *ctl = Ctl{};
    __syncwarp();
    const ws_plan_rec& R = A.B.plans[p];
    char* rec = A.recs + static_cast<int64_t>(A.rec_by_slot ? slot : p) * A.RL.bytes;
    SchedHdr* hdr = reinterpret_cast<SchedHdr*>(rec + A.RL.hdr);
    char* gstate = PHASE ? A.state + static_cast<int64_t>(A.rec_by_slot ? slot : p) * A.state_stride : nullptr;
    SCtx C;
    C.B = &A.B;
    C.R = &R;
    C.F = &A.fit;
    C.L = &A.SL;
    C.sm = smem_dyn + wid * A.warp_smem;
    C.ctl = ctl;
    C.lane = lane;
    C.N = R.n_dev;
    C.M = R.n_mod;
    C.K = 0;
    C.mbase = R.mod_begin;
    const bool decoupled = R.strategy == WS_STRATEGY_DECOUPLED_SEQUENTIAL;
    constexpr bool scoped = SCOPED;  // task-scoped baselines: distmm-mt, task-level-optimus
    bool ok = true;
    WS_PH_START(tg);
    if constexpr (PHASE == 2) {
        // The bisection phase moves only what it touches: it reads the valid
        // sets, levels, level members and curve indices, and writes the
        // discretized bi-points and per-level c*/errors; phase 3 then restores
        // the whole slot (phase 1's state with these spans overwritten).
        int ok_i = 0;
        sched_state_hdr(false, gstate, ctl, ok_i, C.K, lane);
        ok = ok_i != 0;
        if (ok && !decoupled && !scoped && C.K <= 32) {
            const SmLayout& L = A.SL;
            sched_span_io(false, gstate, C.sm, L.valid, L.credit, lane);
            sched_span_io(false, gstate, C.sm, L.level, L.up_n, lane);
            sched_span_io(false, gstate, C.sm, L.lvl_mem, L.absorb, lane);
            sched_span_io(false, gstate, C.sm, L.lvl_begin, L.cstar_sm, lane);
            sched_span_wait();
            s_alloc_concurrent<DM>(C, ctl->i1);
            sched_span_io(true, gstate, C.sm, L.up_n, L.sumlay, lane);
            sched_span_io(true, gstate, C.sm, L.cstar_sm, L.adj, lane);
        }
        return;
    } else if constexpr (PHASE == 3) {  // resume the plan where the previous phases left it
        int ok_i = 0;
        sched_state_io(false, gstate, C.sm, sched_state_bytes(A.SL), ctl, ok_i, C.K, lane);
        ok = ok_i != 0;
    } else {
    if (R.n_mod == 0 && R.n_tasks == 0) {
        ok = false;
        if (lane == 0) ctl->err = WS_E_HOST_PRESET;
    } else if (R.n_dev > MaskTraits<DM>::kBits) {  // wider clusters take the DevMask<4> instance
        ok = false;
        if (lane == 0) ctl->err = WS_E_LIMIT_DEVICES;
    } else if (R.n_mod > A.M_cap) {
        ok = false;
        if (lane == 0) ctl->err = WS_E_LIMIT_MODULES;
    }
    __syncwarp();
    if (ok) ok = s_graph(C);
    WS_PH_STOP(tg, 10);
    // programmatic dependent launch: the graph stage above reads only the batch,
    // so it overlaps k_fit; wait for k_fit's grid (and its memory) before the
    // first fit output is read.  A no-op when launched without the attribute.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (ok) {  // the first k_fit outputs read by k_sched
        int* nmax_of = C.at<int>(C.L->nmax_of);
        const int* gm_of = C.at<int>(C.L->gm_of);
        #pragma unroll 1
        for (int k = lane; k < C.K; k += 32) nmax_of[k] = C.F->nmax[gm_of[k]];
        __syncwarp();
    }
    if (ok) ok = s_fit_status(C);
    if (ok && scoped && !A.scoped_ok) {  // launch built without the task-scoped working set
        ok = false;
        if (lane == 0) ctl->err = WS_E_LIMIT_MODULES;
        __syncwarp();
    }
    if (ok) ok = s_valid<DM>(C, !decoupled && !scoped);
    WS_PH_STOP(tg, 11);
    }
    const bool conc = C.K <= 32;  // every level's bisection at once
    if constexpr (PHASE == 0) {
        if (ok && !decoupled && !scoped && conc) s_alloc_concurrent<DM>(C, ctl->i1);
    }
    if constexpr (PHASE == 1) {  // hand the plan to the next phase
        int ok_i = ok;
        sched_state_io(true, gstate, C.sm, sched_state_bytes(A.SL), ctl, ok_i, C.K, lane);
        return;
    }
    int n_levels = 0, nW = 0, nE = 0, KE = 0, n_pg = 0;
    double lower_bound = 0.0, offset = 0.0;
    if (ok && decoupled) {
        ok = s_decoupled<DM>(C, rec, A.RL, nW, nE, offset, A.caps.W, A.caps.E);
    } else if (ok && scoped) {
        if constexpr (SCOPED) {
            if (R.strategy == WS_STRATEGY_TASK_OPTIMUS)
                ok = s_optimus<DM>(C, rec, A.RL, nW, nE, offset, A.caps.W, A.caps.E, KE, n_pg);
            else
                ok = s_distmm<DM>(C, rec, A.RL, nW, nE, offset, A.caps.W, A.caps.E, KE);
        }
    } else if (ok) {
        n_levels = ctl->i1;
        double* cstar = reinterpret_cast<double*>(rec + A.RL.cstar);
        int* lfw = reinterpret_cast<int*>(rec + A.RL.lvl_fw);
        int* lnw = reinterpret_cast<int*>(rec + A.RL.lvl_nw);
        #pragma unroll 1
        for (int l = 0; l < n_levels && ok; ++l) {
            double cs = 0.0;
            if (conc) {
                const int* aerr = C.at<int>(C.L->aerr);
                cs = C.at<double>(C.L->cstar_sm)[l];
                if (aerr[l]) {
                    if (C.lane == 0) {
                        ctl->err = aerr[l];
                        ctl->x = C.at<double>(C.L->aerr_x)[l];
                        ctl->y = C.at<double>(C.L->aerr_y)[l];
                    }
                    __syncwarp();
                    ok = false;
                } else {
                    ok = s_level_repair<DM>(C, l);
                }
            } else {
                ok = s_level_alloc<DM>(C, l, cs);
            }
            WS_PH_STOP(tg, 12);
            if (!ok) break;
            lower_bound += cs;  // planner.hpp:189
            const int w0 = nW;
            double level_end = offset;
            ok = s_schedule_level<DM>(C, rec, A.RL, l, nW, nE, offset, level_end, A.caps.W, A.caps.E);
            WS_PH_STOP(tg, 13);
            if (!ok) break;
            if (lane == 0) {
                cstar[l] = cs;
                lfw[l] = w0;
                lnw[l] = nW - w0;
            }
            offset = level_end;
        }
    }
    if (!ok) {
        if (lane == 0) {
            write_error(A.results + p, ctl);
            hdr->ok = 0;
        }
        return;
    }
    WS_PH_START(tw);
    // hand the MetaOp (or scoped entity) tables to k_place / emit
    const int K = scoped ? KE : C.K;
    int* r_mod_of = reinterpret_cast<int*>(rec + A.RL.mod_of);
    int* r_level = reinterpret_cast<int*>(rec + A.RL.level);
    int* r_up_n = reinterpret_cast<int*>(rec + A.RL.up_n);
    int* r_up_l = reinterpret_cast<int*>(rec + A.RL.up_l);
    int* r_lo_n = reinterpret_cast<int*>(rec + A.RL.lo_n);
    int* r_lo_l = reinterpret_cast<int*>(rec + A.RL.lo_l);
    int* r_by_rank = reinterpret_cast<int*>(rec + A.RL.by_rank);
    int* r_idrank = reinterpret_cast<int*>(rec + A.RL.idrank);
    uint64_t* r_pred = reinterpret_cast<uint64_t*>(rec + A.RL.pred_r);
    uint64_t* r_succ = reinterpret_cast<uint64_t*>(rec + A.RL.succ_r);
    double* r_frac = reinterpret_cast<double*>(rec + A.RL.e_frac);
    int* r_met = reinterpret_cast<int*>(rec + A.RL.e_met);
    int* r_task = reinterpret_cast<int*>(rec + A.RL.e_task);
    if constexpr (SCOPED) {
        const int* ent_met = C.at<int>(A.SL.ent_met);
        const int* ent_task = C.at<int>(A.SL.ent_task);
        const uint64_t* epred = C.at<uint64_t>(A.SL.epred);
        auto trank = [&](int e) { return A.B.task_rank[R.task_begin + ent_task[e]]; };
        #pragma unroll 1
        for (int e = lane; e < K; e += 32) {
            const int k = ent_met[e];
            r_mod_of[e] = C.at<int>(A.SL.mod_of)[k];
            r_level[e] = C.at<int>(A.SL.level)[k];
            r_up_n[e] = r_up_l[e] = r_lo_n[e] = r_lo_l[e] = 0;
            r_frac[e] = C.at<double>(A.SL.ent_frac)[e];
            r_met[e] = k;
            r_task[e] = ent_task[e];
            int r = 0;  // entity ids "m<k>@<task>" in std::map order
            #pragma unroll 1
            for (int e2 = 0; e2 < K; ++e2) r += scoped_less(ent_met[e2], trank(e2), k, trank(e));
            r_idrank[e] = r;
            r_by_rank[r] = e;
        }
        __syncwarp();
        #pragma unroll 1
        for (int e = lane; e < K; e += 32) {
            uint64_t pr = 0, sr = 0;
            #pragma unroll 1
            for (uint64_t b = epred[e]; b; b &= b - 1) pr |= 1ull << r_idrank[low_bit(b)];
            #pragma unroll 1
            for (int e2 = 0; e2 < K; ++e2)
                if (epred[e2] >> e & 1ull) sr |= 1ull << r_idrank[e2];
            r_pred[e] = pr;
            r_succ[e] = sr;
        }
    } else {
        #pragma unroll 1
        for (int k = lane; k < K; k += 32) {
            r_mod_of[k] = C.at<int>(A.SL.mod_of)[k];
            r_level[k] = C.at<int>(A.SL.level)[k];
            r_up_n[k] = C.at<int>(A.SL.up_n)[k];
            r_up_l[k] = C.at<int>(A.SL.up_l)[k];
            r_lo_n[k] = C.at<int>(A.SL.lo_n)[k];
            r_lo_l[k] = C.at<int>(A.SL.lo_l)[k];
            r_by_rank[k] = C.at<int>(A.SL.by_rank)[k];
            r_idrank[k] = C.at<int>(A.SL.idrank)[k];
            r_pred[k] = C.at<uint64_t>(A.SL.pred_r)[k];
            r_succ[k] = C.at<uint64_t>(A.SL.succ_r)[k];
            r_frac[k] = 1.0;
            r_met[k] = k;
            r_task[k] = -1;
        }
    }
    if (lane == 0) {
        SchedHdr h{};
        h.ok = 1;
        h.K = K;
        h.scoped = scoped ? 1 : 0;
        h.n_pg = n_pg;
        h.n_levels = n_levels;
        h.nW = nW;
        h.nE = nE;
        h.lower_bound = lower_bound;
        h.end_time = offset;
        *hdr = h;
    }
    WS_PH_STOP(tw, 14);
}


// DM: valid-allocation set type (uint64_t: N <= 64; DevMask<4>: N <= 256);
// PHASE: 0 whole, 1..3 the phase-split launches (sched_body)
#ifndef WS_SCHED_MINB
#define WS_SCHED_MINB 0  /* 0: no resident-block target (the compiler picks the register budget) */
#endif
#ifndef WS_SCHED1_MINB
#define WS_SCHED1_MINB WS_SCHED_MINB
#endif
#ifndef WS_SCHED2_MINB
// phase 2 (bisection): 7 blocks per SM (<= 72 registers) -- measured on the
// 100k sweep: unbounded (90 registers, 5 blocks) 4.34 ms k_sched, 6 blocks
// 4.20, 7 blocks 4.13, 8 blocks 4.13, 10 blocks 4.50 (spills)
#define WS_SCHED2_MINB 7
#endif
#ifndef WS_SCHED3_MINB
#define WS_SCHED3_MINB WS_SCHED_MINB
#endif
// resident-block targets per phase kernel (register budgets; tuning builds)
template <int PHASE>
constexpr int sched_minb() {
    return PHASE == 1 ? WS_SCHED1_MINB : PHASE == 2 ? WS_SCHED2_MINB : PHASE == 3 ? WS_SCHED3_MINB : WS_SCHED_MINB;
}
template <class DM = uint64_t, int PHASE = 0>
__global__ void __launch_bounds__(32 * kSchedWarps, sched_minb<PHASE>()) k_sched(SchedArgs A) {
    extern __shared__ __align__(16) char smem_dyn[];
    __shared__ Ctl ctl_s[kSchedWarps];
    sched_body<false, DM, PHASE>(A, smem_dyn, ctl_s);
}

// plan_distmm_mt plans of the batch (the planner instance skips them)
template <class DM = uint64_t>
__global__ void __launch_bounds__(32 * kSchedWarps) k_sched_scoped(SchedArgs A) {
    extern __shared__ __align__(16) char smem_dyn[];
    __shared__ Ctl ctl_s[kSchedWarps];
    sched_body<true, DM>(A, smem_dyn, ctl_s);
}

}  // namespace wsdev
