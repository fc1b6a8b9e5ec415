// sim.cuh — k_sim: plan evaluation on the device, one warp per planned record.
//
// Replaces wavesched::simulate_plan (simulate.hpp:127-324: build_param_groups +
// the event-driven replay) and validate_plan (validate.hpp:27-188, including
// compute_device_memory) for a whole batch of plans.  Lanes own devices
// (lane, lane+32): per-device availability clocks, compute seconds and
// resident bytes live in registers; gang barriers and the global frontier are
// warp max-reductions; flows and waves are walked in the reference's order so
// every double is produced by the same operations in the same order.
// Validation (a verdict plus the first WS_SIM_MAX_VIOLATIONS violation records)
// runs on the same warp; the host rebuilds the reference messages.
//
// Written over the device-mask type DM (mask.cuh): uint64_t for clusters of up
// to 64 devices, DevMask<4> up to 256; a lane then owns devices lane + 32 s,
// s < 2 * kWords, and the record's device words 1..3 come from its ext section.
#pragma once
#include "kcommon.cuh"

namespace wsdev {

struct SimCaps {
    int G, W, IS, K, E;  // groups (param groups + entities), waves, islands, MetaOps, entries
};

struct SimSmLayout {
    int isl;     // [IS] DM  island device masks
    int chg;     // [G]  DM  devices charged per group (compute_device_memory)
    int gmask;   // [G]  DM  devices per group (build_param_groups)
    int gbytes;  // [G]  u64 gradient bytes per group
    int pbytes;  // [G]  u64 pooled bytes per representative group
    int pord;    // [G]  i32 pool representatives in device-list order
    int ord;     // [W]  i32 wave replay order
    int exec;    // [K]  i32 executed layers per MetaOp
    int by_rank; // [K]  i32 MetaOps in id-string order
    int gk;      // [K]  i32 group key per MetaOp
    int efrac;   // [K]  f64 batch_fraction per entity
    int lst;     // [E]  i32 one entity's intervals (validate)
    int vio;     // [WS_SIM_MAX_VIOLATIONS] ws_out_violation
    int bytes;
};

// mb: bytes of one device mask (8: uint64_t, 32: DevMask<4>)
__host__ __device__ inline SimSmLayout make_sim_layout(const SimCaps& c, int mb = 8) {
    SimSmLayout L{};
    int o = 0;
    auto take = [&](int b) {
        const int at = o;
        o = (o + b + 7) & ~7;
        return at;
    };
    L.isl = take(mb * c.IS);
    L.chg = take(mb * c.G);
    L.gmask = take(mb * c.G);
    L.gbytes = take(8 * c.G);
    L.pbytes = take(8 * c.G);
    L.pord = take(4 * c.G);
    L.ord = take(4 * c.W);
    L.exec = take(4 * c.K);
    L.by_rank = take(4 * c.K);
    L.gk = take(4 * c.K);
    L.efrac = take(8 * c.K);
    L.lst = take(4 * c.E);
    L.vio = take(static_cast<int>(sizeof(ws_out_violation)) * WS_SIM_MAX_VIOLATIONS);
    L.bytes = o;
    return L;
}

struct SimArgs {
    ws_batch B;
    const ws_plan_result* plans;  // planned records (device)
    const uint8_t* parena;
    uint8_t* scratch;             // per-entry scratch, mirrors the plan arena offsets
    ws_sim_opts opt;
    SimCaps caps;
    SimSmLayout SL;
    ws_sim_result* out;
    uint8_t* arena;
    unsigned long long* arena_top;
    unsigned long long arena_cap;
    int n_plans;
};

constexpr int kSimWarps = 4;

// ScalingCurve::eval_batch_fraction (scaling.hpp:83-86) over a record's pieces
__device__ __forceinline__ double eval_bf(const ws_out_piece* pc, int np, double c, double w, double n,
                                          double frac) {
    const ws_out_piece* p = pc;
    if (!(n < 1.0)) {
        const double nmax = pc[np - 1].n_hi;
        const double x = n < nmax ? n : nmax;  // std::min(n, n_max_)
        p = pc + np - 1;
        #pragma unroll 1
        for (int i = 0; i < np; ++i)  // locate (scaling.hpp:149-154)
            if (x <= pc[i].n_hi + 1e-9) {
                p = pc + i;
                break;
            }
    }
    return p->alpha + p->beta_c * c + p->beta_w * w * frac / n;
}

// sorted-device-list order of two device masks (std::vector<int> operator<)
__device__ __forceinline__ bool devlist_less(uint64_t a, uint64_t b) {
    const uint64_t diff = a ^ b;
    if (!diff) return false;
    const uint64_t d = diff & (~diff + 1);
    const uint64_t above = ~(d | (d - 1));  // bits strictly above d
    return (a & d) ? (b & above) != 0 : !(a & above);
}

template <int W>
__device__ __forceinline__ bool devlist_less(const DevMask<W>& a, const DevMask<W>& b) {
    const DevMask<W> diff = a ^ b;
    if (!dm_any(diff)) return false;
    const int d = dm_low(diff);
    const DevMask<W> above = ~dm_first<DevMask<W>>(d + 1);  // devices strictly above d
    return dm_test(a, d) ? dm_any(b & above) : !dm_any(a & above);
}

// m |= x on a shared-memory mask, one atomic per nonzero word
__device__ __forceinline__ void dm_atomic_or(uint64_t* p, uint64_t x) {
    atomicOr(reinterpret_cast<unsigned long long*>(p), x);
}
template <int W>
__device__ __forceinline__ void dm_atomic_or(DevMask<W>* p, const DevMask<W>& x) {
    #pragma unroll
    for (int i = 0; i < W; ++i)
        if (x.w[i]) atomicOr(reinterpret_cast<unsigned long long*>(&p->w[i]), x.w[i]);
}

struct SimRec {
    const ws_out_metaop* mo;
    const ws_out_piece* pc;
    const ws_out_edge* ed;
    const ws_out_wave* wv;
    const ws_out_entry* en;
    const ws_out_flow* fl;
    const ws_out_scope* sc;  // task-scoped entities (n_scopes > 0)
    const uint64_t* ext;     // device words 1..3 per entry (records of clusters over 64 devices)
    uint64_t en_off;  // entries section offset inside the record
    uint64_t fl_off;  // flows section offset
    uint64_t ext_off; // ext section offset
};

__device__ __forceinline__ SimRec sim_rec(const ws_plan_result& r, const uint8_t* base) {
    SimRec v;
    uint64_t o = 0;
    v.mo = reinterpret_cast<const ws_out_metaop*>(base + o);
    o += al8(sizeof(ws_out_metaop) * r.n_metaops);
    o += al8(sizeof(ws_out_level) * r.n_levels);
    v.pc = reinterpret_cast<const ws_out_piece*>(base + o);
    o += al8(sizeof(ws_out_piece) * r.n_pieces);
    v.ed = reinterpret_cast<const ws_out_edge*>(base + o);
    o += al8(sizeof(ws_out_edge) * r.n_edges);
    v.wv = reinterpret_cast<const ws_out_wave*>(base + o);
    o += al8(sizeof(ws_out_wave) * r.n_waves);
    v.en = reinterpret_cast<const ws_out_entry*>(base + o);
    v.en_off = o;
    o += al8(sizeof(ws_out_entry) * r.n_entries);
    v.fl = reinterpret_cast<const ws_out_flow*>(base + o);
    v.fl_off = o;
    o += al8(sizeof(ws_out_flow) * r.n_flows);
    v.sc = reinterpret_cast<const ws_out_scope*>(base + o);
    o += al8(sizeof(ws_out_scope) * r.n_scopes);
    v.ext = reinterpret_cast<const uint64_t*>(base + o);
    v.ext_off = o;
    return v;
}

// max over the devices of `mask` of the lane's per-device values (devices
// lane + 32 s), from 0.0
template <class DM, int DPL>
__device__ __forceinline__ double lane_max(const DM& mask, int lane, const double (&a)[DPL]) {
    double t = 0.0;
    #pragma unroll
    for (int s = 0; s < DPL; ++s)
        if (dm_test(mask, lane + 32 * s)) t = s == 0 ? a[0] : ((t < a[s]) ? a[s] : t);
    return warp_max_nonneg(t);
}

#ifndef WS_SIM_MINB
#define WS_SIM_MINB 1
#endif
template <class DM = uint64_t>
__global__ void __launch_bounds__(32 * kSimWarps, WS_SIM_MINB) k_sim(SimArgs A) {
    constexpr int kW = MaskTraits<DM>::kWords;  // 64-bit words per device mask
    constexpr int DPL = 2 * kW;                 // devices per lane: lane + 32 s
    extern __shared__ __align__(16) char sim_smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = blockIdx.x * kSimWarps + wid;
    if (p >= A.n_plans) return;
    const ws_plan_result& R = A.plans[p];
    ws_sim_result* res = A.out + p;
    if (R.status != WS_STATUS_OK || A.B.plans[p].n_dev > MaskTraits<DM>::kBits) {
        if (lane == 0) {  // (the launch picks the mask width for the batch's widest cluster)
            ws_sim_result r{};
            r.status = R.status != WS_STATUS_OK ? R.status : WS_STATUS_LIMIT;
            *res = r;
        }
        return;
    }
    char* sm = sim_smem + wid * A.SL.bytes;
    const ws_batch& B = A.B;
    const ws_plan_rec& P = B.plans[p];
    const SimRec V = sim_rec(R, A.parena + R.offset);
    const int N = P.n_dev, K = R.n_metaops, nW = R.n_waves, nE = R.n_entries, nF = R.n_flows;
    const int G = P.n_groups + K, mbase = P.mod_begin;
    const DM all = dm_first<DM>(N);
    const bool wide_rec = kW > 1 && N > 64;  // the record carries device words 1..3 per entry
    // per-entry / per-flow scratch mirroring the record (one 32-byte slot each):
    // entry: [0] interval end (f64), [1] start (f64), [2] check flags (i32),
    //        [3] plan.devices placement of its (wave, MetaOp) key (u64)
    // flow:  [0] source placement, [1] destination placement, [2] flow_duration
    uint8_t* const s_rec = A.scratch + R.offset;
    auto en_iv = [&](int e) { return reinterpret_cast<double*>(s_rec + V.en_off + 32ull * e); };
    auto en_flags = [&](int e) { return reinterpret_cast<int*>(s_rec + V.en_off + 32ull * e + 16); };
    auto fl_masks = [&](int f) { return reinterpret_cast<uint64_t*>(s_rec + V.fl_off + 32ull * f); };
    // entry e's device set as recorded (word 0 + the ext words of wide records)
    auto raw_mask = [&](int e) {
        DM m = dm_zero<DM>();
        dm_set_word(m, 0, V.en[e].devmask);
        if (wide_rec)
            #pragma unroll
            for (int j = 1; j < kW; ++j) dm_set_word(m, j, V.ext[(kW - 1) * e + j - 1]);
        return m;
    };
    // per-entry placement of its (wave, MetaOp) key: word 0 in the entry's
    // scratch slot, words 1..3 in the scratch mirror of the ext section
    auto pl_set = [&](int e, const DM& m) {
        *reinterpret_cast<uint64_t*>(s_rec + V.en_off + 32ull * e + 24) = dm_word(m, 0);
        if (wide_rec)
            #pragma unroll
            for (int j = 1; j < kW; ++j)
                reinterpret_cast<uint64_t*>(s_rec + V.ext_off)[(kW - 1) * e + j - 1] = dm_word(m, j);
    };
    auto en_pl = [&](int e) {
        DM m = dm_zero<DM>();
        dm_set_word(m, 0, *reinterpret_cast<const uint64_t*>(s_rec + V.en_off + 32ull * e + 24));
        if (wide_rec)
            #pragma unroll
            for (int j = 1; j < kW; ++j)
                dm_set_word(m, j, reinterpret_cast<const uint64_t*>(s_rec + V.ext_off)[(kW - 1) * e + j - 1]);
        return m;
    };
    // a flow's endpoint placements: the masks (u64), or for DevMask the entry
    // indices whose recorded sets they are (-1: none)
    auto fl_end = [&](int f, int h) {
        if constexpr (kW == 1) {
            return fl_masks(f)[h];
        } else {
            const long long i = static_cast<long long>(fl_masks(f)[h]);
            return i < 0 ? dm_zero<DM>() : raw_mask(static_cast<int>(i));
        }
    };
    if (G > A.caps.G || G > 128 || nW > A.caps.W || P.n_islands > A.caps.IS || K > A.caps.K || nE > A.caps.E) {
        if (lane == 0) {
            ws_sim_result r{};
            r.status = WS_STATUS_LIMIT;
            *res = r;
        }
        return;
    }
    DM* islm = reinterpret_cast<DM*>(sm + A.SL.isl);
    DM* chg = reinterpret_cast<DM*>(sm + A.SL.chg);
    DM* gmask = reinterpret_cast<DM*>(sm + A.SL.gmask);
    uint64_t* gbytes = reinterpret_cast<uint64_t*>(sm + A.SL.gbytes);
    uint64_t* pbytes = reinterpret_cast<uint64_t*>(sm + A.SL.pbytes);
    int* pord = reinterpret_cast<int*>(sm + A.SL.pord);
    int* ord = reinterpret_cast<int*>(sm + A.SL.ord);
    int* exec = reinterpret_cast<int*>(sm + A.SL.exec);
    int* by_rank = reinterpret_cast<int*>(sm + A.SL.by_rank);
    int* gk = reinterpret_cast<int*>(sm + A.SL.gk);
    double* efrac = reinterpret_cast<double*>(sm + A.SL.efrac);
    const bool scoped = R.n_scopes > 0;
    int* lst = reinterpret_cast<int*>(sm + A.SL.lst);
    ws_out_violation* vio = reinterpret_cast<ws_out_violation*>(sm + A.SL.vio);

    // ---- per-plan tables ------------------------------------------------
    #pragma unroll 1
    for (int i = 0; i < P.n_islands; ++i) {
        DM m = dm_zero<DM>();
        #pragma unroll 1
        for (int base = 0; base < N; base += 32) {
            const int d = base + lane;
            dm_or_bits32(m, base, __ballot_sync(kFull, d < N && B.dev_island[P.dev_begin + d] == i));
        }
        if (lane == 0) islm[i] = m;
    }
    #pragma unroll 1
    for (int g = lane; g < G; g += 32) {
        chg[g] = dm_zero<DM>();
        gmask[g] = dm_zero<DM>();
        gbytes[g] = 0;
    }
    #pragma unroll 1
    for (int k = lane; k < K; k += 32) {
        const int gm = mbase + V.mo[k].module;
        const int grp = V.mo[k].length == B.mod_layers[gm] ? B.mod_group[gm] : -1;
        const int al = scoped ? -1 : B.mod_alias[gm];
        gk[k] = grp < 0 ? P.n_groups + k : ((al >= 0 && al < K) ? P.n_groups + al : grp);
        exec[k] = 0;
        int r = 0;
        if (scoped) {  // ids "m<metaop>@<task>" (baselines.hpp:49-55)
            const int tk = B.task_rank[P.task_begin + V.sc[k].task];
            #pragma unroll 1
            for (int j = 0; j < K; ++j)
                r += scoped_less(V.sc[j].metaop, B.task_rank[P.task_begin + V.sc[j].task], V.sc[k].metaop, tk);
            int users = 0;  // share_fraction: tasks whose flow routes through the module
            #pragma unroll 1
            for (int t = 0; t < P.n_tasks; ++t) {
                const int tg = P.task_begin + t;
                bool in = false;
                #pragma unroll 1
                for (int i = 0; i < B.task_tok_n[tg] && !in; ++i) in = B.tokens[B.task_tok_off[tg] + i] == V.mo[k].module;
                users += in;
            }
            efrac[k] = users ? 1.0 / static_cast<double>(users) : 1.0;
        } else {
            #pragma unroll 1
            for (int j = 0; j < K; ++j) r += dec_less(j, k);
            efrac[k] = B.mod_frac ? B.mod_frac[gm] : 1.0;
        }
        by_rank[r] = k;
    }
    // replay order: waves by (start, index) (simulate.hpp:208-212)
    bool sorted = true;
    #pragma unroll 1
    for (int w = lane + 1; w < nW; w += 32) sorted &= !(V.wv[w].start < V.wv[w - 1].start);
    sorted = __all_sync(kFull, sorted);
    #pragma unroll 1
    for (int w = lane; w < nW; w += 32) {
        int pos = w;
        if (!sorted) {
            pos = 0;
            const double sw = V.wv[w].start;
            #pragma unroll 1
            for (int j = 0; j < nW; ++j) pos += V.wv[j].start < sw || (V.wv[j].start == sw && j < w);
        }
        ord[pos] = w;
    }
    // plan.devices lookups, resolved once: per entry the placement of its
    // (wave, MetaOp) key (the last placed entry with that key), per flow both
    // endpoints; duplicate keys inside a wave flagged for the validator
    #pragma unroll 1
    for (int w = 0; w < nW; ++w) {
        const int eb = V.wv[w].entry_begin, ne = V.wv[w].n_entries;
        #pragma unroll 1
        for (int i = lane; i < ne; i += 32) {
            const int k = V.en[eb + i].metaop;
            DM m = dm_zero<DM>();
            int flags = 0;
            #pragma unroll 1
            for (int j = 0; j < ne; ++j) {
                const ws_out_entry& x = V.en[eb + j];
                if (x.metaop != k) continue;
                const DM xm = raw_mask(eb + j);
                if (dm_any(xm)) m = xm;
                if (j < i) flags |= 1;  // an earlier entry has this MetaOp
            }
            pl_set(eb + i, m);
            *en_flags(eb + i) = flags;
        }
    }
    __syncwarp();
    #pragma unroll 1
    for (int f = lane; f < nF; f += 32) {
        const ws_out_flow& x = V.fl[f];
        int ia = -1, ib = -1;  // the last placed entry of each endpoint key
        if (x.from_wave >= 0 && x.from_wave < nW)
            #pragma unroll 1
            for (int j = 0; j < V.wv[x.from_wave].n_entries; ++j) {
                const int e = V.wv[x.from_wave].entry_begin + j;
                if (V.en[e].metaop == x.from_metaop && dm_any(raw_mask(e))) ia = e;
            }
        if (x.to_wave >= 0 && x.to_wave < nW)
            #pragma unroll 1
            for (int j = 0; j < V.wv[x.to_wave].n_entries; ++j) {
                const int e = V.wv[x.to_wave].entry_begin + j;
                if (V.en[e].metaop == x.to_metaop && dm_any(raw_mask(e))) ib = e;
            }
        if constexpr (kW == 1) {
            fl_masks(f)[0] = ia < 0 ? 0ull : V.en[ia].devmask;
            fl_masks(f)[1] = ib < 0 ? 0ull : V.en[ib].devmask;
        } else {
            fl_masks(f)[0] = static_cast<uint64_t>(static_cast<long long>(ia));
            fl_masks(f)[1] = static_cast<uint64_t>(static_cast<long long>(ib));
        }
        double dur = 0.0;  // flow_duration (simulate.hpp:96-100)
        if (!A.opt.zero_volumes && x.volume != 0 && x.mode != WS_FLOW_COPY)
            dur = static_cast<double>(x.volume) / (x.mode == WS_FLOW_INTER ? P.inter_bw : P.intra_bw);
        reinterpret_cast<double*>(fl_masks(f))[2] = dur;
    }
    // the first 64 flows' waves stay in registers for the per-wave flow scans
    const int ft0 = lane < nF ? V.fl[lane].to_wave : -1, ff0 = lane < nF ? V.fl[lane].from_wave : -1;
    const int ft1 = lane + 32 < nF ? V.fl[lane + 32].to_wave : -1, ff1 = lane + 32 < nF ? V.fl[lane + 32].from_wave : -1;
    __syncwarp();

    // ---- simulate (simulate.hpp:171-280) ---------------------------------
    const ws_sim_opts& opt = A.opt;
    double av[DPL], bc[DPL];  // availability clocks / compute seconds (per_device_busy) of devices lane + 32 s
    #pragma unroll
    for (int s = 0; s < DPL; ++s) av[s] = 0.0, bc[s] = 0.0;
    DM touched = dm_zero<DM>();  // devices present in per_device_busy
    double frontier = 0.0, fwd_bwd = 0.0, send_recv = 0.0, param_sync = 0.0;
    double transferred = 0.0, inter_bytes = 0.0;
    int timeline = 0;
    auto busy_mask = [&](const DM& m, double t0, double dur) {  // busy(d, t0, dur) for every d in m
        if (dur <= 0.0) {
            #pragma unroll
            for (int s = 0; s < DPL; ++s)
                if (dm_test(m, lane + 32 * s)) av[s] = (av[s] < t0) ? t0 : av[s];
        } else {
            #pragma unroll
            for (int s = 0; s < DPL; ++s)
                if (dm_test(m, lane + 32 * s)) av[s] = t0 + dur;
            timeline += dm_popc(m);
        }
    };
    auto attribute = [&](double& bucket) {
        const double f = lane_max(all, lane, av);
        bucket += f - frontier;
        frontier = f;
    };
    auto run_flow = [&](int fi) {
        const ws_out_flow& f = V.fl[fi];
        const DM ma = fl_end(fi, 0), mb = fl_end(fi, 1);
        if (!dm_any(ma) || !dm_any(mb)) return;
        const double dur = reinterpret_cast<const double*>(fl_masks(fi))[2];
        const DM parties = ma | mb;
        const double t0 = lane_max(parties, lane, av);
        busy_mask(parties, t0, dur);
        if (!opt.zero_volumes) {
            transferred += static_cast<double>(f.volume);
            if (f.mode == WS_FLOW_INTER) inter_bytes += static_cast<double>(f.volume);
        }
    };
    auto run_wave = [&](int w, bool backward) {
        const double scale = backward ? opt.backward_ratio : 1.0;
        const ws_out_wave& wv = V.wv[w];
        DM parts = dm_zero<DM>();
        #pragma unroll 1
        for (int i = lane; i < wv.n_entries; i += 32) parts |= en_pl(wv.entry_begin + i);
        parts = dm_or_reduce(parts);
        const double t0 = lane_max(parts, lane, av);
        #pragma unroll 1
        for (int i = 0; i < wv.n_entries; ++i) {
            const DM m = en_pl(wv.entry_begin + i);
            if (!dm_any(m)) continue;
            const double dur = V.en[wv.entry_begin + i].span * scale;
            busy_mask(m, t0, dur);
            #pragma unroll
            for (int s = 0; s < DPL; ++s)
                if (dm_test(m, lane + 32 * s)) bc[s] += dur;
            touched |= m;
        }
        const double rel = t0 + wv.duration * scale;  // the wave releases its devices together
        #pragma unroll
        for (int s = 0; s < DPL; ++s)
            if (dm_test(parts, lane + 32 * s)) av[s] = (av[s] < rel) ? rel : av[s];
    };
    auto flows_where = [&](bool into, int w) {  // flows_into / flows_out_of, in flow order
        #pragma unroll 1
        for (unsigned b = __ballot_sync(kFull, (into ? ft0 : ff0) == w); b; b &= b - 1) run_flow(__ffs(b) - 1);
        #pragma unroll 1
        for (unsigned b = __ballot_sync(kFull, (into ? ft1 : ff1) == w); b; b &= b - 1) run_flow(32 + __ffs(b) - 1);
        #pragma unroll 1
        for (int base = 64; base < nF; base += 32) {
            const int f = base + lane;
            const bool hit = f < nF && (into ? V.fl[f].to_wave : V.fl[f].from_wave) == w;
            #pragma unroll 1
            for (unsigned b = __ballot_sync(kFull, hit); b; b &= b - 1) run_flow(base + __ffs(b) - 1);
        }
    };
    #pragma unroll 1
    for (int j = 0; j < nW; ++j) {  // forward: transmissions arrive before their consumer wave
        const int w = ord[j];
        flows_where(true, w);
        attribute(send_recv);
        run_wave(w, false);
        attribute(fwd_bwd);
    }
    #pragma unroll 1
    for (int j = nW - 1; j >= 0; --j) {  // backward: reverse order, gradients mirror the flows
        const int w = ord[j];
        run_wave(w, true);
        attribute(fwd_bwd);
        flows_where(false, w);
        attribute(send_recv);
    }
    if (!opt.skip_sync) {  // build_param_groups (simulate.hpp:127-165), group-wise sync (:268-276)
        #pragma unroll 1
        for (int base = 0; base < nE; base += 32) {  // groups: device union and max gradient bytes
            const int e = base + lane;
            int g = -1;
            DM m = dm_zero<DM>();
            uint64_t gb = 0;
            if (e < nE) {
                const int k = V.en[e].metaop;
                m = en_pl(e);
                if (dm_any(m) && k >= 0 && k < K) {
                    const int gm = mbase + V.mo[k].module;
                    const uint64_t pb = static_cast<uint64_t>(static_cast<double>(B.mod_param[gm]) *
                                                              V.mo[k].length / B.mod_layers[gm]);
                    gb = 2ull * pb / static_cast<uint64_t>(B.mod_tp[gm]);
                    g = gk[k];
                }
            }
            if (g >= 0) {
                dm_atomic_or(gmask + g, m);
                atomicMax(reinterpret_cast<unsigned long long*>(gbytes + g), gb);
            }
        }
        __syncwarp();
        // pool entries: one per distinct device set (first group holding it), bytes summed
        int npool = 0;
        #pragma unroll 1
        for (int base = 0; base < G; base += 32) {
            const int g = base + lane;
            bool rep = g < G && dm_any(gmask[g]);
            uint64_t sum = 0;
            if (rep) {
                #pragma unroll 1
                for (int h = 0; h < G; ++h)
                    if (gmask[h] == gmask[g]) {
                        if (h < g) rep = false;
                        sum += gbytes[h];
                    }
            }
            if (rep) pbytes[g] = sum;
            npool += __popc(__ballot_sync(kFull, rep));
            if (g < G) pord[g] = rep ? 1 : 0;  // representative flags
        }
        __syncwarp();
        int rk[4];  // rank of each representative among the distinct sets (G <= 128)
        for (int s = 0; s < 4; ++s) {
            const int g = s * 32 + lane;
            rk[s] = -1;
            if (g < G && pord[g] == 1) {
                int r = 0;
                #pragma unroll 1
                for (int h = 0; h < G; ++h) r += pord[h] == 1 && devlist_less(gmask[h], gmask[g]);
                rk[s] = r;
            }
        }
        __syncwarp();
        for (int s = 0; s < 4; ++s)
            if (rk[s] >= 0) pord[rk[s]] = s * 32 + lane;  // pord reused: rank -> group
        __syncwarp();
        #pragma unroll 1
        for (int r = 0; r < npool; ++r) {
            const int g = pord[r];
            const DM m = gmask[g];
            double dur = 0.0;
            if (dm_popc(m) >= 2) {
                int widest = 0, islands = 0;
                #pragma unroll 1
                for (int base = 0; base < P.n_islands; base += 32) {
                    const int i = base + lane;
                    const int c = i < P.n_islands ? dm_popc(m & islm[i]) : 0;
                    widest = max(widest, static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(c))));
                    islands += __popc(__ballot_sync(kFull, c > 0));
                }
                const double bytes = static_cast<double>(pbytes[g]);
                if (widest >= 2)
                    dur += 2.0 * (static_cast<double>(widest) - 1.0) / static_cast<double>(widest) * bytes / P.intra_bw;
                if (islands >= 2)
                    dur += 2.0 * (static_cast<double>(islands) - 1.0) / static_cast<double>(islands) * bytes /
                           P.inter_bw;
            }
            if (dur <= 0.0) continue;
            const double t0 = lane_max(m, lane, av);
            busy_mask(m, t0, dur);
        }
        attribute(param_sync);
    }
    const double makespan = lane_max(all, lane, av);

    // ---- compute_device_memory (validate.hpp:27-50) -----------------------
    double mem[DPL];
    #pragma unroll
    for (int s = 0; s < DPL; ++s) mem[s] = 0.0;
    #pragma unroll 1
    for (int w = 0; w < nW; ++w) {
        const ws_out_wave& wv = V.wv[w];
        #pragma unroll 1
        for (int i = 0; i < wv.n_entries; ++i) {
            const int e = wv.entry_begin + i;
            const int k = V.en[e].metaop;
            const DM m = en_pl(e);
            if (!dm_any(m) || k < 0 || k >= K) continue;
            const int gm = mbase + V.mo[k].module;
            const uint64_t pb = static_cast<uint64_t>(static_cast<double>(B.mod_param[gm]) * V.mo[k].length /
                                                      B.mod_layers[gm]);
            const DM charged = chg[gk[k]];
            const double pstate = (1.0 + P.grad_mult) * static_cast<double>(pb) / B.mod_tp[gm];
            const double frac = efrac[k];  // PlanEntity::batch_fraction
            const double act = V.en[e].layers * (static_cast<double>(B.mod_act[gm]) * frac / V.en[e].n);
            #pragma unroll
            for (int s = 0; s < DPL; ++s)
                if (dm_test(m, lane + 32 * s)) {
                    if (!dm_test(charged, lane + 32 * s)) mem[s] += pstate;
                    mem[s] += act;
                }
            __syncwarp();
            if (lane == 0) chg[gk[k]] = charged | m;
            __syncwarp();
        }
    }

    // ---- utilization proxy (simulate.hpp:283-300), lanes = MetaOps --------
    double ls[2] = {0.0, 0.0}, ds[2] = {0.0, 0.0}, rate = 0.0;
    bool seen_k[2] = {false, false};
    for (int s = 0; s < 2; ++s) {
        const int k = lane + 32 * s;
        if (k >= K) continue;
        const int gm = mbase + V.mo[k].module;
        const double wk = B.mod_w[gm];
        const double frac = efrac[k];
        #pragma unroll 1
        for (int w = 0; w < nW; ++w)
            #pragma unroll 1
            for (int i = 0; i < V.wv[w].n_entries; ++i) {
                const ws_out_entry& e = V.en[V.wv[w].entry_begin + i];
                if (e.metaop != k) continue;
                ls[s] += wk * frac * e.layers;
                ds[s] += e.span * e.n;
                seen_k[s] = true;
            }
        const double t1 = eval_bf(V.pc + V.mo[k].piece_begin, V.mo[k].piece_count, B.mod_c[gm], wk, 1.0, frac);
        if (t1 > 0.0) {
            const double r = wk * frac / t1;
            rate = (rate < r) ? r : rate;
        }
    }
    const double peak_rate = warp_max_d(rate);
    const uint64_t util_mask = (static_cast<uint64_t>(__ballot_sync(kFull, seen_k[1])) << 32) |
                               __ballot_sync(kFull, seen_k[0]);

    // ---- validate_plan (validate.hpp:58-188) ------------------------------
    // Checks run lane-parallel; violations are appended by lane 0 in the
    // reference's order, so only broken plans pay for the serial emission.
    int nv = 0;  // lane 0 holds the count
    auto fail = [&](int code, int wave, int a, int b, double x, double y) {
        if (nv < WS_SIM_MAX_VIOLATIONS) vio[nv] = ws_out_violation{code, wave, a, b, x, y};
        ++nv;
    };
    const double horizon = R.end_time > 1.0 ? R.end_time : 1.0;  // std::max(1.0, end_time)
    const double tol = 1e-6 * horizon;
    enum { F_DUP = 1, F_UNKNOWN = 2, F_SPAN = 4, F_SPAN_DUR = 8 };
    #pragma unroll 1
    for (int w = 0; w < nW; ++w) {  // per-wave entry checks with recomputed spans
        const ws_out_wave& wv = V.wv[w];
        int used = 0;
        bool any = false;
        #pragma unroll 1
        for (int i = lane; i < wv.n_entries; i += 32) {
            const int e = wv.entry_begin + i;
            const int k = V.en[e].metaop;
            int flags = *en_flags(e) & F_DUP;
            if (k < 0 || k >= K) {
                flags = F_UNKNOWN;
            } else {
                const int gm = mbase + V.mo[k].module;
                const double per_layer =
                    eval_bf(V.pc + V.mo[k].piece_begin, V.mo[k].piece_count, B.mod_c[gm], B.mod_w[gm],
                            static_cast<double>(V.en[e].n), efrac[k]);
                const double span = V.en[e].layers * per_layer;
                const double rec = V.en[e].span;
                if (fabs(span - rec) > tol + 1e-9 * fabs(span)) flags |= F_SPAN;
                if (rec > wv.duration + tol) flags |= F_SPAN_DUR;
                en_iv(e)[0] = wv.start + span;
                en_iv(e)[1] = wv.start;
                atomicAdd(exec + k, V.en[e].layers);
                used += V.en[e].n;
            }
            *en_flags(e) = flags;
            any |= flags != 0;
        }
        used = static_cast<int>(__reduce_add_sync(kFull, static_cast<unsigned>(used)));
        if (__any_sync(kFull, any)) {
            __syncwarp();
            if (lane == 0)
                #pragma unroll 1
                for (int i = 0; i < wv.n_entries; ++i) {
                    const int e = wv.entry_begin + i;
                    const int flags = *en_flags(e), k = V.en[e].metaop;
                    if (flags & F_UNKNOWN) {
                        fail(WS_V_UNKNOWN_ENTITY, w, k, 0, 0, 0);
                        continue;
                    }
                    if (flags & F_DUP) fail(WS_V_DUPLICATE, w, k, 0, 0, 0);
                    if (flags & F_SPAN) {
                        const int gm = mbase + V.mo[k].module;
                        const double span =
                            V.en[e].layers * eval_bf(V.pc + V.mo[k].piece_begin, V.mo[k].piece_count, B.mod_c[gm],
                                                     B.mod_w[gm], static_cast<double>(V.en[e].n),
                                                     efrac[k]);
                        fail(WS_V_SPAN, w, k, 0, V.en[e].span, span);
                    }
                    if (flags & F_SPAN_DUR) fail(WS_V_SPAN_DURATION, w, 0, 0, 0, 0);
                }
        }
        if (lane == 0 && used > N) fail(WS_V_WAVE_DEVICES, w, 0, 0, 0, 0);
    }
    __syncwarp();
    {  // work completion, entities in id order
        bool bad = false;
        #pragma unroll 1
        for (int k = lane; k < K; k += 32) bad |= exec[k] != V.mo[k].length;
        if (__any_sync(kFull, bad) && lane == 0)
            #pragma unroll 1
            for (int r = 0; r < K; ++r) {
                const int k = by_rank[r];
                if (exec[k] != V.mo[k].length) fail(WS_V_WORK, -1, k, exec[k], V.mo[k].length, 0);
            }
    }
    // entry -> (start, end, n) of its interval; known MetaOps only
    auto iv_of = [&](int e, double& s, double& en, int& n) {
        if (V.en[e].metaop < 0 || V.en[e].metaop >= K) return false;
        en = en_iv(e)[0];
        s = en_iv(e)[1];
        n = V.en[e].n;
        return true;
    };
    {  // instantaneous capacity: the first addition event after which active > N
        double bt = 0.0;
        int bn = 0, bi = 0x7fffffff, bact = 0;
        #pragma unroll 1
        for (int i = lane; i < nE; i += 32) {
            double si, ei_, sj, ej;
            int ni, nj;
            if (!iv_of(i, si, ei_, ni)) continue;
            int act = 0;
            #pragma unroll 1
            for (int j = 0; j < nE; ++j) {
                if (!iv_of(j, sj, ej, nj)) continue;
                if (sj < si || (sj == si && (nj < ni || (nj == ni && j <= i)))) act += nj;
                const double rem = sj > ej - tol ? sj : ej - tol;  // std::max(start, end - tol)
                if (rem <= si) act -= nj;
            }
            if (act > N && (bi == 0x7fffffff || si < bt || (si == bt && (ni < bn || (ni == bn && i < bi)))))
                bt = si, bn = ni, bi = i, bact = act;
        }
        #pragma unroll 1
        for (int off = 16; off; off >>= 1) {
            const double ot = __shfl_xor_sync(kFull, bt, off);
            const int on = __shfl_xor_sync(kFull, bn, off), oi = __shfl_xor_sync(kFull, bi, off),
                      oa = __shfl_xor_sync(kFull, bact, off);
            if (oi != 0x7fffffff &&
                (bi == 0x7fffffff || ot < bt || (ot == bt && (on < bn || (on == bn && oi < bi)))))
                bt = ot, bn = on, bi = oi, bact = oa;
        }
        if (lane == 0 && bi != 0x7fffffff) fail(WS_V_CAPACITY, -1, bact, 0, bt, 0);
    }
    {  // same-entity intervals pairwise disjoint, entities in id order; lane per
       // entity walks its intervals in wave order (strictly increasing starts =
       // the sorted order), ties or inversions take the exact std::sort path
        unsigned flag_lo = 0, flag_hi = 0;  // bit per entity: 1 overlap, 2 needs sort
        for (int s = 0; s < 2; ++s) {
            const int k = lane + 32 * s;
            if (k >= K) continue;
            int fl = 0;
            double pe = 0.0, ps = 0.0;
            bool first = true;
            #pragma unroll 1
            for (int w = 0; w < nW && !(fl & 2); ++w)
                #pragma unroll 1
                for (int i = 0; i < V.wv[w].n_entries; ++i) {
                    const int e = V.wv[w].entry_begin + i;
                    if (V.en[e].metaop != k) continue;
                    const double st = en_iv(e)[1], en = en_iv(e)[0];
                    if (!first) {
                        if (!(ps < st)) {
                            fl |= 2;
                            break;
                        }
                        if (pe > st + tol) fl |= 1;
                    }
                    first = false;
                    ps = st;
                    pe = en;
                }
            (s ? flag_hi : flag_lo) = static_cast<unsigned>(fl);
        }
        const bool any = __any_sync(kFull, (flag_lo | flag_hi) != 0);
        if (any) {
            if (lane == 0) {
                #pragma unroll 1
                for (int r = 0; r < K; ++r) {
                    const int k = by_rank[r];
                    int cnt = 0;
                    #pragma unroll 1
                    for (int w = 0; w < nW; ++w)  // by_entity lists keep wave / entry order
                        #pragma unroll 1
                        for (int i = 0; i < V.wv[w].n_entries; ++i)
                            if (V.en[V.wv[w].entry_begin + i].metaop == k) lst[cnt++] = V.wv[w].entry_begin + i;
                    struct ByStart {  // std::sort by interval start (exact libstdc++ emulation)
                        const double* iv;
                        __device__ bool operator()(int a, int b) const { return iv[4 * a + 1] < iv[4 * b + 1]; }
                    } cmp{en_iv(0)};
                    ls_sort(lst, cnt, cmp);
                    #pragma unroll 1
                    for (int i = 0; i + 1 < cnt; ++i)
                        if (en_iv(lst[i])[0] > en_iv(lst[i + 1])[1] + tol) {
                            fail(WS_V_OVERLAP, -1, k, 0, 0, 0);
                            break;
                        }
                }
            }
            __syncwarp();
        }
    }
    #pragma unroll 1
    for (int q = 0; q < R.n_edges; ++q) {  // dependencies, in MetaGraph edge order
        const int from = V.ed[q].from, to = V.ed[q].to;
        double fe = 0.0, ts = horizon * 2;
        bool hf = false, ht = false;
        #pragma unroll 1
        for (int i = lane; i < nE; i += 32) {
            double s, e;
            int n;
            if (!iv_of(i, s, e, n)) continue;
            if (V.en[i].metaop == from) hf = true, fe = (fe < e) ? e : fe;
            if (V.en[i].metaop == to) ht = true, ts = (s < ts) ? s : ts;
        }
        hf = __any_sync(kFull, hf);
        ht = __any_sync(kFull, ht);
        fe = warp_max_d(fe);
        ts = warp_min_d(ts);
        if (lane == 0 && hf && ht && ts + tol < fe) fail(WS_V_DEPENDENCY, -1, from, to, ts, fe);
    }
    bool any_placed = false;
    #pragma unroll 1
    for (int i = lane; i < nE; i += 32) any_placed |= dm_any(raw_mask(i));
    if (__any_sync(kFull, any_placed)) {
        #pragma unroll 1
        for (int w = 0; w < nW; ++w) {  // per wave: placed, sized, disjoint (device-list order)
            const ws_out_wave& wv = V.wv[w];
            bool bad = false;
            DM uni = dm_zero<DM>();
            int sum = 0;
            #pragma unroll 1
            for (int i = lane; i < wv.n_entries; i += 32) {
                const int e = wv.entry_begin + i;
                const DM m = en_pl(e);
                bad |= !dm_any(m) || dm_popc(m) != V.en[e].n || dm_any(m & ~all);
                uni |= m;
                sum += dm_popc(m);
            }
            uni = dm_or_reduce(uni);
            sum = static_cast<int>(__reduce_add_sync(kFull, static_cast<unsigned>(sum)));
            if (!__any_sync(kFull, bad) && sum == dm_popc(uni)) continue;
            if (lane == 0) {
                DM taken = dm_zero<DM>();
                #pragma unroll 1
                for (int i = 0; i < wv.n_entries; ++i) {
                    const int e = wv.entry_begin + i;
                    const DM m = en_pl(e);
                    if (!dm_any(m)) {
                        fail(WS_V_UNPLACED, w, V.en[e].metaop, 0, 0, 0);
                        continue;
                    }
                    int rot = 0;  // the placed entry's rot orders its device list
                    #pragma unroll 1
                    for (int j = 0; j < wv.n_entries; ++j) {
                        const ws_out_entry& x = V.en[wv.entry_begin + j];
                        if (x.metaop == V.en[e].metaop && dm_any(raw_mask(wv.entry_begin + j))) rot = x.rot;
                    }
                    if (dm_popc(m) != V.en[e].n) fail(WS_V_DEVICE_COUNT, w, V.en[e].metaop, dm_popc(m), V.en[e].n, 0);
                    const DM below = dm_first<DM>(rot);
                    const DM order[2] = {m & ~below, m & below};
                    for (int h = 0; h < 2; ++h)
                        #pragma unroll 1
                        for (DM b = order[h]; dm_any(b); b = dm_drop_low(b)) {
                            const int d = dm_low(b);
                            if (d >= N)
                                fail(WS_V_UNKNOWN_DEVICE, -1, d, 0, 0, 0);
                            else if (dm_test(taken, d))
                                fail(WS_V_DEVICE_TWICE, w, d, 0, 0, 0);
                            else
                                taken |= dm_bit<DM>(d);
                        }
                }
            }
            __syncwarp();
        }
        const double cap = static_cast<double>(P.mem_capacity) * (1.0 + 1e-9);
        #pragma unroll
        for (int h = 0; h < DPL; ++h) {  // memory capacity, devices in id order
            const double mv = mem[h];
            const int d = lane + 32 * h;
            const unsigned b = __ballot_sync(kFull, d < N && mv > cap);
            #pragma unroll 1
            for (unsigned q = b; q; q &= q - 1) {
                const int src = __ffs(q) - 1;
                const double x = __shfl_sync(kFull, mv, src);
                if (lane == 0)
                    fail(WS_V_MEMORY, -1, 32 * h + src, 0, x, __longlong_as_double(static_cast<long long>(P.mem_capacity)));
            }
        }
    }
    __syncwarp();

    // ---- write the record ---------------------------------------------------
    nv = __shfl_sync(kFull, nv, 0);
    const int keep = nv < WS_SIM_MAX_VIOLATIONS ? nv : WS_SIM_MAX_VIOLATIONS;
    // busy[N], touched (1 word; 4 for clusters over 64 devices), mem[N], util[K],
    // util_mask, violations: the layout goes by the plan's N (ws_abi.h), not the instance
    const int TW = wide_rec ? kW : 1;
    const uint64_t sz = 16ull * N + 8ull * TW + 8 + 8ull * K + sizeof(ws_out_violation) * keep;
    unsigned long long off = 0;
    if (lane == 0) off = atomicAdd(A.arena_top, static_cast<unsigned long long>(sz));
    off = __shfl_sync(kFull, off, 0);
    if (off + sz > A.arena_cap) {
        if (lane == 0) {
            ws_sim_result r{};
            r.status = WS_STATUS_INTERNAL;
            *res = r;
        }
        return;
    }
    uint8_t* base = A.arena + off;
    double* o_busy = reinterpret_cast<double*>(base);
    double* o_mem = reinterpret_cast<double*>(base + 8ull * N + 8ull * TW);
    double* o_util = reinterpret_cast<double*>(base + 16ull * N + 8ull * TW);
    #pragma unroll
    for (int s = 0; s < DPL; ++s)
        if (lane + 32 * s < N) o_busy[lane + 32 * s] = bc[s], o_mem[lane + 32 * s] = mem[s];
    for (int s = 0; s < 2; ++s) {
        const int k = lane + 32 * s;
        if (k < K)
            o_util[k] = (ds[s] > 0.0 && peak_rate > 0.0) ? (ls[s] / ds[s]) / peak_rate : 0.0;
    }
    ws_out_violation* o_v = reinterpret_cast<ws_out_violation*>(base + 16ull * N + 8ull * TW + 8 + 8ull * K);
    #pragma unroll 1
    for (int i = lane; i < keep; i += 32) o_v[i] = vio[i];
    if (lane == 0) {
        #pragma unroll
        for (int j = 0; j < kW; ++j)
            if (j < TW) reinterpret_cast<uint64_t*>(base + 8ull * N)[j] = dm_word(touched, j);
        *reinterpret_cast<uint64_t*>(base + 16ull * N + 8ull * TW + 8ull * K) = util_mask;
        ws_sim_result r{};
        r.status = WS_STATUS_OK;
        r.valid = nv == 0;
        r.n_violations = nv;
        r.timeline_items = timeline;
        r.makespan = makespan;
        r.fwd_bwd_seconds = fwd_bwd;
        r.param_sync_seconds = param_sync;
        r.send_recv_seconds = send_recv;
        const double span = makespan > 1e-300 ? makespan : 1e-300;  // std::max(makespan, 1e-300)
        r.fwd_bwd_fraction = fwd_bwd / span;
        r.param_sync_fraction = param_sync / span;
        r.send_recv_fraction = send_recv / span;
        r.total_transferred_bytes = transferred;
        r.total_inter_island_bytes = inter_bytes;
        r.offset = off;
        r.size = sz;
        *res = r;
    }
}

}  // namespace wsdev
