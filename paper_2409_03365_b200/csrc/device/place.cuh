// place.cuh — k_place: subsystem (4b) placement (placement.hpp:168-447,
// planner.hpp:99-151) and the output record.  One warp per plan; MetaOp,
// entry, device and group state in dynamic shared memory; lanes score the
// candidate device sets and min-locate the best; the per-wave snapshots the
// backtracking DFS restores from and the flow list live in global memory.
#pragma once
#include "kcommon.cuh"
#include "sched.cuh"

namespace wsdev {

constexpr int kPlaceWarps = 4;

struct PlaceCaps {
    int M, N, W, E, F, G, IS;
};

// The fixed-shape instance of k_place: launches whose caps fit this class use
// a compile-time shared-memory layout, so every table address folds into the
// shared-memory instruction's immediate offset (the runtime layout spends ~8%
// of k_place's instructions recomputing table addresses).  Covers the sweep
// and the BASELINE configs (<= 32 MetaOps, <= 64 devices, <= 16 islands).
constexpr PlaceCaps kFixedPlaceCaps{32, 64, 65, 128, 0, 64, 16};

struct PlSmLayout {
    int by_rank, idrank, lastw, home, lastent, gkey, tp, mod_of;  // [M] i32
    int pred_r, contb, edgeb, memact, parb;                       // [M] u64
    int e_k, e_n, e_l, e_rot, e_prev, e_wave;                     // [E] i32
    int e_mask;                                                   // [E] u64
    int w_eb, w_ec, w_cursor, variant;                            // [W] i32
    int mem;                                                      // [N] f64
    int isl;                                                      // [N] i32
    int islmask;                                                  // [IS] u64
    int isllow;                                                   // [IS] u64 devices below island i
    int islfull;                                                  // [IS] u64 islands of the whole plan
    int glist;                                                    // [W] i32 waves of the current place() call
    int btm;                                                      // [W] int2 backtracking memo (k_place DFS)
    int nwin;                                                     // [IS] i32
    int chg;                                                      // [G] u64
    int fin_src, fin_bytes;                                       // [M+1]
    int disp_mask, disp_bytes, disp_cnt, eorder, va;              // [M]
    int cmask;                                                    // [2N+M+1] candidate device sets
    int used_if;                                                  // [N] f64
    int bytes;
};

// mb: bytes of one device mask (8: uint64_t, N <= 64; 32: DevMask<4>, N <= 256)
__host__ __device__ constexpr PlSmLayout make_pl_layout(const PlaceCaps& c, int mb = 8) {
    PlSmLayout L{};
    int o = 0;
    auto take = [&](int b) {
        const int at = o;
        o = (o + b + 7) & ~7;
        return at;
    };
    const int M = c.M, E = c.E, W = c.W, N = c.N;
    L.by_rank = take(4 * M);
    L.idrank = take(4 * M);
    L.lastw = take(4 * M);
    L.home = take(4 * M);
    L.lastent = take(4 * M);
    L.gkey = take(4 * M);
    L.tp = take(4 * M);
    L.mod_of = take(4 * M);
    L.pred_r = take(8 * M);
    L.contb = take(8 * M);
    L.edgeb = take(8 * M);
    L.memact = take(8 * M);
    L.parb = take(8 * M);
    L.e_k = take(4 * E);
    L.e_n = take(4 * E);
    L.e_l = take(4 * E);
    L.e_rot = take(4 * E);
    L.e_prev = take(4 * E);
    L.e_wave = take(4 * E);
    L.e_mask = take(mb * E);
    L.w_eb = take(4 * W);
    L.w_ec = take(4 * W);
    L.w_cursor = take(4 * W);
    L.variant = take(4 * W);
    L.mem = take(8 * N);
    L.isl = take(4 * N);
    L.islmask = take(mb * c.IS);
    L.isllow = take(mb * c.IS);
    L.islfull = take(mb * c.IS);
    L.glist = take(4 * W);
    L.btm = take(8 * W);
    L.nwin = take(4 * (c.IS + W + 1));  // island window counts, then flows-per-wave marks
    L.chg = take(mb * c.G);
    L.fin_src = take(4 * (M + 1));
    L.fin_bytes = take(8 * (M + 1));
    L.disp_mask = take(mb * M);
    L.disp_bytes = take(8 * M);
    L.disp_cnt = take(4 * M);
    L.eorder = take(4 * M);
    L.va = take(8 * M);
    L.cmask = take(mb * (2 * N + M + 1));
    L.used_if = take(8 * N);
    L.bytes = (o + 15) & ~15;
    return L;
}

struct PlaceArgs {
    ws_batch B;
    FitOut fit;
    PlaceCaps caps;
    RecLayout RL;
    PlSmLayout PL;
    const char* recs;         // schedule records (k_sched)
    uint64_t* flows;          // [n_launch][F][2]: volume, packed meta
    const int32_t* plan_ids;
    const int32_t* n_ids;
    int n_launch;
    int rec_by_slot;          // retry pass: records indexed by launch slot
    ws_plan_result* results;
    uint8_t* arena;
    unsigned long long* arena_top;
    unsigned long long arena_cap;
    // backtracking snapshots: a pool of per-warp slots, each (W+1) states of
    // mem[N] f64 + chg[G] u64, claimed on a plan's first failed wave
    double* snap;             // [snap_slots][snap_stride]
    unsigned* snap_bits;      // claim bitmap, one bit per slot
    int snap_slots;           // 0: no pool (replay only)
    long long snap_stride;    // 8-byte words per slot
    // split emission (k_emit): k_place leaves each plan's placement here
    // (indexed like the schedule records) and k_emit writes the output record
    char* emit_mask;          // [.][caps.E] device masks (sizeof(DM) each)
    int32_t* emit_rot;        // [.][caps.E]
    int32_t* emit_nf;         // [.] flow count, -1: no record (error written)
    int split_emit;
};

template <class DM>
struct PCtx {
    const ws_batch* B;
    const ws_plan_rec* R;
    const FitOut* F;
    const PlSmLayout* L;
    char* sm;
    Ctl* ctl;
    int lane, N, K, mbase, nW, nE, nF, Fcap, G, n_isl;
    int contig;  // every island is one contiguous run of device indices
    int dev_off, dev_cnt;  // device block of the current place() call ([0, N) unless grouped)
    int first_nc;          // candidate count of the wave's first entry (p_wave; 1 << 30: unknown)
    DM all;           // devices of the current place() call
    uint64_t* flows;  // this plan's flow list (2 words per flow)
    // plan options hoisted out of the per-attempt loops (registers, not global loads)
    double gmul1;     // 1 + grad_opt_multiplier
    double cap;       // mem_capacity
    int sequential;
    template <typename T>
    __device__ __forceinline__ T* at(int off) const {
        return reinterpret_cast<T*>(sm + off);
    }
};

// flow packing: word0 = volume; word1 = from_wave | from_k<<16 | to_wave<<32 | to_k<<48 ; mode kept
// in bits 14..15 of the to_k field (k < 2^14)
__device__ __forceinline__ uint64_t pack_flow(int fw, int fk, int tw, int tk, int mode) {
    return static_cast<uint64_t>(fw & 0xffff) | (static_cast<uint64_t>(fk & 0x3fff) << 16) |
           (static_cast<uint64_t>(mode & 3) << 30) | (static_cast<uint64_t>(tw & 0xffff) << 32) |
           (static_cast<uint64_t>(tk & 0xffff) << 48);
}

// One wave: 1 placed, 0 infeasible (caller tries the next variant), -1 error.
template <class DM, bool FIXED = false>
__device__ int p_wave(PCtx<DM>& C, int w, int variant) {
    constexpr PlSmLayout kL = make_pl_layout(kFixedPlaceCaps, 8);
    const PlSmLayout& L = FIXED ? kL : *C.L;
    const ws_plan_rec& R = *C.R;
    const int lane = C.lane, N = C.N;
    const int* w_eb = C.template at<int>(L.w_eb);
    const int* w_ec = C.template at<int>(L.w_ec);
    const int* e_k = C.template at<int>(L.e_k);
    const int* e_n = C.template at<int>(L.e_n);
    const int* e_l = C.template at<int>(L.e_l);
    DM* e_mask = C.template at<DM>(L.e_mask);
    int* e_rot = C.template at<int>(L.e_rot);
    const int* e_wave = C.template at<int>(L.e_wave);
    const int* home = C.template at<int>(L.home);
    const int* lastw = C.template at<int>(L.lastw);
    const int* by_rank = C.template at<int>(L.by_rank);
    const int* idrank = C.template at<int>(L.idrank);
    const uint64_t* pred_r = C.template at<uint64_t>(L.pred_r);
    const uint64_t* contb = C.template at<uint64_t>(L.contb);
    const uint64_t* edgeb = C.template at<uint64_t>(L.edgeb);
    const uint64_t* memact = C.template at<uint64_t>(L.memact);
    const uint64_t* parb = C.template at<uint64_t>(L.parb);
    const int* gkey = C.template at<int>(L.gkey);
    const int* tpk = C.template at<int>(L.tp);
    double* mem = C.template at<double>(L.mem);
    DM* chg = C.template at<DM>(L.chg);
    const int* isl = C.template at<int>(L.isl);
    const DM* islmask = C.template at<DM>(L.islmask);
    const DM* cislm = C.contig ? islmask : nullptr;  // closed-form shard_moves
    const DM* isllow = C.template at<DM>(L.isllow);
    int* nwin = C.template at<int>(L.nwin);
    int* fin_src = C.template at<int>(L.fin_src);
    uint64_t* fin_bytes = C.template at<uint64_t>(L.fin_bytes);
    DM* disp_mask = C.template at<DM>(L.disp_mask);
    double* disp_bytes = C.template at<double>(L.disp_bytes);
    int* disp_cnt = C.template at<int>(L.disp_cnt);
    int* eorder = C.template at<int>(L.eorder);
    uint64_t* va = C.template at<uint64_t>(L.va);
    const int* w_cursor = C.template at<int>(L.w_cursor);
    const int eb = w_eb[w], ec = w_ec[w];
    C.first_nc = 1 << 30;

    WS_PH_START(tw);
    // incoming volume per entry (incoming_flows :188-206), entry order (:208-221)
    #pragma unroll 1
    for (int i = lane; i < ec; i += 32) {
        const int k = e_k[eb + i];
        uint64_t v = 0;
        if (home[k] >= 0) {
            v = contb[k];
        } else {
            #pragma unroll 1
            for (uint64_t pr = pred_r[k]; pr; pr &= pr - 1) {
                const int p = by_rank[low_bit(pr)];
                if (home[p] >= 0) v += edgeb[p];
            }
        }
        va[i] = v;
    }
    __syncwarp();
    #pragma unroll 1
    for (int i = lane; i < ec; i += 32) {
        int pos = i;
        if (!C.sequential) {
            pos = 0;
            const int ki = e_k[eb + i];
            #pragma unroll 1
            for (int j = 0; j < ec; ++j) {
                if (j == i) continue;
                const int kj = e_k[eb + j];
                if (va[j] > va[i] || (va[j] == va[i] && idrank[kj] < idrank[ki])) ++pos;
            }
        }
        eorder[pos] = i;
    }
    __syncwarp();
    WS_PH_STOP(tw, 1);
    DM free = C.all;
    uint64_t placed_now = 0;  // entities placed in this wave (K <= 64)
    int cursor = C.sequential ? w_cursor[w] : 0;
    #pragma unroll 1
    for (int oi = 0; oi < ec; ++oi) {
        const int e = eb + eorder[oi];
        const int k = e_k[e], n = e_n[e], lay = e_l[e];
        // flows_in: the entity's own previous placement, else producers in dep order
        int nfin = 0;
        if (home[k] >= 0) {
            if (lane == 0) fin_src[0] = home[k], fin_bytes[0] = contb[k];
            nfin = 1;
        } else {
            #pragma unroll 1
            for (uint64_t pr = pred_r[k]; pr; pr &= pr - 1) {
                const int p = by_rank[low_bit(pr)];
                if (home[p] < 0) continue;
                if (lane == 0) fin_src[nfin] = home[p], fin_bytes[nfin] = edgeb[p];
                ++nfin;
            }
        }
        // homes this entry could displace (score_candidate :293-305), in id order
        int ndisp = 0;
        #pragma unroll 1
        for (int base = 0; base < C.K; base += 32) {
            const int r = base + lane;
            bool ok = false;
            int e2 = -1;
            if (r < C.K) {
                e2 = by_rank[r];
                ok = e2 != k && lastw[e2] >= w && !(placed_now >> e2 & 1ull) && home[e2] >= 0;
            }
            const unsigned b = __ballot_sync(kFull, ok);
            if (ok) {
                const int slot = ndisp + __popc(b & ((1u << lane) - 1u));
                const DM hm = e_mask[home[e2]];
                disp_mask[slot] = hm;
                disp_bytes[slot] = static_cast<double>(contb[e2]);
                disp_cnt[slot] = dm_popc(hm);
            }
            ndisp += __popc(b);
        }
        WS_PH_STOP(tw, 2);
        // memory_delta constants (:132-140)
        const double A = lay * (static_cast<double>(memact[k]) / n);
        const double Pm = C.gmul1 * static_cast<double>(parb[k]) / tpk[k];
        const DM charged = chg[gkey[k]];
        const double cap = C.cap;
        // device memory if this entry lands there (memory_delta), once per entry
        double* used_if = C.template at<double>(L.used_if);
        #pragma unroll 1
        for (int dv = lane; dv < N; dv += 32) {
            double delta = A;
            if (!dm_test(charged, dv)) delta += Pm;
            used_if[dv] = mem[dv] + delta;
        }
        __syncwarp();

        auto score_of = [&](DM devs, int rot) {
            ScoreT<DM> s;
            s.valid = 1;
            s.devs = devs;
            s.rot = rot;
            s.islands = 0;
            #pragma unroll 1
            for (int i = 0; i < C.n_isl; ++i) s.islands += dm_any(devs & islmask[i]);
            s.displaced = 0.0;
            #pragma unroll 1
            for (int j = 0; j < ndisp; ++j) {
                const int ov = dm_popc(devs & disp_mask[j]);
                if (ov == 0) continue;
                s.displaced += disp_bytes[j] * static_cast<double>(ov) / static_cast<double>(disp_cnt[j]);
            }
            s.feasible = 1;
            double peak = 0.0;
            #pragma unroll 1
            for (DM d = devs; dm_any(d); d = dm_drop_low(d)) {
                const double used = used_if[dm_low(d)];
                peak = (peak < used) ? used : peak;
            }
            s.feasible = !(peak > cap);  // a device above capacity <=> the maximum is
            s.peak = peak;
            s.inter = 0.0;
            s.intra = 0.0;
            #pragma unroll 1
            for (int f = 0; f < nfin; ++f) {
                uint64_t a, b;
                shard_moves(e_mask[fin_src[f]], devs, fin_bytes[f], isl, cislm, isllow, C.n_isl, a, b);
                s.inter += static_cast<double>(b);
                s.intra += static_cast<double>(a);
            }
            return s;
        };

        ScoreT<DM> chosen;
        chosen.valid = 0;
        if (C.sequential) {
            if (dm_popc(free) >= n) {  // rolling cursor block (:350-358), within the device block
                DM m = dm_zero<DM>();
                #pragma unroll 1
                for (int i = 0; i < n; ++i) m |= dm_bit<DM>(C.dev_off + (cursor + i) % C.dev_cnt);
                chosen = score_of(m, C.dev_off + cursor);
                cursor = (cursor + n) % C.dev_cnt;
            }
        } else {
            // candidate_sets (:223-263): predecessor reuse, island windows, global windows
            const int nfree = dm_popc(free);
            if (nfree >= n) {
                int total = nfin;
                #pragma unroll 1
                for (int i = 0; i < C.n_isl; ++i) {
                    const int c = dm_popc(free & islmask[i]);
                    const int nw = c >= n ? c - n + 1 : 0;
                    if (lane == 0) nwin[i] = nw;
                    total += nw;
                }
                total += nfree - n + 1;
                __syncwarp();
                // compact the candidate list first (ballot + popc), so lanes score
                // in lockstep: skipping inside the scoring loop would split the warp
                DM* cmask = C.template at<DM>(L.cmask);
                int ncand = 0;
                #pragma unroll 1
                for (int base = 0; base < total; base += 32) {
                    const int j = base + lane;
                    DM m = dm_zero<DM>();
                    bool keep = false;
                    if (j < nfin) {
                        m = e_mask[fin_src[j]];
                        keep = dm_popc(m) == n && !dm_any(m & ~free);
                    } else if (j < total) {
                        int r = j - nfin;
                        int i = 0;
                        #pragma unroll 1
                        for (; i < C.n_isl && r >= nwin[i]; ++i) r -= nwin[i];
                        keep = true;
                        if (i < C.n_isl) {
                            m = dm_window(free & islmask[i], r, n);
                        } else {
                            m = dm_window(free, r, n);
                            // with contiguous islands a global window inside one island is
                            // that island's window at the same offset: a duplicate (:232)
#ifndef WS_NO_DEDUP
                            keep = !(C.contig && !dm_any(m & ~C.template at<DM>(L.islfull)[isl[dm_low(m)]]));
#endif
                        }
                    }
                    const unsigned bal = __ballot_sync(kFull, keep);
                    if (keep) cmask[ncand + __popc(bal & ((1u << lane) - 1u))] = m;
                    ncand += __popc(bal);
                }
                __syncwarp();
                if (oi == 0) C.first_nc = ncand;
                WS_PH_STOP(tw, 3);
                WS_PH_COUNT(20, 1);
                WS_PH_COUNT(21, ncand);
                WS_PH_COUNT(22, n);
                WS_PH_COUNT(23, ndisp);
                WS_PH_COUNT(24, nfin);
                WS_PH_COUNT(25, C.n_isl);
                WS_PH_COUNT(26, (ncand + 31) / 32);
                WS_PH_COUNT(27, N);
                const int rounds = oi == 0 ? variant + 1 : 1;  // first entry takes scores[variant]
                ScoreT<DM> prev;
                prev.valid = 0;
                #pragma unroll 1
                for (int rd = 0; rd < rounds; ++rd) {
                    ScoreT<DM> best;
                    best.valid = 0;
                    #pragma unroll 1
                    for (int j = lane; j < ncand; j += 32) {
                        const ScoreT<DM> s = score_of(cmask[j], 0);
                        if (prev.valid && !score_less(prev, s)) continue;  // next distinct rank
                        if (!best.valid || score_less(s, best)) best = s;
                    }
                    WS_PH_STOP(tw, 4);
                    best = warp_min_score(best);
                    WS_PH_STOP(tw, 8);
                    if (!best.valid) break;  // fewer distinct candidates than variant+1
                    prev = best;
                    chosen = best;
                }
            }
        }
        WS_PH_STOP(tw, 4);
        if (!chosen.valid || !chosen.feasible) return 0;
        // commit_memory (:142-149), lane per device
        #pragma unroll 1
        for (int dv = lane; dv < N; dv += 32) {
            if (!dm_test(chosen.devs, dv)) continue;
            double delta = A;
            if (!dm_test(charged, dv)) delta += Pm;
            mem[dv] += delta;
        }
        if (lane == 0) {
            chg[gkey[k]] = charged | chosen.devs;
            e_mask[e] = chosen.devs;
            e_rot[e] = chosen.rot;
        }
        // flow records (:376-400), lane 0 appends in order
        #pragma unroll 1
        for (int f = 0; f < nfin; ++f) {
            uint64_t a, b;
            const int src = fin_src[f];
            shard_moves(e_mask[src], chosen.devs, fin_bytes[f], isl, cislm, isllow, C.n_isl, a, b);
            const int need = (a + b == 0) ? 1 : (a > 0) + (b > 0);
            if (C.nF + need > C.Fcap) {
                if (lane == 0) set_err(C.ctl, WS_E_LIMIT_FLOWS);
                __syncwarp();
                return -1;
            }
            if (lane == 0) {
                const int fw = e_wave[src], fk = e_k[src];
                if (a + b == 0) {
                    C.flows[2 * C.nF] = 0;
                    C.flows[2 * C.nF + 1] = pack_flow(fw, fk, w, k, WS_FLOW_COPY);
                } else {
                    int q = C.nF;
                    if (a > 0) C.flows[2 * q] = a, C.flows[2 * q + 1] = pack_flow(fw, fk, w, k, WS_FLOW_INTRA), ++q;
                    if (b > 0) C.flows[2 * q] = b, C.flows[2 * q + 1] = pack_flow(fw, fk, w, k, WS_FLOW_INTER);
                }
            }
            C.nF += need;
        }
        WS_PH_STOP(tw, 5);
        free &= ~chosen.devs;
        placed_now |= 1ull << k;
        __syncwarp();
    }
    return 1;
}

// Where p_emit reads the schedule tables and the placement: shared memory
// inside k_place, or the schedule record + the placement scratch in k_emit.
template <class DM>
struct EmitSrc {
    const int *by_rank, *w_eb, *w_ec, *e_k, *e_n, *e_l, *e_rot;
    const DM* e_mask;
};

template <class DM>
__device__ void p_emit(PCtx<DM>& C, int p, const char* rec, const RecLayout& RL, const SchedHdr& h,
                       const PlaceArgs& A, const EmitSrc<DM>& S) {
    constexpr int kExt = MaskTraits<DM>::kWords - 1;  // device words 1.. of each entry (N > 64)
    const int lane = C.lane, K = C.K;
    const ws_batch& B = *C.B;
    const int* r_mod_of = reinterpret_cast<const int*>(rec + RL.mod_of);
    const int* r_level = reinterpret_cast<const int*>(rec + RL.level);
    const int* r_up_n = reinterpret_cast<const int*>(rec + RL.up_n);
    const int* r_up_l = reinterpret_cast<const int*>(rec + RL.up_l);
    const int* r_lo_n = reinterpret_cast<const int*>(rec + RL.lo_n);
    const int* r_lo_l = reinterpret_cast<const int*>(rec + RL.lo_l);
    const uint64_t* r_succ = reinterpret_cast<const uint64_t*>(rec + RL.succ_r);
    const int* by_rank = S.by_rank;
    int npieces = 0, nedges = 0;
    #pragma unroll 1
    for (int k = lane; k < K; k += 32) {
        npieces += C.F->npieces[C.mbase + r_mod_of[k]];
        nedges += popc64(r_succ[k]);
    }
    npieces = warp_sum(npieces);
    nedges = warp_sum(nedges);
    const int nL = h.n_levels, nW = h.nW, nE = h.nE, nF = C.nF;
    const int nS = h.scoped ? K : 0;  // (MetaOp, task) of each entity
    // the ext section exists for clusters over 64 devices only (a narrow plan of
    // a wide launch has the narrow record layout; readers go by the plan's N)
    const bool ext_on = kExt > 0 && C.R->n_dev > 64;
    const uint64_t sz = al8(sizeof(ws_out_metaop) * K) + al8(sizeof(ws_out_level) * nL) +
                        al8(sizeof(ws_out_piece) * npieces) + al8(sizeof(ws_out_edge) * nedges) +
                        al8(sizeof(ws_out_wave) * nW) + al8(sizeof(ws_out_entry) * nE) + al8(sizeof(ws_out_flow) * nF) +
                        al8(sizeof(ws_out_scope) * nS) + (ext_on ? 8ull * kExt * nE : 0ull);
    unsigned long long off = 0;
    if (lane == 0) off = atomicAdd(A.arena_top, static_cast<unsigned long long>(sz));
    off = __shfl_sync(kFull, off, 0);
    ws_plan_result* res = A.results + p;
    if (off + sz > A.arena_cap) {
        if (lane == 0) {
            ws_plan_result r{};
            r.status = WS_STATUS_INTERNAL;
            r.err_code = WS_E_ARENA_OVERFLOW;
            *res = r;
        }
        return;
    }
    uint8_t* base = A.arena + off;
    uint64_t o = 0;
    auto* mo = reinterpret_cast<ws_out_metaop*>(base + o);
    o += al8(sizeof(ws_out_metaop) * K);
    auto* lv = reinterpret_cast<ws_out_level*>(base + o);
    o += al8(sizeof(ws_out_level) * nL);
    auto* pc = reinterpret_cast<ws_out_piece*>(base + o);
    o += al8(sizeof(ws_out_piece) * npieces);
    auto* ed = reinterpret_cast<ws_out_edge*>(base + o);
    o += al8(sizeof(ws_out_edge) * nedges);
    auto* wv = reinterpret_cast<ws_out_wave*>(base + o);
    o += al8(sizeof(ws_out_wave) * nW);
    auto* en = reinterpret_cast<ws_out_entry*>(base + o);
    o += al8(sizeof(ws_out_entry) * nE);
    auto* fl = reinterpret_cast<ws_out_flow*>(base + o);
    // lane per MetaOp; piece offsets by a warp prefix sum over piece counts
    #pragma unroll 1
    for (int base = 0, pb0 = 0; base < K; base += 32) {
        const int k = base + lane;
        const int gm = k < K ? C.mbase + r_mod_of[k] : 0;
        const int np = k < K ? C.F->npieces[gm] : 0;
        int incl = np;
        #pragma unroll 1
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, off);
            if (lane >= off) incl += v;
        }
        const int pb = pb0 + incl - np;
        pb0 += __shfl_sync(kFull, incl, 31);
        if (k < K) {
            ws_out_metaop x;
            x.module = r_mod_of[k];
            x.level = r_level[k];
            x.first_layer = 0;
            x.length = B.mod_layers[gm];
            x.piece_begin = pb;
            x.piece_count = np;
            x.upper_n = r_up_n[k];
            x.upper_l = r_up_l[k];
            x.lower_n = r_lo_n[k];
            x.lower_l = r_lo_l[k];
            mo[k] = x;
            const double* src = C.F->pieces + 5 * C.F->piece_off[gm];
            #pragma unroll 1
            for (int i = 0; i < np; ++i)
                pc[pb + i] = ws_out_piece{src[5 * i], src[5 * i + 1], src[5 * i + 2], src[5 * i + 3], src[5 * i + 4]};
        }
    }
    const double* cstar = reinterpret_cast<const double*>(rec + RL.cstar);
    const int* lfw = reinterpret_cast<const int*>(rec + RL.lvl_fw);
    const int* lnw = reinterpret_cast<const int*>(rec + RL.lvl_nw);
    #pragma unroll 1
    for (int l = lane; l < nL; l += 32) lv[l] = ws_out_level{cstar[l], lfw[l], lnw[l]};
    // MetaGraph edges in std::set<pair<string,string>> order: lane per source rank
    #pragma unroll 1
    for (int base = 0, ne0 = 0; base < K; base += 32) {
        const int ra = base + lane;
        const int a = ra < K ? by_rank[ra] : 0;
        const uint64_t succ = ra < K ? r_succ[a] : 0;
        const int cnt = popc64(succ);
        int incl = cnt;
        #pragma unroll 1
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, off);
            if (lane >= off) incl += v;
        }
        int ne = ne0 + incl - cnt;
        ne0 += __shfl_sync(kFull, incl, 31);
        #pragma unroll 1
        for (uint64_t s = succ; s; s &= s - 1) ed[ne++] = ws_out_edge{a, by_rank[low_bit(s)]};
    }
    const double* w_start = reinterpret_cast<const double*>(rec + RL.w_start);
    const double* w_dur = reinterpret_cast<const double*>(rec + RL.w_dur);
    const int* w_level = reinterpret_cast<const int*>(rec + RL.w_level);
    const int* w_eb = S.w_eb;
    const int* w_ec = S.w_ec;
    #pragma unroll 1
    for (int w = lane; w < nW; w += 32) {
        ws_out_wave x;
        x.start = w_start[w];
        x.duration = w_dur[w];
        x.level = w_level[w];
        x.entry_begin = w_eb[w];
        x.n_entries = w_ec[w];
        x.pad = 0;
        wv[w] = x;
    }
    const int* e_k = S.e_k;
    const int* e_n = S.e_n;
    const int* e_l = S.e_l;
    const double* e_span = reinterpret_cast<const double*>(rec + RL.e_span);
    const DM* e_mask = S.e_mask;
    const int* e_rot = S.e_rot;
    #pragma unroll 1
    for (int e = lane; e < nE; e += 32) {
        ws_out_entry x;
        x.span = e_span[e];
        x.devmask = dm_word(e_mask[e], 0);
        x.metaop = e_k[e];
        x.n = e_n[e];
        x.layers = e_l[e];
        x.rot = e_rot[e];
        en[e] = x;
    }
    #pragma unroll 1
    for (int f = lane; f < nF; f += 32) {
        const uint64_t meta = C.flows[2 * f + 1];
        ws_out_flow x;
        x.volume = C.flows[2 * f];
        x.from_wave = static_cast<int>(meta & 0xffff);
        x.from_metaop = static_cast<int>((meta >> 16) & 0x3fff);
        x.mode = static_cast<int>((meta >> 30) & 3);
        x.to_wave = static_cast<int>((meta >> 32) & 0xffff);
        x.to_metaop = static_cast<int>((meta >> 48) & 0xffff);
        x.pad = 0;
        fl[f] = x;
    }
    if (nS) {
        auto* sc = reinterpret_cast<ws_out_scope*>(base + o + al8(sizeof(ws_out_flow) * nF));
        const int* r_met = reinterpret_cast<const int*>(rec + RL.e_met);
        const int* r_task = reinterpret_cast<const int*>(rec + RL.e_task);
        #pragma unroll 1
        for (int k = lane; k < nS; k += 32) sc[k] = ws_out_scope{r_met[k], r_task[k]};
    }
    if constexpr (kExt > 0) {  // device words 1..W-1 of entry e at [e * kExt + j - 1] (ws_abi.h)
        if (ext_on) {
            auto* ext = reinterpret_cast<uint64_t*>(base + o + al8(sizeof(ws_out_flow) * nF) +
                                                    al8(sizeof(ws_out_scope) * nS));
            #pragma unroll 1
            for (int i = lane; i < nE * kExt; i += 32) ext[i] = dm_word(e_mask[i / kExt], 1 + i % kExt);
        }
    }
    if (lane == 0) {
        ws_plan_result r{};
        r.status = WS_STATUS_OK;
        r.n_metaops = K;
        r.n_edges = nedges;
        r.n_levels = nL;
        r.n_waves = nW;
        r.n_entries = nE;
        r.n_flows = nF;
        r.n_pieces = npieces;
        r.n_scopes = nS;
        r.lower_bound = h.lower_bound;
        r.end_time = h.end_time;
        r.offset = off;
        r.size = sz;
        *res = r;
    }
}

#ifndef WS_PLACE_MINB
#define WS_PLACE_MINB 4  // measured (no-unroll build): 4 blocks (<=128 regs) 7.29 ms vs 3 blocks 7.60 ms per 100k
#endif
// Snapshot slot claim / release (lane 0): a free bit of the pool bitmap, or -1
// when every slot is taken (the warp then restores by replay).
__device__ int snap_claim(unsigned* bits, int slots, int start) {
    const int words = (slots + 31) >> 5;
    #pragma unroll 1
    for (int t = 0; t < words; ++t) {
        const int w = (start + t) % words;
        const unsigned valid = (w + 1) * 32 <= slots ? ~0u : ((1u << (slots - w * 32)) - 1u);
        unsigned cur = *reinterpret_cast<volatile unsigned*>(bits + w);
        while ((cur & valid) != valid) {
            const int b = __ffs(~cur & valid) - 1;
            const unsigned old = atomicOr(bits + w, 1u << b);
            if (!(old >> b & 1u)) return w * 32 + b;
            cur = old | (1u << b);
        }
    }
    return -1;
}

__device__ __forceinline__ void snap_release(unsigned* bits, int slot) {
    if (slot >= 0) atomicAnd(bits + (slot >> 5), ~(1u << (slot & 31)));
}

// kSnap: backtracking restores from per-wave snapshots (instantiated for
// batches with baseline-strategy plans, whose placements backtrack deep);
// pure wavefront batches backtrack rarely and keep the replay-only kernel.
// DM: device-mask type (uint64_t: N <= 64, 4 warps per block; DevMask<4>: N <= 256,
// one warp per block for the larger shared working set).
template <bool kSnap, class DM = uint64_t, int WARPS = kPlaceWarps, int MINB = WS_PLACE_MINB, bool FIXED = false>
__global__ void __launch_bounds__(32 * WARPS, MINB) k_place(PlaceArgs A) {
    extern __shared__ __align__(16) char smem_dyn[];
    __shared__ Ctl ctl_s[WARPS];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = blockIdx.x * WARPS + wid;
    if (slot >= A.n_launch) return;
    if (A.n_ids && slot >= *A.n_ids) return;
    const int p = A.plan_ids[slot];
    const char* rec = A.recs + static_cast<int64_t>(A.rec_by_slot ? slot : p) * A.RL.bytes;
    const SchedHdr h = *reinterpret_cast<const SchedHdr*>(rec + A.RL.hdr);
    if (!h.ok) return;  // k_sched already wrote the error result
    const int64_t ridx = A.rec_by_slot ? slot : p;
    if (A.split_emit && lane == 0) A.emit_nf[ridx] = -1;  // set to the flow count once placed
    Ctl* ctl = &ctl_s[wid];
    if (lane == 0) *ctl = Ctl{};
    const ws_plan_rec& R = A.B.plans[p];
    PCtx<DM> C;
    C.B = &A.B;
    C.R = &R;
    C.F = &A.fit;
    C.L = &A.PL;
    C.sm = smem_dyn + wid * A.PL.bytes;
    C.ctl = ctl;
    C.lane = lane;
    C.N = R.n_dev;
    C.gmul1 = 1.0 + R.grad_mult;
    C.cap = static_cast<double>(R.mem_capacity);
    C.sequential = R.sequential;
    C.K = h.K;
    C.mbase = R.mod_begin;
    C.nW = h.nW;
    C.nE = h.nE;
    C.nF = 0;
    C.Fcap = A.caps.F;
    C.G = R.n_groups + h.K;
    C.n_isl = R.n_islands;
    C.all = dm_first<DM>(C.N);
    C.flows = A.flows + static_cast<int64_t>(slot) * A.caps.F * 2;
    const ws_batch& B = A.B;
    constexpr PlSmLayout kL = make_pl_layout(kFixedPlaceCaps, 8);
    const PlSmLayout& L = FIXED ? kL : A.PL;
    const int K = C.K, N = C.N, nW = C.nW, nE = C.nE, G = C.G;
    if (C.G > A.caps.G || C.n_isl > A.caps.IS || nE > A.caps.E || nW > A.caps.W || K > A.caps.M) {
        if (lane == 0) {
            set_err(ctl, WS_E_LIMIT_MODULES);
            write_error(A.results + p, ctl);
        }
        return;
    }
    WS_PH_START(tk);
    // load the schedule and build the entity tables (planner.hpp:99-151)
    const int* r_mod_of = reinterpret_cast<const int*>(rec + A.RL.mod_of);
    const int* r_by_rank = reinterpret_cast<const int*>(rec + A.RL.by_rank);
    const int* r_idrank = reinterpret_cast<const int*>(rec + A.RL.idrank);
    const uint64_t* r_pred = reinterpret_cast<const uint64_t*>(rec + A.RL.pred_r);
    const double* r_frac = reinterpret_cast<const double*>(rec + A.RL.e_frac);
    int* by_rank = C.template at<int>(L.by_rank);
    int* idrank = C.template at<int>(L.idrank);
    int* lastw = C.template at<int>(L.lastw);
    int* home = C.template at<int>(L.home);
    int* lastent = C.template at<int>(L.lastent);
    int* gkey = C.template at<int>(L.gkey);
    int* tpk = C.template at<int>(L.tp);
    uint64_t* pred_r = C.template at<uint64_t>(L.pred_r);
    uint64_t* contb = C.template at<uint64_t>(L.contb);
    uint64_t* edgeb = C.template at<uint64_t>(L.edgeb);
    uint64_t* memact = C.template at<uint64_t>(L.memact);
    uint64_t* parb = C.template at<uint64_t>(L.parb);
    // every global load of an iteration first, then the shared stores: the
    // compiler cannot move loads across the (possibly aliasing) generic stores,
    // so interleaving them would serialize one DRAM round trip per field
    #pragma unroll 1
    for (int k = lane; k < K; k += 32) {
        const int rb = r_by_rank[k], ir = r_idrank[k], mo = r_mod_of[k];
        const uint64_t pr = r_pred[k];
        const double frac = r_frac[k];  // batch_fraction (build_memory_model / build_flow_inputs)
        const int gm = C.mbase + mo;
        const int Lk = B.mod_layers[gm];  // one MetaOp per module: length == layers
        const uint64_t par = B.mod_param[gm], act = B.mod_act[gm], out = B.mod_out[gm];
        const int grp0 = B.mod_group[gm], al0 = B.mod_alias[gm], tp = B.mod_tp[gm];
        by_rank[k] = rb;
        idrank[k] = ir;
        pred_r[k] = pr;
        parb[k] = static_cast<uint64_t>(static_cast<double>(par) * Lk / Lk);
        memact[k] = static_cast<uint64_t>(static_cast<double>(act) * frac);
        contb[k] = static_cast<uint64_t>(static_cast<double>(act) * frac);
        const uint64_t edge = out == 0 ? act : out;
        edgeb[k] = static_cast<uint64_t>(static_cast<double>(edge) * frac);
        const int grp = grp0;  // length == layers: the MetaOp covers the whole module
        const int al = h.scoped ? -1 : al0;  // scoped ids "m<k>@<task>" match no param_group
        gkey[k] = grp < 0 ? R.n_groups + k : ((al >= 0 && al < K) ? R.n_groups + al : grp);
        tpk[k] = tp;
        home[k] = -1;
        lastw[k] = -1;
        lastent[k] = -1;
    }
    const int* r_w_eb = reinterpret_cast<const int*>(rec + A.RL.w_eb);
    const int* r_w_ec = reinterpret_cast<const int*>(rec + A.RL.w_ec);
    const int* r_e_k = reinterpret_cast<const int*>(rec + A.RL.e_k);
    const int* r_e_n = reinterpret_cast<const int*>(rec + A.RL.e_n);
    const int* r_e_l = reinterpret_cast<const int*>(rec + A.RL.e_l);
    int* w_eb = C.template at<int>(L.w_eb);
    int* w_ec = C.template at<int>(L.w_ec);
    int* w_cursor = C.template at<int>(L.w_cursor);
    int* variant = C.template at<int>(L.variant);
    int* e_k = C.template at<int>(L.e_k);
    int* e_n = C.template at<int>(L.e_n);
    int* e_l = C.template at<int>(L.e_l);
    int* e_prev = C.template at<int>(L.e_prev);
    int* e_wave = C.template at<int>(L.e_wave);
    DM* e_mask = C.template at<DM>(L.e_mask);
    int* e_rot = C.template at<int>(L.e_rot);
    #pragma unroll 1
    for (int w = lane; w < nW; w += 32) {
        const int eb = r_w_eb[w], ec = r_w_ec[w];
        w_eb[w] = eb;
        w_ec[w] = ec;
        variant[w] = 0;
    }
    #pragma unroll 1
    for (int e = lane; e < nE; e += 32) {
        const int ek = r_e_k[e], en = r_e_n[e], el = r_e_l[e];
        e_k[e] = ek;
        e_n[e] = en;
        e_l[e] = el;
        e_mask[e] = dm_zero<DM>();
        e_rot[e] = 0;
    }
    double* mem = C.template at<double>(L.mem);
    DM* chg = C.template at<DM>(L.chg);
    int* isl = C.template at<int>(L.isl);
    DM* islmask = C.template at<DM>(L.islmask);
    #pragma unroll 1
    for (int d = lane; d < N; d += 32) {
        isl[d] = B.dev_island[R.dev_begin + d];
        mem[d] = 0.0;
    }
    #pragma unroll 1
    for (int g = lane; g < G; g += 32) chg[g] = dm_zero<DM>();
    __syncwarp();
    DM* islfull = C.template at<DM>(L.islfull);
    #pragma unroll 1
    for (int i = 0; i < R.n_islands; ++i) {  // island masks, one ballot per 32 devices
        DM m = dm_zero<DM>();
        #pragma unroll 1
        for (int base = 0; base < N; base += 32) {
            const int d = base + lane;
            dm_or_bits32(m, base, __ballot_sync(kFull, d < N && isl[d] == i));
        }
        if (lane == 0) islfull[i] = m;
    }
    #pragma unroll 1
    for (int w = lane; w < nW; w += 32)
        #pragma unroll 1
        for (int i = 0; i < w_ec[w]; ++i) e_wave[w_eb[w] + i] = w;
    __syncwarp();
    #pragma unroll 1
    for (int e = lane; e < nE; e += 32) {  // previous entry of the same entity
        int pv = -1;
        #pragma unroll 1
        for (int j = e - 1; j >= 0; --j)
            if (e_k[j] == e_k[e]) {
                pv = j;
                break;
            }
        e_prev[e] = pv;
    }
    #pragma unroll 1
    for (int k = lane; k < K; k += 32) {  // last entry / wave of each entity
        #pragma unroll 1
        for (int j = nE - 1; j >= 0; --j)
            if (e_k[j] == k) {
                lastent[k] = j;
                lastw[k] = e_wave[j];
                break;
            }
    }
    __syncwarp();
    WS_PH_STOP(tk, 0);
    // One place() call per placement group: task-level-optimus places every
    // task on its own device block (detail::sub_topology: islands cut to the
    // block) with fresh state; everything else is one group over all waves.
    const int n_pg = h.n_pg;
    const int* r_pg_off = reinterpret_cast<const int*>(rec + A.RL.pg_off);
    const int* r_pg_cnt = reinterpret_cast<const int*>(rec + A.RL.pg_cnt);
    const int* r_pg_wbeg = reinterpret_cast<const int*>(rec + A.RL.pg_wbeg);
    const int* r_pg_wn = reinterpret_cast<const int*>(rec + A.RL.pg_wn);
    const int* r_pg_list = reinterpret_cast<const int*>(rec + A.RL.pg_list);
    int* glist = C.template at<int>(L.glist);
    // backtracking state restore: replay (below) until the plan's first failed
    // wave, then per-wave snapshots in a claimed pool slot (identical doubles:
    // a snapshot holds exactly the state the replay rebuilds)
    int snap_slot = -1;       // claimed pool slot (uniform across the warp)
    int snap_hi = -1;         // snapshots 0..snap_hi of this group are valid
    constexpr int kMW = MaskTraits<DM>::kWords;
    const int snapN = N, snapW = N + G * kMW;  // words per wave state: mem[N], chg[G] (kMW words each)
    auto snap_at = [&](int j) { return A.snap + static_cast<long long>(snap_slot) * A.snap_stride +
                                       static_cast<long long>(j) * snapW; };
    auto snap_save = [&](int j) {  // state before wave j
        double* dst = snap_at(j);
        #pragma unroll 1
        for (int d = lane; d < snapN; d += 32) dst[d] = mem[d];
        #pragma unroll 1
        for (int g = lane; g < G * kMW; g += 32)
            reinterpret_cast<uint64_t*>(dst + snapN)[g] = reinterpret_cast<const uint64_t*>(chg)[g];
    };
    #pragma unroll 1
    for (int grp = 0; grp < (n_pg ? n_pg : 1); ++grp) {
        snap_hi = -1;
        const int goff = n_pg ? r_pg_off[grp] : 0, gcnt = n_pg ? r_pg_cnt[grp] : N;
        const int gn = n_pg ? r_pg_wn[grp] : nW;
        #pragma unroll 1
        for (int i = lane; i < gn; i += 32) glist[i] = n_pg ? r_pg_list[r_pg_wbeg[grp] + i] : i;
        C.dev_off = goff;
        C.dev_cnt = gcnt;
        C.all = dm_range<DM>(goff, gcnt);
        __syncwarp();
        if (lane == 0) {
            int ni = 0, contig = 1;
            #pragma unroll 1
            for (int i = 0; i < R.n_islands; ++i) {  // sub_topology (baselines.hpp:81-93)
                const DM m = islfull[i] & C.all;
                if (!dm_any(m)) continue;
                const int lo = dm_low(m);
                if (m != dm_range<DM>(lo, dm_popc(m))) contig = 0;  // not one run of device indices
                islmask[ni] = m;
                C.template at<DM>(L.isllow)[ni] = dm_first<DM>(lo);
                ++ni;
            }
            int cur = 0;  // sequential-ablation cursor (:331-338) over this call's waves
            #pragma unroll 1
            for (int j = 0; j < gn; ++j) {
                const int w = glist[j];
                w_cursor[w] = cur;
                #pragma unroll 1
                for (int i = 0; i < w_ec[w]; ++i) cur = (cur + e_n[w_eb[w] + i]) % gcnt;
                variant[j] = 0;
            }
            ctl->i0 = contig;
            ctl->i1 = ni;
        }
        __syncwarp();
        C.contig = ctl->i0;
        C.n_isl = ctl->i1;
        #pragma unroll 1
        for (int d = lane; d < N; d += 32) mem[d] = 0.0;
        #pragma unroll 1
        for (int g = lane; g < G; g += 32) chg[g] = dm_zero<DM>();
        #pragma unroll 1
        for (int k = lane; k < K; k += 32) home[k] = -1;
        __syncwarp();
    // depth-first search over per-wave variants with a bounded attempt budget (:409-441).
    // The reference copies the whole state per placed wave; here the state
    // before wave k is rebuilt on demand by replaying the committed entries of
    // waves 0..k-1 (their device masks are still in e_mask): entries of one wave
    // use disjoint devices, so per device the additions happen in the same order
    // and the doubles are identical.  Only the flow count is recorded per wave.
    int* wave_nf = C.template at<int>(L.nwin) + C.n_isl;  // [W+1] after the window counts
    long long attempts = 0, budget = gn;
    #pragma unroll 1
    for (int d = 0; d < R.bt_depth; ++d) budget *= (R.bt_branching > 1 ? R.bt_branching : 1);
    const int branching = R.sequential ? 1 : R.bt_branching;
    int k = 0;
    bool dirty = false;
    if (lane == 0) wave_nf[0] = C.nF;
    // Repeated attempts are skipped, not re-run.  Variant v of wave k takes rank
    // min(v, c - 1) of its first entry's c sorted candidates, so for v >= c it
    // places exactly what variant v - 1 placed from the same state: a failure
    // fails again, and a success re-runs the subtree below it attempt for
    // attempt (deeper variants are back at 0) until it steps back into wave k.
    // Such an attempt only advances the counter: by 1, or by 1 + the subtree's
    // recorded attempt count.  Skips stay within the budget; an attempt that
    // would cross it runs for real, so the exhaustion error names the same wave.
    // btm[k] = {c of wave k's last attempt, -1 if it failed, else the attempt
    // number it succeeded at, turned into the subtree length on the step-back}.
    int2* btm = C.template at<int2>(L.btm);
    const bool memo = budget < (1ll << 30);
    while (k < gn) {
        WS_PH_COUNT(28, 1);
        if (memo && variant[k] >= 1 && variant[k] < branching) {
            const int2 m = btm[k];
            const long long add = m.y >= 0 ? 1ll + m.y : 1ll;
            if (variant[k] >= m.x && attempts + add <= budget) {
                attempts += add;
                __syncwarp();
                if (lane == 0) variant[k]++;
                __syncwarp();
                continue;
            }
        }
        if (++attempts > budget) {
            if (lane == 0) {
                set_err(ctl, WS_E_BT_BUDGET, k);
                write_error(A.results + p, ctl);
                if (kSnap) snap_release(A.snap_bits, snap_slot);
            }
            return;
        }
        WS_PH_START(tr);
        if (kSnap && dirty && snap_hi >= k) {  // restore the state before wave k from its snapshot
            const double* src = snap_at(k);
            #pragma unroll 1
            for (int d = lane; d < N; d += 32) mem[d] = src[d];
            #pragma unroll 1
            for (int g = lane; g < G * kMW; g += 32)
                reinterpret_cast<uint64_t*>(chg)[g] = reinterpret_cast<const uint64_t*>(src + snapN)[g];
            snap_hi = k;
            C.nF = wave_nf[k];
            WS_PH_STOP(tr, 6);
            dirty = false;
            __syncwarp();
        } else if (dirty) {  // rebuild the state before wave k by replay
            if (kSnap && snap_slot < 0 && A.snap_slots > 0) {
                int sl = 0;
                if (lane == 0) sl = snap_claim(A.snap_bits, A.snap_slots, (blockIdx.x * WARPS + wid) >> 5);
                snap_slot = __shfl_sync(kFull, sl, 0);
            }
            #pragma unroll 1
            for (int d = lane; d < N; d += 32) mem[d] = 0.0;
            #pragma unroll 1
            for (int g = lane; g < G; g += 32) chg[g] = dm_zero<DM>();
            __syncwarp();
            WS_PH_COUNT(29, k);
            #pragma unroll 1
            for (int j = 0; j < k; ++j) {
                if (kSnap && snap_slot >= 0) {
                    __syncwarp();
                    snap_save(j);
                }
                const int w = glist[j];
                #pragma unroll 1
                for (int i = 0; i < w_ec[w]; ++i) {
                    const int e = w_eb[w] + i;
                    const int ke = e_k[e];
                    const double Ae = e_l[e] * (static_cast<double>(memact[ke]) / e_n[e]);
                    const double Pe = C.gmul1 * static_cast<double>(parb[ke]) / tpk[ke];
                    const DM charged = chg[gkey[ke]];
                    #pragma unroll 1
                    for (int dv = lane; dv < N; dv += 32) {
                        if (!dm_test(e_mask[e], dv)) continue;
                        double delta = Ae;
                        if (!dm_test(charged, dv)) delta += Pe;
                        mem[dv] += delta;
                    }
                    __syncwarp();
                    if (lane == 0) chg[gkey[ke]] = charged | e_mask[e];
                    __syncwarp();
                }
            }
            if (kSnap && snap_slot >= 0) {
                __syncwarp();
                snap_save(k);
                snap_hi = k;
            }
            C.nF = wave_nf[k];
            WS_PH_STOP(tr, 6);
            dirty = false;
            __syncwarp();
        }
        if (variant[k] >= branching) {
            __syncwarp();
            if (lane == 0) variant[k] = 0;
            if (k == 0) {
                if (lane == 0) {
                    set_err(ctl, WS_E_NO_PLACEMENT_W0);
                    write_error(A.results + p, ctl);
                    if (kSnap) snap_release(A.snap_bits, snap_slot);
                }
                return;
            }
            --k;
            const int wk = glist[k];
            #pragma unroll 1
            for (int i = lane; i < w_ec[wk]; i += 32) {  // home[] back to "before wave k"
                const int e = w_eb[wk] + i;
                home[e_k[e]] = e_prev[e];
            }
            if (lane == 0) {
                btm[k].y = static_cast<int>(attempts) - btm[k].y;  // subtree attempts incl. this step-back
                variant[k]++;
            }
            dirty = true;
            __syncwarp();
            continue;
        }
        const int wk = glist[k];
        WS_PH_COUNT(30, 1);
        const int r = p_wave<DM, FIXED>(C, wk, variant[k]);
        __syncwarp();
        if (lane == 0) btm[k] = make_int2(C.first_nc, r > 0 ? static_cast<int>(attempts) : -1);
        if (r < 0) {
            if (lane == 0) {
                write_error(A.results + p, ctl);
                if (kSnap) snap_release(A.snap_bits, snap_slot);
            }
            return;
        }
        if (r > 0) {
            if (lane == 0) wave_nf[k + 1] = C.nF;  // flows recorded before wave k+1
            #pragma unroll 1
            for (int i = lane; i < w_ec[wk]; i += 32) {
                const int e = w_eb[wk] + i;
                home[e_k[e]] = e;
            }
            ++k;
            if (kSnap && snap_slot >= 0 && k < gn) {  // snapshot mode: state before the next wave
                snap_save(k);
                snap_hi = k;
            }
        } else {
            if (lane == 0) variant[k]++;
            dirty = true;
        }
        __syncwarp();
    }
    }
    if (lane == 0) if (kSnap) snap_release(A.snap_bits, snap_slot);
    WS_PH_START(te);
    if (A.split_emit) {  // k_emit writes the record: leave the placement behind
        DM* gm = reinterpret_cast<DM*>(A.emit_mask) + ridx * A.caps.E;
        int32_t* gr = A.emit_rot + ridx * A.caps.E;
        const DM* sm_mask = C.template at<DM>(L.e_mask);
        const int* sm_rot = C.template at<int>(L.e_rot);
        #pragma unroll 1
        for (int e = lane; e < nE; e += 32) {
            gm[e] = sm_mask[e];
            gr[e] = sm_rot[e];
        }
        if (lane == 0) A.emit_nf[ridx] = C.nF;
    } else {
        EmitSrc<DM> src;
        src.by_rank = C.template at<int>(L.by_rank);
        src.w_eb = C.template at<int>(L.w_eb);
        src.w_ec = C.template at<int>(L.w_ec);
        src.e_k = C.template at<int>(L.e_k);
        src.e_n = C.template at<int>(L.e_n);
        src.e_l = C.template at<int>(L.e_l);
        src.e_rot = C.template at<int>(L.e_rot);
        src.e_mask = C.template at<DM>(L.e_mask);
        p_emit(C, p, rec, A.RL, h, A, src);
    }
    WS_PH_STOP(te, 7);
}

// Output records of the plans k_place placed (split emission): a warp per
// launch slot, no shared working set, so many warps keep the record reads and
// stores in flight; the schedule tables come from the k_sched record and the
// placement from k_place's scratch.
template <class DM = uint64_t>
__global__ void __launch_bounds__(32 * kPlaceWarps) k_emit(PlaceArgs A) {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = blockIdx.x * kPlaceWarps + wid;
    if (slot >= A.n_launch) return;
    if (A.n_ids && slot >= *A.n_ids) return;
    const int p = A.plan_ids[slot];
    const char* rec = A.recs + static_cast<int64_t>(A.rec_by_slot ? slot : p) * A.RL.bytes;
    const SchedHdr h = *reinterpret_cast<const SchedHdr*>(rec + A.RL.hdr);
    if (!h.ok) return;
    const int64_t ridx = A.rec_by_slot ? slot : p;
    const int nf = A.emit_nf[ridx];
    if (nf < 0) return;  // k_place wrote the error result
    const ws_plan_rec& R = A.B.plans[p];
    PCtx<DM> C;
    C.B = &A.B;
    C.R = &R;
    C.F = &A.fit;
    C.L = &A.PL;
    C.lane = lane;
    C.K = h.K;
    C.mbase = R.mod_begin;
    C.nF = nf;
    C.flows = A.flows + static_cast<int64_t>(slot) * A.caps.F * 2;
    EmitSrc<DM> src;
    src.by_rank = reinterpret_cast<const int*>(rec + A.RL.by_rank);
    src.w_eb = reinterpret_cast<const int*>(rec + A.RL.w_eb);
    src.w_ec = reinterpret_cast<const int*>(rec + A.RL.w_ec);
    src.e_k = reinterpret_cast<const int*>(rec + A.RL.e_k);
    src.e_n = reinterpret_cast<const int*>(rec + A.RL.e_n);
    src.e_l = reinterpret_cast<const int*>(rec + A.RL.e_l);
    src.e_rot = A.emit_rot + ridx * A.caps.E;
    src.e_mask = reinterpret_cast<const DM*>(A.emit_mask) + ridx * A.caps.E;
    p_emit(C, p, rec, A.RL, h, A, src);
}

}  // namespace wsdev
