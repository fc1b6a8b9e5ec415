// layout.cuh — per-plan scratch layout of the planner kernel.
//
// One warp plans one problem; its working set lives in a per-plan scratch
// region whose array sizes are set by batch-wide caps (max modules M, max
// devices N, wave/entry/flow caps).  Host and device share this function.
#pragma once
#include <cstdint>

namespace wsdev {

struct Caps {
    int M;   // modules (>= MetaOps)
    int N;   // devices
    int W;   // waves
    int E;   // wave entries
    int F;   // flows
    int G;   // placement group keys (param groups + MetaOps)
    int IS;  // islands
};

struct Layout {
    // module / MetaOp arrays [M]
    int adj, tmask, kofm, indeg, keyrank, modat;
    int mod_of, idrank, by_rank, level, predk, pred_r, succ_r, valid;
    int up_n, up_l, lo_n, lo_l, credit, sumlay;
    int gkey, contb, edgeb, memact, parb, lastw, home, lastent;
    // levels
    int lvl_begin, lvl_mem, cstar, lvl_fw, lvl_nw;
    // tuples [2M] and 3 orders
    int tk, tn, tl, tn2, ord;
    // schedule
    int w_level, w_start, w_dur, w_eb, w_ec, w_cursor;
    int e_k, e_n, e_l, e_span, e_mask, e_rot, e_prev, e_wave;
    int f_vol, f_meta;  // f_meta: 6 ints per flow
    // placement
    int mem, chg, snap_mem, snap_chg, snap_nf, variant;
    int isl, islmask, fin_src, fin_bytes, disp_mask, disp_bytes, disp_cnt, eorder, va;
    int bytes;
};

__host__ __device__ inline int lay_align(int v) { return (v + 15) & ~15; }

__host__ __device__ inline Layout make_layout(const Caps& c) {
    Layout L{};
    int o = 0;
    auto take = [&](int bytes) {
        const int at = o;
        o = lay_align(o + bytes);
        return at;
    };
    const int M = c.M, N = c.N, W = c.W, E = c.E, F = c.F, G = c.G;
    L.adj = take(8 * M);
    L.tmask = take(8 * M);
    L.kofm = take(4 * M);
    L.indeg = take(4 * M);
    L.keyrank = take(4 * M);
    L.modat = take(4 * M);
    L.mod_of = take(4 * M);
    L.idrank = take(4 * M);
    L.by_rank = take(4 * M);
    L.level = take(4 * M);
    L.predk = take(8 * M);
    L.pred_r = take(8 * M);
    L.succ_r = take(8 * M);
    L.valid = take(8 * M);
    L.up_n = take(4 * M);
    L.up_l = take(4 * M);
    L.lo_n = take(4 * M);
    L.lo_l = take(4 * M);
    L.credit = take(8 * M);
    L.sumlay = take(4 * M);
    L.gkey = take(4 * M);
    L.contb = take(8 * M);
    L.edgeb = take(8 * M);
    L.memact = take(8 * M);
    L.parb = take(8 * M);
    L.lastw = take(4 * M);
    L.home = take(4 * M);
    L.lastent = take(4 * M);
    L.lvl_begin = take(4 * (M + 1));
    L.lvl_mem = take(4 * M);
    L.cstar = take(8 * M);
    L.lvl_fw = take(4 * M);
    L.lvl_nw = take(4 * M);
    L.tk = take(4 * 2 * M);
    L.tn = take(4 * 2 * M);
    L.tl = take(4 * 2 * M);
    L.tn2 = take(4 * 2 * M);
    L.ord = take(4 * 3 * 2 * M);
    L.w_level = take(4 * W);
    L.w_start = take(8 * W);
    L.w_dur = take(8 * W);
    L.w_eb = take(4 * W);
    L.w_ec = take(4 * W);
    L.w_cursor = take(4 * W);
    L.e_k = take(4 * E);
    L.e_n = take(4 * E);
    L.e_l = take(4 * E);
    L.e_span = take(8 * E);
    L.e_mask = take(8 * E);
    L.e_rot = take(4 * E);
    L.e_prev = take(4 * E);
    L.e_wave = take(4 * E);
    L.f_vol = take(8 * F);
    L.f_meta = take(4 * 6 * F);
    L.mem = take(8 * N);
    L.chg = take(8 * G);
    L.snap_mem = take(8 * N * (W + 1));
    L.snap_chg = take(8 * G * (W + 1));
    L.snap_nf = take(4 * (W + 1));
    L.variant = take(4 * W);
    L.isl = take(4 * N);
    L.islmask = take(8 * (c.IS > 0 ? c.IS : 1));
    L.fin_src = take(4 * (M + 1));
    L.fin_bytes = take(8 * (M + 1));
    L.disp_mask = take(8 * M);
    L.disp_bytes = take(8 * M);
    L.disp_cnt = take(4 * M);
    L.eorder = take(4 * M);
    L.va = take(8 * M);
    L.bytes = o;
    return L;
}

}  // namespace wsdev
