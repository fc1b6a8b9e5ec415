// kcommon.cuh — pieces shared by the planner kernels k_sched and k_place:
// the per-warp control block, read-only T-table/curve access, the
// reference's numeric kernels (inverse_exact, shard_moves), placement scores
// and warp reductions.
#pragma once
#include "common.cuh"
#include "fit.cuh"
#include "mask.cuh"

namespace wsdev {

struct Ctl {  // per-warp control block (shared memory)
    int err;
    int pad;
    long long a, b;
    double x, y;
    int i0, i1, i2, i3;
    double d0;
};

__device__ __forceinline__ bool set_err(Ctl* ctl, int code, long long a = 0, long long b = 0) {
    if (!ctl->err) {
        ctl->err = code;
        ctl->a = a;
        ctl->b = b;
    }
    return false;
}

__device__ __forceinline__ int status_of(int code) {
    switch (code) {
        case WS_E_FIT_NONPOSITIVE:
        case WS_E_TP_EXCEEDS:
        case WS_E_TASK_NO_VALID:
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

__device__ __forceinline__ void write_error(ws_plan_result* out, const Ctl* ctl) {
    ws_plan_result r{};
    r.err_code = ctl->err;
    r.status = status_of(ctl->err);
    r.err_a = ctl->a;
    r.err_b = ctl->b;
    r.err_x = ctl->x;
    r.err_y = ctl->y;
    *out = r;
}

// ScalingCurve::eval at integer n (scaling.hpp:66-70) through the T-table;
// n above the curve's n_max is OutOfRange.  gm: global module index.
__device__ __forceinline__ double t_at(const FitOut& F, int gm, int n) {
    return __ldg(F.ttab + static_cast<int64_t>(gm) * F.tstride + (n - 1));
}

// T(n) of module gm's fitted curve with the per-device term scaled by `scale`
// (detail::scale_curve, baselines.hpp:40-44: beta_w *= frac, then eval).
__device__ __forceinline__ double t_scaled(const FitOut& F, const ws_batch& B, int gm, int n, double scale) {
    const double* pc = F.pieces + 5 * F.piece_off[gm];
    const int np = F.npieces[gm];
    int i = 0;
    while (i < np - 1 && !(n <= __ldg(pc + 5 * i + 1) + 1e-9)) ++i;  // locate (scaling.hpp:149-154)
    const double bw = __ldg(pc + 5 * i + 4) * scale;
    return __ldg(pc + 5 * i + 2) + __ldg(pc + 5 * i + 3) * B.mod_c[gm] + bw * B.mod_w[gm] / n;
}

struct TErr {  // error-capturing lookup (first error wins)
    const FitOut* F;
    const int* gm_of;    // metaop -> global module (shared)
    const int* nmax_of;  // metaop -> curve n_max (shared)
    Ctl* ctl;
    const double* scale = nullptr;  // per MetaOp beta_w scale (task-scoped baselines), null: none
    const ws_batch* B = nullptr;
    __device__ double operator()(int k, int n) const {
        if (n > nmax_of[k]) {
            if (!ctl->err) {
                ctl->err = WS_E_EVAL_RANGE;
                ctl->x = n;
                ctl->y = nmax_of[k];
            }
            return 1.0;
        }
        return scale ? t_scaled(*F, *B, gm_of[k], n, scale[k]) : t_at(*F, gm_of[k], n);
    }
};

// ScalingCurve::inverse_exact (scaling.hpp:118-137) over fitted pieces
__device__ __forceinline__ double inverse_exact(const double* __restrict__ pc, int np, double c, double w,
                                                double nmax, double target, double scale = 1.0) {
    auto val = [&](int i, double n) {
        return __ldg(pc + 5 * i + 2) + __ldg(pc + 5 * i + 3) * c + __ldg(pc + 5 * i + 4) * scale * w / n;
    };
    if (target <= val(np - 1, nmax)) return nmax;
    #pragma unroll 1
    for (int i = 0; i < np; ++i) {
        const double lo = __ldg(pc + 5 * i + 0), hi = __ldg(pc + 5 * i + 1);
        const double hi_val = val(i, lo);
        const double lo_val = val(i, hi);
        const double b = __ldg(pc + 5 * i + 4) * scale * w;
        const double base = __ldg(pc + 5 * i + 2) + __ldg(pc + 5 * i + 3) * c;
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

// inverse_exact with every target-independent term hoisted out of the
// bisection loop (curves of <= 2 pieces kept in registers; longer curves use
// the generic routine).  Same expressions, so the same doubles.
struct InvPre {
    int np;  // <= 0: generic path
    const double* pc;
    double c, w, nmax, last, scale;
    double lo[2], hi[2], lov[2], thr[2], b[2], base[2];
    // scale: beta_w factor of a scaled curve (detail::scale_curve), 1.0 otherwise
    __device__ __forceinline__ void init(const double* pc_, int np_, double c_, double w_, double nmax_,
                                         double scale_ = 1.0) {
        pc = pc_;
        c = c_;
        w = w_;
        nmax = nmax_;
        scale = scale_;
        if (np_ > 2) {
            np = -np_;
            return;
        }
        np = np_;
        auto val = [&](int i, double n) {
            return __ldg(pc + 5 * i + 2) + __ldg(pc + 5 * i + 3) * c + __ldg(pc + 5 * i + 4) * scale * w / n;
        };
        last = val(np - 1, nmax);
        #pragma unroll 1
        for (int i = 0; i < np; ++i) {
            lo[i] = __ldg(pc + 5 * i + 0);
            hi[i] = __ldg(pc + 5 * i + 1);
            const double hv = val(i, lo[i]);
            thr[i] = hv + 1e-15 * fabs(hv);
            lov[i] = val(i, hi[i]);
            b[i] = __ldg(pc + 5 * i + 4) * scale * w;
            base[i] = __ldg(pc + 5 * i + 2) + __ldg(pc + 5 * i + 3) * c;
        }
    }
    __device__ __forceinline__ double operator()(double target) const {
        if (np <= 0) return inverse_exact(pc, -np, c, w, nmax, target, scale);
        if (target <= last) return nmax;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            if (i >= np) break;
            if (target > thr[i]) {
                if (b[i] <= 0.0) return 0.0;
                return b[i] / (target - base[i]);
            }
            if (target >= lov[i]) {
                if (b[i] <= 0.0) return lo[i];
                if (target <= base[i]) return hi[i];
                const double v = b[i] / (target - base[i]);
                return v < lo[i] ? lo[i] : (hi[i] < v ? hi[i] : v);
            }
        }
        return nmax;
    }
};

// island_matches (common.cuh) over a device-mask type DM (uint64_t or DevMask<W>)
template <class DM>
__device__ __forceinline__ int island_matches_dm(const DM& A, const DM& B, int M, int P, const DM* islm,
                                                 const DM* lowm, int n_isl) {
    int same = 0;
#pragma unroll 1
    for (int a = 0; a < n_isl; ++a) {
        const int ca = dm_popc(A & islm[a]), cb = dm_popc(B & islm[a]);
        if (!ca || !cb) continue;
        const int sa = dm_popc(A & lowm[a]), sb = dm_popc(B & lowm[a]);
        int q = sa > sb + cb ? (sa - sb - cb) / P : 0;
#pragma unroll 1
        for (int off = q * P + sb; off < sa + ca && off < M; off += P) {
            const int lo = sa > off ? sa : off;
            const int hi = (sa + ca) < (off + cb) ? (sa + ca) : (off + cb);
            if (hi > lo) same += hi - lo;
        }
    }
    return same;
}

// shard_moves (placement.hpp:74-103) on device-index bitmasks; isl = island id per device.
// Unit i pairs sources[i % S] with targets[i % T] (both sorted by device id).
// With contiguous islands (islm/lowm given) the island matches are counted in
// closed form (island_matches), otherwise unit by unit.
template <class DM>
__device__ __forceinline__ void shard_moves(const DM& from, const DM& to, uint64_t full, const int* isl,
                                            const DM* islm, const DM* lowm, int n_isl, uint64_t& intra,
                                            uint64_t& inter) {
    intra = inter = 0;
    if (!dm_any(from) || !dm_any(to)) return;
    const DM shared = from & to;
    DM src = from & ~shared, dst = to & ~shared;
    const int pf = dm_popc(from), pt = dm_popc(to);
    const int units = pf > pt ? pf : pt;
    const int moving = units - dm_popc(shared);
    if (moving == 0) return;
    if (!dm_any(src)) src = from;
    if (!dm_any(dst)) dst = to;
    const double unit_bytes = static_cast<double>(full) / static_cast<double>(units);
    const uint64_t bytes = static_cast<uint64_t>(llround(unit_bytes));
    int same = 0;
    if (islm) {
        const int S = dm_popc(src);  // one of S, T equals moving; the other list cycles
        same = S == moving ? island_matches_dm(src, dst, moving, dm_popc(dst), islm, lowm, n_isl)
                           : island_matches_dm(dst, src, moving, S, islm, lowm, n_isl);
    } else {
        DM rs = src, rt = dst;
#pragma unroll 1
        for (int i = 0; i < moving; ++i) {
            const int s = dm_low(rs);
            rs = dm_drop_low(rs);
            if (!dm_any(rs)) rs = src;
            const int t = dm_low(rt);
            rt = dm_drop_low(rt);
            if (!dm_any(rt)) rt = dst;
            same += isl[s] == isl[t];
        }
    }
    intra = static_cast<uint64_t>(same) * bytes;
    inter = static_cast<uint64_t>(moving - same) * bytes;
}

// Score (placement.hpp:265-283)
template <class DM>
struct ScoreT {
    int valid;
    int feasible;
    int islands;
    int rot;
    double inter, intra, displaced, peak;
    DM devs;
};

template <class DM>
__device__ __forceinline__ bool score_less(const ScoreT<DM>& a, const ScoreT<DM>& b) {
    if (a.feasible != b.feasible) return a.feasible;
    if (a.inter != b.inter) return a.inter < b.inter;
    if (a.intra != b.intra) return a.intra < b.intra;
    if (a.displaced != b.displaced) return a.displaced < b.displaced;
    if (a.islands != b.islands) return a.islands < b.islands;
    if (a.peak != b.peak) return a.peak < b.peak;
    return dm_list_less(a.devs, b.devs);  // sorted device-list lexicographic order
}

// Same order as score_less, as a field-by-field elimination over 32-bit words
// with redux.sync: the doubles are all >= +0.0 (sums/maxima of non-negative
// terms starting at 0.0), whose IEEE bit patterns order like the values; the
// sorted device-list order is the unsigned order of ~brev(devs), word by
// word.  Stops as soon as one lane is left; the winner's Score is then
// broadcast once.
template <class DM>
__device__ __forceinline__ ScoreT<DM> warp_min_score(const ScoreT<DM>& s) {
    unsigned cand = __ballot_sync(kFull, s.valid);
    if (!cand) return s;  // no lane holds a candidate (s.valid == 0 everywhere)
    const int lane = threadIdx.x & 31;
    auto stage = [&](unsigned v) {
        const unsigned key = (cand >> lane & 1u) ? v : 0xffffffffu;
        cand &= __ballot_sync(kFull, key == __reduce_min_sync(kFull, key));
        return (cand & (cand - 1u)) == 0u;
    };
    auto hi = [](double d) { return static_cast<unsigned>(__double_as_longlong(d) >> 32); };
    auto lo = [](double d) { return static_cast<unsigned>(__double_as_longlong(d)); };
    bool one = stage(s.feasible ? 0u : 1u) || stage(hi(s.inter)) || stage(lo(s.inter)) || stage(hi(s.intra)) ||
               stage(lo(s.intra)) || stage(hi(s.displaced)) || stage(lo(s.displaced)) ||
               stage(static_cast<unsigned>(s.islands)) || stage(hi(s.peak)) || stage(lo(s.peak));
#pragma unroll
    for (int i = 0; i < 2 * MaskTraits<DM>::kWords; ++i)
        if (!one) one = stage(dm_key_word(s.devs, i));
    const int src = __ffs(cand) - 1;  // equal devs => equal Scores
    ScoreT<DM> o;
    o.valid = 1;
    o.feasible = __shfl_sync(kFull, s.feasible, src);
    o.islands = __shfl_sync(kFull, s.islands, src);
    o.rot = __shfl_sync(kFull, s.rot, src);
    o.inter = __shfl_sync(kFull, s.inter, src);
    o.intra = __shfl_sync(kFull, s.intra, src);
    o.displaced = __shfl_sync(kFull, s.displaced, src);
    o.peak = __shfl_sync(kFull, s.peak, src);
    o.devs = dm_shfl(s.devs, src);
    return o;
}

__device__ __forceinline__ int warp_sum(int v) {
    #pragma unroll 1
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
}

__device__ __forceinline__ int warp_min_i(int v) {
    #pragma unroll 1
    for (int off = 16; off; off >>= 1) {
        const int o = __shfl_xor_sync(kFull, v, off);
        v = o < v ? o : v;
    }
    return v;
}

__device__ __forceinline__ double warp_max_d(double v) {  // std::max fold, NaN-free inputs
    #pragma unroll 1
    for (int off = 16; off; off >>= 1) {
        const double o = __shfl_xor_sync(kFull, v, off);
        v = (v < o) ? o : v;
    }
    return v;
}

// warp max of doubles >= +0.0 (clocks, durations): their IEEE bit patterns
// order like the values, so two redux.sync steps (high word, then low word
// among the lanes holding the maximum high word) give the exact maximum
__device__ __forceinline__ double warp_max_nonneg(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    const unsigned hi = __reduce_max_sync(kFull, static_cast<unsigned>(b >> 32));
    const unsigned lo = __reduce_max_sync(kFull, static_cast<unsigned>(b >> 32) == hi ? static_cast<unsigned>(b) : 0u);
    return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | lo));
}

__device__ __forceinline__ double warp_min_nonneg(double v) {  // same, minimum (+inf allowed)
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    const unsigned hi = __reduce_min_sync(kFull, static_cast<unsigned>(b >> 32));
    const unsigned lo =
        __reduce_min_sync(kFull, static_cast<unsigned>(b >> 32) == hi ? static_cast<unsigned>(b) : 0xffffffffu);
    return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | lo));
}

__device__ __forceinline__ double warp_min_d(double v) {
    #pragma unroll 1
    for (int off = 16; off; off >>= 1) {
        const double o = __shfl_xor_sync(kFull, v, off);
        v = (o < v) ? o : v;
    }
    return v;
}

// kind bytes of module gm followed by "." and optionally a layer number
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
    #pragma unroll 1
    for (int i = 0; i < l; ++i) {
        const unsigned char ca = static_cast<unsigned char>(a.at(i)), cb = static_cast<unsigned char>(b.at(i));
        if (ca != cb) return ca < cb;
    }
    return la < lb;
}

__device__ __forceinline__ uint64_t al8(uint64_t v) { return (v + 7) & ~7ull; }

// Opt-in phase profiler (-DWS_PHASES builds only): SM cycles per planner phase,
// summed over warps (lane 0), read back with ws_debug_phase_cycles().
#ifdef WS_PHASES
__device__ unsigned long long g_phase_cycles[32];
#define WS_PH_START(t) long long t = clock64()
#define WS_PH_STOP(t, idx)                                                                     \
    do {                                                                                       \
        if ((threadIdx.x & 31) == 0)                                                           \
            atomicAdd(&g_phase_cycles[idx], static_cast<unsigned long long>(clock64() - (t))); \
        t = clock64();                                                                         \
    } while (0)
#define WS_PH_COUNT(idx, v) \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase_cycles[idx], static_cast<unsigned long long>(v))
#else
#define WS_PH_START(t) (void)0
#define WS_PH_STOP(t, idx) (void)0
#define WS_PH_COUNT(idx, v) (void)0
#endif

}  // namespace wsdev
