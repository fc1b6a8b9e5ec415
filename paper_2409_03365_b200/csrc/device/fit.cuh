// fit.cuh — K2 `curve_fit_eval`: per-module scalability-curve fit.
//
// One thread per declared module (every kind, planner.hpp:69), over the SoA
// module arrays (coalesced per field).  Restates materialize_truth/all_ns
// (planner.hpp:43-59), synth_profile with zero noise (scaling.hpp:327-339),
// fit_curve (scaling.hpp:229-322) and evaluates T(n) = eval(n) for every
// integer device count n <= min(N, n_max) into the T-table used by K3/K4.
#pragma once
#include "common.cuh"

namespace wsdev {

constexpr int kInlinePieces = 4;   // pieces stored inline per module
constexpr int kMaxDeclared = 64;   // declared truth pieces per module
constexpr int kMaxBounds = WS_MAX_PIECES + 1;

struct FitOut {
    int32_t* err;        // [modules] ws_err of this module's fit (0 = ok)
    int32_t* err_a;      // [modules]
    int32_t* err_b;      // [modules]
    int32_t* npieces;    // [modules]
    int32_t* nmax;       // [modules] curve n_max (integer)
    int64_t* piece_off;  // [modules] index into pieces (5 doubles each)
    double* pieces;      // inline region [modules*kInlinePieces*5] + overflow pool
    unsigned long long* overflow_top;  // pieces allocated in the overflow pool
    int64_t overflow_base;             // first overflow piece index
    int64_t overflow_cap;              // overflow pieces available
    double* ttab;        // [modules*tstride] T(n) at index n-1
    int tstride;
};

struct DPiece {
    double lo, hi, alpha, bc, bw;
};

__device__ __forceinline__ double piece_value(const DPiece& p, double c, double w, double n) {
    return p.alpha + p.bc * c + p.bw * w / n;
}

// ScalingCurve::locate (scaling.hpp:149-154)
__device__ __forceinline__ int locate_piece(const DPiece* p, int np, double n) {
    #pragma unroll 1
    for (int i = 0; i < np; ++i)
        if (n <= p[i].hi + 1e-9) return i;
    return np - 1;
}

struct PieceLoCmp {  // from_pieces sort key (scaling.hpp:45-46)
    const DPiece* p;
    __device__ bool operator()(int a, int b) const { return p[a].lo < p[b].lo; }
};

// Lanes per module: 1 for large batches (one thread per module), kFitWarp for
// small ones (single-plan latency), where the 32 lanes of a warp run the
// serial fit redundantly (identical values, uniform branches) and split the
// per-n evaluations (truth points, integer anchors, T-table) between them
// through shared memory.  Every value is computed by the same expression in
// both modes, so the results are bit-identical.
constexpr int kFitWarp = 32;
constexpr int kFitWarpMaxModules = 4096;  // batches up to this use kFitWarp

// modules [m_begin, m_end) of the batch (a pipelined chunk, or all of them)
template <int kLanes>
__global__ void __launch_bounds__(128) k_fit(ws_batch B, FitOut out, int m_begin, int m_end) {
    // let a k_sched launched with programmatic stream serialization start its
    // graph stage now; it waits (griddepcontrol.wait) before reading our output
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    constexpr int kWarps = kLanes > 1 ? 128 / kLanes : 1;
    __shared__ double s_tv[kWarps][kLanes > 1 ? WS_MAX_DEVICES : 1];  // truth values n = 1..N
    __shared__ double s_fv[kWarps][kLanes > 1 ? 128 : 1];
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int m = m_begin + gt / kLanes;
    const int lane = kLanes > 1 ? gt % kLanes : 0;
    if (m >= m_end) return;  // uniform over a module's lanes
    const ws_plan_rec& R = B.plans[B.mod_plan[m]];
    const int N = R.n_dev;
    const double c = B.mod_c[m], w = B.mod_w[m];
    int err = 0, ea = 0, eb = 0;
    int np = 0, nmax = 1;
    DPiece fp[WS_MAX_PIECES];
    double fv_local[kLanes > 1 ? 1 : 128];  // T(k) of the fitted curve at k = 1..nmax (when cache_fv)
    double* fv = kLanes > 1 ? s_fv[threadIdx.x / kLanes] : fv_local;
    bool cache_fv = false;

    do {
        if (B.mod_pre_err[m]) {
            err = B.mod_pre_err[m];
            break;
        }
        // breakpoints filtered to 1 < b < N (planner.hpp:72-75)
        int bounds[kMaxBounds + 1];
        int nb = 1;
        bounds[0] = 1;
        int nbreak_in = 0;
        const bool has_prof = B.mod_prof_n[m] >= 0;
        const bool has_truth = B.mod_truth_n[m] >= 0;
        // declared truth, materialized (planner.hpp:43-53)
        DPiece tp[kMaxDeclared];
        int ntp = 0;
        if (!has_prof && has_truth) {
            const int nd = B.mod_truth_n[m];
            if (nd > kMaxDeclared) {
                err = WS_E_LIMIT_PIECES;
                break;
            }
            DPiece raw[kMaxDeclared];
            int order[kMaxDeclared];
            #pragma unroll 1
            for (int i = 0; i < nd; ++i) {
                const double* q = B.truth + 5 * (B.mod_truth_off[m] + i);
                DPiece p{q[0], q[1], q[2], q[3], q[4]};
                if (p.lo >= N) continue;
                p.hi = (static_cast<double>(N) < p.hi) ? static_cast<double>(N) : p.hi;  // std::min
                raw[ntp++] = p;
            }
            if (ntp == 0) {
                err = WS_E_TRUTH_RANGE;
                break;
            }
            raw[ntp - 1].hi = N;
            #pragma unroll 1
            for (int i = 0; i < ntp; ++i) order[i] = i;
            PieceLoCmp cmp{raw};
            ls_sort(order, ntp, cmp);
            #pragma unroll 1
            for (int i = 0; i < ntp; ++i) tp[i] = raw[order[i]];
            if (fabs(tp[0].lo - 1.0) > 1e-9) {
                err = WS_E_CURVE_START;
                break;
            }
            bool contig = true;
            #pragma unroll 1
            for (int i = 0; i + 1 < ntp; ++i)
                if (fabs(tp[i].hi - tp[i + 1].lo) > 1e-9) contig = false;
            if (!contig) {
                err = WS_E_CURVE_CONTIG;
                break;
            }
        } else if (!has_prof && !has_truth) {
            err = WS_E_NO_SOURCE;
            ea = m - R.mod_begin;
            break;
        }
        // point source: profile points, or truth.eval(n) for n = 1..N, each
        // truth value evaluated once (a pure function of n) and reused
        const int npts = has_prof ? B.mod_prof_n[m] : N;
        const int poff = has_prof ? B.mod_prof_off[m] : 0;
        double tv_local[kLanes > 1 ? 1 : WS_MAX_DEVICES];
        double* tv = kLanes > 1 ? s_tv[threadIdx.x / kLanes] : tv_local;
        if (!has_prof)
            #pragma unroll 1
            for (int i = lane; i < N && i < WS_MAX_DEVICES; i += kLanes)
                tv[i] = piece_value(tp[locate_piece(tp, ntp, i + 1)], c, w, static_cast<double>(i + 1));
        if (kLanes > 1) __syncwarp();
        auto point = [&](int i, int& n, double& t) {
            if (has_prof) {
                n = B.prof_n[poff + i];
                t = B.prof_t[poff + i];
            } else {
                n = i + 1;
                t = tv[i];
            }
        };
        // fit_curve argument checks (scaling.hpp:231-238)
        if (npts == 0) {
            err = WS_E_FIT_NO_POINTS;
            break;
        }
        #pragma unroll 1
        for (int i = 0; i < npts && !err; ++i) {
            int n;
            double t;
            point(i, n, t);
            if (n < 1) err = WS_E_FIT_BAD_N;
            else if (t <= 0.0) err = WS_E_FIT_BAD_TIME;
            else if (n > nmax) nmax = n;
        }
        if (err) break;
        // breaks: spec breakpoints, else truth piece ends (planner.hpp:72-87)
        if (B.mod_bp_n[m] >= 0) {
            #pragma unroll 1
            for (int i = 0; i < B.mod_bp_n[m] && !err; ++i) {
                const int b = B.bps[B.mod_bp_off[m] + i];
                if (!(b > 1 && b < N)) continue;
                ++nbreak_in;
                if (b <= bounds[nb - 1] || b >= nmax) {
                    err = WS_E_FIT_BREAKPOINT;
                    ea = b;
                } else if (nb >= kMaxBounds) {
                    err = WS_E_LIMIT_PIECES;
                } else {
                    bounds[nb++] = b;
                }
            }
            if (err) break;
        }
        if (nbreak_in == 0 && !has_prof && has_truth) {
            #pragma unroll 1
            for (int i = 0; i + 1 < ntp && !err; ++i) {
                const int b = static_cast<int>(llround(tp[i].hi));
                if (!(b > 1 && b < N)) continue;
                if (b <= bounds[nb - 1] || b >= nmax) {
                    err = WS_E_FIT_BREAKPOINT;
                    ea = b;
                } else if (nb >= kMaxBounds) {
                    err = WS_E_LIMIT_PIECES;
                } else {
                    bounds[nb++] = b;
                }
            }
            if (err) break;
        }
        bounds[nb++] = nmax;
        // per-piece least squares of time vs 1/n (scaling.hpp:175-190, 248-280)
        np = nb - 1;
        #pragma unroll 1
        for (int i = 0; i < np && !err; ++i) {
            const int lo = bounds[i], hi = bounds[i + 1];
            double sx = 0, sy = 0, sxy = 0, sxx = 0;
            int cnt = 0, nlo = 0x7fffffff, nhi = -1;
            // truth points are n = j + 1 in order: only the piece's own range
            // contributes, visited in the same (ascending) order
            const int j0 = has_prof ? 0 : (i == 0 ? lo - 1 : lo), j1 = has_prof ? npts : (hi < npts ? hi : npts);
            #pragma unroll 1
            for (int j = j0 < 0 ? 0 : j0; j < j1; ++j) {
                int n;
                double t;
                point(j, n, t);
                const bool in = i == 0 ? (n >= lo && n <= hi) : (n > lo && n <= hi);
                if (!in) continue;
                const double x = 1.0 / static_cast<double>(n);
                sx += x;
                sy += t;
                sxy += x * t;
                sxx += x * x;
                ++cnt;
                nlo = n < nlo ? n : nlo;
                nhi = n > nhi ? n : nhi;
            }
            if (cnt == 0 || nlo == nhi) {
                err = WS_E_FIT_PIECE_POINTS;
                ea = lo;
                eb = hi;
                break;
            }
            const double mm = static_cast<double>(cnt);
            const double denom = mm * sxx - sx * sx;
            if (fabs(denom) < 1e-18) {
                err = WS_E_FIT_DEGENERATE_X;
                break;
            }
            const double slope = (mm * sxy - sx * sy) / denom;
            const double intercept = (sy - slope * sx) / mm;
            fp[i] = DPiece{static_cast<double>(lo), static_cast<double>(hi), intercept, 0.0, slope / w};
        }
        if (err) break;
        #pragma unroll 1
        for (int i = 1; i < np; ++i) {  // continuity join (scaling.hpp:282-287)
            const double bound = fp[i].lo;
            const double left = fp[i - 1].alpha + fp[i - 1].bw * w / bound;
            const double right = fp[i].alpha + fp[i].bw * w / bound;
            fp[i].alpha += left - right;
        }
        // isotonic check: PAV changes the anchors iff some adjacent pair violates
        // v[k-1] >= v[k] - 1e-15 (scaling.hpp:193-220, first merge is adjacent)
        // T(k) at the integer anchors k = 1..nmax, evaluated once and reused by the
        // isotonic check, the positivity check and the T-table
        cache_fv = nmax <= 128;
        auto fval = [&](int k) {
            return cache_fv ? fv[k - 1] : piece_value(fp[locate_piece(fp, np, k)], c, w, static_cast<double>(k));
        };
        if (cache_fv)
            #pragma unroll 1
            for (int k = 1 + lane; k <= nmax; k += kLanes)
                fv[k - 1] = piece_value(fp[locate_piece(fp, np, k)], c, w, static_cast<double>(k));
        if (kLanes > 1) __syncwarp();
        bool changed = false;
        double prev = 0.0;
        #pragma unroll 1
        for (int k = 1; k <= nmax; ++k) {
            const double v = fval(k);
            if (k > 1 && prev < v - 1e-15) {
                changed = true;
                break;
            }
            prev = v;
        }
        if (changed) {
            if (nmax - 1 > WS_MAX_PIECES || nmax > 128) {
                err = WS_E_LIMIT_PIECES;
                break;
            }
            double vals[128];
            double bsum[128];
            int bcnt[128];
            int nbk = 0;
            #pragma unroll 1
            for (int k = 1; k <= nmax; ++k) vals[k - 1] = fval(k);
            #pragma unroll 1
            for (int k = 0; k < nmax; ++k) {
                bsum[nbk] = vals[k];
                bcnt[nbk] = 1;
                ++nbk;
                while (nbk >= 2) {
                    if (bsum[nbk - 2] / bcnt[nbk - 2] >= bsum[nbk - 1] / bcnt[nbk - 1] - 1e-15) break;
                    bsum[nbk - 2] += bsum[nbk - 1];
                    bcnt[nbk - 2] += bcnt[nbk - 1];
                    --nbk;
                }
            }
            int idx = 0;
            #pragma unroll 1
            for (int b = 0; b < nbk; ++b) {
                const double mean = bsum[b] / bcnt[b];
                #pragma unroll 1
                for (int k = 0; k < bcnt[b]; ++k) vals[idx++] = mean;
            }
            np = nmax - 1;
            #pragma unroll 1
            for (int k = 1; k < nmax; ++k) {
                const double v0 = vals[k - 1], v1 = vals[k];
                const double b = (v0 - v1) / (1.0 / k - 1.0 / (k + 1.0));
                DPiece q;
                q.lo = k;
                q.hi = k + 1;
                q.bw = b / w;
                q.alpha = v0 - b / k;
                q.bc = 0.0;
                fp[k - 1] = q;
            }
            if (kLanes > 1) __syncwarp();  // every lane has read the old anchors
            if (cache_fv)  // the rebuilt curve's anchor values
                #pragma unroll 1
                for (int k = 1 + lane; k <= nmax; k += kLanes)
                    fv[k - 1] = piece_value(fp[locate_piece(fp, np, k)], c, w, static_cast<double>(k));
            if (kLanes > 1) __syncwarp();
        }
        #pragma unroll 1
        for (int k = 1; k <= nmax; ++k) {  // positivity (scaling.hpp:317-320)
            if (fval(k) <= 0.0) {
                err = WS_E_FIT_NONPOSITIVE;
                ea = k;
                break;
            }
        }
    } while (false);

    if (lane == 0) {
        out.err[m] = err;
        out.err_a[m] = ea;
        out.err_b[m] = eb;
    }
    if (err) {
        if (lane == 0) {
            out.npieces[m] = 0;
            out.nmax[m] = 0;
        }
        return;
    }
    int64_t off = static_cast<int64_t>(m) * kInlinePieces;
    if (np > kInlinePieces) {
        unsigned long long o = 0;
        if (lane == 0) o = atomicAdd(out.overflow_top, static_cast<unsigned long long>(np));
        if (kLanes > 1) o = __shfl_sync(0xffffffffu, o, 0);
        if (static_cast<int64_t>(o) + np > out.overflow_cap) {
            if (lane == 0) out.err[m] = WS_E_LIMIT_PIECES;
            return;
        }
        off = out.overflow_base + static_cast<int64_t>(o);
    }
    if (lane == 0) {
        out.piece_off[m] = off;
        out.npieces[m] = np;
        out.nmax[m] = nmax;
    }
    double* dst = out.pieces + 5 * off;
    #pragma unroll 1
    for (int i = lane; i < np; i += kLanes) {
        dst[5 * i + 0] = fp[i].lo;
        dst[5 * i + 1] = fp[i].hi;
        dst[5 * i + 2] = fp[i].alpha;
        dst[5 * i + 3] = fp[i].bc;
        dst[5 * i + 4] = fp[i].bw;
    }
    const int lim = N < nmax ? N : nmax;
    double* tt = out.ttab + static_cast<int64_t>(m) * out.tstride;
    #pragma unroll 1
    for (int n = 1 + lane; n <= lim; n += kLanes)
        tt[n - 1] = cache_fv ? fv[n - 1] : piece_value(fp[locate_piece(fp, np, n)], c, w, static_cast<double>(n));
}

}  // namespace wsdev
