// common.cuh — device helpers shared by the planner kernels (sm_100a).
#pragma once
#include <cstdint>

#include "wsgpu/ws_abi.h"

namespace wsdev {

constexpr unsigned kFull = 0xffffffffu;

__host__ __device__ __forceinline__ int popc64(uint64_t m) {
#ifdef __CUDA_ARCH__
    return __popcll(m);
#else
    return __builtin_popcountll(m);
#endif
}
// index of the lowest set bit; m != 0 (one BREV+FLO on the nonzero half: cheaper than __ffsll)
__device__ __forceinline__ int low_bit(uint64_t m) {
    const unsigned lo = static_cast<unsigned>(m);
    return lo ? __ffs(lo) - 1 : 31 + __ffs(static_cast<unsigned>(m >> 32));
}

// Index of the k-th (0-based) set bit of m; m must hold more than k bits.
__device__ __forceinline__ int select_bit(uint64_t m, int k) {
    int pos = 0;
    uint32_t x = static_cast<uint32_t>(m);
    int c = __popc(x);
    if (k >= c) {
        k -= c;
        x = static_cast<uint32_t>(m >> 32);
        pos = 32;
    }
    c = __popc(x & 0xffffu);
    if (k >= c) { k -= c; x >>= 16; pos += 16; }
    c = __popc(x & 0xffu);
    if (k >= c) { k -= c; x >>= 8; pos += 8; }
    c = __popc(x & 0xfu);
    if (k >= c) { k -= c; x >>= 4; pos += 4; }
    c = __popc(x & 0x3u);
    if (k >= c) { k -= c; x >>= 2; pos += 2; }
    if (k >= static_cast<int>(x & 1u)) pos += 1;
    return pos;
}

__device__ __forceinline__ uint64_t bits_upto(int hi) {  // bits [0, hi]
    return hi >= 63 ? ~0ull : ((1ull << (hi + 1)) - 1ull);
}

// Bits of `pool` from its s-th to its (s+cnt-1)-th set bit (a window of the
// ascending free list, placement.hpp:250-258).
__device__ __forceinline__ uint64_t window_mask(uint64_t pool, int s, int cnt) {
    const int lo = select_bit(pool, s);
    const int hi = select_bit(pool, s + cnt - 1);
    return pool & bits_upto(hi) & ~((1ull << lo) - 1ull);
}

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(kFull, v, src); }
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) { return __shfl_sync(kFull, v, src); }

// "m<a>" < "m<b>" as std::string (a, b >= 0): compare the decimal spellings
// lexicographically.  Equal lengths order numerically; otherwise compare the
// shorter spelling with the same-length prefix of the longer one, and a proper
// prefix sorts first.
__host__ __device__ __forceinline__ int dec_digits(int v) {
    int d = 1;
    while (v >= 10) v /= 10, ++d;
    return d;
}
__host__ __device__ __forceinline__ bool dec_less(int a, int b) {
    const int da = dec_digits(a), db = dec_digits(b);
    if (da == db) return a < b;
    int p = 1;
    #pragma unroll 1
    for (int i = da < db ? db - da : da - db; i; --i) p *= 10;
    return da < db ? a <= b / p : a / p < b;
}

// "m<a>@<task a>" < "m<b>@<task b>" as std::string (ids of the task-scoped
// entities, baselines.hpp:49-55): the decimal spellings compare digit by
// digit, a spelling that is a prefix of the other meets '@' > digit; equal
// MetaOps order by task id (ta, tb: id ranks).
__host__ __device__ __forceinline__ bool scoped_less(int a, int ta, int b, int tb) {
    if (a == b) return ta < tb;
    const int da = dec_digits(a), db = dec_digits(b);
    if (da == db) return a < b;
    int p = 1;
    #pragma unroll 1
    for (int i = da < db ? db - da : da - db; i; --i) p *= 10;
    if (da < db) {
        const int pre = b / p;
        return pre == a ? false : a < pre;
    }
    const int pre = a / p;
    return pre == b ? true : pre < b;
}

// shard_moves' island-match count (placement.hpp:88-97) in closed form for
// islands that are contiguous device ranges.  Unit i (< M) pairs A[i] with
// B[i mod P], A and B the sorted device lists as masks, |A| = M >= |B| = P
// (exactly one of the reference's two lists cycles).  In sorted order the
// members of island a occupy positions [sa, sa+ca) of A and, in every block q
// of B's cycle, [qP+sb, qP+sb+cb): the matches are the overlaps of those runs.
// lowm[a]: devices below island a's first device.
__host__ __device__ __forceinline__ int island_matches(uint64_t A, uint64_t B, int M, int P, const uint64_t* islm,
                                                       const uint64_t* lowm, int n_isl) {
    int same = 0;
    #pragma unroll 1
    for (int a = 0; a < n_isl; ++a) {
        const int ca = popc64(A & islm[a]), cb = popc64(B & islm[a]);
        if (!ca || !cb) continue;
        const int sa = popc64(A & lowm[a]), sb = popc64(B & lowm[a]);
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

// ---------------------------------------------------------------------------
// Exact emulation of libstdc++-13 std::sort (bits/stl_algo.h __sort /
// __introsort_loop / __final_insertion_sort, bits/stl_heap.h heap helpers) on
// an int array with a strict-weak-order comparator.  Needed because the
// reference sorts with ties; serial, run by one lane.
// ---------------------------------------------------------------------------
template <typename Cmp>
__host__ __device__ void ls_push_heap(int* a, int hole, int top, int value, Cmp& comp) {
    int parent = (hole - 1) / 2;
    while (hole > top && comp(a[parent], value)) {
        a[hole] = a[parent];
        hole = parent;
        parent = (hole - 1) / 2;
    }
    a[hole] = value;
}

template <typename Cmp>
__host__ __device__ void ls_adjust_heap(int* a, int hole, int len, int value, Cmp& comp) {
    const int top = hole;
    int child = hole;
    while (child < (len - 1) / 2) {
        child = 2 * (child + 1);
        if (comp(a[child], a[child - 1])) child--;
        a[hole] = a[child];
        hole = child;
    }
    if ((len & 1) == 0 && child == (len - 2) / 2) {
        child = 2 * (child + 1);
        a[hole] = a[child - 1];
        hole = child - 1;
    }
    ls_push_heap(a, hole, top, value, comp);
}

template <typename Cmp>
__host__ __device__ void ls_heap_sort(int* a, int len, Cmp& comp) {  // __partial_sort(first, last, last)
    if (len >= 2) {
        #pragma unroll 1
        for (int parent = (len - 2) / 2;; --parent) {
            ls_adjust_heap(a, parent, len, a[parent], comp);
            if (parent == 0) break;
        }
    }
    #pragma unroll 1
    for (int last = len; last > 1;) {
        --last;
        const int v = a[last];
        a[last] = a[0];
        ls_adjust_heap(a, 0, last, v, comp);
    }
}

template <typename Cmp>
__host__ __device__ void ls_insertion_sort(int* a, int lo, int hi, Cmp& comp) {
    if (lo == hi) return;
    #pragma unroll 1
    for (int i = lo + 1; i < hi; ++i) {
        const int v = a[i];
        if (comp(v, a[lo])) {
            #pragma unroll 1
            for (int j = i; j > lo; --j) a[j] = a[j - 1];
            a[lo] = v;
        } else {
            int j = i;
            while (comp(v, a[j - 1])) {
                a[j] = a[j - 1];
                --j;
            }
            a[j] = v;
        }
    }
}

template <typename Cmp>
__host__ __device__ void ls_sort(int* a, int n, Cmp& comp) {
    if (n <= 1) return;
#ifdef __CUDA_ARCH__
    int lg = 31 - __clz(n);
#else
    int lg = 31 - __builtin_clz(static_cast<unsigned>(n));
#endif
    // explicit stack reproducing the recursion order of __introsort_loop
    int st_f[40], st_l[40], st_d[40];
    int sp = 0;
    st_f[sp] = 0, st_l[sp] = n, st_d[sp] = 2 * lg, ++sp;
    while (sp) {
        --sp;
        int f = st_f[sp], l = st_l[sp], d = st_d[sp];
        while (l - f > 16) {
            if (d == 0) {
                ls_heap_sort(a + f, l - f, comp);
                break;
            }
            --d;
            // __unguarded_partition_pivot: median of (f+1, mid, l-1) to f
            const int mid = f + (l - f) / 2;
            {
                const int ia = f + 1, ib = mid, ic = l - 1;
                int pick;
                if (comp(a[ia], a[ib])) {
                    if (comp(a[ib], a[ic])) pick = ib;
                    else if (comp(a[ia], a[ic])) pick = ic;
                    else pick = ia;
                } else if (comp(a[ia], a[ic])) pick = ia;
                else if (comp(a[ib], a[ic])) pick = ic;
                else pick = ib;
                const int t = a[f];
                a[f] = a[pick];
                a[pick] = t;
            }
            int lo = f + 1, hi = l;
            while (true) {
                while (comp(a[lo], a[f])) ++lo;
                --hi;
                while (comp(a[f], a[hi])) --hi;
                if (!(lo < hi)) break;
                const int t = a[lo];
                a[lo] = a[hi];
                a[hi] = t;
                ++lo;
            }
            const int cut = lo;
            st_f[sp] = f, st_l[sp] = cut, st_d[sp] = d, ++sp;  // continuation [f, cut)
            f = cut;                                          // recurse into [cut, l) first
        }
    }
    // __final_insertion_sort
    if (n > 16) {
        ls_insertion_sort(a, 0, 16, comp);
        #pragma unroll 1
        for (int i = 16; i < n; ++i) {
            const int v = a[i];
            int j = i;
            while (comp(v, a[j - 1])) {
                a[j] = a[j - 1];
                --j;
            }
            a[j] = v;
        }
    } else {
        ls_insertion_sort(a, 0, n, comp);
    }
}

}  // namespace wsdev
