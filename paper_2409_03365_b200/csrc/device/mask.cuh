// mask.cuh — device-set bitmasks for the placement and allocation kernels.
//
// A plan's devices are indices [0, N) in ascending id order; a device set is
// a bitmask over them.  Clusters of up to 64 devices use a plain uint64_t (the
// original, fastest code path); up to 256 devices use DevMask<4>, four words
// with the same operations, so k_sched / k_place are written once over a mask
// type DM and instantiated for both (planner.cu picks by the batch's largest
// cluster).  The reference keeps device lists as std::vector<int> with no cap
// (topology.hpp:15-53); 256 covers the paper's largest planned cluster
// (QWen-VAL on 256 GPUs).
#pragma once
#include <cstdint>

#include "common.cuh"

namespace wsdev {

template <int W>
struct DevMask {
    uint64_t w[W];
};

template <class DM>
struct MaskTraits;
template <>
struct MaskTraits<uint64_t> {
    static constexpr int kWords = 1;
    static constexpr int kBits = 64;
};
template <int W>
struct MaskTraits<DevMask<W>> {
    static constexpr int kWords = W;
    static constexpr int kBits = 64 * W;
};

// ---- uint64_t: thin names over the existing helpers -------------------------
__device__ __forceinline__ bool dm_any(uint64_t m) { return m != 0; }
__device__ __forceinline__ int dm_popc(uint64_t m) { return popc64(m); }
__device__ __forceinline__ int dm_low(uint64_t m) { return low_bit(m); }
__device__ __forceinline__ int dm_high(uint64_t m) { return 63 - __clzll(static_cast<long long>(m)); }
__device__ __forceinline__ uint64_t dm_drop_low(uint64_t m) { return m & (m - 1); }
__device__ __forceinline__ uint64_t dm_lowest(uint64_t m) { return m & (~m + 1); }
__device__ __forceinline__ bool dm_test(uint64_t m, int i) { return m >> i & 1ull; }
__device__ __forceinline__ int dm_select(uint64_t m, int k) { return select_bit(m, k); }
__device__ __forceinline__ uint64_t dm_window(uint64_t pool, int s, int cnt) { return window_mask(pool, s, cnt); }
__device__ __forceinline__ uint64_t dm_shfl(uint64_t m, int src) { return __shfl_sync(kFull, m, src); }
__device__ __forceinline__ uint64_t dm_or_reduce(uint64_t m) {
    const unsigned hi = __reduce_or_sync(kFull, static_cast<unsigned>(m >> 32));
    const unsigned lo = __reduce_or_sync(kFull, static_cast<unsigned>(m));
    return static_cast<uint64_t>(hi) << 32 | lo;
}
// 32-bit words of the sorted-device-list order key (placement.hpp:281):
// a < b iff a holds the lowest differing device, i.e. ~brev(a) < ~brev(b)
__device__ __forceinline__ unsigned dm_key_word(uint64_t m, int i) {
    const uint64_t r = ~__brevll(m);
    return i == 0 ? static_cast<unsigned>(r >> 32) : static_cast<unsigned>(r);
}
// word i of the mask (entry records store words 0 and, for N > 64, 1..W-1)
__device__ __forceinline__ uint64_t dm_word(uint64_t m, int) { return m; }
// m |= bits << base (32 devices [base, base + 32) from one ballot; base % 32 == 0)
__device__ __forceinline__ void dm_or_bits32(uint64_t& m, int base, unsigned bits) {
    m |= static_cast<uint64_t>(bits) << base;
}
__device__ __forceinline__ void dm_set_word(uint64_t& m, int, uint64_t v) { m = v; }

template <class DM>
__device__ __forceinline__ DM dm_zero();
template <>
__device__ __forceinline__ uint64_t dm_zero<uint64_t>() { return 0; }
template <class DM>
__device__ __forceinline__ DM dm_bit(int i);
template <>
__device__ __forceinline__ uint64_t dm_bit<uint64_t>(int i) { return 1ull << i; }
// bits [0, n), n in [0, kBits]
template <class DM>
__device__ __forceinline__ DM dm_first(int n);
template <>
__device__ __forceinline__ uint64_t dm_first<uint64_t>(int n) { return n >= 64 ? ~0ull : ((1ull << n) - 1ull); }
// bits [lo, lo + n)
template <class DM>
__device__ __forceinline__ DM dm_range(int lo, int n) {
    return dm_first<DM>(lo + n) & ~dm_first<DM>(lo);
}

// ---- DevMask<W> ----------------------------------------------------------------
template <int W>
__device__ __forceinline__ DevMask<W> operator&(const DevMask<W>& a, const DevMask<W>& b) {
    DevMask<W> r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.w[i] = a.w[i] & b.w[i];
    return r;
}
template <int W>
__device__ __forceinline__ DevMask<W> operator|(const DevMask<W>& a, const DevMask<W>& b) {
    DevMask<W> r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.w[i] = a.w[i] | b.w[i];
    return r;
}
template <int W>
__device__ __forceinline__ DevMask<W> operator^(const DevMask<W>& a, const DevMask<W>& b) {
    DevMask<W> r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.w[i] = a.w[i] ^ b.w[i];
    return r;
}
template <int W>
__device__ __forceinline__ DevMask<W> operator~(const DevMask<W>& a) {
    DevMask<W> r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.w[i] = ~a.w[i];
    return r;
}
template <int W>
__device__ __forceinline__ DevMask<W>& operator&=(DevMask<W>& a, const DevMask<W>& b) {
    return a = a & b;
}
template <int W>
__device__ __forceinline__ DevMask<W>& operator|=(DevMask<W>& a, const DevMask<W>& b) {
    return a = a | b;
}
template <int W>
__device__ __forceinline__ bool operator==(const DevMask<W>& a, const DevMask<W>& b) {
    bool e = true;
#pragma unroll
    for (int i = 0; i < W; ++i) e &= a.w[i] == b.w[i];
    return e;
}
template <int W>
__device__ __forceinline__ bool operator!=(const DevMask<W>& a, const DevMask<W>& b) {
    return !(a == b);
}
template <int W>
__device__ __forceinline__ bool dm_any(const DevMask<W>& m) {
    uint64_t o = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) o |= m.w[i];
    return o != 0;
}
template <int W>
__device__ __forceinline__ int dm_popc(const DevMask<W>& m) {
    int c = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) c += popc64(m.w[i]);
    return c;
}
template <int W>
__device__ __forceinline__ int dm_low(const DevMask<W>& m) {
#pragma unroll
    for (int i = 0; i < W; ++i)
        if (m.w[i]) return 64 * i + low_bit(m.w[i]);
    return -1;
}
template <int W>
__device__ __forceinline__ int dm_high(const DevMask<W>& m) {
#pragma unroll
    for (int i = W - 1; i >= 0; --i)
        if (m.w[i]) return 64 * i + 63 - __clzll(static_cast<long long>(m.w[i]));
    return -1;
}
template <int W>
__device__ __forceinline__ DevMask<W> dm_lowest(const DevMask<W>& m) {
    DevMask<W> r;
    bool found = false;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        r.w[i] = found ? 0ull : (m.w[i] & (~m.w[i] + 1));
        found |= m.w[i] != 0;
    }
    return r;
}
template <int W>
__device__ __forceinline__ DevMask<W> dm_drop_low(const DevMask<W>& m) {
    DevMask<W> r = m;
    bool done = false;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        if (!done && r.w[i]) {
            r.w[i] &= r.w[i] - 1;
            done = true;
        }
    }
    return r;
}
template <int W>
__device__ __forceinline__ bool dm_test(const DevMask<W>& m, int i) {
    return m.w[i >> 6] >> (i & 63) & 1ull;
}
// index of the k-th (0-based) set bit; m must hold more than k bits
template <int W>
__device__ __forceinline__ int dm_select(const DevMask<W>& m, int k) {
    int base = 0;
    uint64_t x = m.w[W - 1];
#pragma unroll
    for (int i = 0; i < W; ++i) {
        const int c = popc64(m.w[i]);
        if (k < c) {
            x = m.w[i];
            base = 64 * i;
            break;
        }
        k -= c;
    }
    return base + select_bit(x, k);
}
template <int W>
__device__ __forceinline__ DevMask<W> dm_shfl(const DevMask<W>& m, int src) {
    DevMask<W> r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.w[i] = __shfl_sync(kFull, m.w[i], src);
    return r;
}
template <int W>
__device__ __forceinline__ DevMask<W> dm_or_reduce(const DevMask<W>& m) {
    DevMask<W> r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.w[i] = dm_or_reduce(m.w[i]);
    return r;
}
template <int W>
__device__ __forceinline__ unsigned dm_key_word(const DevMask<W>& m, int i) {
    return dm_key_word(m.w[i >> 1], i & 1);
}
template <int W>
__device__ __forceinline__ uint64_t dm_word(const DevMask<W>& m, int i) {
    return m.w[i];
}
template <int W>
__device__ __forceinline__ void dm_set_word(DevMask<W>& m, int i, uint64_t v) {
    m.w[i] = v;
}
template <int W>
__device__ __forceinline__ void dm_or_bits32(DevMask<W>& m, int base, unsigned bits) {
    m.w[base >> 6] |= static_cast<uint64_t>(bits) << (base & 63);
}

template <>
__device__ __forceinline__ DevMask<4> dm_zero<DevMask<4>>() {
    return DevMask<4>{{0, 0, 0, 0}};
}
template <>
__device__ __forceinline__ DevMask<4> dm_bit<DevMask<4>>(int i) {
    DevMask<4> r{{0, 0, 0, 0}};
    r.w[i >> 6] = 1ull << (i & 63);
    return r;
}
template <>
__device__ __forceinline__ DevMask<4> dm_first<DevMask<4>>(int n) {
    DevMask<4> r;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = n - 64 * i;
        r.w[i] = k >= 64 ? ~0ull : (k <= 0 ? 0ull : ((1ull << k) - 1ull));
    }
    return r;
}

// Bits of `pool` from its s-th to its (s+cnt-1)-th set bit (a window of the
// ascending free list, placement.hpp:250-258).
template <int W>
__device__ __forceinline__ DevMask<W> dm_window(const DevMask<W>& pool, int s, int cnt) {
    const int lo = dm_select(pool, s);
    const int hi = dm_select(pool, s + cnt - 1);
    return pool & dm_first<DevMask<W>>(hi + 1) & ~dm_first<DevMask<W>>(lo);
}

// a < b in sorted-device-list order (b != a): a holds the lowest differing device
template <class DM>
__device__ __forceinline__ bool dm_list_less(const DM& a, const DM& b) {
    const DM diff = a ^ b;
    if (!dm_any(diff)) return false;
    return dm_any(a & dm_lowest(diff));
}

}  // namespace wsdev
