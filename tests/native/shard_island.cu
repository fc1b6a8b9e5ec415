// Host check: closed-form island matches (common.cuh island_matches) equal the
// unit-by-unit pairing of shard_moves (placement.hpp:88-97) for contiguous islands.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2409_03365_b200/csrc/device/common.cuh"

static int loop_same(uint64_t src, uint64_t dst, int moving, const std::vector<int>& isl) {
    std::vector<int> s, t;
    for (int d = 0; d < 64; ++d) {
        if (src >> d & 1) s.push_back(d);
        if (dst >> d & 1) t.push_back(d);
    }
    int same = 0;
    for (int i = 0; i < moving; ++i) same += isl[s[i % s.size()]] == isl[t[i % t.size()]];
    return same;
}

using wsdev::island_matches;

int main() {
    std::mt19937_64 rng(11);
    long bad = 0, cases = 0;
    for (int trial = 0; trial < 200000; ++trial) {
        const int N = 1 + rng() % 64;
        // contiguous islands of random sizes, ids in a shuffled order
        std::vector<int> isl(64, -1);
        std::vector<uint64_t> islm, lowm;
        int d = 0;
        while (d < N) {
            const int sz = 1 + rng() % 9;
            uint64_t m = 0;
            for (int k = 0; k < sz && d < N; ++k, ++d) m |= 1ull << d;
            islm.push_back(m);
        }
        std::shuffle(islm.begin(), islm.end(), rng);
        for (size_t a = 0; a < islm.size(); ++a) {
            lowm.push_back((1ull << __builtin_ctzll(islm[a])) - 1);
            for (int x = 0; x < 64; ++x)
                if (islm[a] >> x & 1) isl[x] = static_cast<int>(a);
        }
        const uint64_t all = N == 64 ? ~0ull : ((1ull << N) - 1);
        const uint64_t from = rng() & rng() & all, to = (rng() | (trial & 1 ? 0 : rng())) & all;
        if (!from || !to) continue;
        const uint64_t shared = from & to;
        uint64_t src = from & ~shared, dst = to & ~shared;
        const int pf = __builtin_popcountll(from), pt = __builtin_popcountll(to);
        const int moving = (pf > pt ? pf : pt) - __builtin_popcountll(shared);
        if (moving == 0) continue;
        if (!src) src = from;
        if (!dst) dst = to;
        const int S = __builtin_popcountll(src), T = __builtin_popcountll(dst);
        const int want = loop_same(src, dst, moving, isl);
        const int got = S == moving ? island_matches(src, dst, moving, T, islm.data(), lowm.data(), (int)islm.size())
                                    : island_matches(dst, src, moving, S, islm.data(), lowm.data(), (int)islm.size());
        ++cases;
        if (got != want && bad++ < 5)
            std::printf("mismatch N=%d from=%llx to=%llx want=%d got=%d S=%d T=%d M=%d\n", N,
                        (unsigned long long)from, (unsigned long long)to, want, got, S, T, moving);
    }
    std::printf("%ld cases, %ld mismatches\n", cases, bad);
    return bad != 0;
}
