// Host check of the device std::sort emulation (common.cuh ls_sort) against
// libstdc++ std::sort with tie-heavy comparators.
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2409_03365_b200/csrc/device/common.cuh"

struct KeyCmp {
    const int* key;
    long* calls;
    __host__ __device__ bool operator()(int a, int b) const {
        ++*calls;
        return key[a] < key[b];
    }
};

int main() {
    std::mt19937 rng(7);
    long fails = 0, cases = 0;
    for (int n : {0, 1, 2, 3, 5, 15, 16, 17, 18, 31, 32, 33, 47, 64, 100, 128, 257, 1000}) {
        for (int trial = 0; trial < 300; ++trial) {
            const int range = 1 + rng() % (n + 2);
            std::vector<int> key(n);
            for (int& k : key) k = rng() % range;  // many ties
            if (trial % 7 == 0) std::sort(key.begin(), key.end());           // sorted input
            if (trial % 11 == 0) std::sort(key.rbegin(), key.rend());        // reversed input
            std::vector<int> a(n), b(n);
            for (int i = 0; i < n; ++i) a[i] = b[i] = i;
            long ca = 0, cb = 0;
            std::sort(a.begin(), a.end(), KeyCmp{key.data(), &ca});
            KeyCmp c{key.data(), &cb};
            wsdev::ls_sort(b.data(), n, c);
            ++cases;
            if (a != b || ca != cb) ++fails;
        }
    }
    std::printf("%ld cases, %ld mismatches\n", cases, fails);
    return fails != 0;
}
