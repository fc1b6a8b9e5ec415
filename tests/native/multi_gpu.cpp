// multi_gpu.cpp — the C-ABI multi-GPU entry points (ws_abi.h):
//   ws_plan_batch_multi  one process, a batch sharded over one context per GPU
//                        (two contexts on device 0 when the box has one GPU)
//   ws_best_nccl         one rank per GPU, the 16-byte min-loc over NCCL
// checked against the single-context call (itself pinned to the oracle and the
// reference by the parity tests): identical result headers (offset aside) and
// record bytes for every plan, and the same global best on every rank.
// Built by tests/test_gpu_multi.py: g++ multi_gpu.cpp -lwsgpu -lnccl -lcudart.
#include <cuda_runtime_api.h>
#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "wsgpu/ws_abi.h"
#include "wsgpu/wsx.h"

static bool same_record(const ws_plan_result& a, const uint8_t* aa, const ws_plan_result& b, const uint8_t* ba) {
    ws_plan_result x = a, y = b;
    x.offset = y.offset = 0;
    if (std::memcmp(&x, &y, sizeof x) != 0) return false;
    return a.status != WS_STATUS_OK || (a.size == b.size && std::memcmp(aa + a.offset, ba + b.offset, a.size) == 0);
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 20000;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        std::printf("no GPU\n");
        return 2;
    }
    ws_options o;
    wsx_default_options(&o);
    wsx_set* set = wsx_set_new();
    wsx_add_sweep(set, 0, n, &o);
    const ws_batch* b = wsx_encode(set, 1);
    const uint64_t cap = ws_arena_bound(b);
    std::vector<ws_plan_result> r1(n), rm(n);
    std::vector<uint8_t> a1(cap), am(cap);
    uint64_t u1 = 0, um = 0;
    // reference run: one context on device 0
    ws_ctx* c0 = nullptr;
    if (ws_ctx_create(0, &c0) || ws_plan_batch_host(c0, b, r1.data(), a1.data(), cap, &u1, nullptr)) {
        std::printf("single-context call failed\n");
        return 1;
    }
    // sharded: one context per GPU (at least two)
    const int nctx = ndev > 1 ? ndev : 2;
    std::vector<ws_ctx*> ctxs(nctx);
    for (int i = 0; i < nctx; ++i)
        if (ws_ctx_create(i % ndev, &ctxs[i])) {
            std::printf("ws_ctx_create(%d) failed\n", i % ndev);
            return 1;
        }
    if (ws_plan_batch_multi(ctxs.data(), nctx, b, rm.data(), am.data(), cap, &um)) {
        std::printf("ws_plan_batch_multi failed: %s\n", ws_ctx_last_error(ctxs[0]));
        return 1;
    }
    // warm timings of both host calls (pinned batch in, host records out)
    auto ms = [](auto&& fn) {
        const auto t0 = std::chrono::steady_clock::now();
        fn();
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    const double t1 = ms([&] { ws_plan_batch_host(c0, b, r1.data(), a1.data(), cap, &u1, nullptr); });
    const double tm = ms([&] { ws_plan_batch_multi(ctxs.data(), nctx, b, rm.data(), am.data(), cap, &um); });
    std::printf("host call ms: 1 context %.2f (%.0f plans/s), %d contexts %.2f (%.0f plans/s)\n", t1, n / t1 * 1e3,
                nctx, tm, n / tm * 1e3);
    long bad = 0, ok = 0;
    for (long p = 0; p < n; ++p) {
        bad += !same_record(r1[p], a1.data(), rm[p], am.data());
        ok += r1[p].status == WS_STATUS_OK;
    }
    std::printf("multi: %d contexts on %d GPU(s), %ld plans (%ld planned), %ld mismatches\n", nctx, ndev, n, ok, bad);
    double k1, km;
    int64_t i1, im;
    ws_best_host(r1.data(), n, 0, &k1, &i1);
    ws_best_host(rm.data(), n, 0, &km, &im);
    std::printf("best (gap): single %.17g @%lld, multi %.17g @%lld\n", k1, (long long)i1, km, (long long)im);
    if (bad || k1 != km || i1 != im) return 1;

    // one rank per GPU: block r of the plans is rank r's; NCCL min-loc of the local bests
    std::vector<ncclComm_t> comms(ndev);
    std::vector<int> devs(ndev);
    for (int i = 0; i < ndev; ++i) devs[i] = i;
    if (ncclCommInitAll(comms.data(), ndev, devs.data()) != ncclSuccess) {
        std::printf("ncclCommInitAll failed\n");
        return 1;
    }
    std::vector<double> gk(ndev);
    std::vector<int64_t> gi(ndev);
    std::vector<int> rc(ndev);
    std::vector<std::thread> th;
    for (int r = 0; r < ndev; ++r)
        th.emplace_back([&, r] {
            const long lo = n * r / ndev, hi = n * (r + 1) / ndev;
            double lk;
            int64_t li;
            ws_best_host(r1.data() + lo, hi - lo, 0, &lk, &li);
            rc[r] = ws_best_nccl(ctxs[r], comms[r], ndev, lk, li >= 0 ? lo + li : -1, &gk[r], &gi[r], nullptr);
        });
    for (auto& t : th) t.join();
    bool agree = true;
    for (int r = 0; r < ndev; ++r) {
        if (rc[r]) std::printf("rank %d: %s\n", r, ws_ctx_last_error(ctxs[r]));
        agree &= rc[r] == 0 && gk[r] == k1 && gi[r] == i1;
    }
    std::printf("nccl min-loc over %d rank(s): %.17g @%lld, %s\n", ndev, gk[0], (long long)gi[0],
                agree ? "all ranks agree with the single-context best" : "MISMATCH");
    for (auto c : comms) ncclCommDestroy(c);
    return agree ? 0 : 1;
}
