// dropin_bench.cpp — measures the drop-in through the reference's OWN types
// (wavesched_gpu::plan_workload, include/wsgpu/wavesched_compat.hpp) next to
// the reference planner itself (wavesched::plan_workload, planner.hpp:156-212)
// in the same process: single-plan latency (first call and warm, 4 BASELINE
// configs), N host threads calling the drop-in concurrently vs the reference
// on the same threads, the batched drop-in (plan_workloads), and the host
// encode / decode cost per plan.  Prints one JSON object (bench.py "dropin").
//
// Built in the build container against the reference headers (oracle/Makefile
// target _ref/dropin_bench); the reference is the baseline here, the product
// under test is libwsgpu.so.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "wavesched/planner.hpp"
#include "wavesched/scenarios.hpp"
#include "wsgpu/decode_impl.hpp"
#include "wsgpu/wavesched_compat.hpp"

using namespace wavesched;
using clk = std::chrono::steady_clock;

namespace {

double ms_since(clk::time_point t0) { return std::chrono::duration<double, std::milli>(clk::now() - t0).count(); }

Scenario sweep(long i) {  // SURVEY §8(d) mixture i
    static const char* fam[3] = {"clip-like", "ofasys-like", "qwen-val-like"};
    static const int devs[4] = {8, 16, 32, 64};
    return generate_scenario(fam[i % 3], 2 + static_cast<int>((i / 3) % 15), devs[(i / 45) % 4],
                             static_cast<std::uint64_t>(i));
}

struct Stats {
    double median, p10, p90;
};
Stats stats(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const std::size_t n = v.size();
    return {v[n / 2], v[n / 10], v[(9 * n) / 10]};
}

std::string js(const Stats& s) {
    char b[160];
    std::snprintf(b, sizeof b, "{\"median\": %.6f, \"p10\": %.6f, \"p90\": %.6f}", s.median, s.p10, s.p90);
    return b;
}

// plans [0, n) with `threads` std::threads, each thread pulling indices
template <typename Fn>
double rate(long n, int threads, Fn&& fn) {
    std::atomic<long> next{0};
    const auto t0 = clk::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&] {
            for (long i; (i = next.fetch_add(1)) < n;) fn(i);
        });
    for (auto& th : pool) th.join();
    return n / (ms_since(t0) / 1000.0);
}

}  // namespace

int main(int argc, char** argv) {
    const int reps = argc > 1 ? std::atoi(argv[1]) : 300;
    const long n_sweep = argc > 2 ? std::atol(argv[2]) : 20000;
    const int threads = argc > 3 ? std::atoi(argv[3]) : static_cast<int>(std::thread::hardware_concurrency());
    struct Cfg {
        const char* name;
        const char* fam;
        int tasks, devices;
    };
    const Cfg cfgs[4] = {{"clip4x8", "clip-like", 4, 8},
                         {"clip10x64", "clip-like", 10, 64},
                         {"ofasys7x32", "ofasys-like", 7, 32},
                         {"qwen3x64", "qwen-val-like", 3, 64}};
    std::vector<WorkloadSpec> cspec;
    std::vector<ClusterTopology> ctopo;
    for (const Cfg& c : cfgs) {
        Scenario sc = generate_scenario(c.fam, c.tasks, c.devices, 0);
        cspec.push_back(parse_workload(sc.workload_text));
        ctopo.push_back(parse_topology(sc.topology_text));
    }
    std::string out = "{";
    // ---- cold start: the process's first drop-in call (CUDA context, module
    // load, planning context and page-locked buffers created on the way) ----
    {
        const auto t0 = clk::now();
        PlannerResult r = wavesched_gpu::plan_workload(cspec[0], ctopo[0]);
        const double cold = ms_since(t0);
        const auto t1 = clk::now();
        PlannerResult r2 = wavesched_gpu::plan_workload(cspec[0], ctopo[0]);
        const double second = ms_since(t1);
        char b[200];
        std::snprintf(b, sizeof b, "\"cold_start_ms\": %.3f, \"second_call_ms\": %.3f, ", cold, second);
        out += b;
    }
    // ---- warm single-plan latency per BASELINE config ----
    out += "\"latency_ms\": {";
    for (int c = 0; c < 4; ++c) {
        std::vector<double> gpu, ref, dec;
        bool same = true;
        for (int i = 0; i < 5; ++i) wavesched_gpu::plan_workload(cspec[c], ctopo[c]);
        for (int i = 0; i < reps; ++i) {
            auto t0 = clk::now();
            PlannerResult g = wavesched_gpu::plan_workload(cspec[c], ctopo[c]);
            gpu.push_back(ms_since(t0));
            t0 = clk::now();
            PlannerResult r = plan_workload(cspec[c], ctopo[c]);
            ref.push_back(ms_since(t0));
            if (i == 0) same = write_plan(g.plan) == write_plan(r.plan);
        }
        // host decode alone (record -> reference PlannerResult), same plan
        wsgpu::plan_workload_raw(wavesched_gpu::detail::to_mirror(cspec[c]), wavesched_gpu::detail::to_mirror(ctopo[c]),
                                 {}, [&](const ws_plan_result& res, const std::uint8_t* arena) {
                                     for (int i = 0; i < reps; ++i) {
                                         const auto t0 = clk::now();
                                         PlannerResult x;
                                         wsgpu::detail::decode_into(cspec[c], ctopo[c], 0, 3.0, res, arena, true, x);
                                         dec.push_back(ms_since(t0));
                                     }
                                 });
        char b[96];
        std::snprintf(b, sizeof b, "\"%s\": {\"samples\": %d, \"identical_plan\": %s, ", cfgs[c].name, reps,
                      same ? "true" : "false");
        out += std::string(c ? ", " : "") + b + "\"dropin\": " + js(stats(gpu)) + ", \"decode\": " + js(stats(dec)) +
               ", \"reference_1_thread\": " + js(stats(ref)) + "}";
    }
    out += "}, ";
    // ---- throughput over a sweep sample: T host threads ----
    std::vector<WorkloadSpec> sspec(n_sweep);
    std::vector<ClusterTopology> stopo(n_sweep);
    for (long i = 0; i < n_sweep; ++i) {
        Scenario sc = sweep(i);
        sspec[i] = parse_workload(sc.workload_text);
        stopo[i] = parse_topology(sc.topology_text);
    }
    std::atomic<long> bad_g{0}, bad_r{0};
    rate(std::min<long>(n_sweep, 64 * threads), threads, [&](long i) {  // warm every thread's context
        try {
            wavesched_gpu::plan_workload(sspec[i], stopo[i]);
        } catch (const Error&) {
        }
    });
    const double g_rate = rate(n_sweep, threads, [&](long i) {
        try {
            PlannerResult r = wavesched_gpu::plan_workload(sspec[i], stopo[i]);
        } catch (const Error&) {
            bad_g++;
        }
    });
    const double r_rate = rate(n_sweep, threads, [&](long i) {
        try {
            PlannerResult r = plan_workload(sspec[i], stopo[i]);
        } catch (const Error&) {
            bad_r++;
        }
    });
    // batched drop-in: one device batch, conversion + decode on all threads;
    // streaming (each result handed over and dropped, like the per-call loops)
    // and collected (every PlannerResult kept: ~150 KB each, page-fault bound)
    std::vector<std::pair<const WorkloadSpec*, const ClusterTopology*>> probs(n_sweep);
    for (long i = 0; i < n_sweep; ++i) probs[i] = {&sspec[i], &stopo[i]};
    std::atomic<long> bad_s{0};
    auto each = [&](std::size_t, PlannerResult&& r, std::exception_ptr e) {
        if (e) bad_s++;
        PlannerResult dropped = std::move(r);
    };
    wavesched_gpu::plan_workloads_each(probs, {}, threads, each);  // warm
    bad_s = 0;
    auto t0 = clk::now();
    wavesched_gpu::plan_workloads_each(probs, {}, threads, each);
    const double s_rate = n_sweep / (ms_since(t0) / 1000.0);
    t0 = clk::now();
    std::vector<wavesched_gpu::Outcome> outs = wavesched_gpu::plan_workloads(probs, {}, threads);
    const double b_rate = n_sweep / (ms_since(t0) / 1000.0);
    long bad_b = 0;
    for (const auto& o : outs) bad_b += o.error ? 1 : 0;
    // the batched results are the reference's (spot check: every 97th plan)
    long mism = 0;
    for (long i = 0; i < n_sweep; i += 97) {
        std::string want;
        try {
            want = write_plan(plan_workload(sspec[i], stopo[i]).plan);
        } catch (const Error& e) {
            want = std::string("error ") + e.what();
        }
        std::string got;
        if (outs[i].error) {
            try {
                std::rethrow_exception(outs[i].error);
            } catch (const Error& e) {
                got = std::string("error ") + e.what();
            }
        } else {
            got = write_plan(outs[i].result.plan);
        }
        mism += got != want;
    }
    // ---- host cost per plan, one thread: encode (reference types -> batch) and
    // decode (record -> reference PlannerResult) ----
    const long n_host = std::min<long>(n_sweep, 2000);
    double enc_ms = 0, dec_ms = 0;
    long n_dec = 0;
    {
        std::vector<wsgpu::WorkloadSpec> ms(n_host);
        std::vector<wsgpu::ClusterTopology> mt(n_host);
        std::vector<wsgpu::Problem> mp(n_host);
        auto t = clk::now();
        for (long i = 0; i < n_host; ++i) {
            ms[i] = wavesched_gpu::detail::to_mirror(sspec[i]);
            mt[i] = wavesched_gpu::detail::to_mirror(stopo[i]);
            mp[i] = wsgpu::Problem{&ms[i], &mt[i], {}};
            wsgpu::EncodedBatch e = wsgpu::encode_batch({mp[i]}, false);
        }
        enc_ms = ms_since(t);
        wsgpu::plan_workloads_raw(mp, 1, [&](const ws_plan_result* res, const std::uint8_t* arena) {
            const auto t1 = clk::now();
            for (long i = 0; i < n_host; ++i) {
                if (res[i].status != WS_STATUS_OK) continue;
                PlannerResult x;
                wsgpu::detail::decode_into(sspec[i], stopo[i], 0, 3.0, res[i], arena, true, x);
                ++n_dec;
            }
            dec_ms = ms_since(t1);
        });
    }
    char b[1400];
    std::snprintf(b, sizeof b,
                  "\"throughput\": {\"plans\": %ld, \"threads\": %d, \"dropin_per_thread_calls_plans_per_s\": %.1f, "
                  "\"reference_plans_per_s\": %.1f, \"dropin_batched_streaming_plans_per_s\": %.1f, "
                  "\"dropin_batched_collected_plans_per_s\": %.1f, \"errors\": [%ld, %ld, %ld, %ld], "
                  "\"batched_spot_mismatches\": %ld}, "
                  "\"encode_us_per_plan\": %.3f, \"decode_us_per_plan\": %.3f, \"host_cost_plans\": %ld",
                  n_sweep, threads, g_rate, r_rate, s_rate, b_rate, bad_g.load(), bad_r.load(), bad_s.load(), bad_b, mism,
                  1000.0 * enc_ms / n_host, 1000.0 * dec_ms / std::max<long>(n_dec, 1), n_host);
    out += b;
    out += "}";
    std::printf("%s\n", out.c_str());
    return 0;
}
