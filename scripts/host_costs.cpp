// host_costs.cpp — per-plan host costs of the drop-in around the device planner
// (encode, decode, reference-type conversion), measured on the CPU with the
// oracle standing in for the device (its records are bit-identical).
// Build: make -C oracle _ref/host_costs   Run: oracle/_ref/host_costs [count]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "wavesched/planner.hpp"
#include "wavesched/scenarios.hpp"
#include "wsgpu/decode_impl.hpp"
#include "wsgpu/wavesched_compat.hpp"

extern "C" int wso_plan_batch(const ws_batch* in, ws_plan_result* results, uint8_t* arena, uint64_t arena_cap,
                              uint64_t* arena_used);

using clk = std::chrono::steady_clock;
static wavesched::Scenario ref_sweep(long i) {  // SURVEY §8(d) mixture i
    static const char* fam[3] = {"clip-like", "ofasys-like", "qwen-val-like"};
    static const int devs[4] = {8, 16, 32, 64};
    return wavesched::generate_scenario(fam[i % 3], 2 + static_cast<int>((i / 3) % 15), devs[(i / 45) % 4],
                                        static_cast<std::uint64_t>(i));
}
static double us(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); }

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 1000;
    std::vector<wsgpu::Scenario> sc;
    std::vector<wavesched::WorkloadSpec> rspec;
    std::vector<wavesched::ClusterTopology> rtopo;
    for (int i = 0; i < n; ++i) {
        sc.push_back(wsgpu::sweep_mixture(i));
        wavesched::Scenario r = ref_sweep(i);
        rspec.push_back(wavesched::parse_workload(r.workload_text));
        rtopo.push_back(wavesched::parse_topology(r.topology_text));
    }
    std::vector<wsgpu::Problem> probs;
    for (auto& s : sc) probs.push_back({&s.spec, &s.topo, {}});
    // one batch through the oracle: the records the device would return
    wsgpu::EncodedBatch eb = wsgpu::encode_batch(probs, false);
    std::vector<ws_plan_result> res(n);
    uint64_t cap = ws_arena_bound(&eb.view), used = 0;
    std::vector<uint8_t> arena(cap);
    wso_plan_batch(&eb.view, res.data(), arena.data(), cap, &used);

    // each stage in its own pass over all plans (a batch decode's access pattern)
    double t_enc1 = 0, t_dec_g = 0, t_dec = 0, t_conv = 0, t_mirror = 0, t_ref = 0, t_text = 0, t_direct = 0;
    int ok = 0;
    std::vector<wsgpu::PlannerResult> prs(n), prs2(n);
    auto a = clk::now();
    for (int i = 0; i < n; ++i) wsgpu::EncodedBatch one = wsgpu::encode_batch({probs[i]}, false);
    t_enc1 = us(a, clk::now());
    a = clk::now();
    for (int i = 0; i < n; ++i) {
        wsgpu::WorkloadSpec ms = wavesched_gpu::detail::to_mirror(rspec[i]);
        wsgpu::ClusterTopology mt = wavesched_gpu::detail::to_mirror(rtopo[i]);
    }
    t_mirror = us(a, clk::now());
    for (int i = 0; i < n; ++i) ok += res[i].status == 0;
    a = clk::now();
    for (int i = 0; i < n; ++i)
        if (res[i].status == 0) prs[i] = wsgpu::decode_result(probs[i], res[i], arena.data(), true);
    t_dec_g = us(a, clk::now());
    a = clk::now();
    for (int i = 0; i < n; ++i)
        if (res[i].status == 0) prs2[i] = wsgpu::decode_result(probs[i], res[i], arena.data(), false);
    t_dec = us(a, clk::now());
    a = clk::now();
    for (int i = 0; i < n; ++i)
        if (res[i].status == 0) wavesched::PlannerResult rr = wavesched_gpu::detail::to_ref(prs[i], rtopo[i]);
    t_conv = us(a, clk::now());
    a = clk::now();
    for (int i = 0; i < n; ++i)
        if (res[i].status == 0) {
            wavesched::PlannerResult rr;
            wsgpu::detail::decode_into(rspec[i], rtopo[i], 0, 3.0, res[i], arena.data(), true, rr);
        }
    t_direct = us(a, clk::now());
    a = clk::now();
    for (int i = 0; i < n; ++i)
        if (res[i].status == 0) std::string txt = wsgpu::write_plan(prs2[i].plan);
    t_text = us(a, clk::now());
    a = clk::now();
    for (int i = 0; i < n; ++i) {
        try {
            wavesched::PlannerResult ref = wavesched::plan_workload(rspec[i], rtopo[i]);
        } catch (const wavesched::Error&) {
        }
    }
    t_ref = us(a, clk::now());
    std::printf("plans %d (ok %d)\n", n, ok);
    std::printf("encode_batch (1 plan/call)        %8.2f us/plan\n", t_enc1 / n);
    std::printf("reference types -> mirror         %8.2f us/plan\n", t_mirror / n);
    std::printf("decode_result (graph)             %8.2f us/plan\n", t_dec_g / ok);
    std::printf("decode_result (no graph)          %8.2f us/plan\n", t_dec / ok);
    std::printf("mirror -> reference PlannerResult %8.2f us/plan\n", t_conv / ok);
    std::printf("decode_into reference types       %8.2f us/plan\n", t_direct / ok);
    std::printf("write_plan                        %8.2f us/plan\n", t_text / ok);
    std::printf("reference plan_workload           %8.2f us/plan\n", t_ref / n);
    return 0;
}
