// pin.cpp — parity driver built in the build container against the reference
// headers (read in place).  Compares, byte for byte, the reference planner's
// write_plan() text (or exception class + message) with
//   * the oracle restatement (oracle/ws_oracle.cpp)          [--oracle]
//   * the CUDA planner through the C-ABI (needs a GPU)      [--gpu]
// over the bundled acceptance suite, the named BASELINE configs, the
// acceptance fuzz workloads, option variants, and sweep mixtures.
// Also checks the scenario generator restatement against the reference one.
//
// usage: pin [--oracle] [--gpu] [--sweep N] [--sweep-start S] [--fuzz N] [--quiet]
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "wavesched/planner.hpp"
#include "wavesched/scenarios.hpp"

#define main wsref_acceptance_main
#include "tests/acceptance.cpp"
#undef main

#include "wsgpu/planner.hpp"

extern "C" int wso_plan_batch(const ws_batch* in, ws_plan_result* results, uint8_t* arena, uint64_t arena_cap,
                              uint64_t* arena_used);

namespace ws = wavesched;

namespace {

struct Case {
    std::string name;
    std::string workload, topology;
    ws::PlannerOptions ropt;
    wsgpu::PlannerOptions gopt;
};

std::string ref_outcome(const Case& c) {
    try {
        ws::WorkloadSpec spec = ws::parse_workload(c.workload);
        ws::ClusterTopology topo = ws::parse_topology(c.topology);
        return ws::write_plan(ws::plan_workload(spec, topo, c.ropt).plan);
    } catch (const ws::CyclicWorkload& e) {
        return std::string("error CyclicWorkload: ") + e.what() + "\n";
    } catch (const ws::UnknownModule& e) {
        return std::string("error UnknownModule: ") + e.what() + "\n";
    } catch (const ws::EmptyWorkload& e) {
        return std::string("error EmptyWorkload: ") + e.what() + "\n";
    } catch (const ws::InsufficientProfile& e) {
        return std::string("error InsufficientProfile: ") + e.what() + "\n";
    } catch (const ws::ParseError& e) {
        return std::string("error ParseError: ") + e.what() + "\n";
    } catch (const ws::DegenerateFit& e) {
        return std::string("error DegenerateFit: ") + e.what() + "\n";
    } catch (const ws::NoValidAllocation& e) {
        return std::string("error NoValidAllocation: ") + e.what() + "\n";
    } catch (const ws::PlacementInfeasible& e) {
        return std::string("error PlacementInfeasible: ") + e.what() + "\n";
    } catch (const ws::OutOfRange& e) {
        return std::string("error OutOfRange: ") + e.what() + "\n";
    } catch (const ws::InvariantError& e) {
        return std::string("error InvariantError: ") + e.what() + "\n";
    }
}

wsgpu::PlannerOptions mirror(const ws::PlannerOptions& o) {
    wsgpu::PlannerOptions g;
    g.alloc.eps = o.alloc.eps;
    g.alloc.max_iters = o.alloc.max_iters;
    g.alloc.drop_floor = o.alloc.drop_floor;
    g.placement.sequential = o.placement.sequential;
    g.placement.backtrack_depth = o.placement.backtrack_depth;
    g.placement.backtrack_branching = o.placement.backtrack_branching;
    g.grad_opt_multiplier = o.grad_opt_multiplier;
    g.synth_noise = o.synth_noise;
    g.synth_seed = o.synth_seed;
    return g;
}

Case make_case(const std::string& name, const std::string& w, const std::string& t, const ws::PlannerOptions& o = {}) {
    return Case{name, w, t, o, mirror(o)};
}

std::string first_diff(const std::string& a, const std::string& b) {
    std::size_t i = 0;
    while (i < a.size() && i < b.size() && a[i] == b[i]) ++i;
    std::size_t ls = a.rfind('\n', i == 0 ? 0 : i - 1);
    ls = ls == std::string::npos ? 0 : ls + 1;
    auto line = [&](const std::string& s) {
        std::size_t le = s.find('\n', ls);
        return s.substr(ls, le == std::string::npos ? std::string::npos : le - ls);
    };
    return "  ref : " + line(a) + "\n  mine: " + line(b);
}

}  // namespace

int main(int argc, char** argv) {
    bool use_oracle = false, use_gpu = false, quiet = false;
    long sweep_n = 0, sweep_start = 0;
    int fuzz_n = 1000;
    for (int i = 1; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--oracle")) use_oracle = true;
        else if (!std::strcmp(argv[i], "--gpu")) use_gpu = true;
        else if (!std::strcmp(argv[i], "--quiet")) quiet = true;
        else if (!std::strcmp(argv[i], "--sweep")) sweep_n = std::atol(argv[++i]);
        else if (!std::strcmp(argv[i], "--sweep-start")) sweep_start = std::atol(argv[++i]);
        else if (!std::strcmp(argv[i], "--fuzz")) fuzz_n = std::atoi(argv[++i]);
    }
    if (!use_oracle && !use_gpu) use_oracle = true;

    std::vector<Case> cases;
    // bundled acceptance suite (acceptance.cpp:33-40) and the BASELINE configs
    for (const auto& sc : bundled_suite()) {
        ws::Scenario s = ws::generate_scenario(sc.name, sc.tasks, sc.devices, 0);
        cases.push_back(make_case("suite/" + sc.name + "/" + std::to_string(sc.tasks) + "t/" +
                                      std::to_string(sc.devices) + "d",
                                  s.workload_text, s.topology_text));
        ws::PlannerOptions seq;
        seq.placement.sequential = true;
        cases.push_back(make_case("suite-seq/" + sc.name + "/" + std::to_string(sc.tasks) + "t/" +
                                      std::to_string(sc.devices) + "d",
                                  s.workload_text, s.topology_text, seq));
    }
    struct Cfg {
        const char* n;
        int t, d;
    } cfgs[] = {{"clip-like", 4, 8}, {"clip-like", 10, 64}, {"ofasys-like", 7, 32}, {"qwen-val-like", 3, 64}};
    for (const Cfg& c : cfgs) {
        ws::Scenario s = ws::generate_scenario(c.n, c.t, c.d, 0);
        const std::string base = std::string("config/") + c.n + "/" + std::to_string(c.t) + "t/" + std::to_string(c.d) + "d";
        cases.push_back(make_case(base, s.workload_text, s.topology_text));
        ws::PlannerOptions o1;
        o1.placement.backtrack_depth = 0;
        cases.push_back(make_case(base + "/bt0", s.workload_text, s.topology_text, o1));
        ws::PlannerOptions o2;
        o2.alloc.drop_floor = 0.05;
        o2.alloc.eps = 1e-9;
        cases.push_back(make_case(base + "/drop", s.workload_text, s.topology_text, o2));
        ws::PlannerOptions o3;
        o3.synth_noise = 0.02;
        o3.synth_seed = 7;
        cases.push_back(make_case(base + "/noise", s.workload_text, s.topology_text, o3));
        ws::PlannerOptions o4;
        o4.grad_opt_multiplier = 40.0;
        cases.push_back(make_case(base + "/mem", s.workload_text, s.topology_text, o4));
    }
    // acceptance fuzz workloads (acceptance.cpp:451-456)
    {
        ws::Rng rng(2024);
        for (int i = 0; i < fuzz_n; ++i) {
            ws::WorkloadSpec spec = fuzz_workload(rng);
            const int devices = 2 << rng.next_int(0, 3);
            ws::ClusterTopology topo = ws::make_topology(devices, std::max(2, devices / 2), 100e9, 20e9, 1ull << 50);
            cases.push_back(make_case("fuzz/" + std::to_string(i), ws::dump_workload(spec), ws::dump_topology(topo)));
        }
    }
    // generator restatement check + sweep mixtures
    long gen_mismatch = 0;
    for (long i = sweep_start; i < sweep_start + sweep_n; ++i) {
        static const char* fam[3] = {"clip-like", "ofasys-like", "qwen-val-like"};
        static const int devs[4] = {8, 16, 32, 64};
        ws::Scenario s = ws::generate_scenario(fam[i % 3], 2 + static_cast<int>((i / 3) % 15), devs[(i / 45) % 4],
                                               static_cast<std::uint64_t>(i));
        wsgpu::Scenario mine = wsgpu::sweep_mixture(i);
        if (ws::dump_workload(ws::parse_workload(s.workload_text)) != wsgpu::dump_workload(mine.spec) ||
            ws::dump_topology(ws::parse_topology(s.topology_text)) != wsgpu::dump_topology(mine.topo)) {
            if (gen_mismatch++ < 5) std::printf("GEN MISMATCH sweep %ld\n", i);
        }
        cases.push_back(make_case("sweep/" + std::to_string(i), s.workload_text, s.topology_text));
    }

    // mine: parse with the host mirror, encode, plan, decode
    std::vector<wsgpu::WorkloadSpec> specs(cases.size());
    std::vector<wsgpu::ClusterTopology> topos(cases.size());
    std::vector<wsgpu::Problem> probs(cases.size());
    std::vector<std::string> parse_err(cases.size());
    for (std::size_t i = 0; i < cases.size(); ++i) {
        try {
            specs[i] = wsgpu::parse_workload(cases[i].workload);
        } catch (const std::exception& e) {
            parse_err[i] = e.what();
        }
        topos[i] = wsgpu::parse_topology(cases[i].topology);
        probs[i] = wsgpu::Problem{&specs[i], &topos[i], cases[i].gopt};
    }
    wsgpu::EncodedBatch eb = wsgpu::encode_batch(probs, use_gpu);
    std::vector<ws_plan_result> res(cases.size());
    const uint64_t cap = ws_arena_bound(&eb.view);
    std::vector<uint8_t> arena(cap);
    uint64_t used = 0;
    const auto t0 = std::chrono::steady_clock::now();
    if (use_gpu) {
#ifdef WS_HOST_ONLY
        std::printf("built without the CUDA planner\n");
        return 2;
#else
        ws_ctx* ctx = nullptr;
        if (ws_ctx_create(0, &ctx) != 0) {
            std::printf("ws_ctx_create failed\n");
            return 2;
        }
        if (ws_plan_batch_host(ctx, &eb.view, res.data(), arena.data(), cap, &used, nullptr) != 0) {
            std::printf("ws_plan_batch_host failed: %s\n", ws_ctx_last_error(ctx));
            return 2;
        }
        ws_ctx_destroy(ctx);
#endif
    } else {
        wso_plan_batch(&eb.view, res.data(), arena.data(), cap, &used);
    }
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    long bad = 0, errs = 0;
    for (std::size_t i = 0; i < cases.size(); ++i) {
        const std::string ref = ref_outcome(cases[i]);
        std::string mine;
        if (!parse_err[i].empty())
            mine = "parse error: " + parse_err[i];
        else
            mine = wsgpu::plan_text_or_error(probs[i], res[i], arena.data());
        if (ref.rfind("error", 0) == 0) ++errs;
        if (ref != mine) {
            if (bad++ < 10 || !quiet) {
                std::printf("MISMATCH %s\n%s\n", cases[i].name.c_str(), first_diff(ref, mine).c_str());
            }
        }
    }
    std::printf("%s: %zu cases, %ld mismatches, %ld reference errors, %ld generator mismatches, plan time %.3f s\n",
                use_gpu ? "gpu" : "oracle", cases.size(), bad, errs, gen_mismatch, sec);
    return bad || gen_mismatch ? 1 : 0;
}
