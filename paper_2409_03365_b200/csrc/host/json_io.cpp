// json_io.cpp — structured (JSON) ingestion of the workload / topology schemas
// (cli.hpp:46-110 workload_from_json, topology_from_json): the JSON form of
// the planner's inputs, read with the same JSON library the reference uses.
// Parity anchor: a JSON workload plans exactly like its text-grammar twin
// through the reference (the schema has no out_bytes).
#include <json.hpp>

#include "wsgpu/planner.hpp"

namespace wsgpu {

WorkloadSpec workload_from_json(const std::string& text) {
    nlohmann::json j;
    try {
        j = nlohmann::json::parse(text);
    } catch (const nlohmann::json::exception& e) {
        throw ParseError(std::string("workload json: ") + e.what());
    }
    try {
        WorkloadSpec spec;
        for (const auto& jm : j.value("modules", nlohmann::json::array())) {
            ModuleDecl m;
            m.kind = jm.at("kind").get<std::string>();
            m.layers = jm.at("layers").get<int>();
            m.input.batch = jm.at("B").get<std::int64_t>();
            m.input.seq = jm.value("seq", std::int64_t{1});
            m.input.hidden = jm.value("hidden", std::int64_t{1});
            m.tp_degree = jm.value("tp", 1);
            m.param_group = jm.value("param_group", std::string{});
            m.param_bytes = jm.value("param_bytes", std::uint64_t{0});
            m.flops_proxy = jm.value("w", 1.0);
            m.comm_proxy = jm.value("c", 0.0);
            m.act_bytes = jm.value("act_bytes", std::uint64_t{0});
            if (!spec.modules.emplace(m.kind, m).second)
                throw ParseError("workload json: duplicate module '" + m.kind + "'");
        }
        for (const auto& jt : j.value("tasks", nlohmann::json::array())) {
            TaskDecl t;
            t.id = jt.at("id").get<std::string>();
            t.flow_text = jt.at("flow").get<std::string>();
            t.flow = parse_flow(t.flow_text, "task " + t.id);
            spec.tasks.push_back(t);
        }
        // The reference iterates j.value(...).items() of a temporary, which is
        // destroyed before the loop runs (dangling iteration proxy, pre-C++23):
        // its truth/profiles/breakpoints maps come out empty.  Read them as the
        // schema intends, keeping the temporaries alive.
        const nlohmann::json jtruth = j.value("truth", nlohmann::json::object());
        const nlohmann::json jprof = j.value("profiles", nlohmann::json::object());
        const nlohmann::json jbps = j.value("breakpoints", nlohmann::json::object());
        for (const auto& [kind, arr] : jtruth.items()) {
            for (const auto& jp : arr) {
                CurvePiece p;
                p.n_lo = jp.at("n_lo").get<double>();
                p.n_hi = jp.at("n_hi").get<double>();
                p.alpha = jp.at("alpha").get<double>();
                p.beta_c = jp.value("beta_c", 0.0);
                p.beta_w = jp.value("beta_w", 0.0);
                spec.truth[kind].push_back(p);
            }
        }
        for (const auto& [kind, arr] : jprof.items()) {
            for (const auto& jp : arr) {
                ProfilePoint p;
                p.n = jp.at("n").get<int>();
                p.time = jp.at("time").get<double>();
                p.parallel_config = jp.value("config", std::string{"dp"});
                spec.profiles[kind].push_back(p);
            }
        }
        for (const auto& [kind, arr] : jbps.items())
            spec.breakpoints[kind] = arr.get<std::vector<int>>();
        validate_workload(spec);
        return spec;
    } catch (const nlohmann::json::exception& e) {
        throw ParseError(std::string("workload json: ") + e.what());
    }
}

ClusterTopology topology_from_json(const std::string& text) {
    try {
        nlohmann::json j = nlohmann::json::parse(text);
        ClusterTopology topo;
        for (const auto& island : j.at("islands")) topo.islands.push_back(island.get<std::vector<int>>());
        topo.intra_bw = j.at("intra_bw").get<double>();
        topo.inter_bw = j.at("inter_bw").get<double>();
        topo.mem_capacity = j.at("mem").get<std::uint64_t>();
        topo.finalize();
        return topo;
    } catch (const nlohmann::json::exception& e) {
        throw ParseError(std::string("topology json: ") + e.what());
    }
}

}  // namespace wsgpu
