// sim_text.cpp — host side of the plan-evaluation path: turns the device
// evaluator's records (ws_sim_result + simulation arena, ws_abi.h) into the
// canonical evaluation text, rebuilding validate_plan's exact violation
// messages (validate.hpp:58-188) from their codes and arguments.
//
// Canonical text (shared with oracle/ref/ref_bridge.cpp sim_text):
//   sim makespan=.. fwd_bwd=.. param_sync=.. send_recv=.. fracs=a,b,c transferred=.. inter=.. timeline=n
//   busy <device>=<seconds> ...      SimulationReport::per_device_busy
//   mem <device>=<bytes> ...         SimulationReport::per_device_peak_memory
//   util <id>=<fraction> ...         SimulationReport::per_entity_utilization
//   valid <ok> <violations>
//   v <message>                      (the first WS_SIM_MAX_VIOLATIONS)
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "bounds.h"
#include "wsgpu/planner.hpp"

namespace wsgpu {

namespace {

std::string mid(int k) { return "m" + std::to_string(k); }

std::string violation_text(const ws_out_violation& v, const ClusterTopology& topo,
                           const std::vector<std::string>& names) {
    auto mid = [&](int k) {
        return k >= 0 && k < static_cast<int>(names.size()) ? names[k] : "m" + std::to_string(k);
    };
    const std::string wave = "wave " + std::to_string(v.wave) + ": ";
    auto dev = [&](int d) {
        return d >= 0 && d < static_cast<int>(topo.devices.size()) ? std::to_string(topo.devices[d])
                                                                   : std::to_string(d);
    };
    switch (v.code) {
        case WS_V_UNKNOWN_ENTITY: return wave + "unknown entity " + mid(v.a);
        case WS_V_DUPLICATE: return wave + "entity " + mid(v.a) + " appears twice";
        case WS_V_SPAN:
            return wave + "entity " + mid(v.a) + " recorded span " + fmt_g(v.x) + " != recomputed " + fmt_g(v.y);
        case WS_V_SPAN_DURATION: return wave + "entry span exceeds wave duration";
        case WS_V_WAVE_DEVICES: return wave + "allocations exceed device count";
        case WS_V_WORK:
            return "entity " + mid(v.a) + ": executed " + std::to_string(v.b) + " of " +
                   std::to_string(static_cast<long long>(v.x)) + " layers";
        case WS_V_CAPACITY:
            return "capacity exceeded at t=" + fmt_g(v.x) + ": " + std::to_string(v.a) + " devices";
        case WS_V_OVERLAP: return "entity " + mid(v.a) + ": overlapping execution intervals";
        case WS_V_DEPENDENCY:
            return "dependency " + mid(v.a) + " -> " + mid(v.b) + " violated: consumer starts at " + fmt_g(v.x) +
                   " before producer ends at " + fmt_g(v.y);
        case WS_V_UNPLACED: return wave + "entity " + mid(v.a) + " unplaced";
        case WS_V_DEVICE_COUNT:
            return wave + "entity " + mid(v.a) + " placed on " + std::to_string(v.b) + " devices, needs " +
                   std::to_string(static_cast<long long>(v.x));
        case WS_V_UNKNOWN_DEVICE: return "unknown device " + dev(v.a);
        case WS_V_DEVICE_TWICE: return wave + "device " + dev(v.a) + " assigned twice";
        case WS_V_MEMORY: {
            std::uint64_t cap;  // ClusterTopology::mem_capacity, bit-copied into y
            std::memcpy(&cap, &v.y, 8);
            return "device " + dev(v.a) + " memory " + fmt_g(v.x) + " exceeds capacity " + std::to_string(cap);
        }
        default: return "violation code " + std::to_string(v.code);
    }
}

}  // namespace

std::vector<std::string> record_entity_names(const Problem& prob, const ws_plan_result& r,
                                             const std::uint8_t* plan_arena) {
    std::vector<std::string> names;
    if (r.n_scopes > 0) {  // task-scoped entities "m<metaop>@<task id>": the record's last section
        auto a8 = [](std::size_t v) { return (v + 7) & ~std::size_t(7); };
        const std::size_t off = r.offset + a8(sizeof(ws_out_metaop) * r.n_metaops) +
                                a8(sizeof(ws_out_level) * r.n_levels) + a8(sizeof(ws_out_piece) * r.n_pieces) +
                                a8(sizeof(ws_out_edge) * r.n_edges) + a8(sizeof(ws_out_wave) * r.n_waves) +
                                a8(sizeof(ws_out_entry) * r.n_entries) + a8(sizeof(ws_out_flow) * r.n_flows);
        for (int k = 0; k < r.n_scopes; ++k) {
            ws_out_scope sc;
            std::memcpy(&sc, plan_arena + off + sizeof(ws_out_scope) * k, sizeof(sc));
            names.push_back(mid(sc.metaop) + "@" + prob.spec->tasks[sc.task].id);
        }
    } else {
        for (int k = 0; k < r.n_metaops; ++k) names.push_back(mid(k));
    }
    return names;
}

std::vector<std::string> violation_messages(const ClusterTopology& topo, const ws_plan_result& r,
                                            const ws_sim_result& s, const std::uint8_t* sim_arena,
                                            const std::vector<std::string>& names) {
    std::vector<std::string> out;
    if (s.status != WS_STATUS_OK) return out;
    const std::size_t N = topo.devices.size();
    const std::size_t o_viol = 16ull * N + 8ull * sim_mask_words(N) + 8 + 8ull * r.n_metaops;
    const int nv = std::min(s.n_violations, WS_SIM_MAX_VIOLATIONS);
    for (int i = 0; i < nv; ++i) {
        ws_out_violation v;
        std::memcpy(&v, sim_arena + s.offset + o_viol + sizeof(ws_out_violation) * i, sizeof(v));
        out.push_back(violation_text(v, topo, names));
    }
    return out;
}

std::string sim_text(const Problem& prob, const ws_plan_result& r, const std::uint8_t* plan_arena,
                     const ws_sim_result& s, const std::uint8_t* sim_arena) {
    if (r.status != WS_STATUS_OK) return plan_text_or_error(prob, r, plan_arena);
    return sim_text_named(*prob.topo, r, s, sim_arena, record_entity_names(prob, r, plan_arena));
}

std::string sim_text_named(const ClusterTopology& topo, const ws_plan_result& r, const ws_sim_result& s,
                           const std::uint8_t* sim_arena, const std::vector<std::string>& names) {
    if (s.status != WS_STATUS_OK) return "error Internal: simulation arena overflow\n";
    auto name = [&](int k) { return k < static_cast<int>(names.size()) ? names[k] : mid(k); };
    const int N = static_cast<int>(topo.devices.size()), K = r.n_metaops;
    const std::uint8_t* b = sim_arena + s.offset;
    auto f64 = [&](std::size_t off) {
        double v;
        std::memcpy(&v, b + off, 8);
        return v;
    };
    auto u64 = [&](std::size_t off) {
        std::uint64_t v;
        std::memcpy(&v, b + off, 8);
        return v;
    };
    std::string out = "sim makespan=" + fmt_exact(s.makespan) + " fwd_bwd=" + fmt_exact(s.fwd_bwd_seconds) +
                      " param_sync=" + fmt_exact(s.param_sync_seconds) + " send_recv=" +
                      fmt_exact(s.send_recv_seconds) + " fracs=" + fmt_exact(s.fwd_bwd_fraction) + "," +
                      fmt_exact(s.param_sync_fraction) + "," + fmt_exact(s.send_recv_fraction) +
                      " transferred=" + fmt_exact(s.total_transferred_bytes) +
                      " inter=" + fmt_exact(s.total_inter_island_bytes) +
                      " timeline=" + std::to_string(s.timeline_items) + "\n";
    const std::size_t TW = sim_mask_words(N);  // busy_mask words
    const std::size_t o_busy = 0, o_bmask = 8ull * N, o_mem = 8ull * N + 8 * TW, o_util = 16ull * N + 8 * TW,
                      o_umask = 16ull * N + 8 * TW + 8ull * K;
    const std::uint64_t umask = u64(o_umask);
    out += "busy";
    for (int d = 0; d < N; ++d)
        if (u64(o_bmask + 8ull * (d / 64)) >> (d % 64) & 1ull)
            out += " " + std::to_string(topo.devices[d]) + "=" + fmt_exact(f64(o_busy + 8ull * d));
    out += "\nmem";
    for (int d = 0; d < N; ++d) out += " " + std::to_string(topo.devices[d]) + "=" + fmt_exact(f64(o_mem + 8ull * d));
    out += "\nutil";
    std::vector<int> ids;
    for (int k = 0; k < K; ++k)
        if (umask >> k & 1ull) ids.push_back(k);
    std::sort(ids.begin(), ids.end(), [&](int a, int c) { return name(a) < name(c); });
    for (int k : ids) out += " " + name(k) + "=" + fmt_exact(f64(o_util + 8ull * k));
    out += "\nvalid " + std::to_string(s.valid) + " " + std::to_string(s.n_violations) + "\n";
    for (const std::string& m : violation_messages(topo, r, s, sim_arena, names)) out += "v " + m + "\n";
    return out;
}

}  // namespace wsgpu

extern "C" uint64_t ws_sim_arena_bound(const ws_batch* in) {
    uint64_t total = 0;
    for (int p = 0; p < in->n_plans; ++p) total += wsi_plan_sim_bound(in->plans + p);
    return total + 4096;
}
