// model.cpp — value types, text formats and the plan serializer of the host
// drop-in (include/wsgpu/planner.hpp).  Each function names the reference
// function whose observable behaviour it reproduces.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <sstream>

#include "wsgpu/planner.hpp"

namespace wsgpu {

// common.hpp:103-110 — printf %.*g is the text contract of every dump.
std::string fmt_g(double v, int precision) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.*g", precision, v);
    return buf;
}

namespace {

std::vector<std::string> tokens_of(const std::string& line) {
    std::vector<std::string> out;
    std::istringstream is(line);
    for (std::string t; is >> t;) out.push_back(t);
    return out;
}

std::vector<std::string> split_char(const std::string& s, char sep) {
    std::vector<std::string> parts(1);
    for (char ch : s) {
        if (ch == sep)
            parts.emplace_back();
        else
            parts.back().push_back(ch);
    }
    return parts;
}

bool blank_or_comment(const std::string& line) {
    for (unsigned char ch : line) {
        if (ch == '#') return true;
        if (!std::isspace(ch)) return false;
    }
    return true;
}

// key=value tokens after `first` positional tokens (common.hpp:140-192).
struct Fields {
    std::map<std::string, std::string> kv;
    std::string where;

    Fields(const std::vector<std::string>& toks, std::size_t first, std::string ctx) : where(std::move(ctx)) {
        for (std::size_t i = first; i < toks.size(); ++i) {
            const std::size_t eq = toks[i].find('=');
            if (eq == std::string::npos)
                throw ParseError(where + ": expected key=value token, got '" + toks[i] + "'");
            kv[toks[i].substr(0, eq)] = toks[i].substr(eq + 1);
        }
    }
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    std::string str(const std::string& k) const {
        auto it = kv.find(k);
        if (it == kv.end()) throw ParseError(where + ": missing key '" + k + "'");
        return it->second;
    }
    std::string str_or(const std::string& k, const std::string& d) const { return has(k) ? str(k) : d; }
    std::int64_t num(const std::string& k) const {
        try {
            return std::stoll(str(k));
        } catch (const std::logic_error&) {
            throw ParseError(where + ": key '" + k + "' is not an integer");
        }
    }
    std::int64_t num_or(const std::string& k, std::int64_t d) const { return has(k) ? num(k) : d; }
    double real(const std::string& k) const {
        try {
            return std::stod(str(k));
        } catch (const std::logic_error&) {
            throw ParseError(where + ": key '" + k + "' is not a number");
        }
    }
    double real_or(const std::string& k, double d) const { return has(k) ? real(k) : d; }
};

}  // namespace

// ---- ScalingCurve (scaling.hpp:35-164) -------------------------------------------
ScalingCurve ScalingCurve::from_pieces(std::vector<CurvePiece> pieces, double c, double w) {
    if (pieces.empty()) throw InvariantError("ScalingCurve: no pieces");
    ScalingCurve out;
    std::sort(pieces.begin(), pieces.end(),
              [](const CurvePiece& a, const CurvePiece& b) { return a.n_lo < b.n_lo; });
    if (std::abs(pieces.front().n_lo - 1.0) > 1e-9) throw InvariantError("ScalingCurve: pieces must start at n=1");
    for (std::size_t i = 1; i < pieces.size(); ++i)
        if (std::abs(pieces[i - 1].n_hi - pieces[i].n_lo) > 1e-9)
            throw InvariantError("ScalingCurve: pieces must be contiguous");
    out.n_max_ = pieces.back().n_hi;
    if (std::abs(out.n_max_ - std::llround(out.n_max_)) > 1e-9)
        throw InvariantError("ScalingCurve: n_max must be an integer");
    out.pieces_ = std::move(pieces);
    out.c_ = c;
    out.w_ = w;
    return out;
}

int ScalingCurve::n_max_int() const { return static_cast<int>(std::llround(n_max_)); }

double ScalingCurve::eval(double n) const {
    if (n < 1.0 - 1e-9 || n > n_max_ + 1e-9)
        throw OutOfRange("eval_time: n=" + fmt_g(n) + " outside [1, " + fmt_g(n_max_) + "]");
    const CurvePiece* p = &pieces_.back();
    for (const CurvePiece& q : pieces_)
        if (n <= q.n_hi + 1e-9) {
            p = &q;
            break;
        }
    return p->alpha + p->beta_c * c_ + p->beta_w * w_ / n;
}

double ScalingCurve::inverse_exact(double target) const {
    auto value = [&](const CurvePiece& p, double n) { return p.alpha + p.beta_c * c_ + p.beta_w * w_ / n; };
    if (target <= value(pieces_.back(), n_max_)) return n_max_;
    for (const CurvePiece& p : pieces_) {
        const double top = value(p, p.n_lo);
        const double bottom = value(p, p.n_hi);
        const double b = p.beta_w * w_;
        const double base = p.alpha + p.beta_c * c_;
        if (target > top + 1e-15 * std::abs(top)) return b <= 0.0 ? 0.0 : b / (target - base);
        if (target >= bottom) {
            if (b <= 0.0) return p.n_lo;
            if (target <= base) return p.n_hi;
            return std::clamp(b / (target - base), p.n_lo, p.n_hi);
        }
    }
    return n_max_;
}

std::string ScalingCurve::dump() const {
    std::string out;
    for (const CurvePiece& p : pieces_)
        out += "piece " + fmt_exact(p.n_lo) + " " + fmt_exact(p.n_hi) + " " + fmt_exact(p.alpha) + " " +
               fmt_exact(p.beta_c) + " " + fmt_exact(p.beta_w) + "\n";
    return out;
}

// ---- workload (workload.hpp:61-243) --------------------------------------------------
const ModuleDecl& WorkloadSpec::module(const std::string& kind) const {
    auto it = modules.find(kind);
    if (it == modules.end()) throw UnknownModule("unknown module '" + kind + "'");
    return it->second;
}

std::vector<FlowStep> parse_flow(const std::string& text, const std::string& ctx) {
    std::vector<FlowStep> steps;
    for (const std::string& st : split_char(text, ',')) {
        FlowStep step;
        for (const std::string& br : split_char(st, '+')) {
            FlowBranch branch;
            for (const std::string& mod : split_char(br, '>')) {
                if (mod.empty()) throw ParseError(ctx + ": empty module reference in flow");
                branch.push_back(mod);
            }
            step.push_back(std::move(branch));
        }
        steps.push_back(std::move(step));
    }
    return steps;
}

std::string flow_to_text(const std::vector<FlowStep>& flow) {
    std::string out;
    for (std::size_t s = 0; s < flow.size(); ++s) {
        if (s) out += ',';
        for (std::size_t b = 0; b < flow[s].size(); ++b) {
            if (b) out += '+';
            for (std::size_t m = 0; m < flow[s][b].size(); ++m) {
                if (m) out += '>';
                out += flow[s][b][m];
            }
        }
    }
    return out;
}

// workload.hpp:104-127 — host-side validation, same order and messages.
void validate_workload(const WorkloadSpec& spec) {
    if (spec.tasks.empty()) throw EmptyWorkload("workload declares no tasks");
    std::set<std::string> seen;
    for (const TaskDecl& t : spec.tasks) {
        if (!seen.insert(t.id).second) throw ParseError("duplicate task id '" + t.id + "'");
        for (const FlowStep& step : t.flow)
            for (const FlowBranch& br : step)
                for (const std::string& mod : br) spec.module(mod);
    }
    for (const auto& [kind, m] : spec.modules) {
        if (m.layers < 1) throw ParseError("module '" + kind + "': layers must be >= 1");
        if (m.input.batch < 1 || m.input.seq < 1 || m.input.hidden < 1)
            throw ParseError("module '" + kind + "': input size components must be positive");
        if (m.tp_degree < 1) throw ParseError("module '" + kind + "': tp degree must be >= 1");
        if (m.flops_proxy <= 0.0) throw ParseError("module '" + kind + "': w must be positive");
        if (m.comm_proxy < 0.0) throw ParseError("module '" + kind + "': c must be >= 0");
    }
    for (const auto& [kind, pieces] : spec.truth) {
        spec.module(kind);
        if (pieces.empty()) throw ParseError("module '" + kind + "': empty truth curve");
    }
    for (const auto& kv : spec.profiles) spec.module(kv.first);
    for (const auto& kv : spec.breakpoints) spec.module(kv.first);
}

WorkloadSpec parse_workload(const std::string& text) {
    WorkloadSpec spec;
    std::istringstream is(text);
    std::string line;
    int lineno = 0;
    while (std::getline(is, line)) {
        ++lineno;
        if (blank_or_comment(line)) continue;
        const auto toks = tokens_of(line);
        const std::string ctx = "workload line " + std::to_string(lineno);
        const std::string& head = toks[0];
        if (head == "module") {
            if (toks.size() < 2) throw ParseError(ctx + ": module needs a kind");
            Fields f(toks, 2, ctx);
            ModuleDecl m;
            m.kind = toks[1];
            m.layers = static_cast<int>(f.num("layers"));
            m.input.batch = f.num("B");
            m.input.seq = f.num_or("seq", 1);
            m.input.hidden = f.num_or("hidden", 1);
            m.tp_degree = static_cast<int>(f.num_or("tp", 1));
            m.param_group = f.str_or("param_group", "");
            m.param_bytes = static_cast<std::uint64_t>(f.num_or("param_bytes", 0));
            m.flops_proxy = f.real_or("w", 1.0);
            m.comm_proxy = f.real_or("c", 0.0);
            m.act_bytes = static_cast<std::uint64_t>(f.num_or("act_bytes", 0));
            m.out_bytes = static_cast<std::uint64_t>(f.num_or("out_bytes", 0));
            if (!spec.modules.emplace(m.kind, m).second)
                throw ParseError(ctx + ": duplicate module kind '" + m.kind + "'");
        } else if (head == "task") {
            if (toks.size() < 2) throw ParseError(ctx + ": task needs an id");
            Fields f(toks, 2, ctx);
            TaskDecl t;
            t.id = toks[1];
            t.flow_text = f.str("flow");
            t.flow = parse_flow(t.flow_text, ctx);
            spec.tasks.push_back(std::move(t));
        } else if (head == "truth") {
            if (toks.size() != 8 || toks[2] != "piece")
                throw ParseError(ctx + ": expected 'truth <kind> piece <n_lo> <n_hi> <alpha> <beta_c> <beta_w>'");
            CurvePiece p;
            try {
                p.n_lo = std::stod(toks[3]);
                p.n_hi = std::stod(toks[4]);
                p.alpha = std::stod(toks[5]);
                p.beta_c = std::stod(toks[6]);
                p.beta_w = std::stod(toks[7]);
            } catch (const std::logic_error&) {
                throw ParseError(ctx + ": bad numeric field in truth piece");
            }
            spec.truth[toks[1]].push_back(p);
        } else if (head == "metaop") {
            const std::string pctx = "profile line 1";
            if (toks.size() < 3) throw ParseError(pctx + ": expected 'metaop <id> ...'");
            Fields f(toks, 2, pctx);
            ProfilePoint p;
            p.n = static_cast<int>(f.num("n"));
            p.time = f.real("time");
            p.parallel_config = f.str_or("config", "dp");
            if (p.n < 1 || p.time <= 0.0) throw ParseError(pctx + ": need n >= 1 and time > 0");
            spec.profiles[toks[1]].push_back(p);
        } else if (head == "breakpoints") {
            if (toks.size() < 3) throw ParseError(ctx + ": breakpoints needs a kind and values");
            std::vector<int> bps;
            for (std::size_t i = 2; i < toks.size(); ++i) {
                try {
                    bps.push_back(std::stoi(toks[i]));
                } catch (const std::logic_error&) {
                    throw ParseError(ctx + ": bad breakpoint '" + toks[i] + "'");
                }
            }
            spec.breakpoints[toks[1]] = bps;
        } else {
            throw ParseError(ctx + ": unknown directive '" + head + "'");
        }
    }
    validate_workload(spec);
    return spec;
}

std::string dump_workload(const WorkloadSpec& spec) {
    std::string out;
    for (const auto& [kind, m] : spec.modules) {
        out += "module " + kind + " layers=" + std::to_string(m.layers) + " B=" + std::to_string(m.input.batch) +
               " seq=" + std::to_string(m.input.seq) + " hidden=" + std::to_string(m.input.hidden) +
               " tp=" + std::to_string(m.tp_degree);
        if (!m.param_group.empty()) out += " param_group=" + m.param_group;
        out += " param_bytes=" + std::to_string(m.param_bytes) + " w=" + fmt_exact(m.flops_proxy) +
               " c=" + fmt_exact(m.comm_proxy) + " act_bytes=" + std::to_string(m.act_bytes);
        if (m.out_bytes != 0) out += " out_bytes=" + std::to_string(m.out_bytes);
        out += "\n";
    }
    for (const TaskDecl& t : spec.tasks) out += "task " + t.id + " flow=" + flow_to_text(t.flow) + "\n";
    for (const auto& [kind, pieces] : spec.truth)
        for (const CurvePiece& p : pieces)
            out += "truth " + kind + " piece " + fmt_exact(p.n_lo) + " " + fmt_exact(p.n_hi) + " " +
                   fmt_exact(p.alpha) + " " + fmt_exact(p.beta_c) + " " + fmt_exact(p.beta_w) + "\n";
    for (const auto& [kind, pts] : spec.profiles)
        for (const ProfilePoint& p : pts)
            out += "metaop " + kind + " n=" + std::to_string(p.n) + " config=" + p.parallel_config +
                   " time=" + fmt_exact(p.time) + "\n";
    for (const auto& [kind, bps] : spec.breakpoints) {
        out += "breakpoints " + kind;
        for (int b : bps) out += " " + std::to_string(b);
        out += "\n";
    }
    return out;
}

// ---- topology (topology.hpp:15-113) ------------------------------------------------------
void ClusterTopology::finalize() {
    devices.clear();
    island_of.clear();
    for (std::size_t i = 0; i < islands.size(); ++i) {
        std::sort(islands[i].begin(), islands[i].end());
        for (int d : islands[i]) {
            if (!island_of.emplace(d, static_cast<int>(i)).second)
                throw ParseError("device " + std::to_string(d) + " in two islands");
            devices.push_back(d);
        }
    }
    std::sort(devices.begin(), devices.end());
    if (intra_bw < inter_bw || inter_bw <= 0.0) throw ParseError("topology requires intra_bw >= inter_bw > 0");
    if (devices.empty()) throw ParseError("topology declares no devices");
}

ClusterTopology make_topology(int num_devices, int island_size, double intra_bw, double inter_bw,
                              std::uint64_t mem_capacity) {
    ClusterTopology t;
    t.intra_bw = intra_bw;
    t.inter_bw = inter_bw;
    t.mem_capacity = mem_capacity;
    for (int d = 0; d < num_devices; ++d) {
        if (d % island_size == 0) t.islands.emplace_back();
        t.islands.back().push_back(d);
    }
    t.finalize();
    return t;
}

ClusterTopology parse_topology(const std::string& text) {
    ClusterTopology t;
    std::istringstream is(text);
    std::string line;
    int lineno = 0;
    bool have_bw = false, have_mem = false;
    while (std::getline(is, line)) {
        ++lineno;
        if (blank_or_comment(line)) continue;
        const auto toks = tokens_of(line);
        const std::string ctx = "topology line " + std::to_string(lineno);
        if (toks[0] == "island") {
            if (toks.size() < 3) throw ParseError(ctx + ": island needs an id and device ids");
            std::vector<int> members;
            for (std::size_t i = 2; i < toks.size(); ++i) {
                try {
                    members.push_back(std::stoi(toks[i]));
                } catch (const std::logic_error&) {
                    throw ParseError(ctx + ": bad device id '" + toks[i] + "'");
                }
            }
            t.islands.push_back(std::move(members));
        } else if (toks[0] == "bw") {
            Fields f(toks, 1, ctx);
            t.intra_bw = f.real("intra");
            t.inter_bw = f.real("inter");
            have_bw = true;
        } else if (toks[0] == "mem") {
            if (toks.size() != 2) throw ParseError(ctx + ": expected 'mem <bytes>'");
            try {
                t.mem_capacity = std::stoull(toks[1]);
            } catch (const std::logic_error&) {
                throw ParseError(ctx + ": bad byte count");
            }
            have_mem = true;
        } else {
            throw ParseError(ctx + ": unknown directive '" + toks[0] + "'");
        }
    }
    if (!have_bw || !have_mem) throw ParseError("topology needs 'bw' and 'mem' lines");
    t.finalize();
    return t;
}

// Dynamic re-planning sequence (cmd_dynamic, cli.hpp:283-297).
std::vector<SequencePhase> parse_sequence(const std::string& text) {
    std::vector<SequencePhase> phases;
    std::istringstream is(text);
    std::string line;
    int lineno = 0;
    while (std::getline(is, line)) {
        ++lineno;
        if (blank_or_comment(line)) continue;
        const std::vector<std::string> toks = tokens_of(line);
        const std::string where = "sequence line " + std::to_string(lineno);
        if (toks[0] != "phase") throw ParseError(where + ": expected 'phase ...'");
        Fields f(toks, 1, where);
        phases.push_back({f.str("workload"), static_cast<int>(f.num_or("iters", 1))});
    }
    if (phases.empty()) throw ParseError("dynamic sequence declares no phases");
    return phases;
}

std::string dump_topology(const ClusterTopology& topo) {
    std::string out;
    for (std::size_t i = 0; i < topo.islands.size(); ++i) {
        out += "island " + std::to_string(i) + ":";
        for (int d : topo.islands[i]) out += " " + std::to_string(d);
        out += "\n";
    }
    out += "bw intra=" + fmt_exact(topo.intra_bw) + " inter=" + fmt_exact(topo.inter_bw) + "\n";
    out += "mem " + std::to_string(topo.mem_capacity) + "\n";
    return out;
}

// ---- dumps (graph.hpp:245-254, allocation.hpp:216-227, schedule.hpp:311-322) ----------------
std::string dump_metagraph(const MetaGraph& meta) {
    std::string out;
    for (const auto& [id, m] : meta.metaops)
        out += "node " + id + " kind=" + m.kind + " B=" + std::to_string(m.global_batch) +
               " L=" + std::to_string(m.length) + " level=" + std::to_string(m.level) +
               " tp=" + std::to_string(m.tp_degree) + "\n";
    for (const auto& [a, b] : meta.edges) out += "edge " + a + " " + b + "\n";
    return out;
}

std::string dump_allocation(const AllocationPlan& plan) {
    std::string out;
    for (const auto& [id, pair] : plan.tuples) {
        out += "metaop " + id + " tuple n=" + std::to_string(pair.upper.n) + " l=" +
               std::to_string(pair.upper.layers) + "\n";
        if (pair.lower)
            out += "metaop " + id + " tuple n=" + std::to_string(pair.lower->n) + " l=" +
                   std::to_string(pair.lower->layers) + "\n";
    }
    return out;
}

std::string dump_schedule(const WavefrontSchedule& sched) {
    std::string out;
    for (const Wave& w : sched.waves) {
        out += "wave " + std::to_string(w.index) + " start=" + fmt_g(w.start) + " dur=" + fmt_g(w.duration) + "\n";
        for (const WaveEntry& e : w.entries)
            out += "  entry metaop=" + e.metaop_id + " n=" + std::to_string(e.n) + " l=" + std::to_string(e.layers) +
                   "\n";
    }
    return out;
}

// ---- plan serializer (plan_io.hpp:53-110): byte-level parity artifact ------------------------
std::string write_plan(const ExecutionPlan& plan) {
    std::string out = "# wavesched plan v1\nstrategy " + plan.strategy + "\n";
    out += dump_topology(plan.topo);
    for (const auto& [id, e] : plan.entities) {
        out += "entity " + id + " kind=" + e.kind + " L=" + std::to_string(e.length) +
               " level=" + std::to_string(e.level) + " tp=" + std::to_string(e.tp_degree) +
               " B=" + std::to_string(e.global_batch) + " frac=" + fmt_exact(e.batch_fraction);
        if (!e.param_group.empty()) out += " param_group=" + e.param_group;
        out += " param_bytes=" + std::to_string(e.param_bytes) + " act_bytes=" + std::to_string(e.act_bytes);
        if (e.out_bytes != 0) out += " out_bytes=" + std::to_string(e.out_bytes);
        out += " w=" + fmt_exact(e.w) + " c=" + fmt_exact(e.c);
        if (!e.task_ids.empty()) {
            out += " tasks=";
            bool first = true;
            for (const std::string& t : e.task_ids) {
                if (!first) out += ';';
                out += t;
                first = false;
            }
        }
        out += "\n";
    }
    for (const auto& [id, curve] : plan.curves) {
        for (const CurvePiece& p : curve.pieces())
            out += "curve " + id + " piece " + fmt_exact(p.n_lo) + " " + fmt_exact(p.n_hi) + " " +
                   fmt_exact(p.alpha) + " " + fmt_exact(p.beta_c) + " " + fmt_exact(p.beta_w) + "\n";
        out += "curve " + id + " workload c=" + fmt_exact(curve.c()) + " w=" + fmt_exact(curve.w()) + "\n";
    }
    for (const auto& [a, b] : plan.deps) out += "dep " + a + " " + b + "\n";
    out += "lower_bound " + fmt_exact(plan.lower_bound) + "\n";
    out += "mem_multiplier " + fmt_exact(plan.grad_opt_multiplier) + "\n";
    for (const Wave& w : plan.schedule.waves) {
        out += "wave " + std::to_string(w.index) + " level=" + std::to_string(w.level) + " start=" +
               fmt_exact(w.start) + " dur=" + fmt_exact(w.duration) + "\n";
        for (const WaveEntry& e : w.entries) {
            out += "entry metaop=" + e.metaop_id + " n=" + std::to_string(e.n) + " l=" + std::to_string(e.layers) +
                   " dur=" + fmt_exact(e.span);
            auto it = plan.devices.find({w.index, e.metaop_id});
            if (it != plan.devices.end()) {
                out += " devices=";
                for (std::size_t i = 0; i < it->second.size(); ++i) {
                    if (i) out += ',';
                    out += std::to_string(it->second[i]);
                }
            }
            out += "\n";
        }
    }
    for (const Flow& f : plan.flows)
        out += "flow from=" + std::to_string(f.from_wave) + ":" + f.from_id + " to=" + std::to_string(f.to_wave) +
               ":" + f.to_id + " volume=" + std::to_string(f.volume) + " mode=" + f.mode + "\n";
    out += "end_time " + fmt_exact(plan.schedule.end_time) + "\n";
    return out;
}

// ---- plan parser (plan_io.hpp:112-255): any strategy's plan file back into an ExecutionPlan ----
ExecutionPlan parse_plan(const std::string& text) {
    ExecutionPlan plan;
    plan.strategy.clear();
    std::istringstream is(text);
    std::string line;
    int lineno = 0;
    std::map<std::string, std::vector<CurvePiece>> curve_pieces;
    std::map<std::string, std::pair<double, double>> curve_cw;
    ClusterTopology topo;
    bool saw_bw = false, saw_mem = false, saw_end = false;
    int last_level = -1;
    while (std::getline(is, line)) {
        ++lineno;
        if (blank_or_comment(line)) continue;
        const auto toks = tokens_of(line);
        const std::string ctx = "plan line " + std::to_string(lineno);
        const std::string& head = toks[0];
        try {
            if (head == "strategy") {
                if (toks.size() != 2) throw ParseError(ctx + ": expected 'strategy <name>'");
                plan.strategy = toks[1];
            } else if (head == "island") {
                std::vector<int> members;
                for (std::size_t i = 2; i < toks.size(); ++i) members.push_back(std::stoi(toks[i]));
                topo.islands.push_back(members);
            } else if (head == "bw") {
                Fields kv(toks, 1, ctx);
                topo.intra_bw = kv.real("intra");
                topo.inter_bw = kv.real("inter");
                saw_bw = true;
            } else if (head == "mem") {
                topo.mem_capacity = std::stoull(toks.at(1));
                saw_mem = true;
            } else if (head == "entity") {
                if (toks.size() < 2) throw ParseError(ctx + ": entity needs an id");
                Fields kv(toks, 2, ctx);
                PlanEntity e;
                e.id = toks[1];
                e.kind = kv.str("kind");
                e.length = static_cast<int>(kv.num("L"));
                e.level = static_cast<int>(kv.num_or("level", 0));
                e.tp_degree = static_cast<int>(kv.num_or("tp", 1));
                e.global_batch = kv.num_or("B", 1);
                e.batch_fraction = kv.real_or("frac", 1.0);
                e.param_group = kv.str_or("param_group", "");
                e.param_bytes = static_cast<std::uint64_t>(kv.num_or("param_bytes", 0));
                e.act_bytes = static_cast<std::uint64_t>(kv.num_or("act_bytes", 0));
                e.out_bytes = static_cast<std::uint64_t>(kv.num_or("out_bytes", 0));
                e.w = kv.real_or("w", 1.0);
                e.c = kv.real_or("c", 0.0);
                if (kv.has("tasks"))
                    for (const std::string& t : split_char(kv.str("tasks"), ';')) e.task_ids.insert(t);
                plan.entities[e.id] = e;
            } else if (head == "curve") {
                if (toks.size() < 3) throw ParseError(ctx + ": malformed curve line");
                if (toks[2] == "piece") {
                    if (toks.size() != 8) throw ParseError(ctx + ": curve piece needs 5 numbers");
                    CurvePiece p;
                    p.n_lo = std::stod(toks[3]);
                    p.n_hi = std::stod(toks[4]);
                    p.alpha = std::stod(toks[5]);
                    p.beta_c = std::stod(toks[6]);
                    p.beta_w = std::stod(toks[7]);
                    curve_pieces[toks[1]].push_back(p);
                } else if (toks[2] == "workload") {
                    Fields kv(toks, 3, ctx);
                    curve_cw[toks[1]] = {kv.real("c"), kv.real("w")};
                } else {
                    throw ParseError(ctx + ": unknown curve directive '" + toks[2] + "'");
                }
            } else if (head == "dep") {
                if (toks.size() != 3) throw ParseError(ctx + ": expected 'dep <from> <to>'");
                plan.deps.insert({toks[1], toks[2]});
            } else if (head == "lower_bound") {
                plan.lower_bound = std::stod(toks.at(1));
            } else if (head == "mem_multiplier") {
                plan.grad_opt_multiplier = std::stod(toks.at(1));
            } else if (head == "wave") {
                Fields kv(toks, 2, ctx);
                Wave w;
                w.index = std::stoi(toks.at(1));
                w.level = static_cast<int>(kv.num_or("level", 0));
                w.start = kv.real("start");
                w.duration = kv.real("dur");
                if (w.level != last_level) {
                    plan.schedule.level_boundaries.push_back(w.index);
                    last_level = w.level;
                }
                plan.schedule.waves.push_back(w);
            } else if (head == "entry") {
                if (plan.schedule.waves.empty()) throw ParseError(ctx + ": entry before any wave");
                Fields kv(toks, 1, ctx);
                WaveEntry e;
                e.metaop_id = kv.str("metaop");
                e.n = static_cast<int>(kv.num("n"));
                e.layers = static_cast<int>(kv.num("l"));
                e.span = kv.real("dur");
                Wave& w = plan.schedule.waves.back();
                w.entries.push_back(e);
                if (kv.has("devices")) {
                    std::vector<int> devs;
                    for (const std::string& d : split_char(kv.str("devices"), ','))
                        if (!d.empty()) devs.push_back(std::stoi(d));
                    plan.devices[{w.index, e.metaop_id}] = devs;
                }
            } else if (head == "flow") {
                Fields kv(toks, 1, ctx);
                Flow f;
                const auto from = split_char(kv.str("from"), ':');
                const auto to = split_char(kv.str("to"), ':');
                if (from.size() != 2 || to.size() != 2) throw ParseError(ctx + ": flow endpoints are <wave>:<id>");
                f.from_wave = std::stoi(from[0]);
                f.from_id = from[1];
                f.to_wave = std::stoi(to[0]);
                f.to_id = to[1];
                f.volume = static_cast<std::uint64_t>(kv.num("volume"));
                f.mode = kv.str("mode");
                plan.flows.push_back(f);
            } else if (head == "end_time") {
                plan.schedule.end_time = std::stod(toks.at(1));
                saw_end = true;
            } else {
                throw ParseError(ctx + ": unknown directive '" + head + "'");
            }
        } catch (const ParseError&) {
            throw;
        } catch (const std::logic_error& e) {
            throw ParseError(ctx + ": " + e.what());
        }
    }
    if (plan.strategy.empty()) throw ParseError("plan: missing strategy line");
    if (!saw_bw || !saw_mem) throw ParseError("plan: incomplete topology");
    if (!saw_end) throw ParseError("plan: missing end_time");
    topo.finalize();
    plan.topo = topo;
    for (auto& [id, pieces] : curve_pieces) {
        auto cw = curve_cw.find(id);
        if (cw == curve_cw.end()) throw ParseError("plan: curve '" + id + "' missing workload line");
        plan.curves[id] = ScalingCurve::from_pieces(pieces, cw->second.first, cw->second.second);
    }
    for (const auto& [id, e] : plan.entities)
        if (!plan.curves.count(id)) throw ParseError("plan: entity '" + id + "' has no curve");
    return plan;
}

}  // namespace wsgpu
