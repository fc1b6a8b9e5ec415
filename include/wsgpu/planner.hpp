// planner.hpp — host-side C++ drop-in for the reference planner interface.
//
// Mirrors the value types of the reference planner API
//   WorkloadSpec/ModuleDecl/TaskDecl/InputSize   workload.hpp:16-69
//   CurvePiece/ProfilePoint/ScalingCurve          scaling.hpp:16-164
//   ClusterTopology                               topology.hpp:15-53
//   MetaOp/MetaGraph/ComputationGraph             graph.hpp:13-58
//   AslTuple/TuplePair/AllocationPlan/Options     allocation.hpp:17-46
//   Wave/WaveEntry/WavefrontSchedule              schedule.hpp:15-35
//   Flow/PlacementOptions                         placement.hpp:42-109
//   PlanEntity/ExecutionPlan                      plan_io.hpp:21-51
//   PlannerOptions/PlannerResult/plan_workload    planner.hpp:21-38,156
// with the same field names and meaning, so callers switch by namespace.
// plan_workload() here encodes the inputs into the ws_abi.h batch format,
// runs the sm_100a kernels through the C-ABI and decodes the result; errors
// are rethrown as the same exception classes with the same what() text.
#pragma once

#include <cstdint>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "wsgpu/ws_abi.h"

namespace wsgpu {

// ---- exception taxonomy (common.hpp:20-60) --------------------------------
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : Error {
    using Error::Error;
};
struct InfeasibleError : Error {
    using Error::Error;
};
struct InvariantError : Error {
    using Error::Error;
};
struct CyclicWorkload : ParseError {
    using ParseError::ParseError;
};
struct UnknownModule : ParseError {
    using ParseError::ParseError;
};
struct EmptyWorkload : ParseError {
    using ParseError::ParseError;
};
struct InsufficientProfile : ParseError {
    using ParseError::ParseError;
};
struct DegenerateFit : InfeasibleError {
    using InfeasibleError::InfeasibleError;
};
struct OutOfRange : InvariantError {
    using InvariantError::InvariantError;
};
struct NoValidAllocation : InfeasibleError {
    using InfeasibleError::InfeasibleError;
};
struct EmptyLevel : InvariantError {
    using InvariantError::InvariantError;
};
struct PlacementInfeasible : InfeasibleError {
    using InfeasibleError::InfeasibleError;
};
// Input outside the device limits of this build (ws_abi.h WS_MAX_*).
struct LimitExceeded : Error {
    using Error::Error;
};

std::string fmt_g(double v, int precision = 9);
inline std::string fmt_exact(double v) { return fmt_g(v, 17); }

// ---- curves ------------------------------------------------------------------
struct ProfilePoint {
    int n = 1;
    double time = 0.0;
    std::string parallel_config = "dp";
};

struct CurvePiece {
    double n_lo = 1.0;
    double n_hi = 1.0;
    double alpha = 0.0;
    double beta_c = 0.0;
    double beta_w = 0.0;
};

// Piecewise alpha-beta curve T(n) = alpha + beta_c*c + beta_w*w/n.
class ScalingCurve {
public:
    ScalingCurve() = default;
    static ScalingCurve from_pieces(std::vector<CurvePiece> pieces, double c, double w);
    double n_max() const { return n_max_; }
    int n_max_int() const;
    double c() const { return c_; }
    double w() const { return w_; }
    const std::vector<CurvePiece>& pieces() const { return pieces_; }
    double eval(double n) const;
    double inverse_exact(double target) const;
    std::string dump() const;

private:
    std::vector<CurvePiece> pieces_;
    double c_ = 0.0;
    double w_ = 1.0;
    double n_max_ = 1.0;
};

// ---- workload & topology -------------------------------------------------------
struct InputSize {
    std::int64_t batch = 1;
    std::int64_t seq = 1;
    std::int64_t hidden = 1;
    bool operator==(const InputSize& o) const {
        return batch == o.batch && seq == o.seq && hidden == o.hidden;
    }
};

struct ModuleDecl {
    std::string kind;
    int layers = 1;
    InputSize input;
    int tp_degree = 1;
    std::string param_group;
    std::uint64_t param_bytes = 0;
    double flops_proxy = 1.0;
    double comm_proxy = 0.0;
    std::uint64_t act_bytes = 0;
    std::uint64_t out_bytes = 0;
    std::uint64_t edge_bytes() const { return out_bytes == 0 ? act_bytes : out_bytes; }
};

using FlowBranch = std::vector<std::string>;
using FlowStep = std::vector<FlowBranch>;

struct TaskDecl {
    std::string id;
    std::vector<FlowStep> flow;
    std::string flow_text;
};

struct WorkloadSpec {
    std::map<std::string, ModuleDecl> modules;
    std::vector<TaskDecl> tasks;
    std::map<std::string, std::vector<CurvePiece>> truth;
    std::map<std::string, std::vector<ProfilePoint>> profiles;
    std::map<std::string, std::vector<int>> breakpoints;
    const ModuleDecl& module(const std::string& kind) const;
};

struct ClusterTopology {
    std::vector<int> devices;
    std::vector<std::vector<int>> islands;
    std::map<int, int> island_of;
    double intra_bw = 1.0;
    double inter_bw = 1.0;
    std::uint64_t mem_capacity = 0;
    void finalize();
};

ClusterTopology make_topology(int num_devices, int island_size, double intra_bw, double inter_bw,
                              std::uint64_t mem_capacity);

std::vector<FlowStep> parse_flow(const std::string& text, const std::string& ctx);
std::string flow_to_text(const std::vector<FlowStep>& flow);
void validate_workload(const WorkloadSpec& spec);
WorkloadSpec parse_workload(const std::string& text);
std::string dump_workload(const WorkloadSpec& spec);
ClusterTopology parse_topology(const std::string& text);
std::string dump_topology(const ClusterTopology& topo);

// ---- graph ---------------------------------------------------------------------
struct Operator {
    std::string id;
    std::string kind;
    std::set<std::string> task_ids;
    InputSize input;
    int tp_degree = 1;
    std::string param_group;
};

struct ComputationGraph {
    std::map<std::string, Operator> operators;
    std::set<std::pair<std::string, std::string>> edges;
};

struct MetaOp {
    std::string id;
    std::vector<std::string> member_ops;
    int length = 0;
    std::string kind;
    InputSize input;
    std::int64_t global_batch = 1;
    int tp_degree = 1;
    int level = -1;
    std::string param_group;
    std::set<std::string> task_ids;
};

struct MetaGraph {
    std::map<std::string, MetaOp> metaops;
    std::set<std::pair<std::string, std::string>> edges;
    std::vector<std::vector<std::string>> levels;
};

std::string dump_metagraph(const MetaGraph& meta);

// ---- allocation / schedule / placement ----------------------------------------------
struct AslTuple {
    std::string metaop_id;
    int n = 0;
    double start = -1.0;
    int layers = 0;
};

struct TuplePair {
    AslTuple upper;
    std::optional<AslTuple> lower;
};

struct AllocationPlan {
    int level = 0;
    double c_star = 0.0;
    std::map<std::string, TuplePair> tuples;
};

struct AllocatorOptions {
    double eps = 1e-7;
    int max_iters = 200;
    double drop_floor = 0.0;
};

std::string dump_allocation(const AllocationPlan& plan);

struct WaveEntry {
    std::string metaop_id;
    int n = 0;
    int layers = 0;
    double span = 0.0;
};

struct Wave {
    int index = 0;
    int level = 0;
    double start = 0.0;
    double duration = 0.0;
    std::vector<WaveEntry> entries;
};

struct WavefrontSchedule {
    std::vector<Wave> waves;
    double end_time = 0.0;
    std::vector<int> level_boundaries;
};

std::string dump_schedule(const WavefrontSchedule& sched);

struct Flow {
    int from_wave = 0;
    std::string from_id;
    int to_wave = 0;
    std::string to_id;
    std::uint64_t volume = 0;
    std::string mode;
};

struct PlacementOptions {
    bool sequential = false;
    int backtrack_depth = 2;
    int backtrack_branching = 3;
};

// ---- plan artifact ----------------------------------------------------------------------
struct PlanEntity {
    std::string id;
    std::string kind;
    int length = 1;
    int level = 0;
    int tp_degree = 1;
    std::int64_t global_batch = 1;
    double batch_fraction = 1.0;
    std::string param_group;
    std::uint64_t param_bytes = 0;
    std::uint64_t act_bytes = 0;
    std::uint64_t out_bytes = 0;
    double w = 1.0;
    double c = 0.0;
    std::set<std::string> task_ids;
};

struct ExecutionPlan {
    std::string strategy = "wavefront";
    ClusterTopology topo;
    std::map<std::string, PlanEntity> entities;
    std::map<std::string, ScalingCurve> curves;
    std::set<std::pair<std::string, std::string>> deps;
    WavefrontSchedule schedule;
    std::map<std::pair<int, std::string>, std::vector<int>> devices;
    std::vector<Flow> flows;
    double lower_bound = 0.0;
    double grad_opt_multiplier = 3.0;
};

std::string write_plan(const ExecutionPlan& plan);
// parse_plan (plan_io.hpp:112-255): a plan file of any strategy
ExecutionPlan parse_plan(const std::string& text);
// Structured ingestion (cli.hpp:46-110): the JSON forms of workload and topology
WorkloadSpec workload_from_json(const std::string& text);
ClusterTopology topology_from_json(const std::string& text);

// ---- planner API (planner.hpp:21-38,156) ------------------------------------------------------
struct PlannerOptions {
    AllocatorOptions alloc;
    PlacementOptions placement;
    double grad_opt_multiplier = 3.0;
    double synth_noise = 0.0;
    std::uint64_t synth_seed = 0;
    // Not a reference PlannerOptions field: the plan_for_strategy selector
    // (cli.hpp:163-171) -- ws_strategy, 0 = wavefront (plan_workload).
    int strategy = 0;
};

struct PlannerResult {
    ComputationGraph graph;
    MetaGraph meta;
    std::map<std::string, ScalingCurve> curves;
    std::vector<AllocationPlan> level_plans;
    WavefrontSchedule schedule;
    ExecutionPlan plan;
    double lower_bound = 0.0;
    double predicted_makespan = 0.0;
};

// Drop-in for wavesched::plan_workload: same arguments, same result, same
// exceptions.  Reentrant like the reference: each call checks a
// planning context with its own streams and page-locked staging buffers out of
// a pool for the calling thread's current CUDA device ($WSGPU_DEVICE
// overrides), so concurrent callers plan in parallel.  Throws if the CUDA
// planner cannot run (no fallback).
PlannerResult plan_workload(const WorkloadSpec& spec, const ClusterTopology& topo,
                            const PlannerOptions& opt = {});

// ---- batch encoding (host side of the C-ABI) ---------------------------------------------
// One planning problem of a batch.
struct Problem {
    const WorkloadSpec* spec = nullptr;
    const ClusterTopology* topo = nullptr;
    PlannerOptions opt;
};

// plan_workload over many problems in ONE device batch: the per-problem host
// preparation and the decode into PlannerResult run on `threads` host threads
// (0 = all cores).  Each outcome holds the result or the exception
// plan_workload would have thrown for that problem.
struct PlanOutcome {
    PlannerResult result;
    std::exception_ptr error;
};
std::vector<PlanOutcome> plan_workloads(const std::vector<Problem>& problems, int threads = 0);

// The raw device output of plan_workload / plan_workloads, for callers that
// decode into their own types (wavesched_compat.hpp decodes straight into the
// reference's types with detail::decode_into): `consume` sees the result
// header(s) and record arena, valid only during the call.
void plan_workload_raw(const WorkloadSpec& spec, const ClusterTopology& topo, const PlannerOptions& opt,
                       const std::function<void(const ws_plan_result& res, const std::uint8_t* arena)>& consume);
void plan_workloads_raw(const std::vector<Problem>& problems, int threads,
                        const std::function<void(const ws_plan_result* res, const std::uint8_t* arena)>& consume);

// Owns the memory behind a ws_batch (one contiguous, optionally pinned,
// block = ws_batch.blob).  Host-side validation (validate_workload) runs while
// encoding; a failing problem is recorded in host_error_* and encoded with no
// modules so the batch stays aligned.
class EncodedBatch {
public:
    ws_batch view{};
    std::vector<std::string> host_error_class;  // per plan; empty = encoded
    std::vector<std::string> host_error_msg;
    std::shared_ptr<std::uint8_t> buffer;
    std::size_t nbytes = 0;
    bool pinned = false;
};

EncodedBatch encode_batch(const std::vector<Problem>& problems, bool pinned = false);

// Decoded plan (strings rebuilt).  Throws the reference exception for a failed plan.
PlannerResult decode_result(const Problem& prob, const ws_plan_result& res, const std::uint8_t* arena,
                            bool build_graph = true);
// write_plan() text of a decoded result, or "error <Class>: <what>" for a failure.
std::string plan_text_or_error(const Problem& prob, const ws_plan_result& res, const std::uint8_t* arena);
// Canonical evaluation text (simulate_plan + validate_plan report) of one
// evaluated plan, or the plan's error text; see csrc/host/sim_text.cpp.
std::string sim_text(const Problem& prob, const ws_plan_result& res, const std::uint8_t* plan_arena,
                     const ws_sim_result& sim, const std::uint8_t* sim_arena);
// The same for a record with explicit entity names (index -> id), e.g. a parsed plan file.
std::string sim_text_named(const ClusterTopology& topo, const ws_plan_result& res, const ws_sim_result& sim,
                           const std::uint8_t* sim_arena, const std::vector<std::string>& names);
[[noreturn]] void throw_result_error(const Problem& prob, const ws_plan_result& res);

// Entity ids of a planned record ("m<k>", or "m<k>@<task>" for task-scoped strategies)
// and validate_plan's messages for its evaluation (the first WS_SIM_MAX_VIOLATIONS).
std::vector<std::string> record_entity_names(const Problem& prob, const ws_plan_result& res,
                                             const std::uint8_t* plan_arena);
std::vector<std::string> violation_messages(const ClusterTopology& topo, const ws_plan_result& res,
                                            const ws_sim_result& sim, const std::uint8_t* sim_arena,
                                            const std::vector<std::string>& names);

// ---- strategies, comparison and dynamic re-planning (cli.hpp:163-327) ---------------------
// The strategies in the reference's order (all_strategies, cli.hpp:237-241).
const std::vector<std::string>& all_strategies();
// ws_strategy id of a strategy name; ParseError("unknown strategy '<s>'") otherwise.
int strategy_id(const std::string& strategy);
// Drop-in for plan_for_strategy (cli.hpp:163-171): the plan of one strategy,
// planned on the device through the default context.
ExecutionPlan plan_for_strategy(const std::string& strategy, const WorkloadSpec& spec, const ClusterTopology& topo,
                                const PlannerOptions& opt);

// One strategy's plan and its simulated iteration time (simulate_plan(plan).makespan).
struct StrategyRun {
    std::string strategy;
    ExecutionPlan plan;
    double makespan = 0.0;
};

// cmd_compare (cli.hpp:243-264) without the file I/O: every strategy planned,
// validated and simulated on the device in one batch.  Throws what the
// reference throws, in its order (the first strategy's planning error, or
// InvariantError "strategy <s> produced an invalid plan: <first violation>").
// `table` is compare.csv.
struct CompareReport {
    std::vector<StrategyRun> runs;
    std::string table;
};
CompareReport compare_strategies(const WorkloadSpec& spec, const ClusterTopology& topo, const PlannerOptions& opt);

// Dynamic re-planning (cmd_dynamic, cli.hpp:269-327): a sequence file of
// `phase workload=<path> iters=<k>` lines.
struct SequencePhase {
    std::string workload;
    int iters = 1;
};
std::vector<SequencePhase> parse_sequence(const std::string& text);

// Every (phase, strategy) pair planned in ONE device batch and simulated in one
// k_sim launch.  `table` is dynamic.csv, `summary` cumulative.csv.  A phase
// whose workload failed to load is passed as a null spec with its exception in
// `load_errors[p]`; errors surface in the reference's (phase, strategy) order.
struct DynamicReport {
    std::vector<std::vector<StrategyRun>> phases;
    std::string table;
    std::string summary;
};
DynamicReport dynamic_replan(const std::vector<const WorkloadSpec*>& phases, const std::vector<int>& iters,
                             const ClusterTopology& topo, const PlannerOptions& opt,
                             const std::vector<std::exception_ptr>& load_errors = {});

// The CLI commands themselves (cli.hpp:243-327), with the reference's file
// outputs under `out_dir` (compare.csv; phase<p>.<strategy>.plan.txt, dynamic.csv,
// cumulative.csv).  Paths ending in ".json" load through workload_from_json /
// topology_from_json (cli.hpp:117-130).  Return the text the command prints.
std::string cmd_compare(const std::string& workload_path, const std::string& topology_path,
                        const std::string& out_dir, const PlannerOptions& opt);
std::string cmd_dynamic(const std::string& sequence_path, const std::string& topology_path,
                        const std::string& out_dir, const PlannerOptions& opt);

// Deterministic scenario generator (scenarios.hpp restated): the measurement
// input source.  Returns workload + topology built directly (no text pass).
struct Scenario {
    WorkloadSpec spec;
    ClusterTopology topo;
};
Scenario generate_scenario(const std::string& name, int tasks, int devices, std::uint64_t seed);
// SURVEY §8(d) sweep mixture i.
Scenario sweep_mixture(std::int64_t i);

}  // namespace wsgpu
