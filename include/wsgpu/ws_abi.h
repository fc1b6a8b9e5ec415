/*
 * ws_abi.h — C-ABI of the B200 wavefront planner (drop-in for
 * wavesched::plan_workload, /root/reference/proj/include/wavesched/planner.hpp:156-212).
 *
 * Plain C: fixed-width integers, plain pointers and sizes, no torch or C++
 * types.  A *batch* holds many independent planning problems ("plans") as
 * structure-of-arrays sections; the planner fills one ws_plan_result per plan
 * plus a byte arena holding each plan's variable-length output record.
 *
 * Every declaration below names the reference interface it replaces.
 * The host-side C++ mirror (include/wsgpu/planner.hpp) encodes
 * WorkloadSpec/ClusterTopology/PlannerOptions into this format and decodes the
 * results back into PlannerResult/ExecutionPlan.
 */
#ifndef WSGPU_WS_ABI_H
#define WSGPU_WS_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WS_ABI_VERSION 1

/* Device-side limits of this build (per plan).  A plan exceeding one returns
 * WS_STATUS_LIMIT with err_code naming the limit; nothing falls back to CPU. */
#define WS_MAX_DEVICES 256  /* device sets: one u64 mask up to 64 devices, four words up to 256 */
#define WS_MAX_DEVICES_EVAL 256 /* plan evaluation (simulate/validate, plan files)  */
#define WS_MAX_MODULES 64   /* module DAG adjacency is u64 masks               */
#define WS_MAX_TASKS 64     /* task sets are u64 masks                         */
#define WS_MAX_PIECES 64    /* fitted pieces per curve (isotonic: nmax-1)      */
#define WS_MAX_TUPLES 128   /* pending ASL tuples per level                    */
#define WS_MAX_WAVES 256    /* waves per plan                                  */
#define WS_MAX_ENTRIES 1024 /* wave entries per plan                           */
#define WS_MAX_FLOWS 4096   /* flows per plan                                  */

/* ---- status (maps the exception taxonomy, common.hpp:20-60, cli.hpp:330-344) */
enum ws_status {
    WS_STATUS_OK = 0,
    WS_STATUS_PARSE = 2,      /* ParseError and subclasses       -> exit 2 */
    WS_STATUS_INFEASIBLE = 3, /* InfeasibleError and subclasses  -> exit 3 */
    WS_STATUS_INVARIANT = 4,  /* InvariantError and subclasses   -> exit 4 */
    WS_STATUS_LIMIT = 5,      /* input exceeds a WS_MAX_* limit of this build */
    WS_STATUS_INTERNAL = 6    /* arena overflow or CUDA error */
};

/* ---- leaf error codes; err_a/err_b/err_x/err_y carry the message arguments */
enum ws_err {
    WS_E_NONE = 0,
    WS_E_CYCLIC_WORKLOAD = 1,   /* CyclicWorkload "workload data flows form a cycle" (graph.hpp:145)      */
    WS_E_TRUTH_RANGE = 2,       /* ParseError "truth curve does not cover the device range" (planner.hpp:50) */
    WS_E_CURVE_START = 3,       /* InvariantError "ScalingCurve: pieces must start at n=1" (scaling.hpp:48) */
    WS_E_CURVE_CONTIG = 4,      /* InvariantError "ScalingCurve: pieces must be contiguous" (scaling.hpp:51) */
    WS_E_NO_SOURCE = 5,         /* ParseError "module '<a>' has neither profile points nor a truth curve" */
    WS_E_FIT_NO_POINTS = 6,     /* InsufficientProfile "fit: no profile points" (scaling.hpp:231)         */
    WS_E_FIT_BAD_N = 7,         /* InsufficientProfile "fit: device count must be >= 1"                  */
    WS_E_FIT_BAD_TIME = 8,      /* InsufficientProfile "fit: non-positive time sample"                   */
    WS_E_FIT_BREAKPOINT = 9,    /* ParseError "fit: breakpoint <a> outside point span" (scaling.hpp:243)  */
    WS_E_FIT_PIECE_POINTS = 10, /* InsufficientProfile "fit: piece [<a>, <b>] needs points at >= 2 distinct n" */
    WS_E_FIT_DEGENERATE_X = 11, /* InsufficientProfile "fit: points do not span distinct n" (scaling.hpp:186) */
    WS_E_FIT_NONPOSITIVE = 12,  /* DegenerateFit "fit: non-positive T(<a>)" (scaling.hpp:319)            */
    WS_E_TP_EXCEEDS = 13,       /* NoValidAllocation "metaop 'm<a>': tp degree <b> exceeds device count <N>" */
    WS_E_EVAL_RANGE = 14,       /* OutOfRange "eval_time: n=<x> outside [1, <y>]" (scaling.hpp:68)        */
    WS_E_NO_SCHEDULABLE = 15,   /* InvariantError "schedule_level: no schedulable tuple"                 */
    WS_E_NO_PROGRESS = 16,      /* InvariantError "schedule_level: wave made no progress"                */
    WS_E_BT_BUDGET = 17,        /* PlacementInfeasible "placement backtrack budget exhausted at wave <a>" */
    WS_E_NO_PLACEMENT_W0 = 18,  /* PlacementInfeasible "no feasible placement for wave 0"                */
    WS_E_HOST_PRESET = 19,      /* error detected by the host encoder; message kept host-side           */
    WS_E_TASK_NO_VALID = 20,    /* NoValidAllocation "task '<task a>' has no allocation valid for all its metaops" */
    WS_E_LIMIT_DEVICES = 40,
    WS_E_LIMIT_MODULES = 41,
    WS_E_LIMIT_TASKS = 42,
    WS_E_LIMIT_PIECES = 43,
    WS_E_LIMIT_TUPLES = 44,
    WS_E_LIMIT_WAVES = 45,
    WS_E_LIMIT_ENTRIES = 46,
    WS_E_LIMIT_FLOWS = 47,
    WS_E_ARENA_OVERFLOW = 60,
    WS_E_CUDA = 61
};

/* Flow token encoding (workload.hpp:71-87 grammar "a>b+c,d"):
 *   >= 0           module index local to the plan ('>' chains consecutive modules)
 *   WS_TOK_BRANCH  '+'   WS_TOK_STEP ','                                         */
#define WS_TOK_BRANCH (-1)
#define WS_TOK_STEP (-2)

/* One planning problem: a WorkloadSpec + ClusterTopology + PlannerOptions. */
typedef struct ws_plan_rec {
    int32_t mod_begin, n_mod;    /* modules, sorted by kind (std::map order)           */
    int32_t task_begin, n_tasks; /* tasks in spec order; see ws_batch.task_*           */
    int32_t dev_begin, n_dev;    /* devices in ascending id order; island per device   */
    int32_t n_islands;           /* islands in declaration order                        */
    int32_t n_groups;            /* distinct param_group strings (ids 0..n_groups-1)    */
    int32_t max_iters;           /* AllocatorOptions::max_iters (allocation.hpp:44)     */
    int32_t sequential;          /* PlacementOptions::sequential (placement.hpp:106)    */
    int32_t bt_depth;            /* PlacementOptions::backtrack_depth                   */
    int32_t bt_branching;        /* PlacementOptions::backtrack_branching               */
    uint64_t mem_capacity;       /* ClusterTopology::mem_capacity                       */
    double eps;                  /* AllocatorOptions::eps                               */
    double drop_floor;           /* AllocatorOptions::drop_floor                        */
    double grad_mult;            /* PlannerOptions::grad_opt_multiplier                 */
    double intra_bw, inter_bw;   /* ClusterTopology bandwidths (simulator, flow_duration) */
    int32_t strategy;            /* ws_strategy: plan_for_strategy selector (cli.hpp:163-171) */
    int32_t pad_s;
} ws_plan_rec;

/* Planning strategies (cli.hpp:238-241): the wavefront planner (plan_workload)
 * and the baseline planners of baselines.hpp. */
enum ws_strategy {
    WS_STRATEGY_WAVEFRONT = 0,            /* planner.hpp:156-212                  */
    WS_STRATEGY_DECOUPLED_SEQUENTIAL = 1, /* plan_decoupled_sequential, baselines.hpp:104-131 */
    WS_STRATEGY_DISTMM_MT = 2,            /* plan_distmm_mt, baselines.hpp:323-413          */
    WS_STRATEGY_TASK_OPTIMUS = 3          /* plan_task_level_optimus, baselines.hpp:133-321 */
};

/* Structure-of-arrays batch.  All pointers address the same memory space
 * (host for the oracle and the *_host entry points, device inside the ctx). */
typedef struct ws_batch {
    int32_t n_plans;
    int32_t n_modules;     /* total modules over all plans        */
    int32_t n_task_total;  /* total tasks                         */
    int32_t n_tokens;      /* total flow tokens                   */
    int32_t n_devices;     /* total devices                       */
    int32_t n_pieces;      /* total declared truth pieces         */
    int32_t n_points;      /* total profile points                */
    int32_t n_bps;         /* total breakpoint values             */
    int32_t n_name_bytes;  /* total kind-name bytes               */
    int32_t pad0;
    /* Optional: if non-NULL every section below lies inside [blob, blob +
     * blob_bytes) and the planner moves the batch with one copy. */
    const void* blob;
    uint64_t blob_bytes;
    const ws_plan_rec* plans; /* [n_plans] */
    /* modules (ModuleDecl workload.hpp:27-40 + per-kind curve sources) [n_modules] */
    const int32_t* mod_plan;     /* owning plan                                   */
    const int32_t* mod_layers;   /* layers                                        */
    const int32_t* mod_tp;       /* tp_degree                                     */
    const int32_t* mod_group;    /* param_group id, -1 = empty                    */
    const int32_t* mod_alias;    /* param_group spelled "m<k>": k, else -1        */
    const int64_t* mod_batch;    /* input.batch                                   */
    const uint64_t* mod_param;   /* param_bytes                                   */
    const uint64_t* mod_act;     /* act_bytes                                     */
    const uint64_t* mod_out;     /* out_bytes                                     */
    const double* mod_w;         /* flops_proxy                                   */
    const double* mod_c;         /* comm_proxy                                    */
    const int32_t* mod_name_off; /* kind bytes in names[]                         */
    const int32_t* mod_name_len;
    const int32_t* mod_truth_off; /* declared truth pieces (spec.truth)           */
    const int32_t* mod_truth_n;   /* -1: no truth entry                           */
    const int32_t* mod_prof_off;  /* profile points (spec.profiles)               */
    const int32_t* mod_prof_n;    /* -1: no profile entry                         */
    const int32_t* mod_bp_off;    /* breakpoints (spec.breakpoints)               */
    const int32_t* mod_bp_n;      /* -1: no breakpoints entry                     */
    const int32_t* mod_pre_err;   /* host-detected fit-stage error (ws_err), 0    */
    /* tasks [n_task_total]: token range and rank of the id among the plan's ids */
    const int32_t* task_tok_off;
    const int32_t* task_tok_n;
    const int32_t* task_rank;
    const int32_t* tokens;        /* [n_tokens]                                    */
    const int32_t* dev_island;    /* [n_devices] island index of device i          */
    const double* truth;          /* [n_pieces*5]: n_lo n_hi alpha beta_c beta_w   */
    const int32_t* prof_n;        /* [n_points]                                    */
    const double* prof_t;         /* [n_points]                                    */
    const int32_t* bps;           /* [n_bps]                                       */
    const uint8_t* names;         /* [n_name_bytes]                                */
    /* Optional (plan evaluation of parsed plan files, NULL = 1.0 everywhere):
     * PlanEntity::batch_fraction per module row (plan_io.hpp:36). */
    const double* mod_frac;       /* [n_modules]                                   */
} ws_batch;

/* ---- per-plan result header ------------------------------------------------ */
typedef struct ws_plan_result {
    int32_t status;    /* ws_status                                             */
    int32_t err_code;  /* ws_err                                                */
    int64_t err_a, err_b;
    double err_x, err_y;
    int32_t n_metaops, n_edges, n_levels, n_waves;
    int32_t n_entries, n_flows, n_pieces;
    int32_t n_scopes;   /* task-scoped strategies: entities are (MetaOp, task) pairs */
    double lower_bound; /* PlannerResult::lower_bound (planner.hpp:189)          */
    double end_time;    /* predicted_makespan = schedule.end_time (:193-194)      */
    uint64_t offset;    /* byte offset of this plan's record in the arena        */
    uint64_t size;      /* record bytes                                          */
} ws_plan_result;

/* Arena record of one plan: the sections below, in this order, each 8-byte
 * aligned.  MetaOps are indexed by their number k (id "m<k>", graph.hpp:175). */
typedef struct ws_out_metaop {
    int32_t module;      /* local module index (kind)                          */
    int32_t level;       /* MetaOp::level (graph.hpp:207-226)                  */
    int32_t first_layer; /* first member operator layer                        */
    int32_t length;      /* L_m                                                */
    int32_t piece_begin; /* into the pieces section                            */
    int32_t piece_count;
    int32_t upper_n, upper_l; /* TuplePair::upper (allocation.hpp:31-34)       */
    int32_t lower_n, lower_l; /* lower tuple; lower_l == 0: absent             */
} ws_out_metaop;

typedef struct ws_out_level {
    double c_star;        /* AllocationPlan::c_star                             */
    int32_t first_wave;   /* WavefrontSchedule::level_boundaries                 */
    int32_t n_waves;
} ws_out_level;

typedef struct ws_out_piece {
    double n_lo, n_hi, alpha, beta_c, beta_w; /* CurvePiece (scaling.hpp:25-31) */
} ws_out_piece;

typedef struct ws_out_edge {
    int32_t from, to; /* MetaGraph::edges, std::set<pair<string,string>> order */
} ws_out_edge;

typedef struct ws_out_wave {
    double start, duration; /* Wave (schedule.hpp:22-28) after merge_levels     */
    int32_t level, entry_begin, n_entries, pad;
} ws_out_wave;

typedef struct ws_out_entry {
    double span;         /* layers * T(n)                                        */
    uint64_t devmask;    /* placement device set, devices 0..63 (bit i = i-th device id);
                            devices 64.. of a wider cluster are in the last section */
    int32_t metaop, n, layers;
    int32_t rot;         /* device-list start index (sequential ablation order)  */
} ws_out_entry;

enum ws_flow_mode { WS_FLOW_COPY = 0, WS_FLOW_INTRA = 1, WS_FLOW_INTER = 2 };

typedef struct ws_out_flow {
    uint64_t volume;
    int32_t from_wave, from_metaop, to_wave, to_metaop;
    int32_t mode, pad;
} ws_out_flow;

/* Section after the flows, only for task-scoped strategies (n_scopes > 0):
 * entity k of the record is PlanEntity "m<metaop>@<task id>"
 * (baselines.hpp:49-55); its ws_out_metaop row carries the MetaOp's module,
 * level, length and base curve.
 * Last section, only for clusters of more than 64 devices: 3 uint64_t per
 * entry, words 1..3 of its device set (devices 64..255): entry e's word j at
 * [3 * e + j - 1]. */
typedef struct ws_out_scope {
    int32_t metaop, task; /* task = declaration index within the plan */
} ws_out_scope;

/* ---- plan evaluation: simulate_plan + validate_plan (simulate.hpp, validate.hpp)
 * Evaluates planned records (ws_plan_result + arena, from the planner or any
 * producer of the same layout) on the device. */
typedef struct ws_sim_opts {   /* SimulatorOptions (simulate.hpp:69-73)                */
    double backward_ratio;     /* backward compute as a multiple of forward (2.0)       */
    int32_t zero_volumes;      /* free transmissions                                   */
    int32_t skip_sync;         /* no parameter synchronization                         */
} ws_sim_opts;

typedef struct ws_sim_result {
    int32_t status;         /* WS_STATUS_OK, or the plan's own status (not evaluated)  */
    int32_t valid;          /* ValidationReport::ok (validate.hpp:58-188)              */
    int32_t n_violations;   /* violations found (the first WS_SIM_MAX_VIOLATIONS kept)  */
    int32_t timeline_items; /* SimulationReport::timeline.size()                       */
    double makespan;        /* SimulationReport (simulate.hpp:53-67)                   */
    double fwd_bwd_seconds, param_sync_seconds, send_recv_seconds;
    double fwd_bwd_fraction, param_sync_fraction, send_recv_fraction;
    double total_transferred_bytes, total_inter_island_bytes;
    uint64_t offset;        /* this plan's record in the simulation arena:             */
    uint64_t size;          /*   busy[N] f64, busy_mask (1 u64; 4 when N > 64),         */
                            /*   mem[N] f64, util[K] f64, util_mask u64,               */
                            /*   ws_out_violation[min(n, MAX)]                         */
} ws_sim_result;

#define WS_SIM_MAX_VIOLATIONS 16

/* One ValidationReport::fail() call; the host rebuilds the reference message. */
enum ws_violation {
    WS_V_UNKNOWN_ENTITY = 1, /* "wave <w>: unknown entity m<a>"                               */
    WS_V_DUPLICATE = 2,      /* "wave <w>: entity m<a> appears twice"                          */
    WS_V_SPAN = 3,           /* "wave <w>: entity m<a> recorded span <x> != recomputed <y>"    */
    WS_V_SPAN_DURATION = 4,  /* "wave <w>: entry span exceeds wave duration"                   */
    WS_V_WAVE_DEVICES = 5,   /* "wave <w>: allocations exceed device count"                    */
    WS_V_WORK = 6,           /* "entity m<a>: executed <b> of <x> layers"                      */
    WS_V_CAPACITY = 7,       /* "capacity exceeded at t=<x>: <a> devices"                      */
    WS_V_OVERLAP = 8,        /* "entity m<a>: overlapping execution intervals"                 */
    WS_V_DEPENDENCY = 9,     /* "dependency m<a> -> m<b> violated: consumer starts at <x> ..." */
    WS_V_UNPLACED = 10,      /* "wave <w>: entity m<a> unplaced"                               */
    WS_V_DEVICE_COUNT = 11,  /* "wave <w>: entity m<a> placed on <b> devices, needs <x>"       */
    WS_V_UNKNOWN_DEVICE = 12,/* "unknown device <a>" (a = device index)                        */
    WS_V_DEVICE_TWICE = 13,  /* "wave <w>: device <a> assigned twice" (a = device index)       */
    WS_V_MEMORY = 14         /* "device <a> memory <x> exceeds capacity <y as u64 bits>"       */
};

typedef struct ws_out_violation {
    int32_t code, wave, a, b;
    double x, y;
} ws_out_violation;

/* ---- context & planning --------------------------------------------------- */
typedef struct ws_ctx ws_ctx;

/* Creates a planning context bound to CUDA device `device`.  Returns 0 on
 * success; the ctx owns device buffers and a stream. */
int ws_ctx_create(int device, ws_ctx** out);
void ws_ctx_destroy(ws_ctx* ctx);
/* Text of the last error on this ctx (CUDA failures, bad arguments). */
const char* ws_ctx_last_error(const ws_ctx* ctx);

/* Replaces wavesched::plan_workload over a whole batch (planner.hpp:156-212).
 * `in` points to HOST memory; results and arena are written to HOST memory.
 * The H2D copy, all kernels and the D2H copies run on the ctx stream (or on
 * `stream` if non-NULL, a cudaStream_t).  Never throws; per-plan failures are
 * reported in results[i].status.  Returns 0 unless the call itself failed. */
int ws_plan_batch_host(ws_ctx* ctx, const ws_batch* in, ws_plan_result* results, uint8_t* arena,
                       uint64_t arena_cap, uint64_t* arena_used, void* stream);

/* Device-resident variant for throughput measurement: ws_stage_batch copies a
 * host batch into ctx-owned device memory once; ws_plan_staged then plans it
 * entirely on the device (results stay in device memory until ws_fetch_results). */
int ws_stage_batch(ws_ctx* ctx, const ws_batch* in, void* stream);
int ws_plan_staged(ws_ctx* ctx, void* stream);
int ws_fetch_results(ws_ctx* ctx, ws_plan_result* results, uint8_t* arena, uint64_t arena_cap,
                     uint64_t* arena_used, void* stream);
/* Number of kernel launches issued by the last ws_plan_staged / ws_plan_batch_host. */
int ws_last_launch_count(const ws_ctx* ctx);
/* Plans of the last planning call that overflowed the launch's soft record caps
 * and were re-planned with the hard caps (all of them, any number; valid once
 * the results were fetched).  Diagnostic only: results never depend on it. */
long long ws_last_retry_count(const ws_ctx* ctx);
/* Device time (ms) of each planner kernel in the last planning call, measured
 * with CUDA events on the launching stream: out[0]=k_fit, out[1]=k_sched,
 * out[2]=k_place (including the soft-cap retry pass). */
int ws_last_kernel_ms(const ws_ctx* ctx, double* out, int n);

/* Global best candidate: on-device argmin of key over the staged
 * batch, key = end_time / lower_bound (mode 0), end_time (mode 1), or the
 * simulated makespan of the last ws_simulate_staged (mode 2); infeasible
 * plans count as +inf; ties go to the smaller index.  Writes {key, index}. */
int ws_best_staged(ws_ctx* ctx, int mode, double* key, int64_t* index, void* stream);
/* The candidate search of one workload in one call: plans the HOST batch `in`
 * (its candidate variants), evaluates it when mode == 2 (sim: SimulatorOptions,
 * NULL = defaults), and returns the min-loc as ws_best_staged does.  Batches
 * of up to 512 plans take the small-batch launch (one H2D copy, no retry pass,
 * one 16-byte copy back); the records stay on the device (ws_fetch_results). */
int ws_best_batch_host(ws_ctx* ctx, const ws_batch* in, int mode, const ws_sim_opts* sim, double* key,
                       int64_t* index, void* stream);

/* ---- multi-GPU -------------------------------------------------
 * One process, several GPUs: plans `in` (HOST memory) sharded over n_ctx
 * contexts (one per GPU; the same device twice is allowed) as contiguous
 * blocks of equal estimated cost, each block on its own host thread through
 * the pipelined host call; results/arena as for ws_plan_batch_host (offsets
 * into the one arena, bound ws_arena_bound(in)).  Replaces a loop of
 * wavesched::plan_workload calls (planner.hpp:156-212) spread over the box. */
int ws_plan_batch_multi(ws_ctx* const* ctxs, int n_ctx, const ws_batch* in, ws_plan_result* results,
                        uint8_t* arena, uint64_t arena_cap, uint64_t* arena_used);
/* min-loc over host results: key = end_time / lower_bound (mode 0) or
 * end_time (mode 1); infeasible plans lose; ties -> smaller index. */
int ws_best_host(const ws_plan_result* results, int64_t n, int mode, double* key, int64_t* index);
/* Several processes, one rank per GPU: all-gathers every rank's local best
 * {key, global index} (16 bytes) over the caller's NCCL communicator
 * (`nccl_comm` is an ncclComm_t; NCCL is loaded with dlopen) and returns the
 * global min-loc on every rank (ties -> smaller index; index < 0 = none). */
int ws_best_nccl(ws_ctx* ctx, void* nccl_comm, int nranks, double local_key, int64_t local_index, double* key,
                 int64_t* index, void* stream);

/* Profiling aid: SM cycles per planner phase summed over warps since the last
 * call (k_place 0-7, k_sched 10-14); all zero unless built with -DWS_PHASES. */
int ws_debug_phase_cycles(unsigned long long* out, int n);

/* Arena capacity sufficient for any batch whose plans stay within the limits. */
uint64_t ws_arena_bound(const ws_batch* in);

/* Replaces wavesched::simulate_plan + validate_plan (simulate.hpp:322-324,
 * validate.hpp:58-188) for every planned record of the last ws_plan_staged /
 * ws_plan_batch_host call on this ctx, on the device (plans that failed keep
 * their status and are not evaluated).  Results stay on the device until
 * ws_fetch_sim. */
int ws_simulate_staged(ws_ctx* ctx, const ws_sim_opts* opts, void* stream);
int ws_fetch_sim(ws_ctx* ctx, ws_sim_result* out, uint8_t* arena, uint64_t arena_cap, uint64_t* arena_used,
                 void* stream);
/* Same over plan records supplied from HOST memory (any producer of the
 * ws_plan_result + arena layout, e.g. an edited plan): stages `in` and the
 * records, simulates + validates, and writes HOST results. */
int ws_simulate_batch_host(ws_ctx* ctx, const ws_batch* in, const ws_plan_result* plans, const uint8_t* plan_arena,
                           uint64_t plan_arena_bytes, const ws_sim_opts* opts, ws_sim_result* out, uint8_t* arena,
                           uint64_t arena_cap, uint64_t* arena_used, void* stream);
/* Simulation-arena capacity for a batch (every plan evaluated). */
uint64_t ws_sim_arena_bound(const ws_batch* in);
/* Device time (ms) of the last simulation launch. */
double ws_last_sim_ms(const ws_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* WSGPU_WS_ABI_H */
