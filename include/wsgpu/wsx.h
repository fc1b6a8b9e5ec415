/*
 * wsx.h — host-side helper C-ABI around ws_abi.h for FFI callers (Python
 * ctypes, tests, bench).  Builds problem sets from the reference's own input
 * forms — workload/topology text (workload.hpp:139-210, topology.hpp:59-101),
 * the scenario generator (scenarios.hpp:292) and the SURVEY §8(d) sweep — and
 * turns planner results back into the reference's plan text
 * (plan_io.hpp:53-110) or exception text.
 */
#ifndef WSGPU_WSX_H
#define WSGPU_WSX_H

#include <stdint.h>

#include "wsgpu/ws_abi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* PlannerOptions (planner.hpp:21-27) flattened. */
typedef struct ws_options {
    double eps;         /* AllocatorOptions::eps = 1e-7        */
    int32_t max_iters;  /* AllocatorOptions::max_iters = 200   */
    int32_t sequential; /* PlacementOptions::sequential = 0    */
    double drop_floor;  /* AllocatorOptions::drop_floor = 0    */
    int32_t bt_depth;   /* PlacementOptions::backtrack_depth = 2 */
    int32_t bt_branching; /* PlacementOptions::backtrack_branching = 3 */
    double grad_mult;   /* grad_opt_multiplier = 3             */
    double synth_noise; /* = 0                                 */
    uint64_t synth_seed;/* = 0                                 */
    int32_t strategy;   /* ws_strategy (plan_for_strategy selector) = 0 wavefront */
    int32_t pad;
} ws_options;

void wsx_default_options(ws_options* o);

typedef struct wsx_set wsx_set;
wsx_set* wsx_set_new(void);
void wsx_set_free(wsx_set* s);
int32_t wsx_set_size(const wsx_set* s);
/* Each add returns the problem index, or -1 (see wsx_set_error). */
int32_t wsx_add_text(wsx_set* s, const char* workload, const char* topology, const ws_options* o);
/* JSON workload / topology (cli.hpp:46-110 workload_from_json, topology_from_json);
 * an argument not starting with '{' is read with the text grammar instead. */
int32_t wsx_add_json(wsx_set* s, const char* workload, const char* topology, const ws_options* o);
int32_t wsx_add_scenario(wsx_set* s, const char* name, int32_t tasks, int32_t devices, uint64_t seed,
                         const ws_options* o);
int32_t wsx_add_sweep(wsx_set* s, int64_t start, int64_t count, const ws_options* o);
const char* wsx_set_error(const wsx_set* s);
/* Encodes all problems; the view stays valid until the next encode/free. */
const ws_batch* wsx_encode(wsx_set* s, int32_t pinned);
uint64_t wsx_encoded_bytes(const wsx_set* s);
/* Plan text (write_plan) or "error <Class>: <what>\n" of problem i; free with wsx_free_str. */
char* wsx_result_text(const wsx_set* s, int32_t i, const ws_plan_result* results, const uint8_t* arena);
/* Canonical evaluation text (simulate_plan + validate_plan, see sim_text.cpp)
 * of problem i, or its planner error text; free with wsx_free_str. */
char* wsx_sim_text(const wsx_set* s, int32_t i, const ws_plan_result* results, const uint8_t* arena,
                   const ws_sim_result* sims, const uint8_t* sim_arena);
char* wsx_dump_workload(const wsx_set* s, int32_t i);
char* wsx_dump_topology(const wsx_set* s, int32_t i);
void wsx_free_str(char* p);

/* SURVEY §8(d) compulsory (algorithmic) input/output bytes of the encoded set
 * and its results: the roofline numerator. */
void wsx_algorithmic_bytes(const wsx_set* s, const ws_plan_result* results, const uint8_t* arena,
                           uint64_t* in_bytes, uint64_t* out_bytes);

/* Plan files of any strategy (parse_plan, plan_io.hpp:112-255) as evaluator
 * input: each plan becomes a batch row + a planned record (ws_abi.h layout)
 * that ws_simulate_batch_host evaluates on the device. */
typedef struct wsx_plans wsx_plans;
wsx_plans* wsx_plans_new(void);
void wsx_plans_free(wsx_plans* p);
int32_t wsx_plans_size(const wsx_plans* p);
/* Returns the plan index, or -1 with the ParseError text in wsx_plans_error. */
int32_t wsx_plans_add_text(wsx_plans* p, const char* plan_text);
const char* wsx_plans_error(const wsx_plans* p);
/* Encodes every plan; returns the batch (NULL on an unsupported plan, see
 * wsx_plans_error) and the host records to pass to ws_simulate_batch_host. */
const ws_batch* wsx_plans_encode(wsx_plans* p, int32_t pinned, const ws_plan_result** results,
                                 const uint8_t** arena, uint64_t* arena_bytes);
/* write_plan text of parsed plan i (round trip); canonical evaluation text. */
char* wsx_plans_write(const wsx_plans* p, int32_t i);
char* wsx_plans_sim_text(const wsx_plans* p, int32_t i, const ws_sim_result* sims, const uint8_t* sim_arena);

/* Page-locked host buffers for results/arena (cudaMallocHost; plain malloc
 * when no CUDA device is present).  Not zero-initialized. */
void* wsx_host_alloc(uint64_t bytes);
void wsx_host_free(void* p);

/* Drop-in single-plan call through the process default context:
 * plan text, or "error <Class>: <what>\n". */
char* wsx_plan_workload_text(const char* workload, const char* topology, const ws_options* o);

/* plan_for_strategy (cli.hpp:163-171) on reference text inputs: plan text, or
 * "error <Class>: <what>\n". */
char* wsx_plan_strategy_text(const char* workload, const char* topology, const char* strategy,
                             const ws_options* o);

/* The reference's compare / dynamic commands (cli.hpp:243-327) over the device
 * planner + evaluator: all (phase, strategy) pairs in one planning batch and one
 * evaluation launch.  Writes the reference's files under out_dir and returns the
 * text the command prints, or "error <Class>: <what>\n" (exit codes 2/3/4 by
 * class, cli.hpp:330-344). */
char* wsx_cmd_compare(const char* workload_path, const char* topology_path, const char* out_dir,
                      const ws_options* o);
char* wsx_cmd_dynamic(const char* sequence_path, const char* topology_path, const char* out_dir,
                      const ws_options* o);

#ifdef __cplusplus
}
#endif
#endif /* WSGPU_WSX_H */
