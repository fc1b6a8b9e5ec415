/* bounds.h — per-plan output-arena bounds shared by the host entry points
 * (decode.cpp ws_arena_bound, sim_text.cpp ws_sim_arena_bound) and the
 * pipelined host call (planner.cu), which sums them per chunk in its single
 * pass over the plan records.  Private header. */
#pragma once
#include "wsgpu/ws_abi.h"

/* planning record: MetaOps, levels, pieces, edges, waves, entries, flows */
static inline uint64_t wsi_plan_arena_bound(const ws_plan_rec* r) {
    const uint64_t M = (uint64_t)r->n_mod;
    return 64 + sizeof(ws_out_metaop) * M + sizeof(ws_out_level) * M + sizeof(ws_out_piece) * 4 * M +
           sizeof(ws_out_edge) * M * M + sizeof(ws_out_wave) * 4 * M + sizeof(ws_out_entry) * 8 * M +
           sizeof(ws_out_flow) * 16 * M + (r->n_dev > 64 ? 24 * 8 * M : 0);
}

/* evaluation record: busy/mem per device, utilization per entity, violations */
// words of the busy_mask field of a simulation record (ws_abi.h ws_sim_result)
static inline uint64_t sim_mask_words(uint64_t n_dev) { return n_dev > 64 ? 4 : 1; }

static inline uint64_t wsi_plan_sim_bound(const ws_plan_rec* r) {
    // a batch with a wider cluster evaluates every plan with 4-word masks
    return 16ull * r->n_dev + 8ull * r->n_mod + 8 * 4 + 8 + sizeof(ws_out_violation) * WS_SIM_MAX_VIOLATIONS;
}
