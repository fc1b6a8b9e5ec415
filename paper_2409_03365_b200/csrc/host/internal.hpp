// internal.hpp — host helpers shared by the drop-in entry points (not installed).
#pragma once
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "wsgpu/planner.hpp"

namespace wsgpu::detail {

// Host results of one planning batch: headers + the record arena.
struct Planned {
    std::vector<ws_plan_result> res;
    std::vector<std::uint8_t> arena;
};

// Plans a problem list on `ctx`; plans whose record overflowed the arena are
// re-planned alone with a large arena.  Throws Error if the call itself fails.
Planned plan_on(ws_ctx* ctx, const std::vector<Problem>& probs);

// The process-wide default context (CUDA device 0, or $WSGPU_DEVICE), locked
// for the lifetime of `lock`.  Throws Error when no CUDA planner can run.
ws_ctx* default_ctx_locked(std::unique_lock<std::mutex>& lock);

// "ParseError", "PlacementInfeasible", ... : the most derived reference
// exception class of `e` (the "error <Class>: <what>" convention).
const char* error_class(const std::exception& e);

char* dup_c(const std::string& s);

}  // namespace wsgpu::detail
