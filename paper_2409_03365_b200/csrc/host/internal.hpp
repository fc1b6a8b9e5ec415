// internal.hpp — host helpers shared by the drop-in entry points (not installed).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "wsgpu/planner.hpp"

namespace wsgpu::detail {

// Growable page-locked host buffer (cudaMallocHost), reused across calls so
// the drop-in pays no page-locking per plan.
struct HostBuffer {
    std::uint8_t* p = nullptr;
    std::size_t cap = 0;
    std::vector<std::uint8_t*> retired;  // outgrown blocks, freed with the buffer
    bool ensure(std::size_t bytes);
    ~HostBuffer();
    HostBuffer() = default;
    HostBuffer(const HostBuffer&) = delete;
    HostBuffer& operator=(const HostBuffer&) = delete;
};

// encode_batch into `reuse` (when non-null and it can grow) with the
// per-problem preparation spread over `threads` host threads.
EncodedBatch encode_batch_with(const std::vector<Problem>& problems, bool pinned, HostBuffer* reuse, int threads);

// A planning context plus its reusable page-locked staging buffers, checked out
// of a per-device pool for one call: concurrent callers (one per host thread)
// each hold their own, so drop-in calls run in parallel ("pure and
// reentrant"); idle leases stay pooled for the next call.
struct Lease;
class CtxLease {
public:
    // the calling thread's current CUDA device ($WSGPU_DEVICE overrides);
    // throws Error when no CUDA planner can run (no fallback)
    CtxLease();
    explicit CtxLease(int device);
    ~CtxLease();
    CtxLease(const CtxLease&) = delete;
    CtxLease& operator=(const CtxLease&) = delete;
    ws_ctx* ctx() const;
    HostBuffer& in() const;
    HostBuffer& results() const;
    HostBuffer& arena() const;

private:
    Lease* l_ = nullptr;
    int device_ = 0;
};

// Host results of one planning batch: headers + the record arena.
struct Planned {
    std::vector<ws_plan_result> res;
    std::vector<std::uint8_t> arena;
};

// Plans a problem list on a leased context; plans whose record overflowed the
// arena are re-planned alone with a large arena.  Throws Error if the call
// itself fails.
Planned plan_on(CtxLease& lease, const std::vector<Problem>& probs, int threads = 1);

// One problem planned into the lease's page-locked buffers (no copies): the
// header and its record stay valid until the lease's next call.
struct PlannedOne {
    const ws_plan_result* res;
    const std::uint8_t* arena;
    std::vector<std::uint8_t> own;  // only for a record that overflowed the lease arena
};
PlannedOne plan_one(CtxLease& lease, const Problem& prob);

// "ParseError", "PlacementInfeasible", ... : the most derived reference
// exception class of `e` (the "error <Class>: <what>" convention).
const char* error_class(const std::exception& e);

char* dup_c(const std::string& s);

}  // namespace wsgpu::detail
