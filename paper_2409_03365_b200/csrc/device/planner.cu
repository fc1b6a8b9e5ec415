// planner.cu — C-ABI implementation: planning context, device buffers and the
// launch sequence of the sm_100a planner kernels.
//
//   k_fit    (subsystem 2)        one thread (large batches) or warp (small) per declared module
//   k_sched  (subsystems 1, 3, 4a) one warp per plan, working set in shared memory
//   k_place  (subsystem 4b + out)  one warp per plan, working set in shared memory
//   retry    plans that overflow the soft record caps re-run with the hard
//            caps; the list is built and counted on the device (no host sync)
//   k_best   global-best candidate (min-loc) over the batch
//
// Plans are launched in descending estimated cost (longest-processing-time
// order) so the long plans start first and the tail of each launch is short.
// Replaces wavesched::plan_workload (planner.hpp:156-212) for whole batches.
#include <cuda_runtime.h>

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <limits>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../host/bounds.h"
#include "fit.cuh"
#include "place.cuh"
#include "sched.cuh"
#include "sim.cuh"

using namespace wsdev;

namespace {

constexpr int kRetryMax = 1024;               // plans re-run with hard caps per retry launch
constexpr int64_t kOverflowPieces = 1 << 18;  // isotonic/long curves
constexpr int kSmemLimit = 227 * 1024;
constexpr int kMaxChunks = 16;  // k_sched/k_place pipeline depth
constexpr int kMaxHostChunks = 8;
constexpr int kSplitMin = 2048;
constexpr int kBestBatchMax = 512;  // ws_best_batch_host: batches up to this take the small-batch launch  // launches of at least this many plans run k_sched as three phase kernels
// k_place snapshot slots: only warps of plans that fail a wave claim one (a few
// hundred per 100k sweep), so a small pool serves every resident warp; a warp
// that finds none falls back to replaying the committed waves
constexpr int kSnapSlots = 512;
// arena bound up to which ws_fetch_results copies the whole bound in one go
constexpr uint64_t kOneSyncArena = 256u << 10;  // H2D / compute / D2H pipeline depth of ws_plan_batch_host

// host_tops (page-locked u64 words): [0, 8) chunk arena bases, [8, 16) chunk
// arena tops, [16] final top, [17] fetched top, [18] retry count of a staged
// call, [20, 22) the last min-loc, [24, 32) retry counts of the pipelined chunks
constexpr int kHostTopsWords = 4 * kMaxHostChunks + 8;
constexpr int kHtFinal = 2 * kMaxHostChunks, kHtFetch = kHtFinal + 1, kHtRetry = kHtFinal + 2;
constexpr int kHtBest = kHtFinal + 4;  // [20, 22): {key, index} of k_best
constexpr int kHtChunkRetry = 3 * kMaxHostChunks;

// Makes `device` current for the scope of an entry point and restores the
// caller's device on every exit path (the caller's torch/CUDA state stays put).
struct DevGuard {
    int prev = -1;
    bool ok = true;
    explicit DevGuard(int device) {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
        if (prev != device) ok = cudaSetDevice(device) == cudaSuccess;
    }
    ~DevGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// Device buffer that only grows.  A grown buffer's old block is retired, not
// freed: cudaFree synchronizes the whole device (every other host thread's
// context included), and kernels of this ctx still in flight may use it.
// Growth is geometric (1.5x) so a ctx settles after a few calls.
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    std::vector<void*> retired;
    bool ensure(size_t bytes) {
        if (bytes <= n) return true;
        const size_t want = std::max(bytes, n + n / 2);
        void* q = nullptr;
        if (cudaMalloc(&q, want) != cudaSuccess) {
            cudaGetLastError();
            if (want == bytes || cudaMalloc(&q, bytes) != cudaSuccess) return false;
            n = bytes;
        } else {
            n = want;
        }
        if (p) retired.push_back(p);
        p = q;
        return true;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
        for (void* q : retired) cudaFree(q);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// plans whose soft record caps overflowed get queued for the retry pass: ALL
// of them (ids has room for every plan of the range); the first retry launch
// covers the first kRetryMax without a host round trip, drain_overflow() the rest
__global__ void k_soft_collect(const ws_plan_result* res, int p_begin, int p_end, int32_t* ids, int32_t* count) {
    const int p = p_begin + blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= p_end) return;
    const int e = res[p].err_code;
    if (e == WS_E_LIMIT_WAVES || e == WS_E_LIMIT_ENTRIES || e == WS_E_LIMIT_FLOWS) ids[atomicAdd(count, 1)] = p;
}

// Global min-loc over plan keys; ties -> smaller index.
__global__ void k_best(const ws_plan_result* res, const ws_sim_result* sim, int n, int mode, double* out_key,
                       long long* out_idx) {
    __shared__ double sk[1024];
    __shared__ long long si[1024];
    double bk = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    long long bi = -1;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        const ws_plan_result& r = res[p];
        if (r.status != WS_STATUS_OK || (mode == 2 && sim[p].status != WS_STATUS_OK)) continue;
        const double k = mode == 0 ? r.end_time / r.lower_bound : (mode == 1 ? r.end_time : sim[p].makespan);
        if (bi < 0 || k < bk || (k == bk && p < bi)) bk = k, bi = p;
    }
    sk[threadIdx.x] = bk;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s) {
            const double ok = sk[threadIdx.x + s];
            const long long oi = si[threadIdx.x + s];
            if (oi >= 0 && (si[threadIdx.x] < 0 || ok < sk[threadIdx.x] ||
                            (ok == sk[threadIdx.x] && oi < si[threadIdx.x]))) {
                sk[threadIdx.x] = ok;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *out_key = sk[0];
        *out_idx = si[0];
    }
}

struct LaunchCaps {
    RecCaps rec;
    PlaceCaps pl;
    int M;        // modules (MetaOps) per plan
    int T;        // tasks per plan
    bool scoped;  // the batch has task-scoped baseline plans
    bool baseline;  // the batch has baseline-strategy plans (k_place<true>)
};

// Batch maxima that size a launch (one pass over the plan records).
struct BatchMax {
    int M = 1, N = 1, IS = 1, gmax = 0, T = 1;
    bool scoped = false, baseline = false;
    void add(const ws_plan_rec& r) {
        M = std::max(M, r.n_mod);
        N = std::max(N, r.n_dev);
        IS = std::max(IS, r.n_islands);
        gmax = std::max(gmax, r.n_groups);
        T = std::max(T, r.n_tasks);
        scoped |= r.strategy == WS_STRATEGY_DISTMM_MT || r.strategy == WS_STRATEGY_TASK_OPTIMUS;
        baseline |= r.strategy != WS_STRATEGY_WAVEFRONT;
    }
};

LaunchCaps caps_from(const BatchMax& b, bool hard, bool tiny = false) {
    const int M = std::min(b.M, WS_MAX_MODULES);
    const int N = std::min(b.N, WS_MAX_DEVICES);
    const int IS = std::min(b.IS, N);
    // placement entities: the MetaOps, or up to 64 (MetaOp, task) pairs
    const int ME = b.scoped ? WS_MAX_MODULES : M;
    const int W = std::min(WS_MAX_WAVES, 2 * ME + 1);  // each wave drains a tuple
    int E, F;
    if (hard) {
        E = std::min(WS_MAX_ENTRIES, std::max(64, 2 * ME * ME));
        F = WS_MAX_FLOWS;
    } else if (tiny) {  // $WSGPU_TINY_SOFT_CAPS (tests): nearly every plan overflows
        E = 4;
        F = 2;
    } else {
        E = std::max(32, 4 * ME);
        F = std::max(64, 8 * ME);
    }
    LaunchCaps c;
    c.M = M;
    c.T = std::min(b.T, WS_MAX_TASKS);
    c.scoped = b.scoped;
    c.baseline = b.baseline;
    c.rec = RecCaps{ME, W, E};
    c.pl = PlaceCaps{ME, N, W, E, F, b.gmax + ME, IS};
    return c;
}

LaunchCaps batch_caps(const ws_plan_rec* plans, int P, bool hard, bool tiny = false) {
    BatchMax b;
    for (int p = 0; p < P; ++p) b.add(plans[p]);
    return caps_from(b, hard, tiny);
}

int warps_for(int bytes_per_warp, int want) {
    int w = want;
    while (w > 1 && w * bytes_per_warp > kSmemLimit) --w;
    return w;
}

}  // namespace

struct ws_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    // staged batch
    DevBuf blob, order;
    ws_batch dview{};
    std::vector<int32_t> key_count;              // LPT counting-sort histograms
    std::vector<uint16_t> lpt_keys;              // per-plan LPT key of the pipelined host call
    int32_t* order_pinned = nullptr;             // launch order, page-locked so its H2D
    size_t order_pinned_n = 0;                   //   copies stay asynchronous;
    cudaEvent_t order_ev = nullptr;              //   recorded after the last one (the host
    bool order_ev_pending = false;               //   waits on it before rewriting the buffer)
    LaunchCaps caps{}, caps_hard{};
    // K2 outputs
    DevBuf fit_err, fit_a, fit_b, fit_np, fit_nmax, fit_off, fit_pieces, ttab;
    // records, flows, results
    DevBuf recs, flows, recs_r, flows_r, results, arena, counters, retry_ids, best;
    DevBuf snap, snap_bits;    // k_place backtracking snapshot pool (kSnapSlots slots)
    long long snap_stride = 0; // 8-byte words per slot
    uint64_t arena_cap = 0;
    int launches = 0;
    cudaEvent_t ev[4] = {};
    cudaStream_t stream2 = nullptr;             // k_place side of the pipeline
    cudaEvent_t cev[kMaxChunks + 2] = {};       // chunk hand-offs + fork/join
    int chunks = 1;  // measured: concurrent k_sched/k_place chunks share the I-cache and lose ($WSGPU_CHUNKS)
    double kernel_ms[3] = {0, 0, 0};  // k_fit, k_sched, k_place (+ retry pass)
    bool staged_events = false;       // ev[0..3] bracket the kernels of the last ws_plan_staged
    // plan evaluation (k_sim)
    DevBuf sim_res, sim_arena, sim_scratch, sim_top;
    uint64_t sim_cap = 0;           // ws_sim_arena_bound of the staged batch
    bool records_on_device = false; // the last planning call left its records in ctx memory
    bool sim_valid = false;         // sim_res holds the evaluation of the staged records
    cudaEvent_t sev[2] = {};
    double sim_ms = 0;
    // direct output: kernels write headers/records straight into the caller's
    // page-locked host buffers (zero-copy), set only inside ws_plan_batch_host
    ws_plan_result* d_results = nullptr;
    uint8_t* d_arena = nullptr;
    uint64_t d_cap = 0;
    // pipelined host call: arena top counter / capacity of the chunk in flight
    unsigned long long* top_ptr = nullptr;
    uint64_t top_cap = 0;
    DevBuf chunk_tops;
    cudaStream_t stream3 = nullptr;          // D2H side of the host pipeline (stream2: H2D side)
    cudaStream_t stream4 = nullptr;          // second compute stream of the host pipeline
    cudaStream_t stream5 = nullptr;          // third compute stream ($WSGPU_HOST_STREAMS=3)
    DevBuf recs_r2, flows_r2, recs_r3, flows_r3;  // their retry-pass buffers
    cudaEvent_t join_ev = nullptr;           // joins the third compute stream
    unsigned long long* host_tops = nullptr; // page-locked: chunk bases, chunk tops, final top, retry counts
    // soft-cap overflows beyond the first retry launch (kRetryMax plans): the
    // overflow count is copied back asynchronously and the remaining plans are
    // re-planned at the next call that consumes the staged results
    cudaEvent_t drain_ev = nullptr;
    bool drain_pending = false;
    cudaStream_t drain_stream = nullptr;
    long long last_retry = 0;   // soft-cap overflows of the last planning call (all re-planned)
    bool tiny_soft = false;     // $WSGPU_TINY_SOFT_CAPS: soft caps below every plan (tests of the retry pass)
    bool small_path = true;     // $WSGPU_SMALL_PATH=0: small host batches take the staged path
    bool trace = false;         // $WSGPU_TRACE: host-side timing of the pipelined host call on stderr
    // k_sched as three phase kernels for launches of >= kSplitMin plans
    // ($WSGPU_SCHED_SPLIT: 0 never, 1 default, 2 always); state between them
    int sched_split = 1;
    DevBuf sched_state;
    // output records by k_emit after k_place for launches of >= kSplitMin plans
    // ($WSGPU_EMIT_SPLIT: 0 never, 1 default, 2 always); placement scratch
    int emit_split = 1;
    bool fixed_layout = true;  // $WSGPU_FIXED_LAYOUT=0: always the runtime-layout k_place
    DevBuf emit_mask, emit_rot, emit_nf;
    // measured (100k sweep, ms): one compute stream: 1 chunk 27.8, 2: 27.4, 4: 32.0 (each
    // chunk's k_sched + k_place launch tail outweighs the hidden copies); two compute
    // streams (consecutive chunks fill each other's tails) with completion-order D2H:
    // weights 1,3,1 24.9, 1,3,3,1 22.8, 1,4,4,1 22.8, 1,3,3,3,1 22.8, 1,5,5,1 23.8
    int host_chunks = 4;                     // $WSGPU_HOST_CHUNKS
    int host_streams = 2;                    // $WSGPU_HOST_STREAMS (1 to 3)
    bool force_snap = false;                 // $WSGPU_FORCE_SNAP: k_place<true> for every batch (tuning)
    // k_sched launched programmatic-dependent on k_fit: its graph stage overlaps
    // k_fit (measured: single-plan latency -7..-10%, 100k throughput unchanged);
    // k_fit's time is then reported inside k_sched's.  $WSGPU_PDL=0 disables.
    bool pdl = true;
    // $WSGPU_HOST_WEIGHTS (sets the chunk count).  Measured per 100k (profiles/
    // r2h_host_weights.txt): 1,4,4,2,1 14.4 ms, 2,3,3,2 13.9 ms -- with the heavy
    // backtracking tail gone (k_place attempt memo) a larger first chunk pays
    std::vector<double> host_weights{2, 3, 3, 2};
    ws_plan_result* res_out() { return d_results ? d_results : results.as<ws_plan_result>(); }
    // small host batches stage their zeroed counters with the batch (one H2D copy)
    unsigned long long* small_counters = nullptr;
    unsigned long long* counters_dev() { return small_counters ? small_counters : counters.as<unsigned long long>(); }
    uint8_t* small_host = nullptr;  // page-locked staging of the small-batch path
    size_t small_host_n = 0;
    std::vector<void*> retired_host;  // grown page-locked buffers (cudaFreeHost synchronizes: freed at destroy)
    uint8_t* arena_out() { return d_arena ? d_arena : arena.as<uint8_t>(); }
    uint64_t cap_out() const { return d_arena ? d_cap : arena_cap; }
};

namespace {

// arena top counter / capacity of a pipelined chunk for the launches in scope
struct TopScope {
    ws_ctx* c;
    TopScope(ws_ctx* ctx, unsigned long long* top, uint64_t cap) : c(ctx) {
        c->top_ptr = top;
        c->top_cap = cap;
    }
    ~TopScope() { c->top_ptr = nullptr; }
};

int fail(ws_ctx* c, const std::string& what, cudaError_t e = cudaSuccess) {
    c->err = what;
    if (e != cudaSuccess) c->err += std::string(": ") + cudaGetErrorString(e);
    return 1;
}

#define CK(call)                                            \
    do {                                                    \
        cudaError_t e_ = (call);                            \
        if (e_ != cudaSuccess) return fail(ctx, #call, e_); \
    } while (0)

// The dynamic shared-memory opt-in of every kernel, set ONCE per device to the
// most a block may take.  The attribute is process-wide state of the function:
// setting it per launch to that launch's size would let a concurrent context
// (another host thread) lower it between another launch's set and its launch.
template <typename K>
cudaError_t smem_opt_in(K* fn) {
    cudaFuncAttributes a{};
    cudaError_t e = cudaFuncGetAttributes(&a, fn);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemLimit - static_cast<int>(a.sharedSizeBytes));
}

cudaError_t smem_opt_in_all(int device) {
    static std::once_flag once[64];
    static cudaError_t status[64] = {};
    if (device < 0 || device >= 64) return cudaErrorInvalidDevice;
    std::call_once(once[device], [&] {
        cudaError_t e = smem_opt_in(k_sched<uint64_t>);
        if (e == cudaSuccess) e = smem_opt_in(k_sched<DevMask<4>>);
        if (e == cudaSuccess) e = smem_opt_in(k_sched<uint64_t, 1>);
        if (e == cudaSuccess) e = smem_opt_in(k_sched<uint64_t, 2>);
        if (e == cudaSuccess) e = smem_opt_in(k_sched<uint64_t, 3>);
        if (e == cudaSuccess) e = smem_opt_in(k_sched<DevMask<4>, 1>);
        if (e == cudaSuccess) e = smem_opt_in(k_sched<DevMask<4>, 2>);
        if (e == cudaSuccess) e = smem_opt_in(k_sched<DevMask<4>, 3>);
        if (e == cudaSuccess) e = smem_opt_in(k_sched_scoped<uint64_t>);
        if (e == cudaSuccess) e = smem_opt_in(k_sched_scoped<DevMask<4>>);
        if (e == cudaSuccess) e = smem_opt_in(k_place<true>);
        if (e == cudaSuccess) e = smem_opt_in(k_place<false>);
        if (e == cudaSuccess) e = smem_opt_in(k_place<true, DevMask<4>, 1, 1>);
        if (e == cudaSuccess) e = smem_opt_in(k_place<true, uint64_t, kPlaceWarps, WS_PLACE_MINB, true>);
        if (e == cudaSuccess) e = smem_opt_in(k_place<false, uint64_t, kPlaceWarps, WS_PLACE_MINB, true>);
        if (e == cudaSuccess) e = smem_opt_in(k_place<false, DevMask<4>, 1, 1>);
        if (e == cudaSuccess) e = smem_opt_in(k_sim<uint64_t>);
        if (e == cudaSuccess) e = smem_opt_in(k_sim<DevMask<4>>);
        status[device] = e;
    });
    return status[device];
}

// rebase every section pointer of a host batch into device memory at `dbase`
ws_batch rebase(const ws_batch& h, const void* hbase, char* dbase) {
    ws_batch d = h;
    auto mv = [&](auto* ptr) {
        using P = decltype(ptr);
        if (!ptr) return static_cast<P>(nullptr);
        return reinterpret_cast<P>(dbase + (reinterpret_cast<const char*>(ptr) - static_cast<const char*>(hbase)));
    };
    d.plans = mv(h.plans);
    d.mod_plan = mv(h.mod_plan);
    d.mod_layers = mv(h.mod_layers);
    d.mod_tp = mv(h.mod_tp);
    d.mod_group = mv(h.mod_group);
    d.mod_alias = mv(h.mod_alias);
    d.mod_batch = mv(h.mod_batch);
    d.mod_param = mv(h.mod_param);
    d.mod_act = mv(h.mod_act);
    d.mod_out = mv(h.mod_out);
    d.mod_w = mv(h.mod_w);
    d.mod_c = mv(h.mod_c);
    d.mod_name_off = mv(h.mod_name_off);
    d.mod_name_len = mv(h.mod_name_len);
    d.mod_truth_off = mv(h.mod_truth_off);
    d.mod_truth_n = mv(h.mod_truth_n);
    d.mod_prof_off = mv(h.mod_prof_off);
    d.mod_prof_n = mv(h.mod_prof_n);
    d.mod_bp_off = mv(h.mod_bp_off);
    d.mod_bp_n = mv(h.mod_bp_n);
    d.mod_pre_err = mv(h.mod_pre_err);
    d.task_tok_off = mv(h.task_tok_off);
    d.task_tok_n = mv(h.task_tok_n);
    d.task_rank = mv(h.task_rank);
    d.tokens = mv(h.tokens);
    d.dev_island = mv(h.dev_island);
    d.truth = mv(h.truth);
    d.prof_n = mv(h.prof_n);
    d.prof_t = mv(h.prof_t);
    d.bps = mv(h.bps);
    d.names = mv(h.names);
    d.mod_frac = mv(h.mod_frac);
    d.blob = dbase;
    return d;
}

// launch k_sched + k_place over `n` slots (plan ids from `ids`, count optionally
// on device).  With chunks > 1 the slots are split into consecutive chunks and
// k_place(chunk c) on a second stream overlaps k_sched(chunk c+1): the two
// kernels share the SMs, so each SM has more resident warps to hide latency.
int launch_pair(ws_ctx* ctx, cudaStream_t st, const LaunchCaps& lc, const FitOut& fo, const int32_t* ids,
                const int32_t* n_ids, int n, bool by_slot, char* recs, uint64_t* flows,
                cudaEvent_t mid = nullptr, int chunks = 1, bool pdl = false);

// 8-byte words of one k_place snapshot slot: W wave states of mem[N] doubles +
// chg[G] device masks (1 word each up to 64 devices, 4 above)
long long snap_words(const LaunchCaps& lc) {
    const int mw = lc.pl.N > 64 ? 4 : 1;
    return static_cast<long long>(lc.pl.W) * (lc.pl.N + static_cast<long long>(lc.pl.G) * mw);
}

}  // namespace

namespace {

int launch_pair(ws_ctx* ctx, cudaStream_t st, const LaunchCaps& lc, const FitOut& fo, const int32_t* ids,
                const int32_t* n_ids, int n, bool by_slot, char* recs, uint64_t* flows, cudaEvent_t mid,
                int chunks, bool pdl) {
    if (n <= 0) return 0;
    const ws_batch& B = ctx->dview;
    SchedArgs S{};
    S.B = B;
    S.fit = fo;
    S.caps = lc.rec;
    S.RL = make_rec_layout(lc.rec);
    // clusters over 64 devices: DevMask<4> instances (valid sets and device
    // masks of 4 words), k_place with one warp per block for the wider working set
    const bool wide = lc.pl.N > 64;
    const int mb = wide ? static_cast<int>(sizeof(DevMask<4>)) : 8;
    const int pw = wide ? 1 : kPlaceWarps;
    S.SL = make_sm_layout(lc.M, lc.scoped, lc.T, mb);
    S.warp_smem = S.SL.bytes;
    // (a compile-time layout for k_sched, as k_place has, measured slower: the
    // fixed class's larger working set costs occupancy and phase-state traffic)
    S.scoped_ok = lc.scoped ? 1 : 0;
    S.recs = recs;
    S.n_ids = n_ids;
    S.rec_by_slot = by_slot ? 1 : 0;
    S.M_cap = lc.M;
    S.results = ctx->res_out();
    if (kSchedWarps * S.SL.bytes > kSmemLimit) return fail(ctx, "k_sched working set exceeds shared memory");
    // phase-split k_sched (sched_body): smaller per-kernel instruction footprint;
    // the warp's working set travels through global memory between the phases
    const bool split = !n_ids && !by_slot &&
                       (ctx->sched_split == 2 || (ctx->sched_split == 1 && n >= kSplitMin));
    if (split) {
        S.state_stride = S.SL.bytes + kSchedStateHdr;
        if (!ctx->sched_state.ensure(static_cast<size_t>(S.state_stride) * std::max(B.n_plans, 1)))
            return fail(ctx, "cudaMalloc k_sched phase state");
        S.state = ctx->sched_state.as<char>();
    }

    PlaceArgs P{};
    P.B = B;
    P.fit = fo;
    P.caps = lc.pl;
    // the fixed-shape k_place instance (compile-time shared layout) when the
    // launch's caps fit kFixedPlaceCaps; the placement result does not depend
    // on the caps, only the working-set sizes do
    const PlaceCaps& fc = kFixedPlaceCaps;
    const bool fixed = !wide && ctx->fixed_layout && lc.pl.M <= fc.M && lc.pl.N <= fc.N && lc.pl.W <= fc.W &&
                       lc.pl.E <= fc.E && lc.pl.G <= fc.G && lc.pl.IS <= fc.IS;
    if (fixed) {
        P.caps = fc;
        P.caps.F = lc.pl.F;
    }
    P.RL = S.RL;
    P.PL = make_pl_layout(P.caps, mb);
    P.recs = recs;
    P.flows = flows;
    P.n_ids = n_ids;
    P.rec_by_slot = by_slot ? 1 : 0;
    P.results = ctx->res_out();
    P.arena = ctx->arena_out();
    P.arena_top = ctx->top_ptr ? ctx->top_ptr : ctx->counters_dev();
    P.arena_cap = ctx->top_ptr ? ctx->top_cap : ctx->cap_out();
    const bool snap_ok = ctx->snap_stride >= snap_words(lc);
    P.snap = ctx->snap.as<double>();
    P.snap_bits = ctx->snap_bits.as<unsigned>();
    P.snap_slots = snap_ok ? kSnapSlots : 0;
    P.snap_stride = ctx->snap_stride;
    if (pw * P.PL.bytes > kSmemLimit) return fail(ctx, "k_place working set exceeds shared memory");
    // measured (100k sweep, ms): snapshots cut decoupled-sequential 9.8 -> 7.9 and
    // distmm-mt 81 -> 47, while the extra code costs wavefront 10.6 -> 11.0
    const bool snap = lc.baseline || ctx->force_snap;
    auto* kplace = wide    ? (snap ? k_place<true, DevMask<4>, 1, 1> : k_place<false, DevMask<4>, 1, 1>)
                   : fixed ? (snap ? k_place<true, uint64_t, kPlaceWarps, WS_PLACE_MINB, true>
                                   : k_place<false, uint64_t, kPlaceWarps, WS_PLACE_MINB, true>)
                           : (snap ? k_place<true> : k_place<false>);
    // split emission: k_place leaves the placement, k_emit writes the records
    P.split_emit = !n_ids && !by_slot && (ctx->emit_split == 2 || (ctx->emit_split == 1 && n >= kSplitMin));
    if (P.split_emit) {
        const size_t rows = static_cast<size_t>(std::max(B.n_plans, 1)) * P.caps.E;
        if (!ctx->emit_mask.ensure(rows * mb) || !ctx->emit_rot.ensure(rows * 4) ||
            !ctx->emit_nf.ensure(4ull * std::max(B.n_plans, 1)))
            return fail(ctx, "cudaMalloc placement scratch");
        P.emit_mask = ctx->emit_mask.as<char>();
        P.emit_rot = ctx->emit_rot.as<int32_t>();
        P.emit_nf = ctx->emit_nf.as<int32_t>();
    }
    auto* kemit = wide ? k_emit<DevMask<4>> : k_emit<uint64_t>;
    auto* ksched = wide ? k_sched<DevMask<4>> : k_sched<uint64_t>;
    auto* ksched1 = wide ? k_sched<DevMask<4>, 1> : k_sched<uint64_t, 1>;
    auto* ksched2 = wide ? k_sched<DevMask<4>, 2> : k_sched<uint64_t, 2>;
    auto* ksched3 = wide ? k_sched<DevMask<4>, 3> : k_sched<uint64_t, 3>;

    chunks = std::max(1, std::min(chunks, kMaxChunks));
    if (n_ids || n < 4096) chunks = 1;  // retry pass / small batches: no pipelining
    const int cs = (n + chunks - 1) / chunks;
    cudaStream_t sb = chunks > 1 ? ctx->stream2 : st;
    if (chunks > 1) {
        CK(cudaEventRecord(ctx->cev[kMaxChunks], st));
        CK(cudaStreamWaitEvent(sb, ctx->cev[kMaxChunks], 0));
    }
    for (int c = 0; c < chunks; ++c) {
        const int base = c * cs;
        const int cnt = std::min(cs, n - base);
        if (cnt <= 0) break;
        S.plan_ids = ids + base;
        S.n_launch = cnt;
        SchedArgs S1 = S;  // the first k_sched kernel: the unsplit one, or phase 1
        S1.warp_smem = split ? sched_phase_bytes(S.SL, 1) : S.SL.bytes;
        if (pdl && c == 0) {  // right behind k_fit: programmatic dependent launch
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3((cnt + kSchedWarps - 1) / kSchedWarps);
            cfg.blockDim = dim3(32 * kSchedWarps);
            cfg.dynamicSmemBytes = kSchedWarps * S1.warp_smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, split ? ksched1 : ksched, S1));
        } else {
            (split ? ksched1 : ksched)<<<(cnt + kSchedWarps - 1) / kSchedWarps, 32 * kSchedWarps,
                                         kSchedWarps * S1.warp_smem, st>>>(S1);
        }
        ctx->launches++;
        if (split) {
            SchedArgs S2 = S1, S3 = S1;
            S2.warp_smem = sched_phase_bytes(S.SL, 2);
            S3.warp_smem = S.SL.bytes;
            ksched2<<<(cnt + kSchedWarps - 1) / kSchedWarps, 32 * kSchedWarps, kSchedWarps * S2.warp_smem, st>>>(S2);
            ksched3<<<(cnt + kSchedWarps - 1) / kSchedWarps, 32 * kSchedWarps, kSchedWarps * S3.warp_smem, st>>>(S3);
            ctx->launches += 2;
        }
        if (lc.scoped) {  // the batch's distmm-mt plans (each instance skips the other's plans)
            (wide ? k_sched_scoped<DevMask<4>> : k_sched_scoped<uint64_t>)<<<(cnt + kSchedWarps - 1) / kSchedWarps, 32 * kSchedWarps, kSchedWarps * S.SL.bytes,
                             st>>>(S);
            ctx->launches++;
        }
        if (chunks > 1) {
            CK(cudaEventRecord(ctx->cev[c], st));
            CK(cudaStreamWaitEvent(sb, ctx->cev[c], 0));
        } else if (mid) {
            CK(cudaEventRecord(mid, st));
        }
        P.plan_ids = ids + base;
        P.n_launch = cnt;
        kplace<<<(cnt + pw - 1) / pw, 32 * pw, pw * P.PL.bytes, sb>>>(P);
        ctx->launches++;
        if (P.split_emit) {
            kemit<<<(cnt + kPlaceWarps - 1) / kPlaceWarps, 32 * kPlaceWarps, 0, sb>>>(P);
            ctx->launches++;
        }
    }
    if (chunks > 1) {
        if (mid) CK(cudaEventRecord(mid, st));  // end of the last k_sched chunk
        CK(cudaEventRecord(ctx->cev[kMaxChunks + 1], sb));
        CK(cudaStreamWaitEvent(st, ctx->cev[kMaxChunks + 1], 0));
    }
    return 0;
}

}  // namespace

extern "C" {

int ws_ctx_create(int device, ws_ctx** out) {
    *out = nullptr;
    DevGuard g(device);
    if (!g.ok) return 1;
    auto* c = new ws_ctx();
    c->device = device;
    bool ok = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->stream3, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->stream4, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->stream5, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMallocHost(reinterpret_cast<void**>(&c->host_tops), 8 * kHostTopsWords) == cudaSuccess;
    for (auto& e : c->ev) ok = ok && cudaEventCreate(&e) == cudaSuccess;
    for (auto& e : c->sev) ok = ok && cudaEventCreate(&e) == cudaSuccess;
    for (auto& e : c->cev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->drain_ev, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && smem_opt_in_all(device) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        ws_ctx_destroy(c);
        return 1;
    }
    std::memset(c->host_tops, 0, 8 * kHostTopsWords);
    if (const char* env = std::getenv("WSGPU_CHUNKS")) c->chunks = std::atoi(env);
    if (const char* env = std::getenv("WSGPU_HOST_CHUNKS")) {
        c->host_chunks = std::atoi(env);
        c->host_weights.clear();  // uniform chunks
    }
    if (const char* env = std::getenv("WSGPU_HOST_WEIGHTS")) {
        c->host_weights.clear();
        for (const char* q = env; *q;) {
            char* end = nullptr;
            const double w = std::strtod(q, &end);
            if (end == q) break;
            if (w > 0) c->host_weights.push_back(w);
            q = *end == ',' ? end + 1 : end;
        }
        if (!c->host_weights.empty()) c->host_chunks = static_cast<int>(c->host_weights.size());
    }
    if (const char* env = std::getenv("WSGPU_FORCE_SNAP")) c->force_snap = std::atoi(env) != 0;
    if (const char* env = std::getenv("WSGPU_PDL")) c->pdl = std::atoi(env) != 0;
    if (const char* env = std::getenv("WSGPU_HOST_STREAMS")) c->host_streams = std::max(1, std::min(3, std::atoi(env)));
    if (const char* env = std::getenv("WSGPU_TINY_SOFT_CAPS")) c->tiny_soft = std::atoi(env) != 0;
    if (const char* env = std::getenv("WSGPU_SMALL_PATH")) c->small_path = std::atoi(env) != 0;
    if (const char* env = std::getenv("WSGPU_TRACE")) c->trace = std::atoi(env) != 0;
    if (const char* env = std::getenv("WSGPU_SCHED_SPLIT")) c->sched_split = std::atoi(env);
    if (const char* env = std::getenv("WSGPU_EMIT_SPLIT")) c->emit_split = std::atoi(env);
    if (const char* env = std::getenv("WSGPU_FIXED_LAYOUT")) c->fixed_layout = std::atoi(env) != 0;
    *out = c;
    return 0;
}

void ws_ctx_destroy(ws_ctx* c) {
    if (!c) return;
    DevGuard g(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (cudaEvent_t* e : {c->ev, c->ev + 1, c->ev + 2, c->ev + 3, c->sev, c->sev + 1, &c->order_ev, &c->drain_ev, &c->join_ev})
        if (*e) cudaEventDestroy(*e);
    for (auto& e : c->cev)
        if (e) cudaEventDestroy(e);
    for (cudaStream_t s : {c->stream, c->stream2, c->stream3, c->stream4, c->stream5})
        if (s) cudaStreamDestroy(s);
    if (c->host_tops) cudaFreeHost(c->host_tops);
    if (c->order_pinned) cudaFreeHost(c->order_pinned);
    if (c->small_host) cudaFreeHost(c->small_host);
    for (void* q : c->retired_host) cudaFreeHost(q);
    delete c;  // DevBuf destructors free device memory on c->device (guarded)
}

const char* ws_ctx_last_error(const ws_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

int ws_last_launch_count(const ws_ctx* c) { return c ? c->launches : 0; }

long long ws_last_retry_count(const ws_ctx* c) { return c ? c->last_retry : 0; }

int ws_last_kernel_ms(const ws_ctx* c, double* out, int n) {
    if (!c) return 1;
    double ms3[3] = {c->kernel_ms[0], c->kernel_ms[1], c->kernel_ms[2]};
    if (c->staged_events && cudaEventSynchronize(c->ev[2]) == cudaSuccess) {
        // read the events of the last ws_plan_staged directly (no fetch needed)
        float ms = 0;
        if (cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]) == cudaSuccess) ms3[0] = ms;
        if (cudaEventElapsedTime(&ms, c->ev[1], c->ev[3]) == cudaSuccess) ms3[1] = ms;
        if (cudaEventElapsedTime(&ms, c->ev[3], c->ev[2]) == cudaSuccess) ms3[2] = ms;
    }
    for (int i = 0; i < n && i < 3; ++i) out[i] = ms3[i];
    return 0;
}

namespace {
// device buffers of a planning call sized for the staged batch, and the k_fit output view
int prepare_plan(ws_ctx* ctx, FitOut& fo, cudaStream_t st) {
    const ws_batch& B = ctx->dview;
    const int P = B.n_plans, NM = std::max(B.n_modules, 1);
    const LaunchCaps& lc = ctx->caps;
    const LaunchCaps& lh = ctx->caps_hard;
    const int tstride = lc.pl.N;
    if (!ctx->fit_err.ensure(4ull * NM) || !ctx->fit_a.ensure(4ull * NM) || !ctx->fit_b.ensure(4ull * NM) ||
        !ctx->fit_np.ensure(4ull * NM) || !ctx->fit_nmax.ensure(4ull * NM) || !ctx->fit_off.ensure(8ull * NM) ||
        !ctx->fit_pieces.ensure(40ull * (static_cast<uint64_t>(NM) * kInlinePieces + kOverflowPieces)) ||
        !ctx->ttab.ensure(8ull * NM * tstride))
        return fail(ctx, "cudaMalloc fit buffers");
    const RecLayout RL = make_rec_layout(lc.rec), RLh = make_rec_layout(lh.rec);
    if (!ctx->counters.ensure(64) || !ctx->results.ensure(sizeof(ws_plan_result) * std::max(P, 1)) ||
        !ctx->arena.ensure(ctx->arena_cap) || !ctx->retry_ids.ensure(4ull * std::max(P, 1)) || !ctx->best.ensure(64) ||
        !ctx->recs.ensure(static_cast<size_t>(RL.bytes) * std::max(P, 1)) ||
        !ctx->flows.ensure(16ull * lc.pl.F * std::max(P, 1)) ||
        !ctx->recs_r.ensure(static_cast<size_t>(RLh.bytes) * kRetryMax) ||
        !ctx->flows_r.ensure(16ull * lh.pl.F * kRetryMax))
        return fail(ctx, "cudaMalloc planner buffers");
    // backtracking snapshot pool sized for the larger (retry) caps; the claim
    // bitmap is zeroed only when the pool is (re)allocated -- warps always release
    const long long stride = std::max(snap_words(lc), snap_words(lh));
    // (only k_place<true>, batches with baseline strategies, uses snapshots).
    // A grown pool is a fresh allocation (the old one stays with any k_place of
    // this ctx still running), its bits zeroed on the launch stream.
    if ((lc.baseline || ctx->force_snap) && stride > ctx->snap_stride) {
        if (!ctx->snap.ensure(8ull * stride * kSnapSlots)) return fail(ctx, "cudaMalloc snapshot pool");
        if (ctx->snap_bits.p) ctx->snap_bits.retired.push_back(ctx->snap_bits.p);
        ctx->snap_bits.p = nullptr;
        ctx->snap_bits.n = 0;
        if (!ctx->snap_bits.ensure(4 * ((kSnapSlots + 31) / 32))) return fail(ctx, "cudaMalloc snapshot bits");
        if (cudaMemsetAsync(ctx->snap_bits.p, 0, 4 * ((kSnapSlots + 31) / 32), st) != cudaSuccess)
            return fail(ctx, "cudaMemset snapshot bits");
        ctx->snap_stride = stride;
    }
    auto* counters = ctx->counters_dev();
    fo.err = ctx->fit_err.as<int32_t>();
    fo.err_a = ctx->fit_a.as<int32_t>();
    fo.err_b = ctx->fit_b.as<int32_t>();
    fo.npieces = ctx->fit_np.as<int32_t>();
    fo.nmax = ctx->fit_nmax.as<int32_t>();
    fo.piece_off = ctx->fit_off.as<int64_t>();
    fo.pieces = ctx->fit_pieces.as<double>();
    fo.overflow_top = counters + 1;
    fo.overflow_base = static_cast<int64_t>(NM) * kInlinePieces;
    fo.overflow_cap = kOverflowPieces;
    fo.ttab = ctx->ttab.as<double>();
    fo.tstride = tstride;
    return 0;
}

// Re-plans the soft-cap overflows the first retry launch of the last
// ws_plan_staged did not cover (more than kRetryMax in one batch), in further
// kRetryMax-plan launches on `st`.  Called by every entry point that consumes
// the staged results; waits for the overflow count of that call.
int drain_overflow(ws_ctx* ctx, cudaStream_t st) {
    if (!ctx->drain_pending) return 0;
    ctx->drain_pending = false;
    CK(cudaEventSynchronize(ctx->drain_ev));
    const long long total = static_cast<int32_t>(ctx->host_tops[kHtRetry] & 0xffffffffull);
    ctx->last_retry = total;
    if (total <= kRetryMax) return 0;
    FitOut fo;
    if (prepare_plan(ctx, fo, st)) return 1;
    for (long long b = kRetryMax; b < total; b += kRetryMax) {
        const int n = static_cast<int>(std::min<long long>(kRetryMax, total - b));
        if (launch_pair(ctx, st, ctx->caps_hard, fo, ctx->retry_ids.as<int32_t>() + b, nullptr, n, true,
                        ctx->recs_r.as<char>(), ctx->flows_r.as<uint64_t>()))
            return 1;
    }
    CK(cudaGetLastError());
    return 0;
}

// longest-processing-time launch order: descending modules x devices, stable
constexpr int kLptKeys = (WS_MAX_MODULES + 1) * (WS_MAX_DEVICES + 9);
inline int lpt_key(const ws_plan_rec& r) {
    const int m = std::min(std::max(r.n_mod, 0), WS_MAX_MODULES), d = std::min(std::max(r.n_dev, 0), WS_MAX_DEVICES);
    return kLptKeys - 1 - m * (d + 8);
}

// LPT order of plans [p0, p1) by a stable counting sort (O(plans) on the host)
void lpt_order(ws_ctx* ctx, const ws_plan_rec* plans, int p0, int p1, int32_t* out) {
    ctx->key_count.assign(kLptKeys + 1, 0);
    for (int p = p0; p < p1; ++p) ctx->key_count[lpt_key(plans[p]) + 1]++;
    for (int k = 0; k < kLptKeys; ++k) ctx->key_count[k + 1] += ctx->key_count[k];
    for (int p = p0; p < p1; ++p) out[p0 + ctx->key_count[lpt_key(plans[p])]++] = p;
}

// page-locked launch-order buffer of at least P entries (asynchronous H2D
// copies), safe to rewrite: the previous call's copies have completed
int ensure_order_pinned(ws_ctx* ctx, int P) {
    if (ctx->order_ev_pending) {
        cudaEventSynchronize(ctx->order_ev);
        ctx->order_ev_pending = false;
    }
    if (ctx->order_pinned_n >= static_cast<size_t>(P)) return 0;
    if (ctx->order_pinned) ctx->retired_host.push_back(ctx->order_pinned);
    ctx->order_pinned = nullptr;
    const size_t want = std::max<size_t>({static_cast<size_t>(P), ctx->order_pinned_n * 3 / 2, 1024});
    ctx->order_pinned_n = 0;
    if (cudaMallocHost(reinterpret_cast<void**>(&ctx->order_pinned), 4ull * want) != cudaSuccess)
        return fail(ctx, "cudaMallocHost launch order");
    ctx->order_pinned_n = want;
    return 0;
}
}  // namespace

int ws_stage_batch(ws_ctx* ctx, const ws_batch* in, void* stream) {
    DevGuard dg_(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    if (!in->blob) return fail(ctx, "ws_stage_batch: batch must be contiguous (ws_batch.blob)");
    const int P = in->n_plans;
    if (!ctx->blob.ensure(in->blob_bytes + 256) || !ctx->order.ensure(4ull * std::max(P, 1)))
        return fail(ctx, "cudaMalloc batch");
    CK(cudaMemcpyAsync(ctx->blob.p, in->blob, in->blob_bytes, cudaMemcpyHostToDevice, st));
    ctx->dview = rebase(*in, in->blob, ctx->blob.as<char>());
    ctx->small_counters = nullptr;
    ctx->drain_pending = false;  // results of an earlier staged batch are superseded
    ctx->caps = batch_caps(in->plans, P, false, ctx->tiny_soft);
    ctx->caps_hard = batch_caps(in->plans, P, true);
    ctx->arena_cap = ws_arena_bound(in);
    ctx->sim_cap = ws_sim_arena_bound(in);
    ctx->records_on_device = false;
    ctx->sim_valid = false;
    if (ensure_order_pinned(ctx, P)) return 1;
    lpt_order(ctx, in->plans, 0, P, ctx->order_pinned);
    if (P) {
        CK(cudaMemcpyAsync(ctx->order.p, ctx->order_pinned, 4ull * P, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(ctx->order_ev, st));
        ctx->order_ev_pending = true;
    }
    return 0;
}

// k_fit over modules [m0, m1): a warp per module for small batches (latency),
// a thread per module for large ones (throughput); identical results
// ($WSGPU_FIT_WARP_MAX overrides the 4096-module threshold; 0 = always a thread)
static void launch_fit(const ws_batch& B, const FitOut& fo, int m0, int m1, cudaStream_t s) {
    static const int64_t warp_max = [] {
        const char* env = std::getenv("WSGPU_FIT_WARP_MAX");
        return env ? static_cast<int64_t>(std::atoll(env)) : static_cast<int64_t>(kFitWarpMaxModules);
    }();
    const int64_t nm = m1 - m0;
    if (nm <= warp_max)
        k_fit<kFitWarp><<<static_cast<int>((nm * kFitWarp + 127) / 128), 128, 0, s>>>(B, fo, m0, m1);
    else
        k_fit<1><<<static_cast<int>((nm + 127) / 128), 128, 0, s>>>(B, fo, m0, m1);
}

int ws_plan_staged(ws_ctx* ctx, void* stream) {
    DevGuard dg_(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    const ws_batch& B = ctx->dview;
    const int P = B.n_plans;
    const LaunchCaps& lc = ctx->caps;
    const LaunchCaps& lh = ctx->caps_hard;
    ctx->launches = 0;
    ctx->drain_pending = false;  // this call re-plans every plan of the staged batch
    ctx->last_retry = 0;
    FitOut fo;
    if (prepare_plan(ctx, fo, st)) return 1;
    ctx->small_counters = nullptr;
    auto* counters = ctx->counters_dev();  // [0] arena top [1] overflow top [2] retry count
    CK(cudaMemsetAsync(counters, 0, 64, st));

    CK(cudaEventRecord(ctx->ev[0], st));
    // with programmatic dependent launch k_sched directly follows k_fit (no
    // event in between), so k_fit's time is reported inside k_sched's
    if (ctx->pdl) CK(cudaEventRecord(ctx->ev[1], st));
    if (B.n_modules > 0) {
        launch_fit(B, fo, 0, B.n_modules, st);
        ctx->launches++;
    }
    if (!ctx->pdl) CK(cudaEventRecord(ctx->ev[1], st));
    if (launch_pair(ctx, st, lc, fo, ctx->order.as<int32_t>(), nullptr, P, false, ctx->recs.as<char>(),
                    ctx->flows.as<uint64_t>(), ctx->ev[3], ctx->chunks, ctx->pdl && B.n_modules > 0))
        return 1;
    // retry pass: soft-cap overflows with the hard caps, count read on device;
    // the first kRetryMax run here, any beyond in drain_overflow()
    auto* rcount = reinterpret_cast<int32_t*>(counters + 2);
    if (P > 0) {
        k_soft_collect<<<(P + 255) / 256, 256, 0, st>>>(ctx->res_out(), 0, P,
                                                         ctx->retry_ids.as<int32_t>(), rcount);
        ctx->launches++;
        // retry grid sized for at most min(P, kRetryMax) plans (small batches: one block)
        if (launch_pair(ctx, st, lh, fo, ctx->retry_ids.as<int32_t>(), rcount, std::min(P, kRetryMax), true,
                        ctx->recs_r.as<char>(), ctx->flows_r.as<uint64_t>()))
            return 1;
    }
    CK(cudaEventRecord(ctx->ev[2], st));
    if (P > 0) {
        ctx->host_tops[kHtRetry] = 0;
        CK(cudaMemcpyAsync(ctx->host_tops + kHtRetry, rcount, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(ctx->drain_ev, st));
        ctx->drain_pending = true;
        ctx->drain_stream = st;
    }
    CK(cudaGetLastError());
    ctx->staged_events = P > 0;
    ctx->records_on_device = true;
    ctx->sim_valid = false;
    return 0;
}

int ws_fetch_results(ws_ctx* ctx, ws_plan_result* results, uint8_t* arena, uint64_t arena_cap,
                     uint64_t* arena_used, void* stream) {
    DevGuard dg_(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    if (drain_overflow(ctx, st)) return 1;
    const int P = ctx->dview.n_plans;
    unsigned long long top = 0;
    // small batches (single-plan latency): copy the whole arena bound with the
    // headers and the top counter, one synchronization instead of two
    const bool one_sync = ctx->arena_cap <= kOneSyncArena && ctx->arena_cap <= arena_cap;
    if (P) CK(cudaMemcpyAsync(results, ctx->results.p, sizeof(ws_plan_result) * P, cudaMemcpyDeviceToHost, st));
    unsigned long long* htop = ctx->host_tops + kHtFetch;  // page-locked
    CK(cudaMemcpyAsync(htop, ctx->counters_dev(), sizeof(top), cudaMemcpyDeviceToHost, st));
    if (one_sync && ctx->arena_cap) CK(cudaMemcpyAsync(arena, ctx->arena.p, ctx->arena_cap, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    top = *htop;
    float ms = 0;
    ctx->kernel_ms[1] = ctx->kernel_ms[2] = 0;
    if (cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]) == cudaSuccess) ctx->kernel_ms[0] = ms;
    if (P && cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[3]) == cudaSuccess) ctx->kernel_ms[1] = ms;
    if (P && cudaEventElapsedTime(&ms, ctx->ev[3], ctx->ev[2]) == cudaSuccess) ctx->kernel_ms[2] = ms;
    if (top > ctx->arena_cap) top = ctx->arena_cap;
    if (top > arena_cap) return fail(ctx, "ws_fetch_results: arena buffer too small");
    if (!one_sync && top) {
        CK(cudaMemcpyAsync(arena, ctx->arena.p, top, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    *arena_used = top;
    return 0;
}

extern "C" uint64_t wsi_arena_bound_plans(const ws_plan_rec* plans, int n);

namespace {
constexpr int kSmallBatch = 64;  // host batches planned by plan_small

// Small host batches (single-plan latency, concurrent drop-in callers): the
// batch, its launch order and zeroed counters go to the device in ONE copy,
// the kernels run with the hard record caps (no soft-cap overflow, so no
// retry pass and no host round trip for its count), and the results come back
// in one or two copies: 6-7 CUDA calls per call instead of ~25 (the CUDA
// driver serializes concurrent callers' API calls, so their count bounds the
// multi-threaded drop-in throughput).
// stage + launch of the small-batch path (results stay on the device).
// soft: launch with the soft record caps (the fixed-shape k_place instance
// applies when they fit); the caller re-plans on a soft-cap overflow.
int small_launch(ws_ctx* ctx, const ws_batch* in, cudaStream_t st, bool soft = false) {
    const int P = in->n_plans;
    const uint64_t o_order = 256, o_blob = (o_order + 4ull * P + 255) & ~255ull;
    const uint64_t bytes = o_blob + in->blob_bytes;
    if (ctx->small_host_n < bytes) {
        if (ctx->small_host) ctx->retired_host.push_back(ctx->small_host);
        ctx->small_host = nullptr;
        const size_t want = std::max<size_t>({bytes, ctx->small_host_n * 3 / 2, 256 << 10});
        ctx->small_host_n = 0;
        if (cudaMallocHost(reinterpret_cast<void**>(&ctx->small_host), want) != cudaSuccess)
            return fail(ctx, "cudaMallocHost small-batch staging");
        ctx->small_host_n = want;
    }
    if (!ctx->blob.ensure(bytes + 256)) return fail(ctx, "cudaMalloc batch");
    uint8_t* h = ctx->small_host;
    std::memset(h, 0, 256);  // counters
    auto* order = reinterpret_cast<int32_t*>(h + o_order);
    for (int p = 0; p < P; ++p) order[p] = p;
    std::sort(order, order + P, [&](int a, int b) {  // LPT, stable by index
        const int ka = lpt_key(in->plans[a]), kb = lpt_key(in->plans[b]);
        return ka != kb ? ka < kb : a < b;
    });
    std::memcpy(h + o_blob, in->blob, in->blob_bytes);
    char* d = ctx->blob.as<char>();
    CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    ctx->dview = rebase(*in, in->blob, d + o_blob);
    ctx->drain_pending = false;
    ctx->last_retry = 0;
    ctx->caps = batch_caps(in->plans, P, !soft, ctx->tiny_soft);
    ctx->caps_hard = soft ? batch_caps(in->plans, P, true) : ctx->caps;
    ctx->arena_cap = ws_arena_bound(in);
    ctx->sim_cap = ws_sim_arena_bound(in);
    ctx->sim_valid = false;
    ctx->small_counters = reinterpret_cast<unsigned long long*>(d);
    FitOut fo;
    if (prepare_plan(ctx, fo, st)) return 1;
    ctx->launches = 0;
    const ws_batch& B = ctx->dview;
    if (B.n_modules > 0) {
        launch_fit(B, fo, 0, B.n_modules, st);
        ctx->launches++;
    }
    if (launch_pair(ctx, st, ctx->caps, fo, reinterpret_cast<const int32_t*>(d + o_order), nullptr, P, false,
                    ctx->recs.as<char>(), ctx->flows.as<uint64_t>(), nullptr, 1, ctx->pdl && B.n_modules > 0))
        return 1;
    ctx->staged_events = false;
    ctx->records_on_device = true;
    return 0;
}

int plan_small(ws_ctx* ctx, const ws_batch* in, ws_plan_result* results, uint8_t* arena, uint64_t arena_cap,
               uint64_t* arena_used, cudaStream_t st) {
    const int P = in->n_plans;
    if (small_launch(ctx, in, st, true)) return 1;
    const bool one_sync = ctx->arena_cap <= kOneSyncArena && ctx->arena_cap <= arena_cap;
    if (P) CK(cudaMemcpyAsync(results, ctx->results.p, sizeof(ws_plan_result) * P, cudaMemcpyDeviceToHost, st));
    if (one_sync) CK(cudaMemcpyAsync(arena, ctx->arena.p, ctx->arena_cap, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // a plan over the soft record caps (rare: > 4 entries per MetaOp on average):
    // re-plan the batch on the staged path, whose retry pass uses the hard caps
    for (int p = 0; p < P; ++p) {
        const int e = results[p].err_code;
        if (e == WS_E_LIMIT_WAVES || e == WS_E_LIMIT_ENTRIES || e == WS_E_LIMIT_FLOWS) {
            if (ws_stage_batch(ctx, in, st) || ws_plan_staged(ctx, st)) return 1;
            return ws_fetch_results(ctx, results, arena, arena_cap, arena_used, st);
        }
    }
    uint64_t top = 0;  // records are bump-allocated: the arena top is the furthest record end
    for (int p = 0; p < P; ++p)
        if (results[p].status == WS_STATUS_OK) top = std::max<uint64_t>(top, results[p].offset + results[p].size);
    if (top > arena_cap) return fail(ctx, "ws_plan_batch_host: arena buffer too small");
    if (!one_sync && top) {
        CK(cudaMemcpyAsync(arena, ctx->arena.p, top, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    ctx->kernel_ms[0] = ctx->kernel_ms[1] = ctx->kernel_ms[2] = 0;  // not timed on this path
    *arena_used = top;
    return 0;
}
}  // namespace

// Host batch in, host results out.  Batches of >= 2 x 4096 plans run as a
// pipeline over chunks of plans (default sizes 1:3:3:1, $WSGPU_HOST_WEIGHTS /
// $WSGPU_HOST_CHUNKS): the H2D copy of chunk c+1 (its byte ranges of every SoA
// section: sections are plan-ordered, so a chunk's rows are contiguous) and the
// D2H copy of chunk c-1 (results rows + its own arena region) overlap the
// kernels of chunk c, and consecutive chunks alternate between two compute
// streams so each fills the other's launch tail.  Smaller batches: stage (one
// H2D copy), plan, fetch (two D2H copies).  Kernels always write device memory
// (zero-copy writes into host memory stall k_place on PCIe: measured 20 ms vs
// 11 ms per 100k).
namespace {
// The pipelined host call over plans [P0, P1) of `in`: `results` receives the
// headers of plans P0.. and `arena` the range's records (offsets relative to
// it).  Only the range's rows of every section travel to the device (sections
// are plan-ordered, so they are contiguous); the device blob mirrors the host
// layout, so indices stay absolute.  ws_plan_batch_host runs it over [0, P);
// ws_plan_batch_multi runs one range per context.
int host_range(ws_ctx* ctx, const ws_batch* in, int P0, int P1, ws_plan_result* results, uint8_t* arena,
               uint64_t arena_cap, uint64_t* arena_used, cudaStream_t st) {
    const int P = in->n_plans, n = P1 - P0;
    *arena_used = 0;
    if (n <= 0) return 0;
    using hclk = std::chrono::steady_clock;
    const auto t_enter = hclk::now();
    hclk::time_point t_prep, t_issued;
    int C = ctx->host_chunks;
    C = std::max(1, std::min({C, kMaxHostChunks, n / 4096}));
    if (!ctx->blob.ensure(in->blob_bytes + 256) || !ctx->order.ensure(4ull * P) || !ctx->chunk_tops.ensure(8 * 64))
        return fail(ctx, "cudaMalloc batch");
    char* dblob = ctx->blob.as<char>();
    ctx->dview = rebase(*in, in->blob, dblob);
    ctx->sim_valid = false;
    ctx->drain_pending = false;
    int pb[kMaxHostChunks + 1];
    uint64_t abase[kMaxHostChunks + 1];
    abase[0] = 0;
    if (ensure_order_pinned(ctx, P)) return 1;
    // chunk boundaries: uniform, or proportional to $WSGPU_HOST_WEIGHTS ("1,3,3,1": small
    // first/last chunks shorten the exposed first H2D and last D2H copies)
    double wsum = 0, wacc = 0;
    for (int c = 0; c < C; ++c) wsum += c < static_cast<int>(ctx->host_weights.size()) ? ctx->host_weights[c] : 1.0;
    pb[0] = P0;
    for (int c = 0; c < C; ++c) {
        wacc += c < static_cast<int>(ctx->host_weights.size()) ? ctx->host_weights[c] : 1.0;
        pb[c + 1] = c + 1 == C ? P1
                               : P0 + std::max(pb[c] - P0 + 1, std::min(n - (C - 1 - c), static_cast<int>(n * (wacc / wsum))));
    }
    // Chunk 0's input rows go out first: the DMA runs while the host makes its
    // pass over the plan records below (which only the launch order and the
    // arena bounds depend on)
    auto* tops = ctx->chunk_tops.as<unsigned long long>();
    cudaStream_t sh = ctx->stream2, sd = ctx->stream3;
    cudaEvent_t* h2d = ctx->cev;               // [0, C)
    cudaEvent_t* done = ctx->cev + kMaxHostChunks;  // [C, 2C)
    CK(cudaEventRecord(ctx->ev[0], st));
    CK(cudaStreamWaitEvent(sh, ctx->ev[0], 0));
    const ws_batch& h = *in;
    auto rows = [&](const void* hp, size_t esz, int64_t lo, int64_t hi) -> cudaError_t {
        if (!hp || hi <= lo) return cudaSuccess;
        const size_t off = static_cast<const char*>(hp) - static_cast<const char*>(in->blob) + lo * esz;
        return cudaMemcpyAsync(dblob + off, static_cast<const char*>(hp) + lo * esz, (hi - lo) * esz,
                               cudaMemcpyHostToDevice, sh);
    };
    auto first = [](const int32_t* a, int64_t i, int64_t n, int64_t total) { return i < n ? a[i] : total; };
#define RK(x)                              \
    do {                                   \
        const cudaError_t e_ = (x);        \
        if (e_ != cudaSuccess) return e_;  \
    } while (0)
    auto issue_rows = [&](int c) -> cudaError_t {  // chunk c's input rows (H2D side)
        const int p0 = pb[c], p1 = pb[c + 1];
        const int64_t m0 = h.plans[p0].mod_begin, m1 = p1 < P ? h.plans[p1].mod_begin : h.n_modules;
        const int64_t t0 = h.plans[p0].task_begin, t1 = p1 < P ? h.plans[p1].task_begin : h.n_task_total;
        const int64_t d0 = h.plans[p0].dev_begin, d1 = p1 < P ? h.plans[p1].dev_begin : h.n_devices;
        const int64_t nm = h.n_modules, nt = h.n_task_total;
        RK(rows(h.plans, sizeof(ws_plan_rec), p0, p1));
        for (const int32_t* a : {h.mod_plan, h.mod_layers, h.mod_tp, h.mod_group, h.mod_alias, h.mod_name_off,
                                 h.mod_name_len, h.mod_truth_off, h.mod_truth_n, h.mod_prof_off, h.mod_prof_n,
                                 h.mod_bp_off, h.mod_bp_n, h.mod_pre_err})
            RK(rows(a, 4, m0, m1));
        for (const void* a : {static_cast<const void*>(h.mod_batch), static_cast<const void*>(h.mod_param),
                              static_cast<const void*>(h.mod_act), static_cast<const void*>(h.mod_out),
                              static_cast<const void*>(h.mod_w), static_cast<const void*>(h.mod_c)})
            RK(rows(a, 8, m0, m1));
        for (const int32_t* a : {h.task_tok_off, h.task_tok_n, h.task_rank}) RK(rows(a, 4, t0, t1));
        RK(rows(h.tokens, 4, first(h.task_tok_off, t0, nt, h.n_tokens), first(h.task_tok_off, t1, nt, h.n_tokens)));
        RK(rows(h.dev_island, 4, d0, d1));
        RK(rows(h.truth, 40, first(h.mod_truth_off, m0, nm, h.n_pieces), first(h.mod_truth_off, m1, nm, h.n_pieces)));
        const int64_t q0 = first(h.mod_prof_off, m0, nm, h.n_points), q1 = first(h.mod_prof_off, m1, nm, h.n_points);
        RK(rows(h.prof_n, 4, q0, q1));
        RK(rows(h.prof_t, 8, q0, q1));
        RK(rows(h.bps, 4, first(h.mod_bp_off, m0, nm, h.n_bps), first(h.mod_bp_off, m1, nm, h.n_bps)));
        RK(rows(h.names, 1, first(h.mod_name_off, m0, nm, h.n_name_bytes),
                first(h.mod_name_off, m1, nm, h.n_name_bytes)));
        return cudaSuccess;
    };
#undef RK
    CK(issue_rows(0));
    // ONE pass over the plan records: launch maxima, per-chunk arena bounds, the
    // evaluation bound and per-chunk LPT key histograms; then one scatter pass
    // (the host work before the first copy is exposed in the end-to-end time)
    BatchMax bm;
    uint64_t sim_total = 0;
    ctx->lpt_keys.resize(P);
    ctx->key_count.assign(static_cast<size_t>(C) * (kLptKeys + 1), 0);
    for (int c = 0; c < C; ++c) {
        uint64_t ab = 0;
        int* hist = ctx->key_count.data() + static_cast<size_t>(c) * (kLptKeys + 1);
        for (int p = pb[c]; p < pb[c + 1]; ++p) {
            const ws_plan_rec& r = in->plans[p];
            bm.add(r);
            ab += wsi_plan_arena_bound(&r);
            sim_total += wsi_plan_sim_bound(&r);
            const int key = lpt_key(r);
            ctx->lpt_keys[p] = static_cast<uint16_t>(key);
            hist[key + 1]++;
        }
        abase[c + 1] = abase[c] + ab;
        ctx->host_tops[c] = abase[c];
    }
    for (int c = 0; c < C; ++c) {
        int* hist = ctx->key_count.data() + static_cast<size_t>(c) * (kLptKeys + 1);
        for (int k = 0; k < kLptKeys; ++k) hist[k + 1] += hist[k];
        for (int p = pb[c]; p < pb[c + 1]; ++p) ctx->order_pinned[pb[c] + hist[ctx->lpt_keys[p]]++] = p;
    }
    ctx->caps = caps_from(bm, false, ctx->tiny_soft);
    ctx->caps_hard = caps_from(bm, true);
    ctx->sim_cap = sim_total + 4096;  // == ws_sim_arena_bound(in)
    ctx->arena_cap = abase[C];
    if (ctx->arena_cap > arena_cap) {
        cudaStreamSynchronize(sh);  // chunk 0's copy reads the caller's buffers: done before returning
        return fail(ctx, "ws_plan_batch_host: arena buffer too small");
    }
    ctx->small_counters = nullptr;
    FitOut fo;
    if (prepare_plan(ctx, fo, st)) {
        cudaStreamSynchronize(sh);
        return 1;
    }
    auto* counters = ctx->counters_dev();
    t_prep = hclk::now();
    CK(cudaMemcpyAsync(tops, ctx->host_tops, 8ull * C, cudaMemcpyHostToDevice, sh));
    for (int c = 0; c < C; ++c) {
        const int p0 = pb[c], p1 = pb[c + 1];
        if (c > 0) CK(issue_rows(c));
        CK(cudaMemcpyAsync(ctx->order.as<int32_t>() + p0, ctx->order_pinned + p0, 4ull * (p1 - p0),
                           cudaMemcpyHostToDevice, sh));
        CK(cudaEventRecord(h2d[c], sh));
    }
    CK(cudaEventRecord(ctx->order_ev, sh));
    ctx->order_ev_pending = true;
    ctx->launches = 0;
    CK(cudaMemsetAsync(counters, 0, 64, st));
    const ws_batch& B = ctx->dview;
    // compute streams: chunk c runs on cs[c % S]; chunk c+1's kernels fill chunk c's launch tail
    const int S = ctx->host_streams;
    cudaStream_t cs[3] = {st, ctx->stream4, ctx->stream5};
    if (S > 1) {
        if (!ctx->recs_r2.ensure(ctx->recs_r.n) || !ctx->flows_r2.ensure(ctx->flows_r.n) ||
            (S > 2 && (!ctx->recs_r3.ensure(ctx->recs_r.n) || !ctx->flows_r3.ensure(ctx->flows_r.n))))
            return fail(ctx, "cudaMalloc retry buffers");
        CK(cudaEventRecord(ctx->ev[1], st));
        for (int k = 1; k < S; ++k) CK(cudaStreamWaitEvent(cs[k], ctx->ev[1], 0));
    }
    for (int c = 0; c < C; ++c) {  // compute side
        const int p0 = pb[c], p1 = pb[c + 1];
        const int m0 = in->plans[p0].mod_begin, m1 = p1 < P ? in->plans[p1].mod_begin : in->n_modules;
        const int k = c % S;
        cudaStream_t s = cs[k];
        auto* rcount = reinterpret_cast<int32_t*>(counters + 2 + k);
        int32_t* rids = ctx->retry_ids.as<int32_t>() + p0;  // chunks own disjoint plan ranges
        DevBuf& rrecs = k == 2 ? ctx->recs_r3 : k ? ctx->recs_r2 : ctx->recs_r;
        DevBuf& rflows = k == 2 ? ctx->flows_r3 : k ? ctx->flows_r2 : ctx->flows_r;
        CK(cudaStreamWaitEvent(s, h2d[c], 0));
        TopScope ts(ctx, tops + c, abase[c + 1]);
        if (m1 > m0) {
            launch_fit(B, fo, m0, m1, s);
            ctx->launches++;
        }
        // k_place's flow scratch is indexed by launch slot: each chunk gets its own
        // region (slots of concurrent chunks would otherwise collide)
        int rc = launch_pair(ctx, s, ctx->caps, fo, ctx->order.as<int32_t>() + p0, nullptr, p1 - p0, false,
                             ctx->recs.as<char>(),
                             ctx->flows.as<uint64_t>() + static_cast<int64_t>(p0) * ctx->caps.pl.F * 2, nullptr, 1,
                             ctx->pdl && m1 > m0);
        if (!rc) {
            CK(cudaMemsetAsync(rcount, 0, 4, s));
            k_soft_collect<<<(p1 - p0 + 255) / 256, 256, 0, s>>>(ctx->res_out(), p0, p1, rids, rcount);
            ctx->launches++;
            rc = launch_pair(ctx, s, ctx->caps_hard, fo, rids, rcount, std::min(p1 - p0, kRetryMax), true,
                             rrecs.as<char>(), rflows.as<uint64_t>());
        }
        if (rc) return 1;
        ctx->host_tops[kHtChunkRetry + c] = 0;
        CK(cudaMemcpyAsync(ctx->host_tops + kHtChunkRetry + c, rcount, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(ctx->host_tops + kMaxHostChunks + c, tops + c, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(done[c], s));
    }
    if (S > 1) {  // join the other compute streams
        CK(cudaEventRecord(ctx->ev[3], cs[1]));
        CK(cudaStreamWaitEvent(st, ctx->ev[3], 0));
    }
    if (S > 2) {
        CK(cudaEventRecord(ctx->join_ev, cs[2]));
        CK(cudaStreamWaitEvent(st, ctx->join_ev, 0));
    }
    CK(cudaEventRecord(ctx->ev[2], st));
    t_issued = hclk::now();
    uint64_t used = 0;
    // D2H side, in completion order (chunks on two compute streams finish out of
    // order): poll the chunk events and copy each finished chunk back at once
    bool copied[kMaxHostChunks] = {};
    for (int left = C; left > 0;) {
        bool progressed = false;
        for (int c = 0; c < C; ++c) {
            if (copied[c]) continue;
            const cudaError_t q = cudaEventQuery(done[c]);
            if (q == cudaErrorNotReady) continue;
            CK(q);
            uint64_t top = ctx->host_tops[kMaxHostChunks + c];
            top = std::min<uint64_t>(top, abase[c + 1]);
            CK(cudaMemcpyAsync(results + (pb[c] - P0), ctx->results.as<ws_plan_result>() + pb[c],
                               sizeof(ws_plan_result) * (pb[c + 1] - pb[c]), cudaMemcpyDeviceToHost, sd));
            if (top > abase[c])
                CK(cudaMemcpyAsync(arena + abase[c], ctx->arena.as<uint8_t>() + abase[c], top - abase[c],
                                   cudaMemcpyDeviceToHost, sd));
            used = std::max<uint64_t>(used, top);
            copied[c] = true;
            --left;
            progressed = true;
        }
        if (!progressed) std::this_thread::yield();
    }
    CK(cudaStreamSynchronize(sd));
    CK(cudaStreamSynchronize(st));
    // soft-cap overflows beyond a chunk's first retry launch (more than kRetryMax
    // in one chunk): re-plan the rest now, then copy that chunk back again
    ctx->last_retry = 0;
    for (int c = 0; c < C; ++c) {
        const long long total = static_cast<int32_t>(ctx->host_tops[kHtChunkRetry + c] & 0xffffffffull);
        ctx->last_retry += total;
        if (total <= kRetryMax) continue;
        {
            TopScope ts(ctx, tops + c, abase[c + 1]);
            const int32_t* rids = ctx->retry_ids.as<int32_t>() + pb[c];
            for (long long b = kRetryMax; b < total; b += kRetryMax) {
                const int n = static_cast<int>(std::min<long long>(kRetryMax, total - b));
                if (launch_pair(ctx, st, ctx->caps_hard, fo, rids + b, nullptr, n, true, ctx->recs_r.as<char>(),
                                ctx->flows_r.as<uint64_t>()))
                    return 1;
            }
        }
        CK(cudaMemcpyAsync(ctx->host_tops + kMaxHostChunks + c, tops + c, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const uint64_t top = std::min<uint64_t>(ctx->host_tops[kMaxHostChunks + c], abase[c + 1]);
        CK(cudaMemcpyAsync(results + (pb[c] - P0), ctx->results.as<ws_plan_result>() + pb[c],
                           sizeof(ws_plan_result) * (pb[c + 1] - pb[c]), cudaMemcpyDeviceToHost, st));
        if (top > abase[c])
            CK(cudaMemcpyAsync(arena + abase[c], ctx->arena.as<uint8_t>() + abase[c], top - abase[c],
                               cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        used = std::max<uint64_t>(used, top);
    }
    // the device arena top for a later ws_fetch_results / ws_simulate_staged
    ctx->host_tops[kHtFinal] = used;
    CK(cudaMemcpyAsync(counters, ctx->host_tops + kHtFinal, 8, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0;
    ctx->staged_events = false;
    ctx->kernel_ms[0] = ctx->kernel_ms[1] = 0;  // chunked: only the whole pipeline is timed
    if (cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[2]) == cudaSuccess) ctx->kernel_ms[2] = ms;
    // a sub-range leaves the other plans' device records unset: evaluation and
    // min-loc over the staged batch need a whole-batch call
    ctx->records_on_device = P0 == 0 && P1 == P;
    if (ctx->trace) {
        auto ms = [](hclk::time_point a, hclk::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        std::fprintf(stderr, "[wsgpu] host_range %d plans, %d chunks: host prep %.3f ms, launches issued %.3f ms, "
                             "end %.3f ms, device pipeline %.3f ms\n", n, C, ms(t_enter, t_prep),
                     ms(t_enter, t_issued), ms(t_enter, hclk::now()), ctx->kernel_ms[2]);
    }
    *arena_used = used;
    return 0;
}
}  // namespace

int ws_plan_batch_host(ws_ctx* ctx, const ws_batch* in, ws_plan_result* results, uint8_t* arena,
                       uint64_t arena_cap, uint64_t* arena_used, void* stream) {
    DevGuard dg_(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    const int P = in->n_plans;
    if (P > 0 && P <= kSmallBatch && in->blob && ctx->small_path)
        return plan_small(ctx, in, results, arena, arena_cap, arena_used, st);
    const int C = std::max(1, std::min({ctx->host_chunks, kMaxHostChunks, P / 4096}));
    if (C == 1 || !in->blob) {
        if (ws_stage_batch(ctx, in, stream)) return 1;
        if (ws_plan_staged(ctx, stream)) return 1;
        return ws_fetch_results(ctx, results, arena, arena_cap, arena_used, stream);
    }
    return host_range(ctx, in, 0, P, results, arena, arena_cap, arena_used, st);
}

// One batch over several contexts (typically one per GPU of the box), SURVEY
// §8(e): contiguous plan blocks of equal estimated cost (the LPT key), each
// planned by host_range on its own host thread into its own slice of the
// caller's arena; record offsets are rebased to the whole arena.
int ws_plan_batch_multi(ws_ctx* const* ctxs, int n_ctx, const ws_batch* in, ws_plan_result* results,
                        uint8_t* arena, uint64_t arena_cap, uint64_t* arena_used) {
    if (n_ctx <= 0 || !ctxs) return 1;
    for (int i = 0; i < n_ctx; ++i)
        if (!ctxs[i]) return 1;
    const int P = in->n_plans;
    *arena_used = 0;
    if (!in->blob) return fail(ctxs[0], "ws_plan_batch_multi: batch must be contiguous (ws_batch.blob)");
    if (n_ctx == 1) return ws_plan_batch_host(ctxs[0], in, results, arena, arena_cap, arena_used, nullptr);
    // block boundaries by cumulative cost estimate (modules x (devices + 8))
    std::vector<double> cum(P + 1, 0.0);
    for (int p = 0; p < P; ++p) {
        const ws_plan_rec& r = in->plans[p];
        cum[p + 1] = cum[p] + static_cast<double>(std::max(r.n_mod, 1)) * (std::max(r.n_dev, 0) + 8);
    }
    std::vector<int> pb(n_ctx + 1, P);
    pb[0] = 0;
    for (int s = 1; s < n_ctx; ++s)
        pb[s] = static_cast<int>(std::lower_bound(cum.begin(), cum.end(), cum[P] * s / n_ctx) - cum.begin());
    for (int s = 1; s <= n_ctx; ++s) pb[s] = std::max(pb[s], pb[s - 1]);
    std::vector<uint64_t> abase(n_ctx + 1, 0);
    for (int s = 0; s < n_ctx; ++s)
        abase[s + 1] = abase[s] + wsi_arena_bound_plans(in->plans + pb[s], pb[s + 1] - pb[s]);
    if (abase[n_ctx] > arena_cap) return fail(ctxs[0], "ws_plan_batch_multi: arena buffer too small");
    std::vector<int> rc(n_ctx, 0);
    std::vector<uint64_t> used(n_ctx, 0);
    std::vector<std::thread> pool;
    for (int s = 0; s < n_ctx; ++s)
        pool.emplace_back([&, s] {
            ws_ctx* ctx = ctxs[s];
            DevGuard dg_(ctx->device);
            rc[s] = host_range(ctx, in, pb[s], pb[s + 1], results + pb[s], arena + abase[s], abase[s + 1] - abase[s],
                               &used[s], ctx->stream);
            for (int p = pb[s]; p < pb[s + 1]; ++p)
                if (results[p].status == WS_STATUS_OK) results[p].offset += abase[s];
        });
    for (auto& t : pool) t.join();
    for (int s = 0; s < n_ctx; ++s) {
        if (rc[s]) {
            if (s) ctxs[0]->err = "context " + std::to_string(s) + ": " + ctxs[s]->err;
            return 1;
        }
        if (used[s]) *arena_used = abase[s] + used[s];
    }
    return 0;
}

// min-loc over host results (ties -> smaller index; infeasible plans lose)
int ws_best_host(const ws_plan_result* results, int64_t n, int mode, double* key, int64_t* index) {
    double bk = std::numeric_limits<double>::infinity();
    int64_t bi = -1;
    for (int64_t p = 0; p < n; ++p) {
        const ws_plan_result& r = results[p];
        if (r.status != WS_STATUS_OK) continue;
        const double k = mode == 0 ? r.end_time / r.lower_bound : r.end_time;
        if (bi < 0 || k < bk) bk = k, bi = p;
    }
    *key = bk;
    *index = bi;
    return mode == 0 || mode == 1 ? 0 : 1;
}

// Global best over the ranks of a multi-process job (one rank per GPU), SURVEY
// §8(e): every rank's local best {key, global index} is all-gathered as a
// 16-byte record over the caller's NCCL communicator (NVLink / NVSwitch) and
// min-located on every rank (ties -> smaller index).  NCCL has no MINLOC; the
// library loads NCCL with dlopen (no link-time dependency).
namespace {
using nccl_allgather_fn = int (*)(const void*, void*, size_t, int, void*, cudaStream_t);
using nccl_error_fn = const char* (*)(int);
struct NcclApi {
    nccl_allgather_fn allgather = nullptr;
    nccl_error_fn error = nullptr;
    std::string why;
};
const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = nullptr;
        if (const char* env = std::getenv("WSGPU_NCCL_LIB")) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = "libnccl.so.2 not found (set WSGPU_NCCL_LIB)";
            return a;
        }
        a.allgather = reinterpret_cast<nccl_allgather_fn>(dlsym(h, "ncclAllGather"));
        a.error = reinterpret_cast<nccl_error_fn>(dlsym(h, "ncclGetErrorString"));
        if (!a.allgather) a.why = "ncclAllGather not exported";
        return a;
    }();
    return api;
}
}  // namespace

int ws_best_nccl(ws_ctx* ctx, void* nccl_comm, int nranks, double local_key, int64_t local_index, double* key,
                 int64_t* index, void* stream) {
    DevGuard dg_(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    const NcclApi& api = nccl_api();
    if (!api.allgather) return fail(ctx, "ws_best_nccl: " + api.why);
    if (nranks < 1 || !nccl_comm) return fail(ctx, "ws_best_nccl: bad communicator");
    if (!ctx->best.ensure(16ull * (nranks + 1))) return fail(ctx, "cudaMalloc min-loc records");
    struct Rec {
        double key;
        int64_t index;
    };
    Rec mine{local_index >= 0 ? local_key : std::numeric_limits<double>::infinity(), local_index};
    auto* dev = ctx->best.as<Rec>();
    CK(cudaMemcpyAsync(dev, &mine, sizeof(Rec), cudaMemcpyHostToDevice, st));
    const int r = api.allgather(dev, dev + 1, sizeof(Rec), /*ncclUint8*/ 1, nccl_comm, st);
    if (r != 0) return fail(ctx, std::string("ncclAllGather: ") + (api.error ? api.error(r) : std::to_string(r)));
    std::vector<Rec> all(nranks);
    CK(cudaMemcpyAsync(all.data(), dev + 1, sizeof(Rec) * nranks, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double bk = std::numeric_limits<double>::infinity();
    int64_t bi = -1;
    for (const Rec& x : all) {
        if (x.index < 0 || x.key != x.key) continue;
        if (bi < 0 || x.key < bk || (x.key == bk && x.index < bi)) bk = x.key, bi = x.index;
    }
    *key = bk;
    *index = bi;
    return 0;
}

// Phase cycle counters of a -DWS_PHASES build (zeros otherwise); resets them.
int ws_debug_phase_cycles(unsigned long long* out, int n) {
#ifdef WS_PHASES
    unsigned long long h[32] = {};
    if (cudaMemcpyFromSymbol(h, g_phase_cycles, sizeof(h)) != cudaSuccess) return 1;
    for (int i = 0; i < n && i < 32; ++i) out[i] = h[i];
    const unsigned long long z[32] = {};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
#else
    for (int i = 0; i < n; ++i) out[i] = 0;
#endif
    return 0;
}

// Candidate search in one call: a host batch of up to
// kBestBatchMax plans through the small-batch launch (one H2D copy, hard record
// caps, no retry pass), optionally the device evaluation (mode 2), the on-device
// min-loc and one 16-byte copy back.  The records stay on the device for a later
// ws_fetch_results; larger batches go through stage + plan + best.
int ws_best_batch_host(ws_ctx* ctx, const ws_batch* in, int mode, const ws_sim_opts* sim, double* key,
                       int64_t* index, void* stream) {
    DevGuard dg_(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    const int P = in->n_plans;
    if (P > kBestBatchMax || !in->blob) {
        if (ws_stage_batch(ctx, in, stream) || ws_plan_staged(ctx, stream)) return 1;
    } else if (small_launch(ctx, in, st)) {
        return 1;
    }
    if (mode == 2 && ws_simulate_staged(ctx, sim, stream)) return 1;
    return ws_best_staged(ctx, mode, key, index, stream);
}

int ws_best_staged(ws_ctx* ctx, int mode, double* key, int64_t* index, void* stream) {
    DevGuard dg_(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    if (drain_overflow(ctx, st)) return 1;
    auto* kb = ctx->best.as<double>();
    auto* ib = reinterpret_cast<long long*>(kb + 1);
    if (mode == 2 && !ctx->sim_valid) return fail(ctx, "ws_best_staged: mode 2 needs ws_simulate_staged first");
    k_best<<<1, 1024, 0, st>>>(ctx->results.as<ws_plan_result>(), ctx->sim_res.as<ws_sim_result>(),
                               ctx->dview.n_plans, mode, kb, ib);
    // {key, index} are adjacent: one copy into page-locked host memory
    unsigned long long* hb = ctx->host_tops + kHtBest;
    CK(cudaMemcpyAsync(hb, kb, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::memcpy(key, hb, sizeof(double));
    *index = static_cast<int64_t>(hb[1]);
    return 0;
}



// ---- plan evaluation (simulate_plan + validate_plan) -------------------------
int ws_simulate_staged(ws_ctx* ctx, const ws_sim_opts* opts, void* stream) {
    DevGuard dg_(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    if (!ctx->records_on_device)
        return fail(ctx, "ws_simulate_staged: no device-resident plan records (plan with ws_plan_staged, "
                         "or evaluate host records with ws_simulate_batch_host)");
    if (drain_overflow(ctx, st)) return 1;
    const int P = ctx->dview.n_plans;
    const LaunchCaps& lh = ctx->caps_hard;
    SimArgs A{};
    A.B = ctx->dview;
    A.plans = ctx->results.as<ws_plan_result>();
    A.parena = ctx->arena.as<uint8_t>();
    A.opt = opts ? *opts : ws_sim_opts{2.0, 0, 0};
    A.caps = SimCaps{lh.pl.G, lh.rec.W, lh.pl.IS, lh.rec.M, lh.rec.E};
    const bool wide = lh.pl.N > 64;  // DevMask<4> device sets, as the planning launch
    A.SL = make_sim_layout(A.caps, wide ? static_cast<int>(sizeof(DevMask<4>)) : 8);
    A.n_plans = P;
    if (!ctx->sim_res.ensure(sizeof(ws_sim_result) * std::max(P, 1)) || !ctx->sim_arena.ensure(ctx->sim_cap) ||
        !ctx->sim_scratch.ensure(std::max<uint64_t>(ctx->arena_cap, 8)) || !ctx->sim_top.ensure(64))
        return fail(ctx, "cudaMalloc simulation buffers");
    A.scratch = ctx->sim_scratch.as<uint8_t>();
    A.out = ctx->sim_res.as<ws_sim_result>();
    A.arena = ctx->sim_arena.as<uint8_t>();
    A.arena_top = ctx->sim_top.as<unsigned long long>();
    A.arena_cap = ctx->sim_cap;
    const int smem = kSimWarps * A.SL.bytes;
    if (smem > kSmemLimit) return fail(ctx, "ws_simulate_staged: per-warp working set exceeds shared memory");
    CK(cudaMemsetAsync(A.arena_top, 0, 8, st));
    CK(cudaEventRecord(ctx->sev[0], st));
    if (P > 0)
        (wide ? k_sim<DevMask<4>> : k_sim<uint64_t>)<<<(P + kSimWarps - 1) / kSimWarps, 32 * kSimWarps, smem, st>>>(A);
    CK(cudaEventRecord(ctx->sev[1], st));
    CK(cudaGetLastError());
    ctx->sim_valid = true;
    return 0;
}

int ws_fetch_sim(ws_ctx* ctx, ws_sim_result* out, uint8_t* arena, uint64_t arena_cap, uint64_t* arena_used,
                 void* stream) {
    DevGuard dg_(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    if (!ctx->sim_valid) return fail(ctx, "ws_fetch_sim: nothing simulated");
    const int P = ctx->dview.n_plans;
    unsigned long long top = 0;
    if (P) CK(cudaMemcpyAsync(out, ctx->sim_res.p, sizeof(ws_sim_result) * P, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&top, ctx->sim_top.p, sizeof(top), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0;
    if (cudaEventElapsedTime(&ms, ctx->sev[0], ctx->sev[1]) == cudaSuccess) ctx->sim_ms = ms;
    if (top > ctx->sim_cap) top = ctx->sim_cap;
    if (top > arena_cap) return fail(ctx, "ws_fetch_sim: arena buffer too small");
    if (top) CK(cudaMemcpyAsync(arena, ctx->sim_arena.p, top, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *arena_used = top;
    return 0;
}

int ws_simulate_batch_host(ws_ctx* ctx, const ws_batch* in, const ws_plan_result* plans, const uint8_t* plan_arena,
                           uint64_t plan_arena_bytes, const ws_sim_opts* opts, ws_sim_result* out, uint8_t* arena,
                           uint64_t arena_cap, uint64_t* arena_used, void* stream) {
    DevGuard dg_(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    if (ws_stage_batch(ctx, in, stream)) return 1;
    const int P = in->n_plans;
    ctx->arena_cap = std::max<uint64_t>(plan_arena_bytes, 8);
    if (!ctx->results.ensure(sizeof(ws_plan_result) * std::max(P, 1)) || !ctx->arena.ensure(ctx->arena_cap))
        return fail(ctx, "cudaMalloc plan records");
    if (P) CK(cudaMemcpyAsync(ctx->results.p, plans, sizeof(ws_plan_result) * P, cudaMemcpyHostToDevice, st));
    if (plan_arena_bytes) CK(cudaMemcpyAsync(ctx->arena.p, plan_arena, plan_arena_bytes, cudaMemcpyHostToDevice, st));
    ctx->records_on_device = true;
    if (ws_simulate_staged(ctx, opts, stream)) return 1;
    return ws_fetch_sim(ctx, out, arena, arena_cap, arena_used, stream);
}

double ws_last_sim_ms(const ws_ctx* ctx) { return ctx ? ctx->sim_ms : 0.0; }

}  // extern "C"
