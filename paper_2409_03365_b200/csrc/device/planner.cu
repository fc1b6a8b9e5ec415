// planner.cu — C-ABI implementation: planning context, device buffers and the
// launch sequence of the sm_100a planner kernels.
//
//   k_fit   (K2)           one thread per declared module
//   k_plan  (K1,K3,K4,K5)  one warp per plan; soft-cap overflows re-run in a
//                          device-driven retry launch with the hard caps
//   k_best                 global-best candidate (min-loc) over the batch
//
// Replaces wavesched::plan_workload (planner.hpp:156-212) for whole batches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fit.cuh"
#include "plan.cuh"

using namespace wsdev;

namespace {

constexpr int kRetryMax = 2048;               // plans re-run with hard caps per call
constexpr int64_t kOverflowPieces = 1 << 18;  // isotonic/long curves
constexpr size_t kScratchBudget = size_t(6) << 30;

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    bool ensure(size_t bytes) {
        if (bytes <= n) return true;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        if (cudaMalloc(&p, bytes) != cudaSuccess) return false;
        n = bytes;
        return true;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// k_soft_collect: plans whose soft scratch caps overflowed (waves/entries/flows
// or arena) get queued for the retry launch.
__global__ void k_soft_collect(const ws_plan_result* res, int n, int32_t* ids, int32_t* count) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int e = res[p].err_code;
    if (e == WS_E_LIMIT_WAVES || e == WS_E_LIMIT_ENTRIES || e == WS_E_LIMIT_FLOWS) {
        const int slot = atomicAdd(count, 1);
        if (slot < kRetryMax) ids[slot] = p;
    }
}

__global__ void k_clamp_count(int32_t* count) {
    if (*count > kRetryMax) *count = kRetryMax;
}

// Global min-loc over plan keys; ties -> smaller index.
__global__ void k_best(const ws_plan_result* res, int n, int mode, double* out_key, long long* out_idx) {
    __shared__ double sk[1024];
    __shared__ long long si[1024];
    double bk = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    long long bi = -1;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        const ws_plan_result& r = res[p];
        if (r.status != WS_STATUS_OK) continue;
        const double k = mode == 0 ? r.end_time / r.lower_bound : r.end_time;
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

}  // namespace

struct ws_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    // staged batch
    DevBuf blob;
    ws_batch dview{};
    std::vector<ws_plan_rec> host_plans;
    Caps caps{}, caps_hard{};
    // K2 outputs
    DevBuf fit_err, fit_a, fit_b, fit_np, fit_nmax, fit_off, fit_pieces, ttab;
    // K1/K3/K4/K5
    DevBuf scratch, results, arena, counters, retry_ids, best;
    uint64_t arena_cap = 0;
    int launches = 0;
    cudaEvent_t ev[4] = {};
    double kernel_ms[2] = {0, 0};
};

namespace {

int fail(ws_ctx* c, const std::string& what, cudaError_t e = cudaSuccess) {
    c->err = what;
    if (e != cudaSuccess) c->err += std::string(": ") + cudaGetErrorString(e);
    return 1;
}

#define CK(call)                                               \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return fail(ctx, #call, e_);    \
    } while (0)

Caps batch_caps(const std::vector<ws_plan_rec>& plans, bool hard) {
    Caps c{1, 1, 1, 1, 1, 1, 1};
    int gmax = 0;
    for (const ws_plan_rec& r : plans) {
        c.M = std::max(c.M, r.n_mod);
        c.N = std::max(c.N, r.n_dev);
        c.IS = std::max(c.IS, r.n_islands);
        gmax = std::max(gmax, r.n_groups);
    }
    c.M = std::min(c.M, WS_MAX_MODULES);
    c.N = std::min(c.N, WS_MAX_DEVICES);
    c.G = gmax + c.M;
    c.W = std::min(WS_MAX_WAVES, 2 * c.M + 1);  // each wave drains a tuple
    if (hard) {
        c.E = std::min(WS_MAX_ENTRIES, std::max(64, 2 * c.M * c.M));
        c.F = WS_MAX_FLOWS;
    } else {
        c.E = std::max(32, 4 * c.M);
        c.F = std::max(64, 8 * c.M);
    }
    return c;
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
    d.blob = dbase;
    return d;
}

}  // namespace

extern "C" {

int ws_ctx_create(int device, ws_ctx** out) {
    *out = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    auto* c = new ws_ctx();
    c->device = device;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return 1;
    }
    for (auto& e : c->ev) cudaEventCreate(&e);
    *out = c;
    return 0;
}

void ws_ctx_destroy(ws_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* ws_ctx_last_error(const ws_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

int ws_last_launch_count(const ws_ctx* c) { return c ? c->launches : 0; }

int ws_last_kernel_ms(const ws_ctx* c, double* out, int n) {
    if (!c) return 1;
    for (int i = 0; i < n && i < 2; ++i) out[i] = c->kernel_ms[i];
    return 0;
}

int ws_stage_batch(ws_ctx* ctx, const ws_batch* in, void* stream) {
    cudaSetDevice(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    if (!in->blob) return fail(ctx, "ws_stage_batch: batch must be contiguous (ws_batch.blob)");
    if (!ctx->blob.ensure(in->blob_bytes + 256)) return fail(ctx, "cudaMalloc batch");
    CK(cudaMemcpyAsync(ctx->blob.p, in->blob, in->blob_bytes, cudaMemcpyHostToDevice, st));
    ctx->dview = rebase(*in, in->blob, ctx->blob.as<char>());
    ctx->host_plans.assign(in->plans, in->plans + in->n_plans);
    ctx->caps = batch_caps(ctx->host_plans, false);
    ctx->caps_hard = batch_caps(ctx->host_plans, true);
    ctx->arena_cap = ws_arena_bound(in);
    return 0;
}

int ws_plan_staged(ws_ctx* ctx, void* stream) {
    cudaSetDevice(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    const ws_batch& B = ctx->dview;
    const int P = B.n_plans, NM = std::max(B.n_modules, 1);
    const Caps& caps = ctx->caps;
    ctx->launches = 0;
    // K2 buffers
    const int tstride = caps.N;
    if (!ctx->fit_err.ensure(4ull * NM) || !ctx->fit_a.ensure(4ull * NM) || !ctx->fit_b.ensure(4ull * NM) ||
        !ctx->fit_np.ensure(4ull * NM) || !ctx->fit_nmax.ensure(4ull * NM) || !ctx->fit_off.ensure(8ull * NM) ||
        !ctx->fit_pieces.ensure(40ull * (static_cast<uint64_t>(NM) * kInlinePieces + kOverflowPieces)) ||
        !ctx->ttab.ensure(8ull * NM * tstride))
        return fail(ctx, "cudaMalloc fit buffers");
    if (!ctx->counters.ensure(64) || !ctx->results.ensure(sizeof(ws_plan_result) * std::max(P, 1)) ||
        !ctx->arena.ensure(ctx->arena_cap) || !ctx->retry_ids.ensure(4 * kRetryMax) || !ctx->best.ensure(64))
        return fail(ctx, "cudaMalloc result buffers");
    auto* counters = ctx->counters.as<unsigned long long>();  // [0] arena top [1] overflow top [2] retry count
    CK(cudaMemsetAsync(counters, 0, 64, st));
    FitOut fo;
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

    CK(cudaEventRecord(ctx->ev[0], st));
    if (B.n_modules > 0) {
        k_fit<<<(B.n_modules + 127) / 128, 128, 0, st>>>(B, fo);
        ctx->launches++;
    }
    CK(cudaEventRecord(ctx->ev[1], st));

    PlanArgs A{};
    A.B = B;
    A.fit = fo;
    A.results = ctx->results.as<ws_plan_result>();
    A.arena = ctx->arena.as<uint8_t>();
    A.arena_top = counters;
    A.arena_cap = ctx->arena_cap;
    // main pass (soft caps), chunked by scratch budget
    A.caps = caps;
    A.L = make_layout(caps);
    const size_t per = static_cast<size_t>(A.L.bytes);
    const int chunk = static_cast<int>(std::max<size_t>(1, std::min<size_t>(P, kScratchBudget / per)));
    if (!ctx->scratch.ensure(per * std::max(chunk, 1))) return fail(ctx, "cudaMalloc scratch");
    A.scratch = ctx->scratch.as<char>();
    for (int base = 0; base < P; base += chunk) {
        A.plan_base = base;
        A.n_launch = std::min(chunk, P - base);
        const int blocks = (A.n_launch + kPlanWarps - 1) / kPlanWarps;
        k_plan<<<blocks, 32 * kPlanWarps, 0, st>>>(A);
        ctx->launches++;
    }
    // retry pass: soft-cap overflows with the hard caps, count read on device
    auto* rcount = reinterpret_cast<int32_t*>(counters + 2);
    if (P > 0) {
        k_soft_collect<<<(P + 255) / 256, 256, 0, st>>>(A.results, P, ctx->retry_ids.as<int32_t>(), rcount);
        k_clamp_count<<<1, 1, 0, st>>>(rcount);
        ctx->launches += 2;
        PlanArgs Rr = A;
        Rr.caps = ctx->caps_hard;
        Rr.L = make_layout(Rr.caps);
        const size_t per_h = static_cast<size_t>(Rr.L.bytes);
        const int rchunk = static_cast<int>(std::min<size_t>(kRetryMax, std::max<size_t>(1, kScratchBudget / per_h)));
        if (per_h * rchunk > ctx->scratch.n) {
            // reuse the main scratch when large enough, else grow
            if (!ctx->scratch.ensure(per_h * rchunk)) return fail(ctx, "cudaMalloc retry scratch");
        }
        Rr.scratch = ctx->scratch.as<char>();
        Rr.plan_ids = ctx->retry_ids.as<int32_t>();
        Rr.n_ids = rcount;
        Rr.plan_base = 0;
        Rr.n_launch = rchunk;
        k_plan<<<(rchunk + kPlanWarps - 1) / kPlanWarps, 32 * kPlanWarps, 0, st>>>(Rr);
        ctx->launches++;
    }
    CK(cudaEventRecord(ctx->ev[2], st));
    CK(cudaGetLastError());
    return 0;
}

int ws_fetch_results(ws_ctx* ctx, ws_plan_result* results, uint8_t* arena, uint64_t arena_cap,
                     uint64_t* arena_used, void* stream) {
    cudaSetDevice(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    const int P = ctx->dview.n_plans;
    unsigned long long top = 0;
    CK(cudaMemcpyAsync(results, ctx->results.p, sizeof(ws_plan_result) * P, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&top, ctx->counters.p, sizeof(top), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0;
    if (cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]) == cudaSuccess) ctx->kernel_ms[0] = ms;
    if (cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]) == cudaSuccess) ctx->kernel_ms[1] = ms;
    if (top > ctx->arena_cap) top = ctx->arena_cap;
    if (top > arena_cap) return fail(ctx, "ws_fetch_results: arena buffer too small");
    if (top) CK(cudaMemcpyAsync(arena, ctx->arena.p, top, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *arena_used = top;
    return 0;
}

int ws_plan_batch_host(ws_ctx* ctx, const ws_batch* in, ws_plan_result* results, uint8_t* arena,
                       uint64_t arena_cap, uint64_t* arena_used, void* stream) {
    if (ws_stage_batch(ctx, in, stream)) return 1;
    if (ws_plan_staged(ctx, stream)) return 1;
    return ws_fetch_results(ctx, results, arena, arena_cap, arena_used, stream);
}

int ws_best_staged(ws_ctx* ctx, int mode, double* key, int64_t* index, void* stream) {
    cudaSetDevice(ctx->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    auto* kb = ctx->best.as<double>();
    auto* ib = reinterpret_cast<long long*>(kb + 1);
    k_best<<<1, 1024, 0, st>>>(ctx->results.as<ws_plan_result>(), ctx->dview.n_plans, mode, kb, ib);
    double hk = 0;
    long long hi = -1;
    CK(cudaMemcpyAsync(&hk, kb, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hi, ib, sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *key = hk;
    *index = hi;
    return 0;
}

}  // extern "C"
