// The C-ABI (include/snls_cuda.h): validation with the reference's messages, dispatch to
// the sm_100a kernels, and the per-(device, stream) context.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <string>

#include "common.cuh"
#include "kernels.h"
#include "snls_cuda.h"

using namespace snls_gpu;

struct snls_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int* err = nullptr;  // device-side latch
    void* work = nullptr;
    size_t work_bytes = 0;
    int64_t launches = 0;
    int num_sms = 148;
    int force_generic = 0;
    int search_kernel = 0;
    int last_path = -1;
    int band = -1;  // temporally blocked search raster: -1 auto (search_band), 0 off, > 0 rows
    cudaStream_t aux = nullptr;  // snls_train_bwd: the wpsum backward beside the search backward
    cudaEvent_t fork = nullptr, join = nullptr;
};

namespace snls_capi {

thread_local std::string g_err;

// Record the message of a failure for snls_last_error() (also used by pipeline.cu).
int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// The device error latch of a context (pipeline.cu snapshots it with each clip).
int* ctx_err(snls_ctx* ctx) { return ctx ? ctx->err : nullptr; }
// The device a context's kernels, streams and buffers belong to.
int ctx_device(snls_ctx* ctx) { return ctx ? ctx->device : 0; }

// Read-and-clear of the latch in ONE device operation: latch[1] = atomicExch(latch[0], 0).
// A bit another in-flight stream sets after the exchange stays latched for the next check
// (a separate read then clear could wipe it unreported).
__global__ void latch_take_kernel(int* latch) { latch[1] = atomicExch(latch, 0); }

}  // namespace snls_capi

using snls_capi::fail;
using snls_capi::g_err;

namespace {

int cuda_fail(cudaError_t e, const char* where) {
    return fail(SNLS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int after_launch(snls_ctx* ctx, int launched, const char* where) {
    if (launched > 0) ctx->launches += launched;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, where);
    return SNLS_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// search.cpp:21-32, messages verbatim
int validate(const snls_config* c) {
    if (!c) return fail(SNLS_EARG, "snls: null config");
    if (c->ws < 1 || c->ws % 2 == 0)
        return fail(SNLS_ECONFIG, "SearchConfig: ws must be odd and positive");
    if (c->ps < 1 || c->ps % 2 == 0)
        return fail(SNLS_ECONFIG, "SearchConfig: ps must be odd and positive");
    if (c->wt < 0) return fail(SNLS_ECONFIG, "SearchConfig: wt must be >= 0");
    if (c->stride0 < 1) return fail(SNLS_ECONFIG, "SearchConfig: stride0 must be >= 1");
    if (!(c->stride1 > 0.0) || !std::isfinite(c->stride1))
        return fail(SNLS_ECONFIG, "SearchConfig: stride1 must be positive and finite");
    const long long slots = (2LL * c->wt + 1) * c->ws * c->ws;
    if (c->topl < 1 || c->topl > slots)
        return fail(SNLS_ECONFIG, "SearchConfig: topl must lie in [1, window slots]");
    if (!std::isfinite(c->softmax_scale))
        return fail(SNLS_ECONFIG, "SearchConfig: softmax_scale must be finite");
    if (c->metric != SNLS_METRIC_IP && c->metric != SNLS_METRIC_L2)
        return fail(SNLS_ECONFIG, "SearchConfig: unknown metric");
    return SNLS_OK;
}

int check_dims(snls_dims d) {
    if (d.t < 1 || d.h < 1 || d.w < 1 || d.f < 1)
        return fail(SNLS_EDOMAIN, "VideoTensor: all extents must be at least 1");
    return SNLS_OK;
}

// The kernels load float4 / u64 vectors straight from the base pointers: a misaligned
// pointer would raise cudaErrorMisalignedAddress, which is sticky for the whole context.
int check_aligned(const char* where, std::initializer_list<const void*> ptrs) {
    for (const void* p : ptrs)
        if (p && (reinterpret_cast<uintptr_t>(p) & 15u))
            return fail(SNLS_EARG, std::string(where) + ": tensor pointers must be 16-byte aligned");
    return SNLS_OK;
}

int check_ctx(snls_ctx* ctx) {
    if (!ctx) return fail(SNLS_EARG, "snls: null context");
    return SNLS_OK;
}

// fused_forward's underfull rule (search.cpp:317-325), decided from shapes alone: the
// fewest valid frames any query frame sees, times ws^2.
bool underfull(const snls_config* c, int t, int t0 = 0, int t1 = -1) {
    long long worst = -1;
    if (t1 < 0) t1 = t;
    for (int qt = t0; qt < t1; ++qt) {
        const int lo = qt - c->wt < 0 ? 0 : qt - c->wt;
        const int hi = qt + c->wt > t - 1 ? t - 1 : qt + c->wt;
        const long long valid = (long long)(hi - lo + 1) * c->ws * c->ws;
        if (worst < 0 || valid < worst) worst = valid;
    }
    return worst < c->topl;
}

// Temporally blocked raster for the tiled search (common.cuh band_row): only when the key
// frames one query frame reads overflow about a third of the 126 MB L2; band height such
// that (2wt+2) frames of band rows (plus the window reach) fit that budget.
// SNLS_SEARCH_BAND overrides (0 = plain raster).
int search_band(const snls_ctx* ctx, const snls_config* c, snls_dims d) {
    static const int env = [] {
        const char* e = std::getenv("SNLS_SEARCH_BAND");
        return e ? std::atoi(e) : -1;
    }();
    const int nh = (d.h - 1) / c->stride0 + 1;
    const int forced = ctx->band >= 0 ? ctx->band : env;
    if (forced >= 0) return forced >= nh ? 0 : forced;
    const double row_bytes = double(d.w) * d.f * 4.0;
    const double frames_bytes = (2.0 * c->wt + 1) * d.h * row_bytes;
    const double budget = 42.0e6;
    // key sets that (nearly) fit the 126 MB L2 gain nothing from banding and pay its
    // index arithmetic: c4 (7 frames x 8.4 MB = 59 MB) 3.90 ms plain vs 3.98 ms banded
    if (frames_bytes <= 2.0 * budget) return 0;
    const double px_rows = budget / ((2.0 * c->wt + 2) * row_bytes) - 2.0 * (c->ws / 2 + c->ps / 2 + 4);
    const int band = std::max(4, int(px_rows / c->stride0));
    return band >= nh ? 0 : band;
}

int ensure_work(snls_ctx* ctx, size_t bytes) {
    if (ctx->work_bytes >= bytes) return SNLS_OK;
    if (ctx->work) {
        // the context's stream may have been switched (pipeline chunks): wait for every
        // stream of the device before the old workspace goes away (a rare, growing resize)
        cudaDeviceSynchronize();
        cudaFree(ctx->work);
        ctx->work = nullptr;
        ctx->work_bytes = 0;
    }
    const cudaError_t e = cudaMalloc(&ctx->work, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "snls workspace");
    ctx->work_bytes = bytes;
    return SNLS_OK;
}

}  // namespace

extern "C" {

int snls_abi_version(void) { return SNLS_CUDA_ABI_VERSION; }

const char* snls_last_error(void) { return g_err.c_str(); }

int snls_validate_config(const snls_config* cfg) { return validate(cfg); }

int snls_query_grid(snls_dims dims, int stride0, int64_t* rows, int* nh, int* nw) {
    if (stride0 < 1) return fail(SNLS_ECONFIG, "SearchConfig: stride0 must be >= 1");
    if (int rc = check_dims(dims)) return rc;
    const Dims d = make_dims(dims, stride0);
    if (rows) *rows = d.rows;
    if (nh) *nh = d.nh;
    if (nw) *nw = d.nw;
    return SNLS_OK;
}

// std::mt19937_64 + UniformStream::next_in (rng.hpp:12-24), rounded to fp32.
int snls_uniform_fill_f32(uint64_t seed, double lo, double hi, int64_t n, float* out) {
    if (!out && n > 0) return fail(SNLS_EARG, "snls_uniform_fill_f32: null output");
    uint64_t mt[312];
    mt[0] = seed;
    for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
    int idx = 312;
    for (int64_t i = 0; i < n; ++i) {
        if (idx >= 312) {
            for (int j = 0; j < 312; ++j) {
                const uint64_t x = (mt[j] & 0xFFFFFFFF80000000ULL) | (mt[(j + 1) % 312] & 0x7FFFFFFFULL);
                uint64_t xa = x >> 1;
                if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
                mt[j] = mt[(j + 156) % 312] ^ xa;
            }
            idx = 0;
        }
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        out[i] = float(lo + (hi - lo) * (double(y >> 11) * 0x1.0p-53));
    }
    return SNLS_OK;
}

int snls_ctx_create(int device, void* stream, snls_ctx** out) {
    if (!out) return fail(SNLS_EARG, "snls_ctx_create: null output");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) return fail(SNLS_ECUDA, "snls_ctx_create: no CUDA device visible");
    if (device < 0 || device >= n) return fail(SNLS_EARG, "snls_ctx_create: device index out of range");
    DeviceGuard g(device);
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return cuda_fail(e, "snls_ctx_create");
    if (prop.major != 10)
        return fail(SNLS_ECUDA, std::string("snls_ctx_create: kernels are built for sm_100a, device is ") +
                                    prop.name);
    snls_ctx* ctx = new snls_ctx();
    ctx->device = device;
    ctx->stream = static_cast<cudaStream_t>(stream);
    ctx->num_sms = prop.multiProcessorCount;
    // err[0]: the latch kernels atomicOr into; err[1]: the value taken by sync_check
    if ((e = cudaMalloc(&ctx->err, 2 * sizeof(int))) != cudaSuccess) {
        delete ctx;
        return cuda_fail(e, "snls_ctx_create");
    }
    cudaMemset(ctx->err, 0, 2 * sizeof(int));
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) {
        cudaFree(ctx->err);
        delete ctx;
        return cuda_fail(e, "snls_ctx_create");
    }
    *out = ctx;
    return SNLS_OK;
}

int snls_ctx_destroy(snls_ctx* ctx) {
    if (!ctx) return SNLS_OK;
    DeviceGuard g(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->err) cudaFree(ctx->err);
    if (ctx->work) cudaFree(ctx->work);
    if (ctx->aux) {
        cudaStreamSynchronize(ctx->aux);
        cudaStreamDestroy(ctx->aux);
        cudaEventDestroy(ctx->fork);
        cudaEventDestroy(ctx->join);
    }
    delete ctx;
    return SNLS_OK;
}

int snls_ctx_set_stream(snls_ctx* ctx, void* stream) {
    if (int rc = check_ctx(ctx)) return rc;
    ctx->stream = static_cast<cudaStream_t>(stream);
    return SNLS_OK;
}

int snls_ctx_get_stream(snls_ctx* ctx, void** out) {
    if (int rc = check_ctx(ctx)) return rc;
    if (out) *out = static_cast<void*>(ctx->stream);
    return SNLS_OK;
}

int snls_ctx_launch_count(snls_ctx* ctx, int64_t* out) {
    if (int rc = check_ctx(ctx)) return rc;
    if (out) *out = ctx->launches;
    return SNLS_OK;
}

int snls_ctx_last_search_path(snls_ctx* ctx, int* out) {
    if (int rc = check_ctx(ctx)) return rc;
    if (out) *out = ctx->last_path;
    return SNLS_OK;
}

int snls_ctx_set_search_kernel(snls_ctx* ctx, int kind) {
    if (int rc = check_ctx(ctx)) return rc;
    if (kind < 0 || kind > 2) return fail(SNLS_EARG, "set_search_kernel: kind must be 0, 1 or 2");
    ctx->search_kernel = kind;
    return SNLS_OK;
}

int snls_ctx_set_search_band(snls_ctx* ctx, int band) {
    if (int rc = check_ctx(ctx)) return rc;
    ctx->band = band < 0 ? -1 : band;
    return SNLS_OK;
}

int snls_ctx_force_generic(snls_ctx* ctx, int on) {
    if (int rc = check_ctx(ctx)) return rc;
    ctx->force_generic = on;
    return SNLS_OK;
}

int snls_ctx_sync_check(snls_ctx* ctx) {
    if (int rc = check_ctx(ctx)) return rc;
    DeviceGuard g(ctx->device);
    int host = 0;
    snls_capi::latch_take_kernel<<<1, 1, 0, ctx->stream>>>(ctx->err);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&host, ctx->err + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "snls_ctx_sync_check");
    if (host == 0) return SNLS_OK;
    if (host & kErrFflow) return fail(SNLS_EDOMAIN, "search fflow: flow holds a non-finite value");
    if (host & kErrBflow) return fail(SNLS_EDOMAIN, "search bflow: flow holds a non-finite value");
    if (host & kErrSoftmax) return fail(SNLS_EDOMAIN, "softmax_rows: non-finite input");
    if (host & kErrWpsum)
        return fail(SNLS_EDOMAIN, "wpsum: offsets leave the clip or a pixel has no writers");
    if (host & kErrStack) return fail(SNLS_EDOMAIN, "gather_stack: offsets leave the clip");
    if (host & kErrTopl) return fail(SNLS_EDOMAIN, "top_l: some row has fewer than L valid entries");
    return fail(SNLS_EDOMAIN, "snls: device reported an unknown domain error");
}

int snls_device_alloc(snls_ctx* ctx, uint64_t bytes, void** out) {
    if (int rc = check_ctx(ctx)) return rc;
    if (!out) return fail(SNLS_EARG, "snls_device_alloc: null output");
    DeviceGuard g(ctx->device);
    *out = nullptr;
    if (bytes == 0) return SNLS_OK;
    const cudaError_t e = cudaMalloc(out, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "snls_device_alloc");
    return SNLS_OK;
}

int snls_device_free(snls_ctx* ctx, void* ptr) {
    if (int rc = check_ctx(ctx)) return rc;
    if (!ptr) return SNLS_OK;
    DeviceGuard g(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    const cudaError_t e = cudaFree(ptr);
    if (e != cudaSuccess) return cuda_fail(e, "snls_device_free");
    return SNLS_OK;
}

int snls_copy_h2d(snls_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    if (int rc = check_ctx(ctx)) return rc;
    if (bytes == 0) return SNLS_OK;
    if (!dst || !src) return fail(SNLS_EARG, "snls_copy_h2d: null pointer");
    DeviceGuard g(ctx->device);
    const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "snls_copy_h2d");
    return SNLS_OK;
}

int snls_copy_d2h(snls_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    if (int rc = check_ctx(ctx)) return rc;
    if (bytes == 0) return SNLS_OK;
    if (!dst || !src) return fail(SNLS_EARG, "snls_copy_d2h: null pointer");
    DeviceGuard g(ctx->device);
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "snls_copy_d2h");
    return SNLS_OK;
}

// Stream-ordered copy without a host wait (kind 1 H2D, 2 D2H, 3 D2D); host buffers should be
// pinned (snls_host_register) for the copy to be asynchronous.
int snls_copy_async(snls_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind) {
    if (int rc = check_ctx(ctx)) return rc;
    if (bytes == 0) return SNLS_OK;
    if (!dst || !src) return fail(SNLS_EARG, "snls_copy_async: null pointer");
    const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice
                           : kind == 2 ? cudaMemcpyDeviceToHost
                           : kind == 3 ? cudaMemcpyDeviceToDevice : cudaMemcpyDefault;
    if (kind < 1 || kind > 3) return fail(SNLS_EARG, "snls_copy_async: kind must be 1, 2 or 3");
    DeviceGuard g(ctx->device);
    const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, k, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "snls_copy_async");
    return SNLS_OK;
}

struct snls_event {
    cudaEvent_t ev = nullptr;
    int device = 0;
};

int snls_event_create(snls_ctx* ctx, snls_event** out) {
    if (int rc = check_ctx(ctx)) return rc;
    if (!out) return fail(SNLS_EARG, "snls_event_create: null output");
    DeviceGuard g(ctx->device);
    auto* ev = new snls_event();
    ev->device = ctx->device;
    const cudaError_t e = cudaEventCreateWithFlags(&ev->ev, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        delete ev;
        return cuda_fail(e, "snls_event_create");
    }
    *out = ev;
    return SNLS_OK;
}

int snls_event_record(snls_ctx* ctx, snls_event* ev) {
    if (int rc = check_ctx(ctx)) return rc;
    if (!ev) return fail(SNLS_EARG, "snls_event_record: null event");
    DeviceGuard g(ctx->device);
    const cudaError_t e = cudaEventRecord(ev->ev, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "snls_event_record");
    return SNLS_OK;
}

int snls_event_sync(snls_event* ev) {
    if (!ev) return fail(SNLS_EARG, "snls_event_sync: null event");
    DeviceGuard g(ev->device);
    const cudaError_t e = cudaEventSynchronize(ev->ev);
    if (e != cudaSuccess) return cuda_fail(e, "snls_event_sync");
    return SNLS_OK;
}

int snls_event_destroy(snls_event* ev) {
    if (!ev) return SNLS_OK;
    DeviceGuard g(ev->device);
    cudaEventDestroy(ev->ev);
    delete ev;
    return SNLS_OK;
}

static int search_common_checks(snls_ctx* ctx, const snls_config* cfg, snls_dims dims,
                                const float* q, const float* k, const float* ff, const float* bf) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = validate(cfg)) return rc;
    if (int rc = check_dims(dims)) return rc;
    if (!q || !k) return fail(SNLS_EARG, "search: null query/key tensor");
    if ((ff == nullptr) != (bf == nullptr))
        return fail(SNLS_EARG, "search: pass both flows or neither (nls_forward)");
    return check_aligned("search", {q, k, ff, bf});
}

int snls_search_fwd(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* q,
                    const float* k, const float* ff, const float* bf, int mode, float* sims,
                    float* offsets, float* chains, float* weights) {
    return snls_search_fwd_frames(ctx, cfg, dims, 0, dims.t, q, k, ff, bf, mode, sims, offsets,
                                  chains, weights);
}

int snls_search_fwd_frames(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                           const float* q, const float* k, const float* ff, const float* bf,
                           int mode, float* sims, float* offsets, float* chains, float* weights) {
    if (int rc = search_common_checks(ctx, cfg, dims, q, k, ff, bf)) return rc;
    if (!sims || !offsets) return fail(SNLS_EARG, "search: null output");
    if (t0 < 0 || t1 > dims.t || t0 >= t1) return fail(SNLS_EARG, "search: empty or invalid frame range");
    if (underfull(cfg, dims.t, t0, t1))
        return fail(SNLS_ECONFIG, "search: topl exceeds the valid window entries of some query");
    DeviceGuard g(ctx->device);
    const Dims d = restrict_frames(make_dims(dims, cfg->stride0), t0, t1);
    // validate_forward_inputs (search.cpp:175-183) checks every flow frame; a frame range
    // checks the frames its queries can read, [t0 - wt, t1 + wt) -- the whole clip for the
    // plain entry, and a shard's halo frames are checked by their owner (they may still be
    // in flight while the interior frames run)
    const int f0 = t0 - cfg->wt > 0 ? t0 - cfg->wt : 0;
    const int f1 = t1 + cfg->wt < dims.t ? t1 + cfg->wt : dims.t;
    const int64_t fframe = int64_t(dims.h) * dims.w * 2;
    int launched = launch_flows_check(ff ? ff + f0 * fframe : nullptr, bf ? bf + f0 * fframe : nullptr,
                                      (f1 - f0) * fframe, ctx->err, ctx->stream);
    const float beta = float(cfg->softmax_scale);

    if (mode == SNLS_MODE_FULLGRID) {
        // materialise rows x window_slots scores (search.cpp:351-376) with the same kernel
        // arithmetic as the fused path, then select + emit from the grid (search.cpp:378-406):
        // fused and full-grid results are bitwise identical, as in the reference.
        const int n = (2 * cfg->wt + 1) * cfg->ws * cfg->ws;
        if (int rc = ensure_work(ctx, size_t(d.rows) * n * sizeof(float))) return rc;
        float* grid = static_cast<float*>(ctx->work);
        int produced = 0;
        if (!ctx->force_generic && cfg->stride1 == 1.0) {
            TiledSearch ts{q, k, ff, bf, d, cfg->ws, cfg->wt, cfg->ps, cfg->topl, cfg->metric, beta,
                           sims, offsets, chains, weights, ctx->err, ctx->num_sms, grid, ctx->search_kernel,
                           search_band(ctx, cfg, dims)};
            produced = launch_search_tiled(ts, ctx->stream, nullptr);
            if (produced < 0) return fail(SNLS_ECUDA, "search: tiled kernel launch failed");
        }
        if (produced == 0) {
            GenericSearch gs{q, k, ff, bf, d, cfg->ws, cfg->wt, cfg->ps, cfg->topl, cfg->metric,
                             cfg->stride1, beta, sims, offsets, nullptr, nullptr, grid, nullptr, 0,
                             ctx->err, nullptr};
            if (launch_search_generic(gs, ctx->stream) < 0)
                return fail(SNLS_ECONFIG, "search: window too large for the device search");
            produced = 1;
        }
        GenericSearch sel{q, k, ff, bf, d, cfg->ws, cfg->wt, cfg->ps, cfg->topl, cfg->metric,
                          cfg->stride1, beta, sims, offsets, chains, weights, nullptr, nullptr, 1,
                          ctx->err, grid};
        if (launch_search_generic(sel, ctx->stream) < 0)
            return fail(SNLS_ECONFIG, "search: window too large for the device top_l");
        ctx->last_path = 2;
        return after_launch(ctx, launched + produced + 1, "snls_search_fwd(fullgrid)");
    }

    int tiled = 0, used = 0;
    if (!ctx->force_generic && cfg->stride1 == 1.0) {
        TiledSearch ts{q, k, ff, bf, d, cfg->ws, cfg->wt, cfg->ps, cfg->topl, cfg->metric, beta,
                       sims, offsets, chains, weights, ctx->err, ctx->num_sms, nullptr, ctx->search_kernel,
                       search_band(ctx, cfg, dims)};
        tiled = launch_search_tiled(ts, ctx->stream, &used);
        if (tiled < 0) return fail(SNLS_ECUDA, "search: tiled kernel launch failed");
    }
    if (tiled > 0) {
        launched += tiled;
        ctx->last_path = used == 2 ? 3 : 1;
    } else {
        GenericSearch gs{q, k, ff, bf, d, cfg->ws, cfg->wt, cfg->ps, cfg->topl, cfg->metric,
                         cfg->stride1, beta, sims, offsets, chains, weights, nullptr, nullptr, 1, ctx->err,
                         nullptr};
        if (launch_search_generic(gs, ctx->stream) < 0)
            return fail(SNLS_ECONFIG, "search: window too large for the device search");
        ++launched;
        ctx->last_path = 0;
    }
    return after_launch(ctx, launched, "snls_search_fwd");
}

int snls_search_grid(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* q,
                     const float* k, const float* ff, const float* bf, float* grid,
                     float* grid_offsets) {
    if (int rc = search_common_checks(ctx, cfg, dims, q, k, ff, bf)) return rc;
    if (!grid) return fail(SNLS_EARG, "search_grid: null output");
    DeviceGuard g(ctx->device);
    const Dims d = make_dims(dims, cfg->stride0);
    int launched = launch_flows_check(ff, bf, int64_t(dims.t) * dims.h * dims.w * 2, ctx->err, ctx->stream);
    GenericSearch gs{q, k, ff, bf, d, cfg->ws, cfg->wt, cfg->ps, cfg->topl, cfg->metric,
                     cfg->stride1, 1.f, nullptr, nullptr, nullptr, nullptr, grid, grid_offsets, 0, ctx->err,
                     nullptr};
    if (launch_search_generic(gs, ctx->stream) < 0)
        return fail(SNLS_ECONFIG, "search: window too large for the device search");
    return after_launch(ctx, launched + 1, "snls_search_grid");
}

int snls_topl(snls_ctx* ctx, int64_t rows, int cols, const float* full, const float* full_offsets,
              int topl, float* sel, float* sel_offsets) {
    if (int rc = check_ctx(ctx)) return rc;
    if (rows < 0 || cols < 1) return fail(SNLS_EDOMAIN, "top_l: similarity and offset shapes disagree");
    if (topl < 1 || topl > cols) return fail(SNLS_ECONFIG, "top_l: L out of range");
    if (rows == 0) return SNLS_OK;
    if (!full || !full_offsets || !sel || !sel_offsets) return fail(SNLS_EARG, "top_l: null tensor");
    DeviceGuard g(ctx->device);
    if (launch_topl(rows, cols, full, full_offsets, topl, sel, sel_offsets, ctx->err, ctx->stream) < 0)
        return fail(SNLS_ECONFIG, "top_l: row too long for the device selection");
    return after_launch(ctx, 1, "snls_topl");
}

int snls_replay(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* q,
                const float* k, const float* offsets, float* sims) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = validate(cfg)) return rc;
    if (int rc = check_dims(dims)) return rc;
    if (!q || !k || !offsets || !sims) return fail(SNLS_EARG, "replay_similarities: null tensor");
    DeviceGuard g(ctx->device);
    const Dims d = make_dims(dims, cfg->stride0);
    return after_launch(ctx, launch_replay(q, k, d, cfg->ps, cfg->metric, cfg->topl, offsets, sims, ctx->stream),
                        "snls_replay");
}

int snls_replay64(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                  const float* q, const float* k, const double* centers, int plan, float* sims) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = validate(cfg)) return rc;
    if (int rc = check_dims(dims)) return rc;
    if (!q || !k || !centers || !sims) return fail(SNLS_EARG, "replay_similarities: null tensor");
    if (int rc = check_aligned("replay_similarities", {q, k})) return rc;
    if (t0 < 0 || t1 > dims.t || t0 >= t1) return fail(SNLS_EARG, "replay_similarities: empty or invalid frame range");
    if (plan < -1 || plan > 2) return fail(SNLS_EARG, "replay_similarities: plan must be -1, 0, 1 or 2");
    DeviceGuard g(ctx->device);
    const Dims d = restrict_frames(make_dims(dims, cfg->stride0), t0, t1);
    if (plan == -1)  // the plan the forward takes for this configuration (snls_search_fwd)
        plan = (!ctx->force_generic && cfg->stride1 == 1.0) ? (ctx->search_kernel == 2 ? 2 : 1) : 0;
    TiledSearch ts{q, k, nullptr, nullptr, d, cfg->ws, cfg->wt, cfg->ps, cfg->topl, cfg->metric, 1.f,
                   nullptr, nullptr, nullptr, nullptr, ctx->err, ctx->num_sms, sims, ctx->search_kernel};
    ts.tape = centers;
    ts.d.rows = d.rows * cfg->topl;  // one replay "row" per selected entry
    int n = 0;
    if (plan == 2) {
        if (int rc = ensure_work(ctx, size_t(ts.d.rows) * cfg->ps * cfg->ps * sizeof(float))) return rc;
        ts.grid = static_cast<float*>(ctx->work);
        n = launch_replay_stream(ts, sims, ctx->stream);
        if (n == 0) plan = 1;  // not instantiated for this shape: the forward took the tiled plan
        ts.grid = sims;
    }
    if (plan == 1 && n == 0) {
        n = launch_replay_tiled(ts, ctx->stream);
        if (n == 0) plan = 0;  // the forward took the generic plan
    }
    if (plan == 0 && n == 0) n = launch_replay64(q, k, d, cfg->ps, cfg->metric, cfg->topl, centers, sims, ctx->stream);
    return after_launch(ctx, n, "snls_replay64");
}

int snls_search_bwd(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* grad,
                    const float* offsets, const float* chains, const float* q, const float* k,
                    float* dq, float* dk, float* dff, float* dbf) {
    return snls_search_bwd_frames(ctx, cfg, dims, 0, dims.t, grad, offsets, chains, q, k, dq, dk,
                                  dff, dbf);
}

int snls_search_bwd_frames(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                           const float* grad, const float* offsets, const float* chains,
                           const float* q, const float* k, float* dq, float* dk, float* dff,
                           float* dbf) {
    return snls_search_bwd_ex(ctx, cfg, dims, t0, t1, grad, offsets, chains, nullptr, nullptr, q, k,
                              dq, dk, dff, dbf, 0);
}

int snls_search_bwd_ex(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                       const float* grad, const float* offsets, const float* chains,
                       const double* centers, const double* chains64, const float* q,
                       const float* k, float* dq, float* dk, float* dff, float* dbf, int flags) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = validate(cfg)) return rc;
    if (int rc = check_dims(dims)) return rc;
    if (!grad || !q || !k || !dq || !dk || !dff || !dbf)
        return fail(SNLS_EARG, "shifted_nls_backward: null tensor");
    if (!offsets && !centers)
        return fail(SNLS_EARG, "shifted_nls_backward: the tape needs offsets or centres");
    if (cfg->wt > 1 && (centers ? chains64 == nullptr : chains == nullptr))
        return fail(SNLS_EARG, "shifted_nls_backward: the tape needs chains when wt > 1");
    if (t0 < 0 || t1 > dims.t || t0 >= t1)
        return fail(SNLS_EARG, "shifted_nls_backward: empty or invalid frame range");
    if (flags & ~SNLS_BWD_DETERMINISTIC) return fail(SNLS_EARG, "shifted_nls_backward: unknown flags");
    if (int rc = check_aligned("shifted_nls_backward", {q, k, dq, dk})) return rc;
    DeviceGuard g(ctx->device);
    const Dims d = restrict_frames(make_dims(dims, cfg->stride0), t0, t1);
    const size_t nv = size_t(dims.t) * dims.h * dims.w;
    cudaMemsetAsync(dq, 0, nv * dims.f * sizeof(float), ctx->stream);
    cudaMemsetAsync(dk, 0, nv * dims.f * sizeof(float), ctx->stream);
    const size_t scratch = (size_t(d.rows) * cfg->topl * 2 + nv * 4) * sizeof(double);
    if (flags & SNLS_BWD_DETERMINISTIC) {
        const int n = launch_search_bwd_det(grad, offsets, chains, centers, chains64, q, k, d, cfg->wt,
                                            cfg->ps, cfg->topl, cfg->metric, dq, dk, dff, dbf,
                                            [&](size_t bytes) -> void* {
                                                return ensure_work(ctx, bytes) ? nullptr : ctx->work;
                                            },
                                            ctx->stream);
        if (n < 0) return fail(SNLS_ECUDA, "shifted_nls_backward: deterministic workspace");
        return after_launch(ctx, n, "snls_search_bwd(deterministic)");
    }
    if (int rc = ensure_work(ctx, scratch)) return rc;
    cudaMemsetAsync(ctx->work, 0, scratch, ctx->stream);
    const int n = launch_search_bwd_impl(grad, offsets, chains, centers, chains64, q, k, d, cfg->wt,
                                         cfg->ps, cfg->topl, cfg->metric, dq, dk, dff, dbf,
                                         static_cast<double*>(ctx->work), ctx->stream);
    return after_launch(ctx, n, "snls_search_bwd");
}

int snls_search_tape64(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                       const float* ff, const float* bf, const float* offsets, double* centers,
                       double* chains64) {
    if (!centers) return fail(SNLS_EARG, "search_tape64: null tensor");
    return snls_search_results64(ctx, cfg, dims, t0, t1, ff, bf, nullptr, offsets, nullptr, nullptr,
                                 centers, chains64);
}

int snls_search_results64(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                          const float* ff, const float* bf, const float* sims, const float* offsets,
                          double* sims64, double* offsets64, double* centers, double* chains64) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = validate(cfg)) return rc;
    if (int rc = check_dims(dims)) return rc;
    if ((ff == nullptr) != (bf == nullptr))
        return fail(SNLS_EARG, "search: pass both flows or neither (nls_forward)");
    if (!offsets) return fail(SNLS_EARG, "search_results64: null offsets");
    if (sims64 && !sims) return fail(SNLS_EARG, "search_results64: sims64 needs sims");
    if (chains64 && cfg->wt <= 1) chains64 = nullptr;
    if (t0 < 0 || t1 > dims.t || t0 >= t1) return fail(SNLS_EARG, "search_results64: empty or invalid frame range");
    DeviceGuard g(ctx->device);
    const Dims d = restrict_frames(make_dims(dims, cfg->stride0), t0, t1);
    return after_launch(ctx,
                        launch_tape64(ff, bf, d, cfg->ws, cfg->wt, cfg->topl, cfg->stride1, offsets,
                                      centers, chains64, sims, sims64, offsets64, ctx->stream),
                        "snls_search_results64");
}

int snls_softmax_rows(snls_ctx* ctx, int64_t rows, int l, double beta, const float* sims, float* weights) {
    if (int rc = check_ctx(ctx)) return rc;
    if (rows < 0 || l < 1) return fail(SNLS_EDOMAIN, "softmax_rows: bad shape");
    if (rows == 0) return SNLS_OK;
    if (!sims || !weights) return fail(SNLS_EARG, "softmax_rows: null tensor");
    DeviceGuard g(ctx->device);
    return after_launch(ctx, launch_softmax(rows, l, float(beta), sims, weights, ctx->err, ctx->stream),
                        "snls_softmax_rows");
}

// check_agg_inputs (aggregate.cpp:47-66)
static int agg_checks(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* v,
                      const float* w, const float* o) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = validate(cfg)) return rc;
    if (!((cfg->ps - 1) / 2 < cfg->stride0))
        return fail(SNLS_ECONFIG, "aggregate: (ps-1)/2 < stride0 is required for hole-free output");
    if (int rc = check_dims(dims)) return rc;
    if (!v || !w || !o) return fail(SNLS_EARG, "aggregate: null tensor");
    return check_aligned("aggregate", {v, w, o});
}

int snls_wpsum_fwd(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* v,
                   const float* weights, const float* offsets, float* out, int32_t* counts) {
    return snls_wpsum_fwd_frames(ctx, cfg, dims, 0, dims.t, v, weights, offsets, out, counts);
}

int snls_wpsum_fwd_frames(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                          const float* v, const float* weights, const float* offsets, float* out,
                          int32_t* counts) {
    if (int rc = agg_checks(ctx, cfg, dims, v, weights, offsets)) return rc;
    if (!out) return fail(SNLS_EARG, "wpsum: null output");
    if (t0 < 0 || t1 > dims.t || t0 >= t1) return fail(SNLS_EARG, "wpsum: empty or invalid frame range");
    DeviceGuard g(ctx->device);
    AggArgs a{v, weights, offsets, restrict_frames(make_dims(dims, cfg->stride0), t0, t1), cfg->ps,
              cfg->topl, ctx->err, cfg->wt};
    return after_launch(ctx, launch_wpsum(a, out, counts, ctx->stream), "snls_wpsum_fwd");
}

int snls_gather_stack(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* v,
                      const float* weights, const float* offsets, float* out) {
    if (int rc = agg_checks(ctx, cfg, dims, v, weights, offsets)) return rc;
    if (!out) return fail(SNLS_EARG, "gather_stack: null output");
    DeviceGuard g(ctx->device);
    AggArgs a{v, weights, offsets, make_dims(dims, cfg->stride0), cfg->ps, cfg->topl, ctx->err, cfg->wt};
    return after_launch(ctx, launch_gather_stack(a, out, ctx->stream), "snls_gather_stack");
}

int snls_wpsum_bwd(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* grad_out,
                   const int32_t* counts, const float* v, const float* weights, const float* offsets,
                   float* dv, float* dw) {
    return snls_wpsum_bwd_frames(ctx, cfg, dims, 0, dims.t, grad_out, counts, v, weights, offsets,
                                 dv, dw);
}

int snls_wpsum_bwd_frames(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                          const float* grad_out, const int32_t* counts, const float* v,
                          const float* weights, const float* offsets, float* dv, float* dw) {
    return snls_wpsum_bwd_ex(ctx, cfg, dims, t0, t1, grad_out, counts, v, weights, offsets, dv, dw, 0);
}

int snls_wpsum_bwd_ex(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                      const float* grad_out, const int32_t* counts, const float* v,
                      const float* weights, const float* offsets, float* dv, float* dw, int flags) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = validate(cfg)) return rc;
    if (int rc = check_dims(dims)) return rc;
    if (!grad_out || !counts || !v || !weights || !offsets || !dv || !dw)
        return fail(SNLS_EARG, "wpsum_backward: null tensor");
    if (t0 < 0 || t1 > dims.t || t0 >= t1)
        return fail(SNLS_EARG, "wpsum_backward: empty or invalid frame range");
    if (flags & ~SNLS_BWD_DETERMINISTIC) return fail(SNLS_EARG, "wpsum_backward: unknown flags");
    if (int rc = check_aligned("wpsum_backward", {grad_out, v, weights, offsets, dv, dw})) return rc;
    DeviceGuard g(ctx->device);
    const Dims d = restrict_frames(make_dims(dims, cfg->stride0), t0, t1);
    cudaMemsetAsync(dv, 0, size_t(dims.t) * dims.h * dims.w * dims.f * sizeof(float), ctx->stream);
    cudaMemsetAsync(dw, 0, size_t(d.rows) * cfg->topl * sizeof(float), ctx->stream);
    AggArgs a{v, weights, offsets, d, cfg->ps, cfg->topl, ctx->err, cfg->wt};
    if (flags & SNLS_BWD_DETERMINISTIC) {
        const int n = launch_wpsum_bwd_det(a, grad_out, counts, dv, dw,
                                           [&](size_t bytes) -> void* {
                                               return ensure_work(ctx, bytes) ? nullptr : ctx->work;
                                           },
                                           ctx->stream);
        if (n < 0) return fail(SNLS_ECUDA, "wpsum_backward: deterministic workspace");
        return after_launch(ctx, n, "snls_wpsum_bwd(deterministic)");
    }
    return after_launch(ctx, launch_wpsum_bwd(a, grad_out, counts, dv, dw, ctx->stream), "snls_wpsum_bwd");
}

// ---- frame-alignment pieces (flow.cpp:114-175, tensor.cpp:79-99) ---------------------
int snls_block_match(snls_ctx* ctx, snls_dims dims, const float* a, const float* b, int block,
                     int radius, float* flow) {
    if (int rc = check_ctx(ctx)) return rc;
    if (block < 1 || block % 2 == 0)
        return fail(SNLS_ECONFIG, "estimate_flow_block_matching: block must be odd and positive");
    if (radius < 0) return fail(SNLS_ECONFIG, "estimate_flow_block_matching: radius must be >= 0");
    if (int rc = check_dims(dims)) return rc;
    if (!a || !b || !flow) return fail(SNLS_EARG, "estimate_flow_block_matching: null tensor");
    DeviceGuard g(ctx->device);
    const int n = launch_block_match(a, b, dims.t, dims.h, dims.w, dims.f, block, radius, flow, ctx->stream);
    if (n < 0) return fail(SNLS_ECONFIG, "estimate_flow_block_matching: block too large for the device");
    return after_launch(ctx, n, "snls_block_match");
}

int snls_psnr_frames(snls_ctx* ctx, snls_dims dims, const float* a, const float* b, double peak,
                     double* psnr_host) {
    if (int rc = check_ctx(ctx)) return rc;
    if (!(peak > 0.0)) return fail(SNLS_ECONFIG, "psnr: peak must be positive");
    if (int rc = check_dims(dims)) return rc;
    if (!a || !b || !psnr_host) return fail(SNLS_EARG, "psnr: null tensor");
    DeviceGuard g(ctx->device);
    const size_t nd = psnr_scratch_doubles(dims.t) + size_t(dims.t);
    if (int rc = ensure_work(ctx, nd * sizeof(double))) return rc;
    double* part = static_cast<double*>(ctx->work);
    double* out = part + psnr_scratch_doubles(dims.t);
    const int n = launch_psnr(a, b, dims.t, size_t(dims.h) * dims.w * dims.f, peak, part, out, ctx->stream);
    if (int rc = after_launch(ctx, n, "snls_psnr_frames")) return rc;
    cudaError_t e = cudaMemcpyAsync(psnr_host, out, size_t(dims.t) * sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "snls_psnr_frames");
    return SNLS_OK;
}

// GaussianStream (rng.hpp:30-53) + add_gaussian_noise (tensor.cpp:92-99) on the host, fp64
// like the reference, the result rounded to fp32.
int snls_gaussian_noise_f32(uint64_t seed, double sigma, int64_t n, const float* in, float* out) {
    if (sigma < 0.0) return fail(SNLS_ECONFIG, "add_gaussian_noise: sigma must be non-negative");
    if (n > 0 && (!in || !out)) return fail(SNLS_EARG, "add_gaussian_noise: null buffer");
    if (sigma == 0.0) {
        if (out != in) std::memcpy(out, in, size_t(n) * sizeof(float));
        return SNLS_OK;
    }
    uint64_t mt[312];
    mt[0] = seed;
    for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
    int idx = 312;
    auto next = [&]() {
        if (idx >= 312) {
            for (int j = 0; j < 312; ++j) {
                const uint64_t x = (mt[j] & 0xFFFFFFFF80000000ULL) | (mt[(j + 1) % 312] & 0x7FFFFFFFULL);
                uint64_t xa = x >> 1;
                if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
                mt[j] = mt[(j + 156) % 312] ^ xa;
            }
            idx = 0;
        }
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        return y;
    };
    const double kPi = 3.14159265358979323846;
    for (int64_t i = 0; i < n; i += 2) {
        const double u1 = (double(next() >> 11) + 1.0) * 0x1.0p-53;  // (0,1]
        const double u2 = double(next() >> 11) * 0x1.0p-53;          // [0,1)
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double ang = 2.0 * kPi * u2;
        out[i] = float(double(in[i]) + sigma * (r * std::cos(ang)));
        if (i + 1 < n) out[i + 1] = float(double(in[i + 1]) + sigma * (r * std::sin(ang)));
    }
    return SNLS_OK;
}

static int train_bwd_concurrent() {
    static const int on = [] {
        const char* e = std::getenv("SNLS_TRAIN_BWD_CONCURRENT");
        return e ? std::atoi(e) : 1;
    }();
    return on;
}

int snls_train_bwd(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* grad_sims,
                   const float* grad_out, const int32_t* counts, const float* offsets,
                   const float* chains, const double* centers, const double* chains64,
                   const float* q, const float* k, const float* v, const float* weights, float* dq,
                   float* dk, float* dv, float* dweights, float* dfflow, float* dbflow, int flags) {
    // the two operators (a single fused kernel for v == k was measured slower: 168 registers
    // and three shared-memory patches per warp, 12 warps/SM -- c3 backward 0.80 vs 0.585 ms,
    // profiles/r01_plans.txt).  Their outputs are disjoint, so the wpsum backward (bound by
    // its dV reductions through L2) runs on a second stream beside the search backward
    // (issue-bound); with aliased outputs they run one after the other.
    auto search = [&] {
        return snls_search_bwd_ex(ctx, cfg, dims, 0, dims.t, grad_sims, centers ? nullptr : offsets,
                                  centers ? nullptr : chains, centers, chains64, q, k, dq, dk, dfflow,
                                  dbflow, flags);
    };
    const bool disjoint = dv != dk && dv != dq && (void*)dweights != (void*)dk && (void*)dweights != (void*)dq;
    if (disjoint && (flags & ~SNLS_BWD_DETERMINISTIC) == 0 && ctx && cfg && train_bwd_interleavable(cfg->ps, dims.f)) {
        // one interleaved phase-1 launch (search_bwd.cu train_bwd_interleaved); the checks of
        // both operators first (snls_wpsum_bwd_frames, snls_search_bwd_ex)
        if (int rc = check_ctx(ctx)) return rc;
        if (int rc = validate(cfg)) return rc;
        if (int rc = check_dims(dims)) return rc;
        if (!grad_sims || !q || !k || !dq || !dk || !dfflow || !dbflow || !grad_out || !counts || !v ||
            !weights || !offsets || !dv || !dweights)
            return fail(SNLS_EARG, "train_backward: null tensor");
        if (cfg->wt > 1 && (centers ? chains64 == nullptr : chains == nullptr))
            return fail(SNLS_EARG, "shifted_nls_backward: the tape needs chains when wt > 1");
        if (int rc = check_aligned("train_backward", {q, k, v, dq, dk, grad_out, weights, offsets, dv, dweights}))
            return rc;
        DeviceGuard g(ctx->device);
        const Dims d = make_dims(dims, cfg->stride0);
        const size_t nv = size_t(dims.t) * dims.h * dims.w;
        cudaMemsetAsync(dq, 0, nv * dims.f * sizeof(float), ctx->stream);
        cudaMemsetAsync(dk, 0, nv * dims.f * sizeof(float), ctx->stream);
        cudaMemsetAsync(dv, 0, nv * dims.f * sizeof(float), ctx->stream);
        cudaMemsetAsync(dweights, 0, size_t(d.rows) * cfg->topl * sizeof(float), ctx->stream);
        if (flags & SNLS_BWD_DETERMINISTIC) {
            // both operators in fixed point, one interleaved phase-1 launch: the search
            // backward's workspace first, the wpsum backward's after it
            WpsumBwdArgs wp{AggArgs{v, weights, offsets, d, cfg->ps, cfg->topl, ctx->err, cfg->wt}, grad_out,
                            counts, dv, dweights, nullptr, nullptr, nullptr};
            const size_t wbytes = wpsum_bwd_det_bytes(wp.a);
            auto work = [&](size_t bytes) -> void* {
                const size_t head = (bytes + 255) & ~size_t(255);
                if (ensure_work(ctx, head + wbytes)) return nullptr;
                wpsum_bwd_det_prep(wp.a, grad_out, static_cast<char*>(ctx->work) + head, wp, ctx->stream);
                return ctx->work;
            };
            const int n = launch_search_bwd_det(grad_sims, centers ? nullptr : offsets, centers ? nullptr : chains,
                                                centers, chains64, q, k, d, cfg->wt, cfg->ps, cfg->topl,
                                                cfg->metric, dq, dk, dfflow, dbflow, work, ctx->stream, &wp);
            if (n < 0) return fail(SNLS_ECUDA, "train_backward: deterministic workspace");
            wpsum_bwd_det_finish(wp.a, wp, /*dw written directly by the channel-pair body*/ true, ctx->stream);
            return after_launch(ctx, n + 5, "snls_train_bwd(deterministic)");
        }
        const size_t scratch = (size_t(d.rows) * cfg->topl * 2 + nv * 4) * sizeof(double);
        if (int rc = ensure_work(ctx, scratch)) return rc;
        cudaMemsetAsync(ctx->work, 0, scratch, ctx->stream);
        const WpsumBwdArgs wp{AggArgs{v, weights, offsets, d, cfg->ps, cfg->topl, ctx->err, cfg->wt}, grad_out,
                              counts, dv, dweights};
        const int n = launch_train_bwd_interleaved(grad_sims, centers ? nullptr : offsets, centers ? nullptr : chains,
                                                   centers, chains64, q, k, d, cfg->wt, cfg->ps, cfg->topl,
                                                   cfg->metric, dq, dk, dfflow, dbflow,
                                                   static_cast<double*>(ctx->work), wp, ctx->stream);
        return after_launch(ctx, n, "snls_train_bwd");
    }
    // deterministic: both operators in fixed-point mode, one after the other (they share the
    // context's workspace)
    if (!disjoint || !train_bwd_concurrent() || (flags & SNLS_BWD_DETERMINISTIC)) {
        if (int rc = snls_wpsum_bwd_ex(ctx, cfg, dims, 0, dims.t, grad_out, counts, v, weights, offsets, dv,
                                       dweights, flags))
            return rc;
        return search();
    }
    if (int rc = check_ctx(ctx)) return rc;
    DeviceGuard g(ctx->device);
    if (!ctx->aux) {
        cudaError_t e = cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "snls_train_bwd: stream");
    }
    cudaStream_t main = ctx->stream;
    cudaEventRecord(ctx->fork, main);
    cudaStreamWaitEvent(ctx->aux, ctx->fork, 0);
    ctx->stream = ctx->aux;
    int rc = snls_wpsum_bwd(ctx, cfg, dims, grad_out, counts, v, weights, offsets, dv, dweights);
    ctx->stream = main;
    cudaEventRecord(ctx->join, ctx->aux);
    const int rs = rc == SNLS_OK ? search() : rc;
    cudaStreamWaitEvent(main, ctx->join, 0);  // (also on failure: nothing outlives the call)
    return rs;
}

}  // extern "C"
