// Host-buffer pipeline: search + fused softmax + wpsum over a whole clip from HOST memory,
// with the host->device input copies, the frame-chunked kernels and the device->host result
// copies overlapped on separate CUDA streams.
//
// This is the search -> softmax_rows -> wpsum core of the reference's align_frames /
// run_benchmark (harness.cpp:105-154, 242-283) as one native call over host buffers.  It is
// built only from the public C-ABI (snls_search_fwd_frames / snls_wpsum_fwd_frames, which
// run on the context's stream -- switched per chunk here) plus the CUDA runtime:
//
//   copy stream   : frame 0, 1, ..., T-1 of every distinct input (aliased Q = K = V copied
//                   once), one event per frame
//   compute [2]   : chunk [a, b) waits for the event of frame min(T, b + wt) - 1 (the last
//                   key/value frame its queries can reach, search.cpp:300; wpsum reads
//                   v at qt + dt, aggregate.cpp:108) and runs search + wpsum for the chunk's
//                   query frames; chunks alternate between two streams so one chunk's tail
//                   overlaps the next chunk's head
//   result stream : after chunk c, its sims / offsets / weights rows and out / counts frames
//
// The call is synchronous like the reference API: it returns when every result is in host
// memory and the device error latch has been checked.  Host buffers should be pinned
// (snls_host_register) for the copies to overlap; pageable buffers still work.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "snls_cuda.h"

namespace snls_capi {
int fail(int code, const std::string& msg);  // capi.cu: sets snls_last_error()
}

struct snls_pipeline {
    snls_ctx* ctx = nullptr;
    int device = 0;
    snls_config cfg{};
    snls_dims dims{};
    int chunk = 1;
    int64_t nq = 0;  // query rows per frame
    cudaStream_t copy = nullptr, result = nullptr, comp[2] = {nullptr, nullptr};
    cudaEvent_t start = nullptr, done_copy = nullptr, done_result = nullptr, done_comp[2] = {};
    std::vector<cudaEvent_t> frame_in, chunk_out;
    // device buffers
    float *q = nullptr, *k = nullptr, *v = nullptr, *ff = nullptr, *bf = nullptr;
    float *sims = nullptr, *offs = nullptr, *wts = nullptr, *out = nullptr;
    int32_t* counts = nullptr;
    int alias_key = -1;  // which of k / v alias q or k (decides the input buffers)
};

namespace {

int pfail(int code, const std::string& msg) { return snls_capi::fail(code, msg); }

int pcuda(cudaError_t e, const char* where) {
    return pfail(SNLS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

void free_buffers(snls_pipeline* p) {
    if (p->k == p->q) p->k = nullptr;  // aliased input buffers are freed once
    if (p->v == p->q || p->v == p->k) p->v = nullptr;
    float* fs[] = {p->q, p->k, p->v, p->ff, p->bf, p->sims, p->offs, p->wts, p->out};
    for (float* f : fs)
        if (f) cudaFree(f);
    if (p->counts) cudaFree(p->counts);
    p->q = p->k = p->v = p->ff = p->bf = p->sims = p->offs = p->wts = p->out = nullptr;
    p->counts = nullptr;
}

template <class T>
int alloc(T** ptr, size_t bytes, const char* what) {
    const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), bytes ? bytes : 4);
    if (e != cudaSuccess) return pcuda(e, what);
    return SNLS_OK;
}

}  // namespace

extern "C" {

int snls_host_register(void* ptr, uint64_t bytes) {
    if (!ptr || !bytes) return SNLS_OK;
    const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable);
    if (e != cudaSuccess && e != cudaErrorHostMemoryAlreadyRegistered) return pcuda(e, "snls_host_register");
    cudaGetLastError();
    return SNLS_OK;
}

int snls_host_unregister(void* ptr) {
    if (!ptr) return SNLS_OK;
    const cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess && e != cudaErrorHostMemoryNotRegistered) return pcuda(e, "snls_host_unregister");
    cudaGetLastError();
    return SNLS_OK;
}

int snls_pipeline_create(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int chunk_frames,
                         snls_pipeline** out) {
    if (!out) return pfail(SNLS_EARG, "snls_pipeline_create: null output");
    *out = nullptr;
    if (!ctx || !cfg) return pfail(SNLS_EARG, "snls_pipeline_create: null context or config");
    if (int rc = snls_validate_config(cfg)) return pfail(rc, snls_last_error());
    if (dims.t < 1 || dims.h < 1 || dims.w < 1 || dims.f < 1)
        return pfail(SNLS_EDOMAIN, "VideoTensor: all extents must be at least 1");
    int64_t rows = 0;
    int nh = 0, nw = 0;
    if (int rc = snls_query_grid(dims, cfg->stride0, &rows, &nh, &nw)) return pfail(rc, snls_last_error());
    int dev = 0;
    cudaGetDevice(&dev);
    auto* p = new snls_pipeline();
    p->ctx = ctx;
    p->device = dev;
    p->cfg = *cfg;
    p->dims = dims;
    p->nq = int64_t(nh) * nw;
    p->chunk = chunk_frames > 0 ? chunk_frames : 1;
    if (p->chunk > dims.t) p->chunk = dims.t;
    const int nchunks = (dims.t + p->chunk - 1) / p->chunk;
    cudaError_t e = cudaSuccess;
    auto mk_stream = [&](cudaStream_t* s) {
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    };
    auto mk_event = [&](cudaEvent_t* ev) {
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    };
    mk_stream(&p->copy);
    mk_stream(&p->result);
    mk_stream(&p->comp[0]);
    mk_stream(&p->comp[1]);
    mk_event(&p->start);
    mk_event(&p->done_copy);
    mk_event(&p->done_result);
    mk_event(&p->done_comp[0]);
    mk_event(&p->done_comp[1]);
    p->frame_in.assign(dims.t, nullptr);
    p->chunk_out.assign(nchunks, nullptr);
    for (auto& ev : p->frame_in) mk_event(&ev);
    for (auto& ev : p->chunk_out) mk_event(&ev);
    if (e != cudaSuccess) {
        snls_pipeline_destroy(p);
        return pcuda(e, "snls_pipeline_create");
    }
    const size_t vid = size_t(dims.t) * dims.h * dims.w * dims.f * sizeof(float);
    const size_t flw = size_t(dims.t) * dims.h * dims.w * 2 * sizeof(float);
    const size_t sel = size_t(rows) * cfg->topl * sizeof(float);
    int rc = SNLS_OK;
    if (!rc) rc = alloc(&p->q, vid, "snls_pipeline_create: q");
    if (!rc) rc = alloc(&p->ff, flw, "snls_pipeline_create: fflow");
    if (!rc) rc = alloc(&p->bf, flw, "snls_pipeline_create: bflow");
    if (!rc) rc = alloc(&p->sims, sel, "snls_pipeline_create: sims");
    if (!rc) rc = alloc(&p->offs, sel * 3, "snls_pipeline_create: offsets");
    if (!rc) rc = alloc(&p->wts, sel, "snls_pipeline_create: weights");
    if (!rc) rc = alloc(&p->out, vid, "snls_pipeline_create: out");
    if (!rc) rc = alloc(&p->counts, size_t(dims.t) * dims.h * dims.w * sizeof(int32_t), "snls_pipeline_create: counts");
    if (rc) {
        snls_pipeline_destroy(p);
        return rc;
    }
    *out = p;
    return SNLS_OK;
}

int snls_pipeline_destroy(snls_pipeline* p) {
    if (!p) return SNLS_OK;
    if (p->copy) cudaStreamSynchronize(p->copy);
    if (p->result) cudaStreamSynchronize(p->result);
    for (auto s : p->comp)
        if (s) cudaStreamSynchronize(s);
    free_buffers(p);
    for (auto ev : p->frame_in)
        if (ev) cudaEventDestroy(ev);
    for (auto ev : p->chunk_out)
        if (ev) cudaEventDestroy(ev);
    cudaEvent_t evs[] = {p->start, p->done_copy, p->done_result, p->done_comp[0], p->done_comp[1]};
    for (auto ev : evs)
        if (ev) cudaEventDestroy(ev);
    cudaStream_t ss[] = {p->copy, p->result, p->comp[0], p->comp[1]};
    for (auto s : ss)
        if (s) cudaStreamDestroy(s);
    delete p;
    return SNLS_OK;
}

// q, k, v: HOST T x H x W x F (k and/or v may alias q or each other: each distinct buffer
// is copied once); fflow, bflow: HOST T x H x W x 2 or both NULL (nls_forward).  Outputs
// (HOST, each may be NULL to skip its copy-back): sims rows x L, offsets rows x L x 3,
// weights rows x L, out T x H x W x F, counts T x H x W.  The whole call is ordered after
// the context's stream and joined back into it (record events on it to time the call).
int snls_pipeline_run(snls_pipeline* p, const float* q, const float* k,
                      const float* v, const float* fflow, const float* bflow, float* sims,
                      float* offsets, float* weights, float* out, int32_t* counts) {
    if (!p) return pfail(SNLS_EARG, "snls_pipeline_run: null pipeline");
    if (!q || !k || !v) return pfail(SNLS_EARG, "snls_pipeline_run: null video");
    if ((fflow == nullptr) != (bflow == nullptr))
        return pfail(SNLS_EARG, "snls_pipeline_run: pass both flows or neither");
    const snls_dims d = p->dims;
    const int T = d.t;
    const size_t frame = size_t(d.h) * d.w * d.f, fframe = size_t(d.h) * d.w * 2;
    const int key = (k == q ? 0 : (k == v ? 2 : 1)) * 4 + (v == q ? 0 : (v == k ? 1 : 2));
    if (key != p->alias_key) {  // (re)allocate the distinct input buffers
        if (p->k && p->k != p->q) cudaFree(p->k);
        if (p->v && p->v != p->q && p->v != p->k) cudaFree(p->v);
        p->k = p->v = nullptr;
        const size_t vid = size_t(T) * frame * sizeof(float);
        if (k == q) {
            p->k = p->q;
        } else if (int rc = alloc(&p->k, vid, "snls_pipeline_run: k")) {
            return rc;
        }
        if (v == q) {
            p->v = p->q;
        } else if (v == k) {
            p->v = p->k;
        } else if (int rc = alloc(&p->v, vid, "snls_pipeline_run: v")) {
            return rc;
        }
        p->alias_key = key;
    }
    void* user_stream = nullptr;
    snls_ctx_get_stream(p->ctx, &user_stream);
    cudaStream_t user = static_cast<cudaStream_t>(user_stream);
    cudaError_t e;
#define PCHECK(x, where)                                    \
    do {                                                    \
        if ((e = (x)) != cudaSuccess) return pcuda(e, where); \
    } while (0)
    // everything is ordered after the caller's stream
    PCHECK(cudaEventRecord(p->start, user), "snls_pipeline_run: start");
    cudaStream_t ss[] = {p->copy, p->result, p->comp[0], p->comp[1]};
    for (auto s : ss) PCHECK(cudaStreamWaitEvent(s, p->start, 0), "snls_pipeline_run: order");

    // ---- host -> device, frame by frame
    for (int t = 0; t < T; ++t) {
        const size_t o = size_t(t) * frame;
        PCHECK(cudaMemcpyAsync(p->q + o, q + o, frame * sizeof(float), cudaMemcpyHostToDevice, p->copy), "h2d q");
        if (p->k != p->q) PCHECK(cudaMemcpyAsync(p->k + o, k + o, frame * sizeof(float), cudaMemcpyHostToDevice, p->copy), "h2d k");
        if (p->v != p->q && p->v != p->k)
            PCHECK(cudaMemcpyAsync(p->v + o, v + o, frame * sizeof(float), cudaMemcpyHostToDevice, p->copy), "h2d v");
        if (fflow) {
            const size_t fo = size_t(t) * fframe;
            PCHECK(cudaMemcpyAsync(p->ff + fo, fflow + fo, fframe * sizeof(float), cudaMemcpyHostToDevice, p->copy), "h2d fflow");
            PCHECK(cudaMemcpyAsync(p->bf + fo, bflow + fo, fframe * sizeof(float), cudaMemcpyHostToDevice, p->copy), "h2d bflow");
        }
        PCHECK(cudaEventRecord(p->frame_in[t], p->copy), "h2d event");
    }

    // ---- frame chunks: search (+ fused softmax) and wpsum, then their copy-back
    const int L = p->cfg.topl;
    const int nchunks = (T + p->chunk - 1) / p->chunk;
    int rc = SNLS_OK;
    for (int c = 0; c < nchunks && rc == SNLS_OK; ++c) {
        const int a = c * p->chunk, b = (a + p->chunk < T) ? a + p->chunk : T;
        const int need = (b + p->cfg.wt < T ? b + p->cfg.wt : T) - 1;
        cudaStream_t cs = p->comp[c & 1];
        PCHECK(cudaStreamWaitEvent(cs, p->frame_in[need], 0), "chunk wait");
        snls_ctx_set_stream(p->ctx, cs);
        const int64_t r0 = int64_t(a) * p->nq;
        rc = snls_search_fwd_frames(p->ctx, &p->cfg, d, a, b, p->q, p->k, fflow ? p->ff : nullptr,
                                    fflow ? p->bf : nullptr, SNLS_MODE_FUSED, p->sims + r0 * L,
                                    p->offs + r0 * L * 3, nullptr, p->wts + r0 * L);
        if (rc == SNLS_OK)
            rc = snls_wpsum_fwd_frames(p->ctx, &p->cfg, d, a, b, p->v, p->wts + r0 * L, p->offs + r0 * L * 3,
                                       p->out + size_t(a) * frame, p->counts + size_t(a) * d.h * d.w);
        if (rc != SNLS_OK) {
            pfail(rc, snls_last_error());
            break;
        }
        PCHECK(cudaEventRecord(p->chunk_out[c], cs), "chunk event");
        PCHECK(cudaStreamWaitEvent(p->result, p->chunk_out[c], 0), "result wait");
        const int64_t nr = int64_t(b - a) * p->nq;
        if (sims) PCHECK(cudaMemcpyAsync(sims + r0 * L, p->sims + r0 * L, nr * L * sizeof(float), cudaMemcpyDeviceToHost, p->result), "d2h sims");
        if (offsets) PCHECK(cudaMemcpyAsync(offsets + r0 * L * 3, p->offs + r0 * L * 3, nr * L * 3 * sizeof(float), cudaMemcpyDeviceToHost, p->result), "d2h offsets");
        if (weights) PCHECK(cudaMemcpyAsync(weights + r0 * L, p->wts + r0 * L, nr * L * sizeof(float), cudaMemcpyDeviceToHost, p->result), "d2h weights");
        if (out) PCHECK(cudaMemcpyAsync(out + size_t(a) * frame, p->out + size_t(a) * frame, size_t(b - a) * frame * sizeof(float), cudaMemcpyDeviceToHost, p->result), "d2h out");
        if (counts) PCHECK(cudaMemcpyAsync(counts + size_t(a) * d.h * d.w, p->counts + size_t(a) * d.h * d.w, size_t(b - a) * d.h * d.w * sizeof(int32_t), cudaMemcpyDeviceToHost, p->result), "d2h counts");
    }
    // ---- join everything back into the caller's stream, then report
    PCHECK(cudaEventRecord(p->done_copy, p->copy), "join");
    PCHECK(cudaEventRecord(p->done_result, p->result), "join");
    PCHECK(cudaEventRecord(p->done_comp[0], p->comp[0]), "join");
    PCHECK(cudaEventRecord(p->done_comp[1], p->comp[1]), "join");
    cudaEvent_t joins[] = {p->done_copy, p->done_result, p->done_comp[0], p->done_comp[1]};
    for (auto ev : joins) PCHECK(cudaStreamWaitEvent(user, ev, 0), "join");
    snls_ctx_set_stream(p->ctx, user);
#undef PCHECK
    if (rc != SNLS_OK) {
        cudaStreamSynchronize(user);
        return rc;
    }
    // synchronises the caller's stream; latched device-side domain errors surface here
    if (int r = snls_ctx_sync_check(p->ctx)) return pfail(r, snls_last_error());
    return SNLS_OK;
}

}  // extern "C"
