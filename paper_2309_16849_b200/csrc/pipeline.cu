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
// snls_pipeline_run is synchronous like the reference API: it returns when every result is
// in host memory and the device error latch has been checked.  snls_pipeline_submit /
// snls_pipeline_wait stream clips: up to kSlots = 3 clips in flight on three buffer slots, so
// the next clip's H2D overlaps this clip's compute and this clip's D2H tail overlaps the next
// clip's head.  With two slots the H2D of clip n+2 had to wait for the D2H of clip n (same
// buffers), which made the period (C + D2H + H2D) / 2 whenever the transfers outlast the
// compute C (c4: 5.08 ms per clip vs 4.66 ms of compute); a third slot decouples them.  Host buffers should be pinned (snls_host_register) for the copies to
// overlap; pageable buffers still work.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "snls_cuda.h"

namespace snls_capi {
int fail(int code, const std::string& msg);  // capi.cu: sets snls_last_error()
int* ctx_err(snls_ctx* ctx);                 // capi.cu: the context's device error latch
int ctx_device(snls_ctx* ctx);               // capi.cu: the context's device
}

#ifndef SNLS_D2H_AFTER_H2D
#define SNLS_D2H_AFTER_H2D 1
#endif
constexpr bool kD2HAfterH2D = SNLS_D2H_AFTER_H2D != 0;

// One set of device buffers and events: a clip in flight.
struct PipeSlot {
    float *q = nullptr, *k = nullptr, *v = nullptr, *ff = nullptr, *bf = nullptr;
    float *sims = nullptr, *offs = nullptr, *wts = nullptr, *out = nullptr;
    int32_t* counts = nullptr;
    int alias_key = -1;  // which of k / v alias q or k (decides the input buffers)
    std::vector<cudaEvent_t> frame_in, chunk_out;
    cudaEvent_t done = nullptr;
    bool allocated = false, busy = false;
    // pinned snapshot of the context's error latch, copied on the result stream after the
    // clip's results: wait() reads it without a blocking device read of its own (which would
    // queue behind the next clip's D2H on the copy engine and stall the stream)
    int* err_snap = nullptr;
    // SNLS_PIPE_TRACE=1: timing events (submit, H2D done, compute start/end, D2H done)
    cudaEvent_t tr[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    int clip = -1;
};

struct snls_pipeline {
    snls_ctx* ctx = nullptr;
    int device = 0;
    snls_config cfg{};
    snls_dims dims{};
    int chunk = 1;
    int64_t nq = 0, rows = 0;  // query rows per frame, per clip
    cudaStream_t copy = nullptr, result = nullptr, comp[2] = {nullptr, nullptr};
    cudaEvent_t start = nullptr;
    bool trace = false;
    cudaEvent_t trace0 = nullptr;
    int nsubmit = 0;
    static constexpr int kSlots = 3;
    PipeSlot slot[kSlots];
    int next = 0;          // slot of the next submit
    int pending[kSlots];   // FIFO of in-flight slots
    int npending = 0;
};

namespace {

int pfail(int code, const std::string& msg) { return snls_capi::fail(code, msg); }

// Every entry point runs on the context's device: streams, events and buffers are created
// there and the chunk kernels (DeviceGuard'ed in capi.cu) launch there.
struct PipeDevice {
    int prev = -1;
    explicit PipeDevice(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~PipeDevice() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int pcuda(cudaError_t e, const char* where) {
    return pfail(SNLS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

template <class T>
int alloc(T** ptr, size_t bytes, const char* what) {
    const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), bytes ? bytes : 4);
    if (e != cudaSuccess) return pcuda(e, what);
    return SNLS_OK;
}

void free_slot(PipeSlot& s) {
    if (s.k == s.q) s.k = nullptr;  // aliased input buffers are freed once
    if (s.v == s.q || s.v == s.k) s.v = nullptr;
    float* fs[] = {s.q, s.k, s.v, s.ff, s.bf, s.sims, s.offs, s.wts, s.out};
    for (float* f : fs)
        if (f) cudaFree(f);
    if (s.counts) cudaFree(s.counts);
    if (s.err_snap) cudaFreeHost(s.err_snap);
    s.err_snap = nullptr;
    for (auto& ev : s.tr) {
        if (ev) cudaEventDestroy(ev);
        ev = nullptr;
    }
    s.q = s.k = s.v = s.ff = s.bf = s.sims = s.offs = s.wts = s.out = nullptr;
    s.counts = nullptr;
    for (auto ev : s.frame_in)
        if (ev) cudaEventDestroy(ev);
    for (auto ev : s.chunk_out)
        if (ev) cudaEventDestroy(ev);
    if (s.done) cudaEventDestroy(s.done);
    s.frame_in.clear();
    s.chunk_out.clear();
    s.done = nullptr;
    s.allocated = false;
}

int alloc_slot(snls_pipeline* p, PipeSlot& s) {
    const snls_dims d = p->dims;
    const int nchunks = (d.t + p->chunk - 1) / p->chunk;
    cudaError_t e = cudaSuccess;
    auto mk_event = [&](cudaEvent_t* ev) {
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    };
    s.frame_in.assign(d.t, nullptr);
    s.chunk_out.assign(nchunks, nullptr);
    for (auto& ev : s.frame_in) mk_event(&ev);
    for (auto& ev : s.chunk_out) mk_event(&ev);
    mk_event(&s.done);
    if (e != cudaSuccess) return pcuda(e, "snls_pipeline: events");
    const size_t vid = size_t(d.t) * d.h * d.w * d.f * sizeof(float);
    const size_t flw = size_t(d.t) * d.h * d.w * 2 * sizeof(float);
    const size_t sel = size_t(p->rows) * p->cfg.topl * sizeof(float);
    int rc = SNLS_OK;
    if (!rc) rc = alloc(&s.q, vid, "snls_pipeline: q");
    if (!rc) rc = alloc(&s.ff, flw, "snls_pipeline: fflow");
    if (!rc) rc = alloc(&s.bf, flw, "snls_pipeline: bflow");
    if (!rc) rc = alloc(&s.sims, sel, "snls_pipeline: sims");
    if (!rc) rc = alloc(&s.offs, sel * 3, "snls_pipeline: offsets");
    if (!rc) rc = alloc(&s.wts, sel, "snls_pipeline: weights");
    if (!rc) rc = alloc(&s.out, vid, "snls_pipeline: out");
    if (!rc) rc = alloc(&s.counts, size_t(d.t) * d.h * d.w * sizeof(int32_t), "snls_pipeline: counts");
    if (!rc) {
        const cudaError_t he = cudaHostAlloc(reinterpret_cast<void**>(&s.err_snap), sizeof(int), cudaHostAllocDefault);
        if (he != cudaSuccess) rc = pcuda(he, "snls_pipeline: error snapshot");
        else *s.err_snap = 0;
    }
    if (rc == SNLS_OK) s.allocated = true;
    return rc;
}

// Block until the oldest in-flight clip is done; report its (or an earlier-latched)
// device-side domain error.
int wait_oldest(snls_pipeline* p) {
    if (p->npending == 0) return SNLS_OK;
    PipeSlot& s = p->slot[p->pending[0]];
    for (int i = 0; i + 1 < p->npending; ++i) p->pending[i] = p->pending[i + 1];
    --p->npending;
    const cudaError_t e = cudaEventSynchronize(s.done);
    s.busy = false;
    if (e != cudaSuccess) return pcuda(e, "snls_pipeline_wait");
    if (p->trace && s.tr[0]) {
        float t[5];
        for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], p->trace0, s.tr[i]);
        std::fprintf(stderr, "clip %d: enq %.3f h2d_done %.3f comp %.3f-%.3f d2h_done %.3f\n", s.clip, t[0], t[1],
                     t[2], t[3], t[4]);
    }
    // the latch is per context: an error of a clip still in flight may surface one wait
    // early, never later or not at all.  The full check (message, reset) runs only when the
    // clip's snapshot of the latch is set.
    if (*s.err_snap != 0)
        if (int r = snls_ctx_sync_check(p->ctx)) return pfail(r, snls_last_error());
    return SNLS_OK;
}

// Enqueue one clip on slot `si` (see the file comment for the stream graph).
int enqueue(snls_pipeline* p, int si, const float* q, const float* k, const float* v,
            const float* fflow, const float* bflow, float* sims, float* offsets, float* weights,
            float* out, int32_t* counts) {
    PipeSlot& S = p->slot[si];
    const snls_dims d = p->dims;
    const int T = d.t;
    const size_t frame = size_t(d.h) * d.w * d.f, fframe = size_t(d.h) * d.w * 2;
    const int key = (k == q ? 0 : (k == v ? 2 : 1)) * 4 + (v == q ? 0 : (v == k ? 1 : 2));
    if (key != S.alias_key) {  // (re)allocate the distinct input buffers
        if (S.k && S.k != S.q) cudaFree(S.k);
        if (S.v && S.v != S.q && S.v != S.k) cudaFree(S.v);
        S.k = S.v = nullptr;
        const size_t vid = size_t(T) * frame * sizeof(float);
        if (k == q) {
            S.k = S.q;
        } else if (int rc = alloc(&S.k, vid, "snls_pipeline: k")) {
            return rc;
        }
        if (v == q) {
            S.v = S.q;
        } else if (v == k) {
            S.v = S.k;
        } else if (int rc = alloc(&S.v, vid, "snls_pipeline: v")) {
            return rc;
        }
        S.alias_key = key;
    }
    void* user_stream = nullptr;
    snls_ctx_get_stream(p->ctx, &user_stream);
    cudaStream_t user = static_cast<cudaStream_t>(user_stream);
    cudaError_t e;
#define PCHECK(x, where)                                      \
    do {                                                      \
        if ((e = (x)) != cudaSuccess) return pcuda(e, where); \
    } while (0)
    // everything is ordered after the caller's stream
    PCHECK(cudaEventRecord(p->start, user), "snls_pipeline: start");
    cudaStream_t ss[] = {p->copy, p->result, p->comp[0], p->comp[1]};
    for (auto s : ss) PCHECK(cudaStreamWaitEvent(s, p->start, 0), "snls_pipeline: order");
    if (p->trace) {
        if (!S.tr[0])
            for (auto& ev : S.tr) cudaEventCreate(&ev);
        S.clip = p->nsubmit++;
        cudaEventRecord(S.tr[0], p->copy);
    }

    // ---- host -> device, one copy per tensor per chunk's new frames [t0, t1) (frames up to
    // the last key/value frame the chunk can reach), videos first: an H2D command queued
    // behind an in-flight D2H waits for it, so fewer, larger copies overlap the previous
    // clip's copy-back (c2: 15 per-frame copies 0.84 ms vs 3 copies 0.58 ms next to a D2H)
    {
        const int nch = (T + p->chunk - 1) / p->chunk;
        int t0 = 0;
        for (int c = 0; c < nch && t0 < T; ++c) {
            const int b = (c + 1) * p->chunk < T ? (c + 1) * p->chunk : T;
            const int t1 = b + p->cfg.wt < T ? b + p->cfg.wt : T;
            if (t1 <= t0) continue;
            const size_t o = size_t(t0) * frame, n = size_t(t1 - t0) * frame * sizeof(float);
            PCHECK(cudaMemcpyAsync(S.q + o, q + o, n, cudaMemcpyHostToDevice, p->copy), "h2d q");
            if (S.k != S.q) PCHECK(cudaMemcpyAsync(S.k + o, k + o, n, cudaMemcpyHostToDevice, p->copy), "h2d k");
            if (S.v != S.q && S.v != S.k)
                PCHECK(cudaMemcpyAsync(S.v + o, v + o, n, cudaMemcpyHostToDevice, p->copy), "h2d v");
            if (fflow) {
                const size_t fo = size_t(t0) * fframe, fn = size_t(t1 - t0) * fframe * sizeof(float);
                PCHECK(cudaMemcpyAsync(S.ff + fo, fflow + fo, fn, cudaMemcpyHostToDevice, p->copy), "h2d fflow");
                PCHECK(cudaMemcpyAsync(S.bf + fo, bflow + fo, fn, cudaMemcpyHostToDevice, p->copy), "h2d bflow");
            }
            PCHECK(cudaEventRecord(S.frame_in[t1 - 1], p->copy), "h2d event");
            t0 = t1;
        }
    }
    if (p->trace) cudaEventRecord(S.tr[1], p->copy);

    // the copy-back starts after the clip's last H2D: a D2H command in flight would hold up
    // the H2D commands queued behind it (the same copy-engine ordering as above)
    if (kD2HAfterH2D) PCHECK(cudaStreamWaitEvent(p->result, S.frame_in[T - 1], 0), "result order");

    // ---- frame chunks: search (+ fused softmax) and wpsum, then their copy-back
    const int L = p->cfg.topl;
    const int nchunks = (T + p->chunk - 1) / p->chunk;
    int rc = SNLS_OK;
    for (int c = 0; c < nchunks && rc == SNLS_OK; ++c) {
        const int a = c * p->chunk, b = (a + p->chunk < T) ? a + p->chunk : T;
        const int need = (b + p->cfg.wt < T ? b + p->cfg.wt : T) - 1;
        cudaStream_t cs = p->comp[c & 1];
        PCHECK(cudaStreamWaitEvent(cs, S.frame_in[need], 0), "chunk wait");
        if (p->trace && c == 0) cudaEventRecord(S.tr[2], cs);
        snls_ctx_set_stream(p->ctx, cs);
        const int64_t r0 = int64_t(a) * p->nq;
        rc = snls_search_fwd_frames(p->ctx, &p->cfg, d, a, b, S.q, S.k, fflow ? S.ff : nullptr,
                                    fflow ? S.bf : nullptr, SNLS_MODE_FUSED, S.sims + r0 * L,
                                    S.offs + r0 * L * 3, nullptr, S.wts + r0 * L);
        if (rc == SNLS_OK)
            rc = snls_wpsum_fwd_frames(p->ctx, &p->cfg, d, a, b, S.v, S.wts + r0 * L, S.offs + r0 * L * 3,
                                       S.out + size_t(a) * frame, S.counts + size_t(a) * d.h * d.w);
        if (rc != SNLS_OK) {
            pfail(rc, snls_last_error());
            break;
        }
        PCHECK(cudaEventRecord(S.chunk_out[c], cs), "chunk event");
        if (p->trace && c == nchunks - 1) cudaEventRecord(S.tr[3], cs);
        PCHECK(cudaStreamWaitEvent(p->result, S.chunk_out[c], 0), "result wait");
        const int64_t nr = int64_t(b - a) * p->nq;
        if (sims) PCHECK(cudaMemcpyAsync(sims + r0 * L, S.sims + r0 * L, nr * L * sizeof(float), cudaMemcpyDeviceToHost, p->result), "d2h sims");
        if (offsets) PCHECK(cudaMemcpyAsync(offsets + r0 * L * 3, S.offs + r0 * L * 3, nr * L * 3 * sizeof(float), cudaMemcpyDeviceToHost, p->result), "d2h offsets");
        if (weights) PCHECK(cudaMemcpyAsync(weights + r0 * L, S.wts + r0 * L, nr * L * sizeof(float), cudaMemcpyDeviceToHost, p->result), "d2h weights");
        if (out) PCHECK(cudaMemcpyAsync(out + size_t(a) * frame, S.out + size_t(a) * frame, size_t(b - a) * frame * sizeof(float), cudaMemcpyDeviceToHost, p->result), "d2h out");
        if (counts) PCHECK(cudaMemcpyAsync(counts + size_t(a) * d.h * d.w, S.counts + size_t(a) * d.h * d.w, size_t(b - a) * d.h * d.w * sizeof(int32_t), cudaMemcpyDeviceToHost, p->result), "d2h counts");
    }
    snls_ctx_set_stream(p->ctx, user);
    // the result stream waited for every chunk: its latch snapshot and `done` cover the clip
    PCHECK(cudaMemcpyAsync(S.err_snap, snls_capi::ctx_err(p->ctx), sizeof(int), cudaMemcpyDeviceToHost,
                           p->result), "error snapshot");
    PCHECK(cudaEventRecord(S.done, p->result), "done event");
    if (p->trace) cudaEventRecord(S.tr[4], p->result);
#undef PCHECK
    return rc;
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
    const int dev = snls_capi::ctx_device(ctx);
    PipeDevice guard(dev);
    auto* p = new snls_pipeline();
    p->ctx = ctx;
    p->device = dev;
    p->cfg = *cfg;
    p->dims = dims;
    p->nq = int64_t(nh) * nw;
    p->rows = rows;
    p->chunk = chunk_frames > 0 ? chunk_frames : 1;
    if (p->chunk > dims.t) p->chunk = dims.t;
    cudaError_t e = cudaSuccess;
    auto mk_stream = [&](cudaStream_t* s) {
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    };
    mk_stream(&p->copy);
    mk_stream(&p->result);
    mk_stream(&p->comp[0]);
    mk_stream(&p->comp[1]);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->start, cudaEventDisableTiming);
    {
        const char* tr = std::getenv("SNLS_PIPE_TRACE");
        p->trace = tr && tr[0] == '1';
        if (p->trace && e == cudaSuccess) {
            e = cudaEventCreate(&p->trace0);
            if (e == cudaSuccess) e = cudaEventRecord(p->trace0, 0);
        }
    }
    if (e != cudaSuccess) {
        snls_pipeline_destroy(p);
        return pcuda(e, "snls_pipeline_create");
    }
    if (int rc = alloc_slot(p, p->slot[0])) {  // the other slots are allocated on first use
        snls_pipeline_destroy(p);
        return rc;
    }
    *out = p;
    return SNLS_OK;
}

int snls_pipeline_destroy(snls_pipeline* p) {
    if (!p) return SNLS_OK;
    PipeDevice guard(p->device);
    cudaStream_t ss[] = {p->copy, p->result, p->comp[0], p->comp[1]};
    for (auto s : ss)
        if (s) cudaStreamSynchronize(s);
    for (auto& sl : p->slot) free_slot(sl);
    if (p->start) cudaEventDestroy(p->start);
    for (auto s : ss)
        if (s) cudaStreamDestroy(s);
    delete p;
    return SNLS_OK;
}

// Streaming form: enqueue a clip and return (at most kSlots in flight: one more submit first
// waits for the oldest).  Host buffers must stay untouched until the matching wait.
int snls_pipeline_submit(snls_pipeline* p, const float* q, const float* k, const float* v,
                         const float* fflow, const float* bflow, float* sims, float* offsets,
                         float* weights, float* out, int32_t* counts) {
    if (!p) return pfail(SNLS_EARG, "snls_pipeline_submit: null pipeline");
    if (!q || !k || !v) return pfail(SNLS_EARG, "snls_pipeline_submit: null video");
    if ((fflow == nullptr) != (bflow == nullptr))
        return pfail(SNLS_EARG, "snls_pipeline_submit: pass both flows or neither");
    PipeDevice guard(p->device);
    const int si = p->next;
    PipeSlot& S = p->slot[si];
    if (S.busy)
        if (int rc = wait_oldest(p)) return rc;
    if (!S.allocated)
        if (int rc = alloc_slot(p, S)) return rc;
    const int rc = enqueue(p, si, q, k, v, fflow, bflow, sims, offsets, weights, out, counts);
    S.busy = true;
    p->pending[p->npending++] = si;
    p->next = (si + 1) % snls_pipeline::kSlots;
    if (rc != SNLS_OK) {
        const std::string msg = snls_last_error();
        while (p->npending) wait_oldest(p);
        return pfail(rc, msg);
    }
    return SNLS_OK;
}

// Wait for the oldest submitted clip: its results are in host memory afterwards.
int snls_pipeline_wait(snls_pipeline* p) {
    if (!p) return pfail(SNLS_EARG, "snls_pipeline_wait: null pipeline");
    PipeDevice guard(p->device);
    return wait_oldest(p);
}

// q, k, v: HOST T x H x W x F (k and/or v may alias q or each other: each distinct buffer
// is copied once); fflow, bflow: HOST T x H x W x 2 or both NULL (nls_forward).  Outputs
// (HOST, each may be NULL to skip its copy-back): sims rows x L, offsets rows x L x 3,
// weights rows x L, out T x H x W x F, counts T x H x W.  Synchronous: returns when the
// results are in host memory; the work is joined back into the context's stream, so
// events recorded on it around the call time the whole clip.
int snls_pipeline_run(snls_pipeline* p, const float* q, const float* k, const float* v,
                      const float* fflow, const float* bflow, float* sims, float* offsets,
                      float* weights, float* out, int32_t* counts) {
    if (!p) return pfail(SNLS_EARG, "snls_pipeline_run: null pipeline");
    PipeDevice guard(p->device);
    while (p->npending)  // drain any streamed clips first
        if (int rc = wait_oldest(p)) return rc;
    if (int rc = snls_pipeline_submit(p, q, k, v, fflow, bflow, sims, offsets, weights, out, counts))
        return rc;
    void* user_stream = nullptr;
    snls_ctx_get_stream(p->ctx, &user_stream);
    const int last = p->pending[p->npending - 1];
    cudaStreamWaitEvent(static_cast<cudaStream_t>(user_stream), p->slot[last].done, 0);
    return wait_oldest(p);
}

}  // extern "C"
