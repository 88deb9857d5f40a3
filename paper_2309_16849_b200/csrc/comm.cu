// Frame sharding of one video across GPUs (BASELINE configs[4]) on raw
// NCCL, behind the C-ABI: the shard plan, the forward wt-frame halo exchange and the
// backward's reverse halo (partial gradients of halo frames sent back to their owners and
// added).  No PyTorch on this path; a C++ caller of the drop-in can shard frames with it.
//
// A query at frame t reads key/value frames t-wt .. t+wt and the flow frames in between
// (search.cpp:84-101, 300) and wpsum writes only into the query's own frame
// (aggregate.cpp:197-198), so rank r owns query frames [a, b) and holds the slab
// [lo, hi) = [a-wt, b+wt) n [0, T): the halo frames come from their owners by point-to-point
// ncclSend / ncclRecv inside one ncclGroupStart/End on the communicator's stream, ordered
// after the context's stream by an event and joined back into it by another -- the caller
// enqueues the interior frames (which need no halo) in between, so the transfer overlaps them.
//
// NCCL is loaded at snls_comm_init time (dlopen "libnccl.so.2": the one the process already
// has, e.g. torch's, else the system's), so the library itself has no link-time NCCL
// dependency and every other entry point works without it.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

#include "common.cuh"
#include "snls_cuda.h"

namespace snls_capi {
int fail(int code, const std::string& msg);
int ctx_device(snls_ctx* ctx);
}

namespace {

using snls_capi::fail;

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    bool ok = false;
    std::string why;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("NCCL not loadable: ") + dlerror();
            return;
        }
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            return f != nullptr;
        };
        n.ok = sym(n.GetUniqueId, "ncclGetUniqueId") && sym(n.CommInitRank, "ncclCommInitRank") &&
               sym(n.CommDestroy, "ncclCommDestroy") && sym(n.CommCount, "ncclCommCount") &&
               sym(n.Send, "ncclSend") && sym(n.Recv, "ncclRecv") && sym(n.GroupStart, "ncclGroupStart") &&
               sym(n.GroupEnd, "ncclGroupEnd") && sym(n.GetErrorString, "ncclGetErrorString") &&
               sym(n.GetVersion, "ncclGetVersion");
        if (!n.ok) n.why = "NCCL library lacks a required symbol";
    });
    return n;
}

int nfail(ncclResult_t r, const char* where) {
    return fail(SNLS_ECUDA, std::string(where) + ": " + nccl().GetErrorString(r));
}

// ---- the shard plan (host only; mirrors paper_2309_16849_b200/shard.py) --------------------
void owned_range(int T, int world, int rank, int& a, int& b) {
    const int per = T / world, rem = T % world;
    a = rank * per + (rank < rem ? rank : rem);
    b = a + per + (rank < rem ? 1 : 0);
}

struct Plan {
    int a, b, lo, hi;
};

Plan make_plan(int T, int world, int rank, int wt) {
    Plan p;
    owned_range(T, world, rank, p.a, p.b);
    p.lo = p.a - wt > 0 ? p.a - wt : 0;
    p.hi = p.b + wt < T ? p.b + wt : T;
    return p;
}

struct Transfer {
    int peer, lo, hi, recv;  // recv: 1 = frames [lo, hi) come from peer; 0 = go to peer
};

// Peers in ascending order, receive before send per peer (the same order on every rank, so
// the grouped calls pair up): a peer's frames inside my slab are received, my frames inside
// a peer's slab are sent.  Any shard length (a halo may span several owners).
std::vector<Transfer> transfers(int T, int world, int rank, int wt) {
    std::vector<Transfer> out;
    const Plan me = make_plan(T, world, rank, wt);
    for (int peer = 0; peer < world; ++peer) {
        if (peer == rank) continue;
        int pa, pb;
        owned_range(T, world, peer, pa, pb);
        int lo = me.lo > pa ? me.lo : pa, hi = me.hi < pb ? me.hi : pb;
        if (lo < hi) out.push_back({peer, lo, hi, 1});
        const Plan q = make_plan(T, world, peer, wt);
        lo = q.lo > me.a ? q.lo : me.a;
        hi = q.hi < me.b ? q.hi : me.b;
        if (lo < hi) out.push_back({peer, lo, hi, 0});
    }
    return out;
}

int check_plan_args(int T, int world, int rank, int wt) {
    if (world < 1 || rank < 0 || rank >= world) return fail(SNLS_EARG, "shard: bad rank / world");
    if (T < 1 || wt < 0) return fail(SNLS_EARG, "shard: bad T / wt");
    if (world > T) return fail(SNLS_ECONFIG, "frame sharding needs at least one frame per rank");
    return SNLS_OK;
}

__global__ void add_kernel(float* __restrict__ dst, const float* __restrict__ src, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        dst[i] += src[i];
}

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DevGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace

struct snls_comm {
    snls_ctx* ctx = nullptr;
    int device = 0, rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;  // the communicator's stream
    cudaEvent_t ready = nullptr, done = nullptr;
    void* scratch = nullptr;  // reverse-halo receive buffer
    size_t scratch_bytes = 0;
    bool pending = false;  // an exchange was started and not yet joined
};

extern "C" {

int snls_shard_plan(int T, int world, int rank, int wt, int* out4) {
    if (int rc = check_plan_args(T, world, rank, wt)) return rc;
    if (!out4) return fail(SNLS_EARG, "snls_shard_plan: null output");
    const Plan p = make_plan(T, world, rank, wt);
    out4[0] = p.a;
    out4[1] = p.b;
    out4[2] = p.lo;
    out4[3] = p.hi;
    return SNLS_OK;
}

int snls_shard_transfers(int T, int world, int rank, int wt, int capacity, int* peer, int* lo,
                         int* hi, int* recv, int* count) {
    if (int rc = check_plan_args(T, world, rank, wt)) return rc;
    if (!count) return fail(SNLS_EARG, "snls_shard_transfers: null count");
    const auto tr = transfers(T, world, rank, wt);
    *count = int(tr.size());
    if (int(tr.size()) > capacity) return fail(SNLS_EARG, "snls_shard_transfers: capacity too small");
    for (size_t i = 0; i < tr.size(); ++i) {
        if (peer) peer[i] = tr[i].peer;
        if (lo) lo[i] = tr[i].lo;
        if (hi) hi[i] = tr[i].hi;
        if (recv) recv[i] = tr[i].recv;
    }
    return SNLS_OK;
}

int snls_comm_unique_id(void* id_out) {
    if (!id_out) return fail(SNLS_EARG, "snls_comm_unique_id: null output");
    Nccl& n = nccl();
    if (!n.ok) return fail(SNLS_ECUDA, n.why);
    ncclUniqueId id;
    if (ncclResult_t r = n.GetUniqueId(&id); r != ncclSuccess) return nfail(r, "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
    return SNLS_OK;
}

int snls_comm_init(snls_ctx* ctx, const void* unique_id, int rank, int world, snls_comm** out) {
    if (!out) return fail(SNLS_EARG, "snls_comm_init: null output");
    *out = nullptr;
    if (!ctx || !unique_id) return fail(SNLS_EARG, "snls_comm_init: null context or id");
    if (world < 1 || rank < 0 || rank >= world) return fail(SNLS_EARG, "snls_comm_init: bad rank / world");
    Nccl& n = nccl();
    if (!n.ok) return fail(SNLS_ECUDA, n.why);
    auto* c = new snls_comm();
    c->ctx = ctx;
    c->device = snls_capi::ctx_device(ctx);
    c->rank = rank;
    c->world = world;
    DevGuard g(c->device);
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    if (ncclResult_t r = n.CommInitRank(&c->comm, world, id, rank); r != ncclSuccess) {
        delete c;
        return nfail(r, "ncclCommInitRank");
    }
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        snls_comm_destroy(c);
        return fail(SNLS_ECUDA, std::string("snls_comm_init: ") + cudaGetErrorString(e));
    }
    *out = c;
    return SNLS_OK;
}

int snls_comm_destroy(snls_comm* c) {
    if (!c) return SNLS_OK;
    DevGuard g(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm) nccl().CommDestroy(c->comm);
    if (c->scratch) cudaFree(c->scratch);
    if (c->ready) cudaEventDestroy(c->ready);
    if (c->done) cudaEventDestroy(c->done);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return SNLS_OK;
}

// nranks as NCCL reports it (evidence of the communicator size) and the NCCL version in use.
int snls_comm_info(snls_comm* c, int* nranks, int* nccl_version) {
    if (!c) return fail(SNLS_EARG, "snls_comm_info: null communicator");
    if (nranks)
        if (ncclResult_t r = nccl().CommCount(c->comm, nranks); r != ncclSuccess) return nfail(r, "ncclCommCount");
    if (nccl_version)
        if (ncclResult_t r = nccl().GetVersion(nccl_version); r != ncclSuccess) return nfail(r, "ncclGetVersion");
    return SNLS_OK;
}

// Start the forward halo exchange of `nslabs` persistent frame-major slabs [lo, hi) (owned
// frames [a, b) in place; frame_bytes[i] = bytes per frame of slab i; aliased slabs are the
// caller's to pass once).  Enqueued on the communicator's stream after everything already on
// the context's stream; returns without blocking.  snls_halo_wait joins it back.
int snls_halo_exchange_async(snls_comm* c, int T, int wt, int nslabs, void* const* slabs,
                             const int64_t* frame_bytes) {
    if (!c) return fail(SNLS_EARG, "snls_halo_exchange: null communicator");
    if (int rc = check_plan_args(T, c->world, c->rank, wt)) return rc;
    if (nslabs < 0 || (nslabs > 0 && (!slabs || !frame_bytes))) return fail(SNLS_EARG, "snls_halo_exchange: bad slabs");
    if (c->pending) return fail(SNLS_EARG, "snls_halo_exchange: previous exchange not joined (snls_halo_wait)");
    Nccl& n = nccl();
    DevGuard g(c->device);
    void* user = nullptr;
    snls_ctx_get_stream(c->ctx, &user);
    cudaEventRecord(c->ready, static_cast<cudaStream_t>(user));
    cudaStreamWaitEvent(c->stream, c->ready, 0);
    const Plan p = make_plan(T, c->world, c->rank, wt);
    const auto tr = transfers(T, c->world, c->rank, wt);
    if (!tr.empty()) {
        if (ncclResult_t r = n.GroupStart(); r != ncclSuccess) return nfail(r, "ncclGroupStart");
        for (int s = 0; s < nslabs; ++s) {
            char* base = static_cast<char*>(slabs[s]);
            const int64_t fb = frame_bytes[s];
            for (const auto& t : tr) {
                char* ptr = base + (t.lo - p.lo) * fb;
                const size_t bytes = size_t(t.hi - t.lo) * size_t(fb);
                const ncclResult_t r = t.recv ? n.Recv(ptr, bytes, ncclUint8, t.peer, c->comm, c->stream)
                                              : n.Send(ptr, bytes, ncclUint8, t.peer, c->comm, c->stream);
                if (r != ncclSuccess) {
                    n.GroupEnd();
                    return nfail(r, t.recv ? "ncclRecv" : "ncclSend");
                }
            }
        }
        if (ncclResult_t r = n.GroupEnd(); r != ncclSuccess) return nfail(r, "ncclGroupEnd");
    }
    cudaEventRecord(c->done, c->stream);
    c->pending = true;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SNLS_ECUDA, std::string("snls_halo_exchange: ") + cudaGetErrorString(e));
    return SNLS_OK;
}

// Order the context's stream after the started exchange (a stream wait, not a host block).
int snls_halo_wait(snls_comm* c) {
    if (!c) return fail(SNLS_EARG, "snls_halo_wait: null communicator");
    if (!c->pending) return SNLS_OK;
    DevGuard g(c->device);
    void* user = nullptr;
    snls_ctx_get_stream(c->ctx, &user);
    cudaStreamWaitEvent(static_cast<cudaStream_t>(user), c->done, 0);
    c->pending = false;
    return SNLS_OK;
}

// The backward's halo step: the partial gradients this rank accumulated
// in its halo frames (dK / dV / dFlow land in frames qt + dt, search.cpp:584-666;
// aggregate.cpp:412-460) are sent to the owners of those frames, and the partial sums the
// peers hold for my owned frames come back and are added in place.  fp32 slabs [lo, hi),
// frame_elems[i] floats per frame.  Ordered after the context's stream and joined back into
// it before returning (no host block).
int snls_reverse_halo_add(snls_comm* c, int T, int wt, int nslabs, float* const* slabs,
                          const int64_t* frame_elems) {
    if (!c) return fail(SNLS_EARG, "snls_reverse_halo_add: null communicator");
    if (int rc = check_plan_args(T, c->world, c->rank, wt)) return rc;
    if (nslabs < 0 || (nslabs > 0 && (!slabs || !frame_elems))) return fail(SNLS_EARG, "snls_reverse_halo_add: bad slabs");
    if (c->pending) return fail(SNLS_EARG, "snls_reverse_halo_add: previous exchange not joined (snls_halo_wait)");
    Nccl& n = nccl();
    DevGuard g(c->device);
    const Plan p = make_plan(T, c->world, c->rank, wt);
    const auto tr = transfers(T, c->world, c->rank, wt);
    // one receive buffer per (slab, incoming range): my frames' partial sums from the peers
    size_t need = 0;
    for (int s = 0; s < nslabs; ++s)
        for (const auto& t : tr)
            if (!t.recv) need += size_t(t.hi - t.lo) * size_t(frame_elems[s]) * sizeof(float);
    if (need > c->scratch_bytes) {
        if (c->scratch) {
            cudaStreamSynchronize(c->stream);
            cudaFree(c->scratch);
        }
        c->scratch = nullptr;
        c->scratch_bytes = 0;
        if (cudaMalloc(&c->scratch, need) != cudaSuccess) return fail(SNLS_ECUDA, "snls_reverse_halo_add: scratch");
        c->scratch_bytes = need;
    }
    void* user = nullptr;
    snls_ctx_get_stream(c->ctx, &user);
    const cudaStream_t us = static_cast<cudaStream_t>(user);
    cudaEventRecord(c->ready, us);
    cudaStreamWaitEvent(c->stream, c->ready, 0);
    struct Add {
        float* dst;
        const float* src;
        int64_t n;
    };
    std::vector<Add> adds;
    if (!tr.empty()) {
        if (ncclResult_t r = n.GroupStart(); r != ncclSuccess) return nfail(r, "ncclGroupStart");
        float* buf = static_cast<float*>(c->scratch);
        for (int s = 0; s < nslabs; ++s) {
            const int64_t fe = frame_elems[s];
            for (const auto& t : tr) {
                float* view = slabs[s] + (t.lo - p.lo) * fe;
                const size_t count = size_t(t.hi - t.lo) * size_t(fe);
                ncclResult_t r;
                if (t.recv) {  // halo frames of mine = the peer's owned frames: send my partials
                    r = n.Send(view, count, ncclFloat32, t.peer, c->comm, c->stream);
                } else {  // the peer's partials for my owned frames
                    r = n.Recv(buf, count, ncclFloat32, t.peer, c->comm, c->stream);
                    adds.push_back({view, buf, int64_t(count)});
                    buf += count;
                }
                if (r != ncclSuccess) {
                    n.GroupEnd();
                    return nfail(r, "reverse halo send/recv");
                }
            }
        }
        if (ncclResult_t r = n.GroupEnd(); r != ncclSuccess) return nfail(r, "ncclGroupEnd");
    }
    for (const auto& a : adds) {
        const int64_t blocks = (a.n + 255) / 256;
        add_kernel<<<unsigned(blocks < 4096 ? blocks : 4096), 256, 0, c->stream>>>(a.dst, a.src, a.n);
    }
    cudaEventRecord(c->done, c->stream);
    cudaStreamWaitEvent(us, c->done, 0);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SNLS_ECUDA, std::string("snls_reverse_halo_add: ") + cudaGetErrorString(e));
    return SNLS_OK;
}

// NCCL self-check on one device: a grouped ncclSend / ncclRecv of `bytes` from `src` to
// `dst` with this rank as its own peer, on the communicator's stream (joined into the
// context's stream).  Proves the NCCL path executes on a single-GPU lease.
int snls_comm_loopback(snls_comm* c, const void* src, void* dst, uint64_t bytes) {
    if (!c || !src || !dst) return fail(SNLS_EARG, "snls_comm_loopback: null argument");
    Nccl& n = nccl();
    DevGuard g(c->device);
    void* user = nullptr;
    snls_ctx_get_stream(c->ctx, &user);
    const cudaStream_t us = static_cast<cudaStream_t>(user);
    cudaEventRecord(c->ready, us);
    cudaStreamWaitEvent(c->stream, c->ready, 0);
    if (ncclResult_t r = n.GroupStart(); r != ncclSuccess) return nfail(r, "ncclGroupStart");
    ncclResult_t r = n.Send(src, bytes, ncclUint8, c->rank, c->comm, c->stream);
    if (r == ncclSuccess) r = n.Recv(dst, bytes, ncclUint8, c->rank, c->comm, c->stream);
    const ncclResult_t r2 = n.GroupEnd();
    if (r != ncclSuccess) return nfail(r, "loopback send/recv");
    if (r2 != ncclSuccess) return nfail(r2, "ncclGroupEnd");
    cudaEventRecord(c->done, c->stream);
    cudaStreamWaitEvent(us, c->done, 0);
    return SNLS_OK;
}

}  // extern "C"
