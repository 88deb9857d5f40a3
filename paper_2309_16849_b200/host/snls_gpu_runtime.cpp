#include "snls_gpu_runtime.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include <omp.h>
#include <sys/mman.h>


#include "snls/search.hpp"

namespace snls::gpu {

void check(int status) {
    if (status == SNLS_OK) return;
    const std::string msg = snls_last_error();
    if (status == SNLS_ECONFIG) throw ConfigError(msg);
    if (status == SNLS_EDOMAIN) throw DomainError(msg);
    throw std::runtime_error("snls_cuda: " + msg);
}

namespace {
struct ThreadContext {
    snls_ctx* ctx = nullptr;
    ~ThreadContext() {
        if (ctx) snls_ctx_destroy(ctx);
    }
};
thread_local ThreadContext t_ctx;
}  // namespace

snls_ctx* context() {
    if (!t_ctx.ctx) {
        const char* env = std::getenv("SNLS_DEVICE");
        const int device = env ? std::atoi(env) : 0;
        check(snls_ctx_create(device, nullptr, &t_ctx.ctx));
    }
    return t_ctx.ctx;
}

DeviceBuffer::~DeviceBuffer() {
    if (ptr_ && t_ctx.ctx) snls_device_free(t_ctx.ctx, ptr_);
}

void* DeviceBuffer::reserve(std::uint64_t bytes) {
    if (bytes <= bytes_ && ptr_) return ptr_;
    if (ptr_) check(snls_device_free(context(), ptr_));
    ptr_ = nullptr;
    bytes_ = 0;
    check(snls_device_alloc(context(), bytes ? bytes : 4, &ptr_));
    bytes_ = bytes ? bytes : 4;
    return ptr_;
}

namespace {
// Pinned (page-locked) fp32 staging for the fp64 <-> fp32 conversions: grow-only, one per
// thread, so the copies run at full PCIe rate and the conversion never page-faults.
struct Staging {
    float* ptr = nullptr;
    std::uint64_t n = 0;
    ~Staging() {
        if (ptr) {
            snls_host_unregister(ptr);
            std::free(ptr);
        }
    }
    float* get(std::uint64_t want) {
        if (want <= n && ptr) return ptr;
        if (ptr) {
            snls_host_unregister(ptr);
            std::free(ptr);
        }
        n = want > 0 ? want : 1;
        ptr = static_cast<float*>(std::aligned_alloc(4096, ((n * sizeof(float) + 4095) / 4096) * 4096));
        if (!ptr) throw std::bad_alloc();
        check(snls_host_register(ptr, n * sizeof(float)));
        return ptr;
    }
};
thread_local Staging t_stage;
}  // namespace

float* staging(std::uint64_t n) { return t_stage.get(n); }

float* upload(DeviceBuffer& buf, const double* host, std::uint64_t n) {
    float* tmp = staging(n);
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < std::int64_t(n); ++i) tmp[i] = float(host[i]);
    float* d = buf.f32(n);
    check(snls_copy_h2d(context(), d, tmp, n * sizeof(float)));
    // the staging buffer is reused: the copy must have landed
    check(snls_ctx_sync_check(context()));
    return d;
}

float* upload(DeviceBuffer& buf, const std::vector<double>& host) {
    return upload(buf, host.data(), host.size());
}

std::int32_t* upload_i32(DeviceBuffer& buf, const std::vector<std::int32_t>& host) {
    std::int32_t* d = buf.i32(host.size());
    check(snls_copy_h2d(context(), d, host.data(), host.size() * sizeof(std::int32_t)));
    check(snls_ctx_sync_check(context()));
    return d;
}

void size_for_fill(std::vector<double>& host, std::uint64_t n);

void download(std::vector<double>& host, const float* dev, std::uint64_t n) {
    float* tmp = staging(n);
    check(snls_copy_d2h(context(), tmp, dev, n * sizeof(float)));
    size_for_fill(host, n);
    double* h = host.data();
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < std::int64_t(n); ++i) h[i] = double(tmp[i]);
}

void download_i32(std::vector<std::int32_t>& host, const std::int32_t* dev, std::uint64_t n) {
    host.resize(n);
    check(snls_copy_d2h(context(), host.data(), dev, n * sizeof(std::int32_t)));
}

namespace {
// Two pinned halves for the pipelined copies, with an event per half (reuse waits for the
// copy that last used it).  Grow-only, one per thread.
struct Pipe {
    static constexpr std::uint64_t kChunkBytes = 16u << 20;
    char* half[2] = {nullptr, nullptr};
    snls_event* ev[2] = {nullptr, nullptr};
    bool busy[2] = {false, false};
    Pipe() {
        for (int i = 0; i < 2; ++i) {
            half[i] = static_cast<char*>(std::aligned_alloc(4096, kChunkBytes));
            if (!half[i]) throw std::bad_alloc();
            check(snls_host_register(half[i], kChunkBytes));
            check(snls_event_create(context(), &ev[i]));
        }
    }
    ~Pipe() {
        for (int i = 0; i < 2; ++i) {
            snls_event_destroy(ev[i]);
            if (half[i]) {
                snls_host_unregister(half[i]);
                std::free(half[i]);
            }
        }
    }
    char* acquire(int i) {  // wait until half i's previous copy is done
        if (busy[i]) check(snls_event_sync(ev[i]));
        busy[i] = false;
        return half[i];
    }
    void release(int i) {
        check(snls_event_record(context(), ev[i]));
        busy[i] = true;
    }
};
thread_local Pipe* t_pipe = nullptr;
Pipe& pipe() {
    if (!t_pipe) t_pipe = new Pipe();  // (per thread, lives as long as the thread's context)
    return *t_pipe;
}
}  // namespace

float* upload_async(DeviceBuffer& buf, const double* host, std::uint64_t n) {
    snls_ctx* ctx = context();
    float* d = buf.f32(n);
    Pipe& p = pipe();
    const std::uint64_t per = Pipe::kChunkBytes / sizeof(float);
    int h = 0;
    for (std::uint64_t i0 = 0; i0 < n; i0 += per, h ^= 1) {
        const std::uint64_t m = std::min(per, n - i0);
        float* tmp = reinterpret_cast<float*>(p.acquire(h));
        const double* src = host + i0;
#pragma omp parallel for schedule(static)
        for (std::int64_t i = 0; i < std::int64_t(m); ++i) tmp[i] = float(src[i]);
        check(snls_copy_async(ctx, d + i0, tmp, m * sizeof(float), 1));
        p.release(h);
    }
    return d;
}

void size_for_fill(std::vector<double>& host, std::uint64_t n) {
    // std::vector zero-fills on resize, and the first touch of hundreds of MB of fresh pages
    // is the slow part (4 KB page faults, one thread): ask for transparent huge pages on the
    // reserved region and fault it in in parallel first -- bytes inside capacity() that
    // resize() then value-initialises -- so the zero-fill runs at memset speed (and the
    // caller's later free unmaps 2 MB pages)
    if (host.capacity() < n && n * sizeof(double) >= (std::uint64_t(32) << 20)) {  // (small: plain resize)
        host.reserve(n);
        char* base = reinterpret_cast<char*>(host.data() + host.size());
        const std::int64_t bytes = std::int64_t((n - host.size()) * sizeof(double));
        const std::uintptr_t lo = (reinterpret_cast<std::uintptr_t>(base) + (2u << 20) - 1) & ~std::uintptr_t((2u << 20) - 1);
        const std::uintptr_t hi = (reinterpret_cast<std::uintptr_t>(base) + bytes) & ~std::uintptr_t((2u << 20) - 1);
        if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
        volatile char* vb = base;
        if (omp_in_parallel()) {
            for (std::int64_t off = 0; off < bytes; off += 4096) vb[off] = 0;
        } else {
#pragma omp parallel for schedule(static)
            for (std::int64_t off = 0; off < bytes; off += 4096) vb[off] = 0;
        }
    }
    host.resize(n);
}

void download64(std::vector<double>& host, const double* dev, std::uint64_t n) {
    snls_ctx* ctx = context();
    size_for_fill(host, n);
    profile_mark("  vector sized");
    Pipe& p = pipe();
    const std::uint64_t per = Pipe::kChunkBytes / sizeof(double);
    const std::uint64_t nch = (n + per - 1) / per;
    // chunk c lands in half c % 2; chunk c+1's copy is in flight while chunk c is copied out
    auto start = [&](std::uint64_t c) {
        const std::uint64_t i0 = c * per, m = std::min(per, n - i0);
        char* tmp = p.acquire(int(c & 1));
        check(snls_copy_async(ctx, tmp, dev + i0, m * sizeof(double), 2));
        p.release(int(c & 1));
    };
    if (nch) start(0);
    for (std::uint64_t c = 0; c < nch; ++c) {
        if (c + 1 < nch) start(c + 1);
        check(snls_event_sync(p.ev[c & 1]));
        const std::uint64_t i0 = c * per, m = std::min(per, n - i0);
        const double* src = reinterpret_cast<const double*>(p.half[c & 1]);
        double* dst = host.data() + i0;
#pragma omp parallel for schedule(static)
        for (std::int64_t b = 0; b < std::int64_t((m + 4095) / 4096); ++b) {
            const std::uint64_t j0 = std::uint64_t(b) * 4096, cnt = std::min<std::uint64_t>(4096, m - j0);
            std::memcpy(dst + j0, src + j0, cnt * sizeof(double));
        }
        p.busy[c & 1] = false;
    }
    profile_mark("  vector filled");
}

void profile_mark(const char* stage) {
    static const bool on = [] {
        const char* e = std::getenv("SNLS_ADAPTER_PROFILE");
        return e && e[0] == '1';
    }();
    if (!on) return;
    using clk = std::chrono::steady_clock;
    thread_local clk::time_point last = clk::now();
    const clk::time_point now = clk::now();
    std::fprintf(stderr, "[adapter] %-28s %8.3f ms\n", stage,
                 std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

snls_config to_abi(const SearchConfig& c) {
    snls_config a;
    a.ws = c.ws;
    a.wt = c.wt;
    a.ps = c.ps;
    a.stride0 = c.stride0;
    a.stride1 = c.stride1;
    a.topl = c.topl;
    a.metric = c.metric == Metric::kInnerProduct ? SNLS_METRIC_IP : SNLS_METRIC_L2;
    a.softmax_scale = c.softmax_scale;
    return a;
}

}  // namespace snls::gpu
