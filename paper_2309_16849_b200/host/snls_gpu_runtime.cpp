#include "snls_gpu_runtime.hpp"

#include <cstdlib>
#include <stdexcept>

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

void download(std::vector<double>& host, const float* dev, std::uint64_t n) {
    float* tmp = staging(n);
    check(snls_copy_d2h(context(), tmp, dev, n * sizeof(float)));
    host.resize(n);
    double* h = host.data();
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < std::int64_t(n); ++i) h[i] = double(tmp[i]);
}

void download_i32(std::vector<std::int32_t>& host, const std::int32_t* dev, std::uint64_t n) {
    host.resize(n);
    check(snls_copy_d2h(context(), host.data(), dev, n * sizeof(std::int32_t)));
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
