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

float* upload(DeviceBuffer& buf, const double* host, std::uint64_t n) {
    std::vector<float> tmp(n);
    for (std::uint64_t i = 0; i < n; ++i) tmp[i] = float(host[i]);
    float* d = buf.f32(n);
    check(snls_copy_h2d(context(), d, tmp.data(), n * sizeof(float)));
    // the staging vector must outlive the async copy
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
    std::vector<float> tmp(n);
    check(snls_copy_d2h(context(), tmp.data(), dev, n * sizeof(float)));
    host.resize(n);
    for (std::uint64_t i = 0; i < n; ++i) host[i] = double(tmp[i]);
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
