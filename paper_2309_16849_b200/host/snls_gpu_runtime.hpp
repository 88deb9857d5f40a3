// Host runtime of the drop-in adapter: a per-thread device context, grow-only device
// buffers, fp64 <-> fp32 staging, and the status -> exception mapping of the reference
// (errors.hpp:9-17).  Everything device-side goes through the C-ABI in include/snls_cuda.h.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "snls/errors.hpp"
#include "snls/search.hpp"
#include "snls_cuda.h"

namespace snls::gpu {

// Throws the reference's exception type for a C-ABI status (same message text).
void check(int status);

// Context for the calling thread: device from $SNLS_DEVICE (default 0), default stream.
snls_ctx* context();

// A device allocation that only grows; one per role so repeated calls reuse memory.
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    ~DeviceBuffer();
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;

    void* reserve(std::uint64_t bytes);
    float* f32(std::uint64_t n) { return static_cast<float*>(reserve(n * sizeof(float))); }
    std::int32_t* i32(std::uint64_t n) {
        return static_cast<std::int32_t*>(reserve(n * sizeof(std::int32_t)));
    }

private:
    void* ptr_ = nullptr;
    std::uint64_t bytes_ = 0;
};

// fp64 host data -> fp32 device buffer (the reference computes in fp64, the kernels in
// fp32; fp32-representable inputs round-trip exactly).
float* upload(DeviceBuffer& buf, const std::vector<double>& host);
float* upload(DeviceBuffer& buf, const double* host, std::uint64_t n);
std::int32_t* upload_i32(DeviceBuffer& buf, const std::vector<std::int32_t>& host);
void download(std::vector<double>& host, const float* dev, std::uint64_t n);
// The calling thread's pinned fp32 staging buffer (>= n floats; reused by upload/download).
float* staging(std::uint64_t n);
void download_i32(std::vector<std::int32_t>& host, const std::int32_t* dev, std::uint64_t n);

snls_config to_abi(const snls::SearchConfig& cfg);

// Pipelined fp64 -> fp32 upload: the host converts chunk i (OpenMP) into one half of a pinned
// double buffer while chunk i-1's H2D copy runs; returns with every copy enqueued (the
// buffer reuse is ordered by events, the caller's later kernels by the stream).
float* upload_async(DeviceBuffer& buf, const double* host, std::uint64_t n);
// fp64 device data -> std::vector<double>: the vector is sized (zero-filled by std::vector),
// then filled from pinned staging chunks (D2H of chunk i+1 overlaps the parallel copy of i).
void download64(std::vector<double>& host, const double* dev, std::uint64_t n);
// Size a result vector for a bulk fill (transparent huge pages, parallel first touch, then
// std::vector's zero-fill); download64 calls it, callers may run it ahead on other threads.
void size_for_fill(std::vector<double>& host, std::uint64_t n);
// Stage timing for SNLS_ADAPTER_PROFILE=1 (stderr): mark("name") after each stage.
void profile_mark(const char* stage);

}  // namespace snls::gpu
