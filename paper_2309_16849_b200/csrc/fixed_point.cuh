// Deterministic accumulation helpers (the reference's ExecPolicy::deterministic,
// search.cpp:687-696, aggregate.cpp:439-450): sums as int64 fixed point with a power-of-two
// scale chosen per call from exact maxima, so integer atomics give the same bits in any order.
#pragma once

#include <cstdint>

namespace snls_gpu {
namespace {

// Non-negative float maxima (|q|, |k|, |grad|) as uint bit patterns: atomicMax on the bits
// is exact and order-independent, so the scales below are the same on every run.
__global__ void absmax_kernel(const float* __restrict__ a, int64_t n, unsigned* out) {
    float m = 0.f;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        m = fmaxf(m, fabsf(a[i]));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out, __float_as_uint(m));
}

// 2^(61 - ceil(log2(bound))): |any partial sum| <= bound < 2^61 / scale, so no int64 overflow.
__device__ __forceinline__ double pow2_scale(double bound) {
    if (!(bound > 0.0) || !isfinite(bound)) return 1.0;
    int ex;
    frexp(bound, &ex);  // bound < 2^ex
    return ldexp(1.0, 61 - ex);
}

__global__ void fixed_to_float_kernel(const unsigned long long* __restrict__ a, const double* scale,
                                      float* __restrict__ out, int64_t n) {
    const double inv = 1.0 / *scale;  // a power of two: exact
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = float(double(static_cast<long long>(a[i])) * inv);
}

__device__ __forceinline__ void fixed_add(unsigned long long* a, double v, double scale) {
    atomicAdd(a, static_cast<unsigned long long>(__double2ll_rn(v * scale)));
}

}  // namespace
}  // namespace snls_gpu
