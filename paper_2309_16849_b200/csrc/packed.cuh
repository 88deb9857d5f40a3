// Packed fp32x2 arithmetic on sm_100a (PTX .f32x2 -> FFMA2 / FADD2 / FMUL2): two FP32 operations
// per issued instruction at the same FMA-pipe rate as the scalar forms
// (scripts/micro/ffma2_peak.cu: 74.1 vs 72.2 TFLOP/s), i.e. half the issue slots for the same
// arithmetic.  A `u64` is one register pair (lo, hi); P4 is a float4 as two pairs.
#pragma once

#include <cuda_runtime.h>

namespace snls_gpu {

using u64 = unsigned long long;
__device__ __forceinline__ u64 pk2(float x, float y) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ float2 upk2(u64 v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// a float4 as two channel pairs (x, y) and (z, w)
struct P4 {
    u64 lo, hi;
};
__device__ __forceinline__ P4 ldp4(const float4* p) {
    const float4 v = __ldg(p);
    return {pk2(v.x, v.y), pk2(v.z, v.w)};
}

}  // namespace snls_gpu
