// wpsum_backward on channel pairs (aggregate.cpp:351-460): shared by aggregate.cu (the
// wpsum_bwd_pairs kernel) and search_bwd.cu (the interleaved training backward).
#pragma once

#include "common.cuh"
#include "kernels.h"
#include "packed.cuh"
#include "fixed_point.cuh"

namespace snls_gpu {
namespace {

__device__ __forceinline__ int clampi(int d, int half) { return d < -half ? -half : (d > half ? half : d); }

__device__ __forceinline__ void cell_span(int gi, int stride, int n, int extent, int& lo, int& hi) {
    const int a = (stride - 1) / 2;  // aggregate.cpp:71-75
    lo = gi == 0 ? 0 : gi * stride - a;
    hi = gi == n - 1 ? extent - 1 : gi * stride + (stride - 1 - a);
}

// red.global.add.v2.f32: two channels' contributions in one vector reduction (FTZ, as the
// scalar float atomicAdd on global memory)
__device__ __forceinline__ void red2(float* p, u64 v) {
    const float2 f = upk2(v);
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(f.x), "f"(f.y) : "memory");
}

// wpsum_backward with channel PAIRS per lane (F = 2 NL channels over NL lanes, one row per
// lane group): packed FFMA2 arithmetic, 64-bit loads of V and vector reductions into dV --
// half the instructions of the one-channel-per-lane wpsum_bwd_rows for the same bytes.  The
// folded upstream gradient patch is parked in shared memory (one u64 per lane and pixel).
// The same per-(row, l) formulas as wpsum_bwd_rows (aggregate.cpp:351-460).
// LS > 1: the neighbours of a row are dealt round-robin to LS lane groups (each folds its own
// copy of the gradient patch): dW entries are independent and dV is a sum of atomics, so the
// split only adds warps to hide the per-neighbour load latency.
// The body takes its block index and dynamic shared memory explicitly, so the interleaved
// training backward (search_bwd.cu train_bwd_interleaved) can run it beside the search backward.
// DET (deterministic mode): dV (and, where an entry has several writers, dW) accumulate as
// int64 fixed point (fixed_point.cuh): dvi / dwi with the scales scale[0] / scale[1].  In this
// kernel dW has one writer per entry in either mode.
struct WbwdFixed {
    unsigned long long* dvi;
    unsigned long long* dwi;
    const double* scale;
};
template <int P, int NL, int LS, bool DET = false>
__device__ __forceinline__ void wpsum_bwd_pairs_body(const AggArgs& a, const float* __restrict__ go,
                                                     const int32_t* __restrict__ counts,
                                                     float* __restrict__ dv, float* __restrict__ dw,
                                                     unsigned bid, u64* s_gs2,  // [128 / NL groups][P * P][NL]
                                                     WbwdFixed fxp = {nullptr, nullptr, nullptr}) {
    constexpr int HP = P / 2, F = 2 * NL, GPW = 32 / NL;  // lane groups (rows) per warp
    const int lane = threadIdx.x & 31, c = lane % NL;
    const int grp = threadIdx.x / NL;
    const int64_t unit = int64_t(bid) * (128 / NL) + grp;
    const int64_t row = unit / LS;
    const int l_first = int(unit % LS);
    if (row >= a.d.rows) return;  // (whole lane groups)
    const unsigned gmask = GPW == 1 ? 0xffffffffu : (((1u << NL) - 1u) << (lane / NL * NL));
    int ti, qy, qx;
    row_coords(a.d, row, ti, qy, qx);
    const int H = a.d.h, W = a.d.w, st = a.d.stride0;
    const size_t rowF = size_t(W) * F, frameF = size_t(H) * rowF;
    u64* sgs = s_gs2 + size_t(grp) * P * P * NL + c;
    // ---- fold the upstream gradient (grad_out / count) onto the patch pixels
    const u64* gob = reinterpret_cast<const u64*>(go + size_t(ti - a.d.t0) * frameF) + c;
    const int32_t* cb = counts + size_t(ti - a.d.t0) * H * W;
    auto gval = [&](int y, int x) {
        const int pix = y * W + x;
        const float s = 1.f / float(__ldg(cb + pix));
        return mul2(__ldg(gob + size_t(pix) * NL), pk2(s, s));
    };
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const int y = qy + i - HP, x = qx + j - HP;
            sgs[(i * P + j) * NL] = (y >= 0 && y < H && x >= 0 && x < W) ? gval(y, x) : 0ull;
        }
    int ylo, yhi, xlo, xhi;  // the query's stride cell (aggregate.cpp:68-100)
    cell_span(qy / st, st, a.d.nh, H, ylo, yhi);
    cell_span(qx / st, st, a.d.nw, W, xlo, xhi);
    if (ylo < qy - HP || yhi > qy + HP || xlo < qx - HP || xhi > qx + HP) {  // cell completion
        for (int y = ylo; y <= yhi; ++y)
            for (int x = xlo; x <= xhi; ++x) {
                if (abs(y - qy) <= HP && abs(x - qx) <= HP) continue;
                u64& slot = sgs[((clampi(y - qy, HP) + HP) * P + clampi(x - qx, HP) + HP) * NL];
                const float2 s = upk2(slot), v = upk2(gval(y, x));
                slot = pk2(s.x + v.x, s.y + v.y);
            }
    }
    // ---- per neighbour: dW and the dV block scatter
    for (int l = l_first; l < a.topl; l += LS) {
        const int64_t e = row * a.topl + l;
        const float* o = a.offsets + size_t(e) * 3;
        const int kt = ti + int(roundf(__ldg(o)));
        if (kt < 0 || kt >= a.d.t) {  // "offsets leave the clip" (aggregate.cpp:108-109)
            if (c == 0) latch(a.err, kErrWpsum);
            continue;
        }
        const float oy = __ldg(o + 1), ox = __ldg(o + 2);
        const float fly = floorf(oy), flx = floorf(ox);
        const float fy = oy - fly, fx = ox - flx;
        const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx;
        const float w10 = fy * (1.f - fx), w11 = fy * fx;
        const u64 W00 = pk2(w00, w00), W01 = pk2(w01, w01), W10 = pk2(w10, w10), W11 = pk2(w11, w11);
        const float wv = __ldg(a.weights + e);
        const u64 WV = pk2(wv, wv);
        const int by = qy - HP + int_base(fly), bx = qx - HP + int_base(flx);
        const u64* vb = reinterpret_cast<const u64*>(a.v + size_t(kt) * frameF) + c;
        const size_t dvo = size_t(kt) * frameF + 2 * c;  // this lane's first channel of frame kt
        const double fsc = DET ? *fxp.scale : 0.0;
        auto scatter = [&](size_t idx, u64 val) {  // idx: element index of the pair's first channel
            if constexpr (DET) {
                const float2 f = upk2(val);
                fixed_add(fxp.dvi + idx, f.x, fsc);
                fixed_add(fxp.dvi + idx + 1, f.y, fsc);
            } else {
                red2(dv + idx, val);
            }
        };
        u64 dwl = 0ull;
        // FAST (block inside the frame): one row base, immediate column offsets j * NL; else
        // reflected rows / columns (tensor.cpp:23-48), the columns resolved once per neighbour
        auto body = [&](auto fast_tag) {
            constexpr bool FAST = decltype(fast_tag)::value;
            unsigned bcol[FAST ? 1 : P + 1];
            if constexpr (!FAST) {
#pragma unroll
                for (int j = 0; j <= P; ++j) bcol[j] = unsigned(reflect_near(bx + j, W)) * NL;
            }
            auto colo = [&](int j) -> unsigned { return FAST ? unsigned(j * NL) : bcol[FAST ? 0 : j]; };
            const size_t rowstride = size_t(W) * NL;
            auto rowo = [&](int r) -> size_t {
                return FAST ? size_t(by + r) * rowstride + size_t(bx) * NL : size_t(reflect_near(by + r, H)) * rowstride;
            };
            u64 ra[P + 1], rb[P + 1], ka[P + 1], kn[P + 1];
            size_t roa = rowo(0), rob = rowo(1);
#pragma unroll
            for (int j = 0; j <= P; ++j) {
                ra[j] = __ldg(vb + roa + colo(j));
                rb[j] = __ldg(vb + rob + colo(j));
                ka[j] = 0ull;
            }
#pragma unroll 1
            for (int i = 0; i < P; ++i) {
                u64 rn[P + 1];
                const size_t ron = rowo(i + 2);
                if (i + 1 < P) {
#pragma unroll
                    for (int j = 0; j <= P; ++j) rn[j] = __ldg(vb + ron + colo(j));
                }
#pragma unroll
                for (int j = 0; j <= P; ++j) kn[j] = 0ull;
                const u64* gi = sgs + i * P * NL;
#pragma unroll
                for (int j = 0; j < P; ++j) {
                    const u64 smp = fma2(W11, rb[j + 1], fma2(W10, rb[j], fma2(W01, ra[j + 1], mul2(W00, ra[j]))));
                    const u64 gij = gi[j * NL];
                    dwl = fma2(gij, smp, dwl);
                    const u64 gv = mul2(gij, WV);
                    ka[j] = fma2(gv, W00, ka[j]);
                    ka[j + 1] = fma2(gv, W01, ka[j + 1]);
                    kn[j] = fma2(gv, W10, kn[j]);
                    kn[j + 1] = fma2(gv, W11, kn[j + 1]);
                }
#pragma unroll
                for (int j = 0; j <= P; ++j) scatter(dvo + 2 * (roa + colo(j)), ka[j]);
#pragma unroll
                for (int j = 0; j <= P; ++j) {
                    ra[j] = rb[j];
                    if (i + 1 < P) rb[j] = rn[j];
                    ka[j] = kn[j];
                }
                roa = rob;
                rob = ron;
            }
#pragma unroll
            for (int j = 0; j <= P; ++j) scatter(dvo + 2 * (roa + colo(j)), ka[j]);
        };
        if (by >= 0 && by + P < H && bx >= 0 && bx + P < W)  // uniform per lane group
            body(std::true_type{});
        else
            body(std::false_type{});
        const float2 d2 = upk2(dwl);
        float dws = d2.x + d2.y;
#pragma unroll
        for (int m = NL / 2; m >= 1; m >>= 1) dws += __shfl_xor_sync(gmask, dws, m);
        if (c == 0) dw[e] = dws;  // the entry's only writer (dw was zeroed: same as an add)
    }
}

template <int P, int NL, int LS, bool DET = false>
__global__ void __launch_bounds__(128, 4) wpsum_bwd_pairs(AggArgs a, const float* __restrict__ go,
                                                          const int32_t* __restrict__ counts,
                                                          float* __restrict__ dv, float* __restrict__ dw,
                                                          WbwdFixed fxp) {
    extern __shared__ u64 s_gs2[];
    wpsum_bwd_pairs_body<P, NL, LS, DET>(a, go, counts, dv, dw, blockIdx.x, s_gs2, fxp);
}

}  // namespace
}  // namespace snls_gpu
