// Aggregation kernels: softmax_rows, the deterministic wpsum gather, gather_stack and the
// wpsum backward (aggregate.cpp).
//
// wpsum is evaluated as the reference's fixed-order GATHER (aggregate.cpp:124-203): every
// output pixel is owned by exactly one thread group, which visits its contributing query
// units in the reference order (footprint py/px ascending, then the owning query's cell
// completion) -- deterministic, no atomics, every output element written once, coalesced
// C-vectorised (float4) reads of V.  The backward scatters through 4 bilinear taps, so it
// uses atomics (the reference's non-deterministic mode, aggregate.cpp:451-458).
#include <cstdlib>
#include <functional>
#include <mutex>
#include <set>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "packed.cuh"
#include "fixed_point.cuh"
#include "wpsum_bwd_pairs.cuh"

namespace snls_gpu {

namespace {

__device__ __forceinline__ int owner_index(int coord, int stride, int n) {  // aggregate.hpp:91-95
    int gi = (coord + (stride - 1) / 2) / stride;
    return gi > n - 1 ? n - 1 : gi;
}


// One (query row, patch pixel) unit restricted to neighbour range [l0, l1): accumulate the
// softmax-weighted bilinear samples of V (aggregate.cpp:104-122) for channels [c, c+VEC).
template <int VEC>
__device__ __forceinline__ bool add_unit(const AggArgs& a, int64_t row, int ti, int qy, int qx,
                                         int pyu, int pxu, int l0, int l1, int c, float* acc) {
    for (int li = l0; li < l1; ++li) {
        const size_t e = size_t(row) * a.topl + li;
        const float* o = a.offsets + e * 3;
        const int kt = ti + int(roundf(__ldg(o)));
        if (kt < 0 || kt >= a.d.t) return false;
        int iy, ix;
        float fy, fx;
        split_pos(qy + pyu, __ldg(o + 1), iy, fy, a.d.h);
        split_pos(qx + pxu, __ldg(o + 2), ix, fx, a.d.w);
        const Taps t = taps_from(iy, fy, ix, fx, a.d.h, a.d.w);
        const float wv = __ldg(a.weights + e);
        const float* p00 = a.v + vidx(a.d, kt, t.y0, t.x0) + c;
        const float* p01 = a.v + vidx(a.d, kt, t.y0, t.x1) + c;
        const float* p10 = a.v + vidx(a.d, kt, t.y1, t.x0) + c;
        const float* p11 = a.v + vidx(a.d, kt, t.y1, t.x1) + c;
        if (VEC == 4) {
            const float4 A = __ldg(reinterpret_cast<const float4*>(p00));
            const float4 B = __ldg(reinterpret_cast<const float4*>(p01));
            const float4 C = __ldg(reinterpret_cast<const float4*>(p10));
            const float4 D = __ldg(reinterpret_cast<const float4*>(p11));
            acc[0] = fmaf(wv, blend(t, A.x, B.x, C.x, D.x), acc[0]);
            acc[1] = fmaf(wv, blend(t, A.y, B.y, C.y, D.y), acc[1]);
            acc[2] = fmaf(wv, blend(t, A.z, B.z, C.z, D.z), acc[2]);
            acc[3] = fmaf(wv, blend(t, A.w, B.w, C.w, D.w), acc[3]);
        } else {
            acc[0] = fmaf(wv, blend(t, __ldg(p00), __ldg(p01), __ldg(p10), __ldg(p11)), acc[0]);
        }
    }
    return true;
}

// Fixed-order gather of one pixel (aggregate.cpp:156-188).  Returns the unit count, or -1
// when an offset leaves the clip.
template <int VEC>
__device__ int gather_pixel(const AggArgs& a, int ti, int y, int x, int l0, int l1, int c,
                            float* acc) {
    const int st = a.d.stride0, half = a.ps / 2;
    const int qmax_y = (a.d.nh - 1) * st, qmax_x = (a.d.nw - 1) * st;
    int cnt = 0;
    for (int py = -half; py <= half; ++py) {
        const int qy = y - py;
        if (qy < 0 || qy > qmax_y || qy % st != 0) continue;
        for (int px = -half; px <= half; ++px) {
            const int qx = x - px;
            if (qx < 0 || qx > qmax_x || qx % st != 0) continue;
            const int64_t row = (int64_t(ti) * a.d.nh + qy / st) * a.d.nw + qx / st - a.d.row0;
            if (!add_unit<VEC>(a, row, ti, qy, qx, py, px, l0, l1, c, acc)) return -1;
            ++cnt;
        }
    }
    const int qy = owner_index(y, st, a.d.nh) * st;
    const int qx = owner_index(x, st, a.d.nw) * st;
    if (abs(y - qy) > half || abs(x - qx) > half) {
        const int64_t row = (int64_t(ti) * a.d.nh + qy / st) * a.d.nw + qx / st - a.d.row0;
        if (!add_unit<VEC>(a, row, ti, qy, qx, clampi(y - qy, half), clampi(x - qx, half), l0,
                           l1, c, acc))
            return -1;
        ++cnt;
    }
    return cnt;
}

template <int VEC>
__global__ void __launch_bounds__(256) wpsum_kernel(AggArgs a, float* __restrict__ out,
                                                    int32_t* __restrict__ counts) {
    const int groups = a.d.f / VEC;
    const int64_t npix = int64_t(a.d.nt) * a.d.h * a.d.w;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= npix * groups) return;
    const int64_t pix = idx / groups;  // local to the frame range
    const int c = int(idx % groups) * VEC;
    const int x = int(pix % a.d.w);
    const int y = int((pix / a.d.w) % a.d.h);
    const int ti = a.d.t0 + int(pix / (int64_t(a.d.w) * a.d.h));
    float acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
    const int cnt = gather_pixel<VEC>(a, ti, y, x, 0, a.topl, c, acc);
    if (cnt <= 0) {
        latch(a.err, kErrWpsum);
        return;
    }
    if (c == 0 && counts) counts[pix] = cnt;
    const float inv = 1.f / float(cnt);
    float* o = out + size_t(pix) * a.d.f + c;
    if (VEC == 4) {
        *reinterpret_cast<float4*>(o) =
            make_float4(acc[0] / float(cnt), acc[1] / float(cnt), acc[2] / float(cnt), acc[3] / float(cnt));
    } else {
        o[0] = acc[0] / float(cnt);
    }
    (void)inv;
}

template <int VEC>
__global__ void __launch_bounds__(256) gather_stack_kernel(AggArgs a, float* __restrict__ out) {
    const int groups = a.d.f / VEC;
    const int64_t npix = int64_t(a.d.nt) * a.d.h * a.d.w;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= npix * groups * a.topl) return;
    const int li = int(idx / (npix * groups));
    const int64_t r = idx % (npix * groups);
    const int64_t pix = r / groups;
    const int c = int(r % groups) * VEC;
    const int x = int(pix % a.d.w);
    const int y = int((pix / a.d.w) % a.d.h);
    const int ti = a.d.t0 + int(pix / (int64_t(a.d.w) * a.d.h));
    float acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
    if (gather_pixel<VEC>(a, ti, y, x, li, li + 1, c, acc) < 0) latch(a.err, kErrStack);
    float* o = out + (size_t(li) * npix + size_t(pix)) * a.d.f + c;
    if (VEC == 4)
        *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    else
        o[0] = acc[0];
}

// ---- tiled gather -----------------------------------------------------------------------
// A CTA owns a run of PPC consecutive output pixels of one row (t, y) and all channels
// (G = F/4 lanes per pixel, float4 each).  Phase 1 turns every (query, neighbour) that can
// write into the run into a sample descriptor in shared memory: frame, integer offset and
// the four bilinear weights pre-multiplied by the softmax weight.  Phase 2 is the
// reference's fixed-order gather (footprint py/px ascending, then the owning query's cell
// completion; neighbours ascending), each unit costing 2 LDS + 4 coalesced LDG.128 + 16 FFMA
// per lane instead of re-deriving taps from the offsets in every channel lane.
// One (query, neighbour) of a tile: the sample frame's first pixel index (kt*H*W), the integer
// offset (and its pixel-index form oy*W + ox) and the softmax-weighted bilinear weights.
struct SampleDesc {
    uint32_t kbase;
    int oy, ox, doff;
    float w00, w01, w10, w11;
};

struct TileGeom {
    int gy_lo, nqy, gx_lo, nqx;
};

__device__ __forceinline__ TileGeom tile_geom(const AggArgs& a, int y, int x0, int ppc) {
    const int st = a.d.stride0;
    TileGeom g;
    // any query writing pixel y lies within s0-1 rows of it (footprint: half < s0; cell
    // completion: the owner, possibly clamped to the last grid row)
    const int lo_y = max(0, (y - (st - 1) + st - 1) / st - 1);
    const int hi_y = min(a.d.nh - 1, (y + st - 1) / st);
    g.gy_lo = max(0, lo_y);
    g.nqy = hi_y - g.gy_lo + 1;
    const int x1 = min(x0 + ppc, a.d.w) - 1;
    g.gx_lo = max(0, (x0 - (st - 1)) / st - 1);
    const int hi_x = min(a.d.nw - 1, (x1 + st - 1) / st);
    g.nqx = hi_x - g.gx_lo + 1;
    return g;
}

__device__ void build_descs(const AggArgs& a, int ti, const TileGeom& g, SampleDesc* desc,
                            int* err_bit, int err_code) {
    const int n = g.nqy * g.nqx * a.topl;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int l = i % a.topl, qi = i / a.topl;
        const int gy = g.gy_lo + qi / g.nqx, gx = g.gx_lo + qi % g.nqx;
        const int64_t row = (int64_t(ti) * a.d.nh + gy) * a.d.nw + gx - a.d.row0;
        const size_t e = size_t(row) * a.topl + l;
        const float* o = a.offsets + e * 3;
        SampleDesc d;
        int kt = ti + int(roundf(__ldg(o)));
        if (kt < 0 || kt >= a.d.t) {
            latch(err_bit, err_code);
            kt = ti;
        }
        d.kbase = uint32_t(kt) * uint32_t(a.d.h) * uint32_t(a.d.w);
        const float oy = __ldg(o + 1), ox = __ldg(o + 2);
        const float fly = floorf(oy), flx = floorf(ox);
        d.oy = int_base(fly);
        d.ox = int_base(flx);
        d.doff = d.oy * a.d.w + d.ox;
        const float fy = oy - fly, fx = ox - flx;
        const float wv = __ldg(a.weights + e);
        d.w00 = wv * ((1.f - fy) * (1.f - fx));
        d.w01 = wv * ((1.f - fy) * fx);
        d.w10 = wv * (fy * (1.f - fx));
        d.w11 = wv * (fy * fx);
        desc[i] = d;
    }
}

// Accumulate one unit (query at grid (gy, gx), sample at y + dy, x + dx where (dy, dx) is
// the pixel's displacement inside the query's patch) for neighbours [l0, l1).
#ifndef SNLS_AGG_UNROLL
#define SNLS_AGG_UNROLL 4
#endif
constexpr int kAggUnroll = SNLS_AGG_UNROLL;
// G = float4 groups per pixel (compile time); c4 = this lane's float4 group.  Addresses are
// pixel indices (frame base + (sy, sx) + offset) times G: one wide multiply per tap set.
template <int G>
__device__ __forceinline__ void add_unit_tiled(const AggArgs& a, const SampleDesc* desc,
                                               const TileGeom& g, int gy, int gx, int sy, int sx,
                                               int l0, int l1, int c4, float4& acc) {
    const SampleDesc* dq = desc + ((gy - g.gy_lo) * g.nqx + (gx - g.gx_lo)) * a.topl;
    const int H = a.d.h, W = a.d.w;
    const float4* vb = reinterpret_cast<const float4*>(a.v) + c4;
    const int pix = sy * W + sx;
#pragma unroll kAggUnroll
    for (int l = l0; l < l1; ++l) {
        const SampleDesc d = dq[l];
        const int iy = sy + d.oy, ix = sx + d.ox;
        const float4 *p00, *p01, *p10, *p11;
        if (unsigned(iy) < unsigned(H - 1) && unsigned(ix) < unsigned(W - 1)) {
            p00 = vb + size_t(d.kbase + uint32_t(pix + d.doff)) * G;
            p01 = p00 + G;
            p10 = p00 + size_t(W) * G;
            p11 = p10 + G;
        } else {  // reflected border taps (tensor.cpp:31-48)
            const int y0 = reflect(iy, H), y1 = reflect(iy + 1, H);
            const int x0 = reflect(ix, W), x1 = reflect(ix + 1, W);
            p00 = vb + size_t(d.kbase + uint32_t(y0 * W + x0)) * G;
            p01 = vb + size_t(d.kbase + uint32_t(y0 * W + x1)) * G;
            p10 = vb + size_t(d.kbase + uint32_t(y1 * W + x0)) * G;
            p11 = vb + size_t(d.kbase + uint32_t(y1 * W + x1)) * G;
        }
        const float4 A = __ldg(p00);
        const float4 B = __ldg(p01);
        const float4 C = __ldg(p10);
        const float4 D = __ldg(p11);
        acc.x = fmaf(d.w11, D.x, fmaf(d.w10, C.x, fmaf(d.w01, B.x, fmaf(d.w00, A.x, acc.x))));
        acc.y = fmaf(d.w11, D.y, fmaf(d.w10, C.y, fmaf(d.w01, B.y, fmaf(d.w00, A.y, acc.y))));
        acc.z = fmaf(d.w11, D.z, fmaf(d.w10, C.z, fmaf(d.w01, B.z, fmaf(d.w00, A.z, acc.z))));
        acc.w = fmaf(d.w11, D.w, fmaf(d.w10, C.w, fmaf(d.w01, B.w, fmaf(d.w00, A.w, acc.w))));
    }
}

// Footprint units along one axis: the patch offsets p in [-half, half] with coord - p on the
// query grid {0, s0, ..., qmax}.  Since half < s0 there are at most two, p = m and p = m - s0
// with m = coord mod s0 (ascending p order, as the reference loops, aggregate.cpp:161-166).
struct AxisUnits {
    int n, p0, p1;
};
__device__ __forceinline__ AxisUnits axis_units(int coord, int s0, int half, int qmax) {
    const int m = coord % s0;
    AxisUnits u;
    u.n = 0;
    u.p0 = u.p1 = 0;
    const int cand[2] = {m - s0, m};  // ascending
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int p = cand[i], q = coord - p;
        if (p >= -half && p <= half && q >= 0 && q <= qmax) {
            if (u.n == 0) u.p0 = p; else u.p1 = p;
            ++u.n;
        }
    }
    return u;
}

// One pixel's fixed-order gather over neighbours [l0, l1) (aggregate.cpp:156-188), with the
// footprint units enumerated without division in the inner loop.
template <int G>
__device__ int gather_tiled(const AggArgs& a, const SampleDesc* desc, const TileGeom& g,
                            const AxisUnits& uy, int y, int x, int l0, int l1, int c4,
                            float4& acc) {
    const int st = a.d.stride0, half = a.ps / 2;
    const AxisUnits ux = axis_units(x, st, half, (a.d.nw - 1) * st);
    int cnt = 0;
    for (int iy = 0; iy < uy.n; ++iy) {
        const int py = iy == 0 ? uy.p0 : uy.p1;
        for (int ix = 0; ix < ux.n; ++ix) {
            const int px = ix == 0 ? ux.p0 : ux.p1;
            // footprint unit: sample at qy + off + py = y + off
            add_unit_tiled<G>(a, desc, g, (y - py) / st, (x - px) / st, y, x, l0, l1, c4, acc);
            ++cnt;
        }
    }
    const int gy = owner_index(y, st, a.d.nh), gx = owner_index(x, st, a.d.nw);
    const int qy = gy * st, qx = gx * st;
    if (abs(y - qy) > half || abs(x - qx) > half) {
        add_unit_tiled<G>(a, desc, g, gy, gx, qy + clampi(y - qy, half), qx + clampi(x - qx, half),
                          l0, l1, c4, acc);
        ++cnt;
    }
    return cnt;
}

template <int G>
__global__ void __launch_bounds__(256) wpsum_tiled_kernel(AggArgs a, float* __restrict__ out,
                                                          int32_t* __restrict__ counts,
                                                          int stack) {
    extern __shared__ SampleDesc s_desc[];
    constexpr int PPC = 256 / G;
    const int tiles_x = (a.d.w + PPC - 1) / PPC;
    const int tx = blockIdx.x % tiles_x;
    const int y = (blockIdx.x / tiles_x) % a.d.h;
    const int ti = a.d.t0 + int(blockIdx.x / (tiles_x * a.d.h));
    const int x0 = tx * PPC;
    const TileGeom g = tile_geom(a, y, x0, PPC);
    build_descs(a, ti, g, s_desc, a.err, stack ? kErrStack : kErrWpsum);
    __syncthreads();
    const int p = threadIdx.x / G, c = (threadIdx.x % G) * 4;
    const int x = x0 + p;
    if (x >= a.d.w) return;
    const AxisUnits uy = axis_units(y, a.d.stride0, a.ps / 2, (a.d.nh - 1) * a.d.stride0);
    const size_t pix = (size_t(ti - a.d.t0) * a.d.h + y) * a.d.w + x;  // local output pixel
    if (!stack) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const int cnt = gather_tiled<G>(a, s_desc, g, uy, y, x, 0, a.topl, c / 4, acc);
        if (cnt <= 0) {
            latch(a.err, kErrWpsum);
            return;
        }
        if (c == 0 && counts) counts[pix] = cnt;
        const float fc = float(cnt);
        *reinterpret_cast<float4*>(out + pix * a.d.f + c) =
            make_float4(acc.x / fc, acc.y / fc, acc.z / fc, acc.w / fc);
    } else {
        const size_t plane = size_t(a.d.nt) * a.d.h * a.d.w * a.d.f;
        for (int l = 0; l < a.topl; ++l) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            gather_tiled<G>(a, s_desc, g, uy, y, x, l, l + 1, c / 4, acc);
            *reinterpret_cast<float4*>(out + l * plane + pix * a.d.f + c) = acc;
        }
    }
}

template <int G>
int launch_tiled_agg(const AggArgs& a, float* out, int32_t* counts, int stack, cudaStream_t st) {
    constexpr int PPC = 256 / G;
    const int s0 = a.d.stride0;
    const int nqy = 3 + 1, nqx = (PPC + 2 * s0) / s0 + 3;
    const size_t smem = size_t(nqy) * nqx * a.topl * sizeof(SampleDesc);
    if (smem > 200 * 1024) return 0;
    ensure_smem(wpsum_tiled_kernel<G>, smem);
    const int tiles_x = (a.d.w + PPC - 1) / PPC;
    const unsigned blocks = unsigned(int64_t(a.d.nt) * a.d.h * tiles_x);
    wpsum_tiled_kernel<G><<<blocks, 256, smem, st>>>(a, out, counts, stack);
    return 1;
}

int launch_tiled_agg_any(const AggArgs& a, float* out, int32_t* counts, int stack, cudaStream_t st) {
    if (a.d.f % 4 != 0) return 0;
    if (int64_t(a.d.t) * a.d.h * a.d.w >= (int64_t(1) << 32)) return 0;  // 32-bit pixel indices
    switch (a.d.f / 4) {
        case 1: return launch_tiled_agg<1>(a, out, counts, stack, st);
        case 2: return launch_tiled_agg<2>(a, out, counts, stack, st);
        case 4: return launch_tiled_agg<4>(a, out, counts, stack, st);
        case 8: return launch_tiled_agg<8>(a, out, counts, stack, st);
        case 16: return launch_tiled_agg<16>(a, out, counts, stack, st);
        case 32: return launch_tiled_agg<32>(a, out, counts, stack, st);
        default: return 0;
    }
}

// ---- query-centric wpsum ----------------------------------------------------------------
#ifndef SNLS_WQ_MINB
#define SNLS_WQ_MINB 2
#endif
// A CTA owns a TY x TX output tile of one frame (all channels).  Phase A: every query whose
// write set (footprint + stride-cell remainder, aggregate.cpp:80-100) can meet the tile is
// handled by one group of G lanes (float4 of channels each); for each neighbour l it reads the
// (ps+1)^2 raw V block ONCE and accumulates all ps^2 softmax-weighted bilinear samples in
// registers -- (ps+1)^2 loads per (query, l) instead of the 4*ps^2 of a per-pixel gather --
// then parks the ps^2 patch in shared memory.  Phase B: each output pixel sums the parked
// patches of its contributing units in the reference's fixed order (footprint py, px
// ascending, then the owning query's cell completion; aggregate.cpp:156-188), divides by the
// count and writes once.  Deterministic, no atomics, one barrier.
// FG = F / 4 float4 per pixel; a CTA covers G of them (channel slice blockIdx.y), so wide
// videos (F = 64) split their channels over two CTAs and keep the parked patches, and the
// shared memory per CTA, at the F = 32 size (two resident CTAs per SM instead of one).
template <int P, int G, int FG, int TY, int TX>
__global__ void __launch_bounds__(256, SNLS_WQ_MINB) wpsum_query_kernel(AggArgs a, float* __restrict__ out,
                                                          int32_t* __restrict__ counts) {
    extern __shared__ float4 s_patch[];  // [query][P*P][G]
    constexpr int HP = P / 2, NQG = 256 / G;
    const int H = a.d.h, W = a.d.w, st = a.d.stride0;
    const int tiles_x = (W + TX - 1) / TX, tiles_y = (H + TY - 1) / TY;
    const int tx0 = (blockIdx.x % tiles_x) * TX;
    const int ty0 = ((blockIdx.x / tiles_x) % tiles_y) * TY;
    const int ti = a.d.t0 + int(blockIdx.x / (tiles_x * tiles_y));
    // any query writing inside the tile lies within s0-1 of it
    const int gy_lo = ty0 / st, gy_hi = min(a.d.nh - 1, (ty0 + TY - 1 + st - 1) / st);
    const int gx_lo = tx0 / st, gx_hi = min(a.d.nw - 1, (tx0 + TX - 1 + st - 1) / st);
    const int nqx = gx_hi - gx_lo + 1, nq = (gy_hi - gy_lo + 1) * nqx;
    const int grp = threadIdx.x / G, gl = threadIdx.x % G;
    const unsigned row4 = unsigned(W) * FG;
    const int cg0 = int(blockIdx.y) * G;  // first float4 channel group of this CTA
    const float4* vbase = reinterpret_cast<const float4*>(a.v) + cg0 + gl;

    for (int qi = grp; qi < nq; qi += NQG) {
        const int gy = gy_lo + qi / nqx, gx = gx_lo + qi % nqx;
        const int qy = gy * st, qx = gx * st;
        const int64_t row = (int64_t(ti) * a.d.nh + gy) * a.d.nw + gx - a.d.row0;
        float4 acc[P][P];
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) acc[i][j] = make_float4(0.f, 0.f, 0.f, 0.f);
        auto unit = [&](int l) {
            const size_t e = size_t(row) * a.topl + l;
            const float* o = a.offsets + e * 3;
            int kt = ti + int(roundf(__ldg(o)));
            if (kt < 0 || kt >= a.d.t) {  // "offsets leave the clip" (aggregate.cpp:108-109)
                latch(a.err, kErrWpsum);
                kt = ti;
            }
            const float oy = __ldg(o + 1), ox = __ldg(o + 2);
            const float fly = floorf(oy), flx = floorf(ox);
            const float fy = oy - fly, fx = ox - flx;
            const float wv = __ldg(a.weights + e);
            const float w00 = wv * ((1.f - fy) * (1.f - fx)), w01 = wv * ((1.f - fy) * fx);
            const float w10 = wv * (fy * (1.f - fx)), w11 = wv * (fy * fx);
            // sample (i, j) sits between raw rows by+i, by+i+1 and cols bx+j, bx+j+1
            const int by = qy - HP + int_base(fly), bx = qx - HP + int_base(flx);
            const float4* vf = vbase + size_t(kt) * H * row4;
            float4 blk[P + 1][P + 1];
            if (by >= 0 && by + P < H && bx >= 0 && bx + P < W) {
                const float4* p0 = vf + (unsigned(by) * row4 + unsigned(bx) * FG);
#pragma unroll
                for (int i = 0; i <= P; ++i)
#pragma unroll
                    for (int j = 0; j <= P; ++j) blk[i][j] = __ldg(p0 + i * row4 + j * FG);
            } else {  // reflected border taps (tensor.cpp:31-48)
#pragma unroll
                for (int i = 0; i <= P; ++i) {
                    const unsigned r = unsigned(reflect_near(by + i, H)) * row4;
#pragma unroll
                    for (int j = 0; j <= P; ++j)
                        blk[i][j] = __ldg(vf + (r + unsigned(reflect_near(bx + j, W)) * FG));
                }
            }
#pragma unroll
            for (int i = 0; i < P; ++i)
#pragma unroll
                for (int j = 0; j < P; ++j) {
                    float4& c = acc[i][j];
                    const float4 &A = blk[i][j], &B = blk[i][j + 1], &C = blk[i + 1][j], &D = blk[i + 1][j + 1];
                    c.x = fmaf(w11, D.x, fmaf(w10, C.x, fmaf(w01, B.x, fmaf(w00, A.x, c.x))));
                    c.y = fmaf(w11, D.y, fmaf(w10, C.y, fmaf(w01, B.y, fmaf(w00, A.y, c.y))));
                    c.z = fmaf(w11, D.z, fmaf(w10, C.z, fmaf(w01, B.z, fmaf(w00, A.z, c.z))));
                    c.w = fmaf(w11, D.w, fmaf(w10, C.w, fmaf(w01, B.w, fmaf(w00, A.w, c.w))));
                }
        };
        for (int l = 0; l < a.topl; ++l) unit(l);
        float4* dst = s_patch + size_t(qi) * P * P * G + gl;
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) dst[(i * P + j) * G] = acc[i][j];
    }
    __syncthreads();

    // phase B: fixed-order gather from the parked patches
    for (int idx = threadIdx.x; idx < TY * TX * G; idx += 256) {
        const int pix = idx / G, c = idx % G;
        const int y = ty0 + pix / TX, x = tx0 + pix % TX;
        if (y >= H || x >= W) continue;
        float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
        int cnt = 0;
        auto add = [&](int gy, int gx, int si, int sj) {
            const float4 v = s_patch[(size_t((gy - gy_lo) * nqx + (gx - gx_lo)) * P * P + si * P + sj) * G + c];
            sum.x += v.x;
            sum.y += v.y;
            sum.z += v.z;
            sum.w += v.w;
            ++cnt;
        };
        const AxisUnits uy = axis_units(y, st, HP, (a.d.nh - 1) * st);
        const AxisUnits ux = axis_units(x, st, HP, (a.d.nw - 1) * st);
        for (int iy = 0; iy < uy.n; ++iy) {
            const int py = iy == 0 ? uy.p0 : uy.p1;
            for (int ix = 0; ix < ux.n; ++ix) {
                const int px = ix == 0 ? ux.p0 : ux.p1;
                add((y - py) / st, (x - px) / st, py + HP, px + HP);
            }
        }
        const int gy = owner_index(y, st, a.d.nh), gx = owner_index(x, st, a.d.nw);
        if (abs(y - gy * st) > HP || abs(x - gx * st) > HP)
            add(gy, gx, clampi(y - gy * st, HP) + HP, clampi(x - gx * st, HP) + HP);
        const size_t gp = (size_t(ti - a.d.t0) * H + y) * W + x;  // local output pixel
        if (cnt <= 0) {
            latch(a.err, kErrWpsum);
            continue;
        }
        const float fc = float(cnt);
        reinterpret_cast<float4*>(out + gp * a.d.f)[cg0 + c] = make_float4(sum.x / fc, sum.y / fc, sum.z / fc, sum.w / fc);
        if (c == 0 && cg0 == 0 && counts) counts[gp] = cnt;
    }
}

#ifndef SNLS_WQ_TILE
#define SNLS_WQ_TILE 16
#endif
template <int P, int G, int FG>
int launch_wpsum_query(const AggArgs& a, float* out, int32_t* counts, cudaStream_t st) {
    constexpr int TY = SNLS_WQ_TILE, TX = SNLS_WQ_TILE;
    const int s0 = a.d.stride0;
    // grid rows meeting a tile aligned to TY (tiles start at multiples of TY)
    const int nqy = (TY + s0 - 2) / s0 + (TY % s0 == 0 ? 1 : 2);
    const int nqx = (TX + s0 - 2) / s0 + (TX % s0 == 0 ? 1 : 2);
    const int nq = nqy * nqx;
    const size_t smem = size_t(nq) * P * P * G * sizeof(float4);
    if (smem > 200 * 1024) return 0;
    ensure_smem(wpsum_query_kernel<P, G, FG, TY, TX>, smem);
    const int tiles = ((a.d.w + TX - 1) / TX) * ((a.d.h + TY - 1) / TY);
    const dim3 grid(unsigned(int64_t(a.d.nt) * tiles), FG / G);
    wpsum_query_kernel<P, G, FG, TY, TX><<<grid, 256, smem, st>>>(a, out, counts);
    return 1;
}

// ---- two-pass patch wpsum (wide patches: ps 5 / 7) --------------------------------------
// Pass 1, wpsum_patch_kernel: NL lanes per query (one channel pair each, packed FFMA2) sum the
// softmax-weighted bilinear samples of all L neighbours over the query's ps x ps patch in
// registers -- each (query, l) reads its (ps+1)^2 raw V block once, row by row -- and store
// the summed patch to a stream-ordered scratch [row][ps*ps][F].  RS > 1 splits the patch
// rows over RS lane groups (fewer registers, (ps+RS)/ps the block loads).  Pass 2,
// wpsum_combine_kernel: every output pixel sums its contributing patch pixels in the
// reference's fixed order (aggregate.cpp:156-188) and divides by the count.  The same
// arithmetic in the same order as wpsum_query_kernel (pass 1 = its phase A, pass 2 = its
// phase B), without its per-tile recomputation of the patches that straddle tiles (ps 7 at
// s0 4: 36 queries meet a 16 x 16 tile that owns 16) or parking 49 patch pixels x F per
// query in shared memory (which does not fit at ps 7, F 64).
#ifndef SNLS_WPP_MINB
#define SNLS_WPP_MINB 3
#endif
template <int P, int NL, int RS>
__global__ void __launch_bounds__(256, SNLS_WPP_MINB) wpsum_patch_kernel(AggArgs a, float* __restrict__ patch) {
    constexpr int HP = P / 2, R = (P + RS - 1) / RS, F = 2 * NL;
    const int64_t unit = (int64_t(blockIdx.x) * 256 + threadIdx.x) / NL;
    const int c = threadIdx.x % NL;  // this lane's channel pair
    const bool valid = unit / RS < a.d.rows;
    const int64_t row = valid ? unit / RS : a.d.rows - 1;  // (idle lanes still shuffle)
    const int i0 = int(unit % RS) * R;  // first patch row of this lane group
    int qt, qy, qx;
    row_coords(a.d, row, qt, qy, qx);
    const int H = a.d.h, W = a.d.w;
    const unsigned rowp = unsigned(W) * NL;  // u64 (channel pairs) per image row
    const u64* vbase = reinterpret_cast<const u64*>(a.v) + c;
    u64 acc[R][P];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < P; ++j) acc[i][j] = 0ull;
    for (int l0 = 0; l0 < a.topl; l0 += NL) {
        // lane c decodes neighbour l0 + c (frame, integer corner, softmax-weighted bilinear
        // weights) once; the group then walks the neighbours in order through shuffles, so
        // the V loads of a neighbour wait on no offset load
        int dkt = qt, dby = 0, dbx = 0;
        float d00 = 0.f, d01 = 0.f, d10 = 0.f, d11 = 0.f;
        if (l0 + c < a.topl) {
            const size_t e = size_t(row) * a.topl + l0 + c;
            const float* o = a.offsets + e * 3;
            dkt = qt + int(roundf(__ldg(o)));
            if (dkt < 0 || dkt >= a.d.t) {  // "offsets leave the clip" (aggregate.cpp:108-109)
                if (valid) latch(a.err, kErrWpsum);
                dkt = qt;
            }
            const float oy = __ldg(o + 1), ox = __ldg(o + 2);
            const float fly = floorf(oy), flx = floorf(ox);
            const float fy = oy - fly, fx = ox - flx;
            const float wv = __ldg(a.weights + e);
            d00 = wv * ((1.f - fy) * (1.f - fx));
            d01 = wv * ((1.f - fy) * fx);
            d10 = wv * (fy * (1.f - fx));
            d11 = wv * (fy * fx);
            // sample (i, j) sits between raw rows by+i, by+i+1 and cols bx+j, bx+j+1
            dby = qy - HP + int_base(fly) + i0;
            dbx = qx - HP + int_base(flx);
        }
        const int nl = min(NL, a.topl - l0);
        for (int k = 0; k < nl; ++k) {
            const int kt = __shfl_sync(0xffffffffu, dkt, k, NL);
            const int by = __shfl_sync(0xffffffffu, dby, k, NL), bx = __shfl_sync(0xffffffffu, dbx, k, NL);
            const float w00 = __shfl_sync(0xffffffffu, d00, k, NL), w01 = __shfl_sync(0xffffffffu, d01, k, NL);
            const float w10 = __shfl_sync(0xffffffffu, d10, k, NL), w11 = __shfl_sync(0xffffffffu, d11, k, NL);
            const u64 W00 = pk2(w00, w00), W01 = pk2(w01, w01), W10 = pk2(w10, w10), W11 = pk2(w11, w11);
            const u64* vf = vbase + size_t(kt) * H * rowp;
            const bool inside = by >= 0 && by + R < H && bx >= 0 && bx + P < W;
            auto load_row = [&](int i, u64* dst) {
                if (inside) {
                    const u64* p0 = vf + (unsigned(by + i) * rowp + unsigned(bx) * NL);
#pragma unroll
                    for (int j = 0; j <= P; ++j) dst[j] = __ldg(p0 + j * NL);
                } else {  // reflected border taps (tensor.cpp:31-48)
                    const unsigned r = unsigned(reflect_near(by + i, H)) * rowp;
#pragma unroll
                    for (int j = 0; j <= P; ++j) dst[j] = __ldg(vf + (r + unsigned(reflect_near(bx + j, W)) * NL));
                }
            };
            u64 top[P + 1], bot[P + 1];
            load_row(0, top);
#pragma unroll
            for (int i = 0; i < R; ++i) {
                if (RS > 1 && P % R != 0 && i0 + i >= P) break;  // the last group's short slice
                load_row(i + 1, bot);
#pragma unroll
                for (int j = 0; j < P; ++j)
                    acc[i][j] = fma2(W11, bot[j + 1], fma2(W10, bot[j], fma2(W01, top[j + 1], fma2(W00, top[j], acc[i][j]))));
#pragma unroll
                for (int j = 0; j <= P; ++j) top[j] = bot[j];
            }
        }
    }
    if (!valid) return;
    u64* dst = reinterpret_cast<u64*>(patch + (size_t(row) * P + i0) * P * F) + c;
#pragma unroll
    for (int i = 0; i < R; ++i)
        if (RS == 1 || i0 + i < P)
#pragma unroll
            for (int j = 0; j < P; ++j) dst[(i * P + j) * NL] = acc[i][j];
}

// S0 > 0: the stride as a compile-time constant (its divisions become multiplies); patch
// indices are 32-bit (the launcher checks rows * ps^2 * FG < 2^31).
template <int P, int FG, int S0>
__global__ void __launch_bounds__(256) wpsum_combine_kernel(AggArgs a, const float* __restrict__ patch,
                                                            float* __restrict__ out,
                                                            int32_t* __restrict__ counts) {
    constexpr int HP = P / 2;
    const int H = a.d.h, W = a.d.w, st = S0 > 0 ? S0 : a.d.stride0;
    // grid: x = pixels of one image row (FG lanes each), y = frame * H + row
    const int idx = int(blockIdx.x) * 256 + threadIdx.x;
    const int x = idx / FG, c = idx % FG;
    if (x >= W) return;
    const int y = int(blockIdx.y % unsigned(H));
    const int ti = a.d.t0 + int(blockIdx.y / unsigned(H));
    const int64_t gp = (int64_t(ti - a.d.t0) * H + y) * W + x;  // local output pixel
    const float4* pv = reinterpret_cast<const float4*>(patch) + c;
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    int cnt = 0;
    const unsigned frame_rows = unsigned(ti - a.d.t0) * unsigned(a.d.nh * a.d.nw);
    auto add = [&](int gy, int gx, int si, int sj) {
        const unsigned row = frame_rows + unsigned(gy * a.d.nw + gx);
        const float4 v = __ldg(pv + ((row * P + unsigned(si)) * P + unsigned(sj)) * FG);
        sum.x += v.x;
        sum.y += v.y;
        sum.z += v.z;
        sum.w += v.w;
        ++cnt;
    };
    const AxisUnits uy = axis_units(y, st, HP, (a.d.nh - 1) * st);
    const AxisUnits ux = axis_units(x, st, HP, (a.d.nw - 1) * st);
    for (int iy = 0; iy < uy.n; ++iy) {
        const int py = iy == 0 ? uy.p0 : uy.p1;
        for (int ix = 0; ix < ux.n; ++ix) {
            const int px = ix == 0 ? ux.p0 : ux.p1;
            add((y - py) / st, (x - px) / st, py + HP, px + HP);
        }
    }
    const int gy = owner_index(y, st, a.d.nh), gx = owner_index(x, st, a.d.nw);
    if (abs(y - gy * st) > HP || abs(x - gx * st) > HP)
        add(gy, gx, clampi(y - gy * st, HP) + HP, clampi(x - gx * st, HP) + HP);
    if (cnt <= 0) {
        latch(a.err, kErrWpsum);
        return;
    }
    const float fc = float(cnt);
    reinterpret_cast<float4*>(out + gp * a.d.f)[c] = make_float4(sum.x / fc, sum.y / fc, sum.z / fc, sum.w / fc);
    if (c == 0 && counts) counts[gp] = cnt;
}

// The patch scratch comes from the device's stream-ordered pool (cudaMallocAsync /
// cudaFreeAsync on the launching stream): no shared workspace, so two pipeline chunks on
// different streams never race on it, and with the pool's release threshold raised the
// allocation is a pool hit after the first call.
inline void keep_pool(cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex m;
    static std::set<int> done;
    std::lock_guard<std::mutex> lk(m);
    if (done.count(dev)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done.insert(dev);
    (void)st;
}

template <int P, int NL, int RS>
int launch_wpsum_patch(const AggArgs& a, float* out, int32_t* counts, cudaStream_t st) {
    keep_pool(st);
    const size_t bytes = size_t(a.d.rows) * P * P * a.d.f * sizeof(float);
    void* patch = nullptr;
    if (cudaMallocAsync(&patch, bytes, st) != cudaSuccess) {
        cudaGetLastError();
        return 0;  // caller falls back to the one-pass gather
    }
    const int64_t threads = a.d.rows * RS * NL;
    wpsum_patch_kernel<P, NL, RS><<<unsigned((threads + 255) / 256), 256, 0, st>>>(a, static_cast<float*>(patch));
    constexpr int FG = NL / 2;
    const dim3 cgrid(unsigned((a.d.w * FG + 255) / 256), unsigned(a.d.nt * a.d.h));
    const float* pp = static_cast<const float*>(patch);
    if (a.d.stride0 == 4)
        wpsum_combine_kernel<P, FG, 4><<<cgrid, 256, 0, st>>>(a, pp, out, counts);
    else
        wpsum_combine_kernel<P, FG, 0><<<cgrid, 256, 0, st>>>(a, pp, out, counts);
    cudaFreeAsync(patch, st);
    return 2;
}

int wpsum_patch_rs() {
    static const int rs = [] {
        const char* e = std::getenv("SNLS_WPSUM_RS");  // A/B: 0 = one-pass gather, 1 / 2 / 4 slices
        return e ? std::atoi(e) : 4;
    }();
    return rs;
}

int wpsum_patch3() {
    static const int on = [] {
        const char* e = std::getenv("SNLS_WPSUM_PATCH3");
        return e ? std::atoi(e) : 0;
    }();
    return on;
}

int launch_wpsum_patch_any(const AggArgs& a, float* out, int32_t* counts, cudaStream_t st) {
    const int rs = wpsum_patch_rs();
    if (rs <= 0 || int64_t(a.d.nt) * a.d.h > 65535) return 0;  // (combine grid.y)
    if (a.d.rows * a.ps * a.ps * (a.d.f / 4) >= (int64_t(1) << 31)) return 0;  // 32-bit patch index
    if (a.ps == 7 && a.d.f == 64)
        return rs == 4   ? launch_wpsum_patch<7, 32, 4>(a, out, counts, st)
               : rs == 2 ? launch_wpsum_patch<7, 32, 2>(a, out, counts, st)
                         : launch_wpsum_patch<7, 32, 1>(a, out, counts, st);
    if (a.ps == 7 && a.d.f == 32)
        return rs == 4   ? launch_wpsum_patch<7, 16, 4>(a, out, counts, st)
               : rs == 2 ? launch_wpsum_patch<7, 16, 2>(a, out, counts, st)
                         : launch_wpsum_patch<7, 16, 1>(a, out, counts, st);
    if (a.ps == 3 && wpsum_patch3()) {  // A/B: the query-centric kernel is the default at ps 3
        if (a.d.f == 32) return launch_wpsum_patch<3, 16, 1>(a, out, counts, st);
        if (a.d.f == 64) return launch_wpsum_patch<3, 32, 1>(a, out, counts, st);
    }
    if (a.ps == 5 && a.d.f == 64) return launch_wpsum_patch<5, 32, 1>(a, out, counts, st);
    if (a.ps == 5 && a.d.f == 32) return launch_wpsum_patch<5, 16, 1>(a, out, counts, st);
    return 0;
}

int launch_wpsum_query_any(const AggArgs& a, float* out, int32_t* counts, cudaStream_t st) {
    if (a.d.f % 4 != 0) return 0;
    const int FG = a.d.f / 4;
    // channel slices of 8 float4 (128 B per pixel): slices of 4 measured slower (c4 0.54 ->
    // 0.71 ms, c5 19.0 -> 25.2 ms), one 16-wide slice holds 1 CTA/SM (c5 27.3 ms)
    if (a.ps == 3) {
        if (FG == 8) return launch_wpsum_query<3, 8, 8>(a, out, counts, st);
        if (FG == 16) return launch_wpsum_query<3, 8, 16>(a, out, counts, st);  // two channel slices
        if (FG == 4) return launch_wpsum_query<3, 4, 4>(a, out, counts, st);
        if (FG == 2) return launch_wpsum_query<3, 2, 2>(a, out, counts, st);
    }
    if (a.ps == 1) {
        if (FG == 8) return launch_wpsum_query<1, 8, 8>(a, out, counts, st);
        if (FG == 16) return launch_wpsum_query<1, 8, 16>(a, out, counts, st);
    }
    return 0;
}

// softmax_rows (aggregate.cpp:16-37): one thread per row.
__global__ void softmax_kernel(int64_t rows, int l, float beta, const float* __restrict__ sims,
                               float* __restrict__ w, int* err) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* s = sims + size_t(r) * l;
    float m = -INFINITY;
    for (int j = 0; j < l; ++j) {
        const float z = beta * s[j];
        if (!isfinite(z)) latch(err, kErrSoftmax);
        m = fmaxf(m, z);
    }
    float sum = 0.f;
    for (int j = 0; j < l; ++j) {
        const float e = __expf(beta * s[j] - m);
        w[size_t(r) * l + j] = e;
        sum += e;
    }
    const float inv = 1.f / sum;
    for (int j = 0; j < l; ++j) w[size_t(r) * l + j] *= inv;
}

// wpsum backward (aggregate.cpp:351-408): one thread per (row, neighbour, channel group);
// dW partial sums reduced with one atomic per thread, dV scattered through the 4 taps.
template <int VEC, bool DET = false>
__global__ void __launch_bounds__(256) wpsum_bwd_kernel(AggArgs a, const float* __restrict__ go,
                                                        const int32_t* __restrict__ counts,
                                                        float* __restrict__ dv,
                                                        float* __restrict__ dw, WbwdFixed fxp) {
    const int groups = a.d.f / VEC;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= a.d.rows * a.topl * groups) return;
    const int64_t e = idx / groups;
    const int c = int(idx % groups) * VEC;
    const int64_t row = e / a.topl;
    int ti, qy, qx;
    row_coords(a.d, row, ti, qy, qx);
    const int st = a.d.stride0, half = a.ps / 2;
    const float* o = a.offsets + size_t(e) * 3;
    const int kt = ti + int(roundf(o[0]));
    const float oy = o[1], ox = o[2];
    const float wv = a.weights[e];
    float dw_acc = 0.f;
    int ylo, yhi, xlo, xhi;
    cell_span(qy / st, st, a.d.nh, a.d.h, ylo, yhi);
    cell_span(qx / st, st, a.d.nw, a.d.w, xlo, xhi);
    const int side = 2 * half + 1, nfoot = side * side;
    const int cw = xhi - xlo + 1, ncell = (yhi - ylo + 1) * cw;
    for (int it = 0; it < nfoot + ncell; ++it) {
        int y, x, pyu, pxu;
        if (it < nfoot) {  // for_each_write (aggregate.cpp:81-100)
            pyu = it / side - half;
            pxu = it % side - half;
            y = qy + pyu;
            x = qx + pxu;
            if (y < 0 || y >= a.d.h || x < 0 || x >= a.d.w) continue;
        } else {
            const int j = it - nfoot;
            y = ylo + j / cw;
            x = xlo + j % cw;
            if (abs(y - qy) <= half && abs(x - qx) <= half) continue;
            pyu = clampi(y - qy, half);
            pxu = clampi(x - qx, half);
        }
        const float inv_cnt = 1.f / float(counts[(size_t(ti - a.d.t0) * a.d.h + y) * a.d.w + x]);
        int iy, ix;
        float fy, fx;
        split_pos(qy + pyu, oy, iy, fy, a.d.h);
        split_pos(qx + pxu, ox, ix, fx, a.d.w);
        const Taps t = taps_from(iy, fy, ix, fx, a.d.h, a.d.w);
        const float* gp = go + vidx(a.d, ti - a.d.t0, y, x) + c;
        const size_t i00 = vidx(a.d, kt, t.y0, t.x0) + c, i01 = vidx(a.d, kt, t.y0, t.x1) + c;
        const size_t i10 = vidx(a.d, kt, t.y1, t.x0) + c, i11 = vidx(a.d, kt, t.y1, t.x1) + c;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const float g = __ldg(gp + j) * inv_cnt;
            const float sample = blend(t, __ldg(a.v + i00 + j), __ldg(a.v + i01 + j),
                                       __ldg(a.v + i10 + j), __ldg(a.v + i11 + j));
            dw_acc = fmaf(g, sample, dw_acc);
            const float gv = g * wv;
            if constexpr (DET) {
                const double sv = fxp.scale[0];
                fixed_add(fxp.dvi + i00 + j, gv * t.w00, sv);
                fixed_add(fxp.dvi + i01 + j, gv * t.w01, sv);
                fixed_add(fxp.dvi + i10 + j, gv * t.w10, sv);
                fixed_add(fxp.dvi + i11 + j, gv * t.w11, sv);
            } else {
                atomicAdd(dv + i00 + j, gv * t.w00);
                atomicAdd(dv + i01 + j, gv * t.w01);
                atomicAdd(dv + i10 + j, gv * t.w10);
                atomicAdd(dv + i11 + j, gv * t.w11);
            }
        }
    }
    if constexpr (DET) fixed_add(fxp.dwi + e, dw_acc, fxp.scale[1]);
    else atomicAdd(dw + e, dw_acc);
}

// Row-centric wpsum backward (aggregate.cpp:351-460): one warp per (query row, 32-channel
// slice), lane = channel.  Every write of a query (footprint pixel, or cell-completion
// pixel through its clamped patch pixel, aggregate.cpp:80-100) samples V at a patch pixel
// (i, j) of that query, so the upstream gradient is first folded per patch pixel:
// Gs[i][j] = sum over the writes mapped to (i, j) of grad_out / count -- independent of the
// neighbour l.  Then per neighbour: dW = sum Gs * sample (warp-reduced, one atomic per
// slice) and dV gets w * Gs through the taps, pre-reduced on the (ps+1)^2 raw block two rows
// at a time ((ps+1)^2 coalesced atomics per entry instead of 4 x writes).
#ifndef SNLS_WBWD_GSSM
#define SNLS_WBWD_GSSM 1
#endif
constexpr bool kGsSm = SNLS_WBWD_GSSM != 0;
#ifndef SNLS_WBWD_ROLL
#define SNLS_WBWD_ROLL 1
#endif

// FT > 0: compile-time channel count; raw blocks inside the frame use immediate column
// offsets from one row base (no reflection / per-element address math), as search_bwd_rows.
template <int P, int FT = 0, bool DET = false>
__global__ void __launch_bounds__(128, kGsSm ? 4 : 3) wpsum_bwd_rows(AggArgs a, const float* __restrict__ go,
                                                         const int32_t* __restrict__ counts,
                                                         float* __restrict__ dv, float* __restrict__ dw,
                                                         WbwdFixed fxp) {
    constexpr int HP = P / 2;
    const int slices = (a.d.f + 31) / 32;
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= a.d.rows * slices) return;  // warp-uniform
    const int64_t row = wid / slices;
    const int c = int(wid % slices) * 32 + lane;
    const bool act = c < a.d.f;
    const int cc = act ? c : 0;
    int ti, qy, qx;
    row_coords(a.d, row, ti, qy, qx);
    const int H = a.d.h, W = a.d.w, st = a.d.stride0;
    const size_t F = size_t(a.d.f), rowF = size_t(W) * F, frameF = size_t(H) * rowF;
    // ---- fold the upstream gradient onto the patch pixels (kGsSm: parked in shared memory,
    // each lane its own channel, no barrier)
    __shared__ float s_gs[kGsSm ? 4 : 1][kGsSm ? P * P : 1][32];
    float* sgs = &s_gs[kGsSm ? threadIdx.x >> 5 : 0][0][lane];
    float gs[P][P];
    // grad_out / counts hold the output frames [t0, t0 + nt) (frame-range form)
    const float* gob = go + size_t(ti - a.d.t0) * frameF + cc;
    const int32_t* cb = counts + size_t(ti - a.d.t0) * H * W;
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const int y = qy + i - HP, x = qx + j - HP;
            float v = 0.f;
            if (act && y >= 0 && y < H && x >= 0 && x < W) {
                const int pix = y * W + x;
                v = __ldg(gob + size_t(pix) * F) * (1.f / float(__ldg(cb + pix)));
            }
            gs[i][j] = v;
        }
    int ylo, yhi, xlo, xhi;  // the query's stride cell (aggregate.cpp:68-100)
    cell_span(qy / st, st, a.d.nh, H, ylo, yhi);
    cell_span(qx / st, st, a.d.nw, W, xlo, xhi);
    if (ylo < qy - HP || yhi > qy + HP || xlo < qx - HP || xhi > qx + HP) {  // cell completion
        for (int y = ylo; y <= yhi; ++y)
            for (int x = xlo; x <= xhi; ++x) {
                if (abs(y - qy) <= HP && abs(x - qx) <= HP) continue;
                const int pi = clampi(y - qy, HP) + HP, pj = clampi(x - qx, HP) + HP;
                const int pix = y * W + x;
                const float v = act ? __ldg(gob + size_t(pix) * F) * (1.f / float(__ldg(cb + pix))) : 0.f;
#pragma unroll
                for (int i = 0; i < P; ++i)
#pragma unroll
                    for (int j = 0; j < P; ++j) gs[i][j] += (i == pi && j == pj) ? v : 0.f;
            }
    }
    if constexpr (kGsSm) {
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
            for (int j = 0; j < P; ++j) sgs[(i * P + j) * 32] = gs[i][j];
    }
    auto gsv = [&](int i, int j) { return kGsSm ? sgs[(i * P + j) * 32] : gs[i][j]; };
    // ---- per neighbour: dW and the dV block scatter
    for (int l = 0; l < a.topl; ++l) {
        const int64_t e = row * a.topl + l;
        const float* o = a.offsets + size_t(e) * 3;
        const int kt = ti + int(roundf(__ldg(o)));
        if (kt < 0 || kt >= a.d.t) {  // "offsets leave the clip" (aggregate.cpp:108-109)
            if (lane == 0) latch(a.err, kErrWpsum);
            continue;
        }
        const float oy = __ldg(o + 1), ox = __ldg(o + 2);
        const float fly = floorf(oy), flx = floorf(ox);
        const float fy = oy - fly, fx = ox - flx;
        const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx;
        const float w10 = fy * (1.f - fx), w11 = fy * fx;
        const float wv = __ldg(a.weights + e);
        const int by = qy - HP + int_base(fly), bx = qx - HP + int_base(flx);
        const float* __restrict__ vb = a.v + size_t(kt) * frameF + cc;
        const size_t dvo = size_t(kt) * frameF + cc;
        const double fsv = DET ? fxp.scale[0] : 0.0;
        auto put = [&](size_t idx, float val) {
            if constexpr (DET) fixed_add(fxp.dvi + idx, val, fsv);
            else atomicAdd(dv + idx, val);
        };
        float dwl = 0.f;
        auto body = [&](auto fast_tag) {
            constexpr bool FAST = decltype(fast_tag)::value;
            unsigned bcol[FAST ? 1 : P + 1];
            if constexpr (!FAST) {
#pragma unroll
                for (int j = 0; j <= P; ++j) bcol[j] = unsigned(reflect_near(bx + j, W)) * unsigned(a.d.f);
            }
            auto colo = [&](int j) -> size_t { return FAST ? size_t(j) * FT : size_t(bcol[FAST ? 0 : j]); };
            const size_t xo = FAST ? size_t(bx) * FT : 0;
            auto rowo = [&](int r) -> size_t {
                return FAST ? size_t(by + r) * rowF + xo : size_t(reflect_near(by + r, H)) * rowF;
            };
            float ra[P + 1], rb[P + 1], ka[P + 1], kn[P + 1];
            size_t roa = rowo(0), rob = rowo(1);
#pragma unroll
            for (int j = 0; j <= P; ++j) {
                ra[j] = act ? __ldg(vb + roa + colo(j)) : 0.f;
                rb[j] = act ? __ldg(vb + rob + colo(j)) : 0.f;
                ka[j] = 0.f;
            }
            // rolled for wide patches: unrolled, the two block bodies of ps 7 are ~10k SASS
            // instructions and the warps wait on instruction fetch
            constexpr bool kRoll = SNLS_WBWD_ROLL && kGsSm && P > 3;
#pragma unroll(kRoll ? 1 : P)
            for (int i = 0; i < P; ++i) {
                // raw row i+2 is loaded one row ahead (its latency overlaps row i's arithmetic)
                float rn[P + 1];
                const size_t ron = rowo(i + 2);
                if (i + 1 < P) {
#pragma unroll
                    for (int j = 0; j <= P; ++j) rn[j] = act ? __ldg(vb + ron + colo(j)) : 0.f;
                }
#pragma unroll
                for (int j = 0; j <= P; ++j) kn[j] = 0.f;
#pragma unroll
                for (int j = 0; j < P; ++j) {
                    const float smp = w00 * ra[j] + w01 * ra[j + 1] + w10 * rb[j] + w11 * rb[j + 1];
                    const float gij = gsv(i, j);
                    dwl = fmaf(gij, smp, dwl);
                    const float gv = gij * wv;
                    ka[j] += gv * w00;
                    ka[j + 1] += gv * w01;
                    kn[j] += gv * w10;
                    kn[j + 1] += gv * w11;
                }
                if (act) {
#pragma unroll
                    for (int j = 0; j <= P; ++j) put(dvo + roa + colo(j), ka[j]);
                }
#pragma unroll
                for (int j = 0; j <= P; ++j) {
                    ra[j] = rb[j];
                    if (i + 1 < P) rb[j] = rn[j];
                    ka[j] = kn[j];
                }
                roa = rob;
                rob = ron;
            }
            if (act) {
#pragma unroll
                for (int j = 0; j <= P; ++j) put(dvo + roa + colo(j), ka[j]);
            }
        };
        if (FT > 0 && by >= 0 && by + P < H && bx >= 0 && bx + P < W)  // uniform: one row per warp
            body(std::integral_constant<bool, (FT > 0)>{});
        else
            body(std::false_type{});
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) dwl += __shfl_xor_sync(0xffffffffu, dwl, m);
        if (lane == 0) {
            if constexpr (DET) fixed_add(fxp.dwi + e, dwl, fxp.scale[1]);
            else atomicAdd(dw + e, dwl);
        }
    }
}

// A/B (SNLS_WBWD_WIN=1): the north star's shared-memory pre-reduction for the dV scatter.  One
// warp per (row, 32-channel slice) as wpsum_bwd_rows; the row's neighbours are taken frame by
// frame, and when two or more of a frame's raw blocks (all inside the frame) fit a WS x WS
// window, their contributions are summed in a per-warp shared window (lane = channel, no
// conflicts) and each touched pixel gets ONE global reduction -- a query's neighbours cluster
// (scripts/micro/prereduce_potential.py: per (query, frame) the block union is ~half the
// contributions).  Other blocks scatter directly.  Non-deterministic mode only.
template <int P, int FT, int WS>
__global__ void __launch_bounds__(128, 2) wpsum_bwd_win(AggArgs a, const float* __restrict__ go,
                                                        const int32_t* __restrict__ counts,
                                                        float* __restrict__ dv, float* __restrict__ dw) {
    constexpr int HP = P / 2, F = FT, SL = FT / 32;
    extern __shared__ float s_wb[];  // [4][P*P][32] gradient patch, then [4][WS*WS][32] windows
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (wid >= a.d.rows * SL) return;  // warp-uniform
    const int64_t row = wid / SL;
    const int c = int(wid % SL) * 32 + lane;
    float* sgs = s_wb + size_t(warp) * P * P * 32 + lane;
    float* win = s_wb + size_t(4) * P * P * 32 + size_t(warp) * WS * WS * 32 + lane;
    int ti, qy, qx;
    row_coords(a.d, row, ti, qy, qx);
    const int H = a.d.h, W = a.d.w, st = a.d.stride0;
    const size_t rowF = size_t(W) * F, frameF = size_t(H) * rowF;
    const float* gob = go + size_t(ti - a.d.t0) * frameF + c;
    const int32_t* cb = counts + size_t(ti - a.d.t0) * H * W;
    for (int i = 0; i < P; ++i)
        for (int j = 0; j < P; ++j) {
            const int y = qy + i - HP, x = qx + j - HP;
            float v = 0.f;
            if (y >= 0 && y < H && x >= 0 && x < W) {
                const int pix = y * W + x;
                v = __ldg(gob + size_t(pix) * F) * (1.f / float(__ldg(cb + pix)));
            }
            sgs[(i * P + j) * 32] = v;
        }
    int ylo, yhi, xlo, xhi;
    cell_span(qy / st, st, a.d.nh, H, ylo, yhi);
    cell_span(qx / st, st, a.d.nw, W, xlo, xhi);
    if (ylo < qy - HP || yhi > qy + HP || xlo < qx - HP || xhi > qx + HP) {
        for (int y = ylo; y <= yhi; ++y)
            for (int x = xlo; x <= xhi; ++x) {
                if (abs(y - qy) <= HP && abs(x - qx) <= HP) continue;
                const int pix = y * W + x;
                sgs[((clampi(y - qy, HP) + HP) * P + clampi(x - qx, HP) + HP) * 32] +=
                    __ldg(gob + size_t(pix) * F) * (1.f / float(__ldg(cb + pix)));
            }
    }
    // lane l < topl decodes neighbour l
    int dkt = -1, dby = 0, dbx = 0;
    if (lane < a.topl) {
        const float* o = a.offsets + size_t(row * a.topl + lane) * 3;
        dkt = ti + int(roundf(__ldg(o)));
        if (dkt < 0 || dkt >= a.d.t) {
            latch(a.err, kErrWpsum);
            dkt = -1;
        } else {
            dby = qy - HP + int_base(floorf(__ldg(o + 1)));
            dbx = qx - HP + int_base(floorf(__ldg(o + 2)));
        }
    }
    const bool inside = dkt >= 0 && dby >= 0 && dby + P < H && dbx >= 0 && dbx + P < W;
    unsigned remaining = __ballot_sync(0xffffffffu, dkt >= 0);
    while (remaining) {
        const int kt0 = __shfl_sync(0xffffffffu, dkt, __ffs(remaining) - 1);
        const unsigned members = __ballot_sync(0xffffffffu, dkt == kt0) & remaining;
        remaining &= ~members;
        const unsigned fm = __ballot_sync(0xffffffffu, inside) & members;
        const bool mine = (fm >> lane) & 1u;
        const int y0 = __reduce_min_sync(0xffffffffu, mine ? dby : 0x7fffffff);
        const int y1 = __reduce_max_sync(0xffffffffu, mine ? dby : -0x7fffffff);
        const int x0 = __reduce_min_sync(0xffffffffu, mine ? dbx : 0x7fffffff);
        const int x1 = __reduce_max_sync(0xffffffffu, mine ? dbx : -0x7fffffff);
        const int BY = y1 - y0 + P + 1, BX = x1 - x0 + P + 1;
        const bool use_win = __popc(fm) >= 2 && BY <= WS && BX <= WS;
        if (use_win)
            for (int k = 0; k < BY * WS; ++k) win[k * 32] = 0.f;
        for (unsigned mm = members; mm; mm &= mm - 1) {
            const int l = __ffs(mm) - 1;
            const int64_t e = row * a.topl + l;
            const float* o = a.offsets + size_t(e) * 3;
            const float oy = __ldg(o + 1), ox = __ldg(o + 2);
            const float fly = floorf(oy), flx = floorf(ox);
            const float fy = oy - fly, fx = ox - flx;
            const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx;
            const float w10 = fy * (1.f - fx), w11 = fy * fx;
            const float wv = __ldg(a.weights + e);
            const int by = __shfl_sync(0xffffffffu, dby, l), bx = __shfl_sync(0xffffffffu, dbx, l);
            const bool fast = (fm >> l) & 1u;
            const bool towin = use_win && fast;
            const float* __restrict__ vb = a.v + size_t(kt0) * frameF + c;
            const size_t dvo = size_t(kt0) * frameF + c;
            float dwl = 0.f;
            unsigned bcol[P + 1];
#pragma unroll
            for (int j = 0; j <= P; ++j) bcol[j] = unsigned(fast ? bx + j : reflect_near(bx + j, W)) * unsigned(F);
            auto rowo = [&](int r) -> size_t { return size_t(fast ? by + r : reflect_near(by + r, H)) * rowF; };
            auto put = [&](int r, size_t ro, int j, float val) {
                if (towin) win[((by - y0 + r) * WS + (bx - x0 + j)) * 32] += val;
                else atomicAdd(dv + dvo + ro + bcol[j], val);
            };
            float ra[P + 1], rb[P + 1], ka[P + 1], kn[P + 1];
            size_t roa = rowo(0), rob = rowo(1);
#pragma unroll
            for (int j = 0; j <= P; ++j) {
                ra[j] = __ldg(vb + roa + bcol[j]);
                rb[j] = __ldg(vb + rob + bcol[j]);
                ka[j] = 0.f;
            }
#pragma unroll 1
            for (int i = 0; i < P; ++i) {
                float rn[P + 1];
                const size_t ron = rowo(i + 2);
                if (i + 1 < P) {
#pragma unroll
                    for (int j = 0; j <= P; ++j) rn[j] = __ldg(vb + ron + bcol[j]);
                }
#pragma unroll
                for (int j = 0; j <= P; ++j) kn[j] = 0.f;
#pragma unroll
                for (int j = 0; j < P; ++j) {
                    const float smp = w00 * ra[j] + w01 * ra[j + 1] + w10 * rb[j] + w11 * rb[j + 1];
                    const float gij = sgs[(i * P + j) * 32];
                    dwl = fmaf(gij, smp, dwl);
                    const float gv = gij * wv;
                    ka[j] += gv * w00;
                    ka[j + 1] += gv * w01;
                    kn[j] += gv * w10;
                    kn[j + 1] += gv * w11;
                }
#pragma unroll
                for (int j = 0; j <= P; ++j) put(i, roa, j, ka[j]);
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
            for (int j = 0; j <= P; ++j) put(P, roa, j, ka[j]);
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) dwl += __shfl_xor_sync(0xffffffffu, dwl, m);
            if (lane == 0) atomicAdd(dw + e, dwl);
        }
        if (use_win) {  // one reduction per touched pixel of the window
            float* drow = dv + size_t(kt0) * frameF + c;
            for (int r = 0; r < BY; ++r)
                for (int j = 0; j < BX; ++j) {
                    const float val = win[(r * WS + j) * 32];
                    if (val != 0.f) atomicAdd(drow + size_t(y0 + r) * rowF + size_t(x0 + j) * F, val);
                }
        }
    }
}

#ifndef SNLS_WBWD_PAIRS
#define SNLS_WBWD_PAIRS 1
#endif
#ifndef SNLS_WBWD_WIN
#define SNLS_WBWD_WIN 0
#endif
#ifndef SNLS_WBWD_WS
#define SNLS_WBWD_WS 12
#endif
#ifndef SNLS_WBWD_LSPLIT
#define SNLS_WBWD_LSPLIT 1
#endif

template <int P, bool DET>
void launch_wpsum_bwd_rows(const AggArgs& a, const float* go, const int32_t* counts, float* dv,
                           float* dw, WbwdFixed fxp, cudaStream_t st) {
    // channel pairs for wide patches (and for every ps in deterministic mode: one dW writer
    // per entry); the one-channel-per-lane kernel otherwise
    if constexpr (SNLS_WBWD_WIN != 0 && !DET && P >= 5) {  // A/B build only (measured slower)
      if ((a.d.f == 64 || a.d.f == 32) && a.topl <= 32) {
        constexpr int WS = SNLS_WBWD_WS;
          auto go3 = [&](auto kern) {
              const size_t smem = size_t(4) * (P * P + WS * WS) * 32 * sizeof(float);
              ensure_smem(kern, smem);
              const int64_t warps = a.d.rows * (a.d.f / 32);
              kern<<<unsigned((warps + 3) / 4), 128, smem, st>>>(a, go, counts, dv, dw);
          };
          if (a.d.f == 64) go3(wpsum_bwd_win<P, 64, WS>);
          else go3(wpsum_bwd_win<P, 32, WS>);
          return;
      }
    }
    if (SNLS_WBWD_PAIRS && (P >= 5 || DET) && (a.d.f == 64 || a.d.f == 32)) {
        constexpr int LS = SNLS_WBWD_LSPLIT;
        auto go2 = [&](auto kern, int nl) {
            const size_t smem = size_t(128 / nl) * P * P * nl * sizeof(u64);
            ensure_smem(kern, smem);
            const int64_t units = a.d.rows * LS;
            const unsigned blocks = unsigned((units + 128 / nl - 1) / (128 / nl));
            kern<<<blocks, 128, smem, st>>>(a, go, counts, dv, dw, fxp);
        };
        if (a.d.f == 64) go2(wpsum_bwd_pairs<P, 32, LS, DET>, 32);
        else go2(wpsum_bwd_pairs<P, 16, LS, DET>, 16);
        return;
    }
    const int64_t warps = a.d.rows * ((a.d.f + 31) / 32);
    const unsigned blocks = unsigned((warps + 3) / 4);
    if (a.d.f == 64) wpsum_bwd_rows<P, 64, DET><<<blocks, 128, 0, st>>>(a, go, counts, dv, dw, fxp);
    else if (a.d.f == 32) wpsum_bwd_rows<P, 32, DET><<<blocks, 128, 0, st>>>(a, go, counts, dv, dw, fxp);
    else wpsum_bwd_rows<P, 0, DET><<<blocks, 128, 0, st>>>(a, go, counts, dv, dw, fxp);
}

template <bool DET>
void launch_wpsum_bwd_any(const AggArgs& a, const float* grad_out, const int32_t* counts, float* dv,
                          float* dw, WbwdFixed fxp, cudaStream_t st) {
    switch (a.ps) {
        case 1: launch_wpsum_bwd_rows<1, DET>(a, grad_out, counts, dv, dw, fxp, st); return;
        case 3: launch_wpsum_bwd_rows<3, DET>(a, grad_out, counts, dv, dw, fxp, st); return;
        case 5: launch_wpsum_bwd_rows<5, DET>(a, grad_out, counts, dv, dw, fxp, st); return;
        case 7: launch_wpsum_bwd_rows<7, DET>(a, grad_out, counts, dv, dw, fxp, st); return;
        default: break;
    }
    if (a.d.f % 4 == 0) {
        const int64_t n = a.d.rows * a.topl * (a.d.f / 4);
        wpsum_bwd_kernel<4, DET><<<unsigned((n + 255) / 256), 256, 0, st>>>(a, grad_out, counts, dv, dw, fxp);
    } else {
        const int64_t n = a.d.rows * a.topl * a.d.f;
        wpsum_bwd_kernel<1, DET><<<unsigned((n + 255) / 256), 256, 0, st>>>(a, grad_out, counts, dv, dw, fxp);
    }
}

// bounds[0..2] = max|grad_out|, max|weights|, max|v| (bits).  Every partial sum of dV is a sum
// of (row, l, written pixel) terms |g * w * tap| <= max|go| * max|w| (count >= 1, taps <= 1)
// over at most ps^2 + s0^2 written pixels per (row, l); a dW entry sums <= (ps^2 + s0^2) F
// terms |g * sample| <= max|go| * max|v|.
__global__ void wbwd_scales_kernel(const unsigned* bounds, int64_t entries, int ps, int s0, int f,
                                   double* scales) {
    const double gm = __uint_as_float(bounds[0]), wm = __uint_as_float(bounds[1]);
    const double vm = __uint_as_float(bounds[2]);
    const double px = double(ps) * ps + double(s0) * s0;
    scales[0] = pow2_scale(double(entries) * px * gm * wm * 1.001);
    scales[1] = pow2_scale(px * f * gm * vm * 1.001);
}

}  // namespace

int launch_softmax(int64_t rows, int l, float beta, const float* sims, float* weights, int* err,
                   cudaStream_t st) {
    softmax_kernel<<<unsigned((rows + 127) / 128), 128, 0, st>>>(rows, l, beta, sims, weights, err);
    return 1;
}

int launch_wpsum(const AggArgs& a, float* out, int32_t* counts, cudaStream_t st) {
    if (int64_t(a.d.t) * a.d.h * a.d.w < (int64_t(1) << 31))
        if (int n = launch_wpsum_patch_any(a, out, counts, st)) return n;
    if (int n = launch_wpsum_query_any(a, out, counts, st)) return n;
    if (int n = launch_tiled_agg_any(a, out, counts, 0, st)) return n;
    const int64_t npix = int64_t(a.d.nt) * a.d.h * a.d.w;
    if (a.d.f % 4 == 0) {
        const int64_t n = npix * (a.d.f / 4);
        wpsum_kernel<4><<<unsigned((n + 255) / 256), 256, 0, st>>>(a, out, counts);
    } else {
        const int64_t n = npix * a.d.f;
        wpsum_kernel<1><<<unsigned((n + 255) / 256), 256, 0, st>>>(a, out, counts);
    }
    return 1;
}

int launch_gather_stack(const AggArgs& a, float* out, cudaStream_t st) {
    if (int n = launch_tiled_agg_any(a, out, nullptr, 1, st)) return n;
    const int64_t npix = int64_t(a.d.nt) * a.d.h * a.d.w;
    if (a.d.f % 4 == 0) {
        const int64_t n = npix * (a.d.f / 4) * a.topl;
        gather_stack_kernel<4><<<unsigned((n + 255) / 256), 256, 0, st>>>(a, out);
    } else {
        const int64_t n = npix * a.d.f * a.topl;
        gather_stack_kernel<1><<<unsigned((n + 255) / 256), 256, 0, st>>>(a, out);
    }
    return 1;
}

int launch_wpsum_bwd(const AggArgs& a, const float* grad_out, const int32_t* counts, float* dv,
                     float* dw, cudaStream_t st) {
    launch_wpsum_bwd_any<false>(a, grad_out, counts, dv, dw, WbwdFixed{nullptr, nullptr, nullptr}, st);
    return 1;
}

// Deterministic mode (aggregate.cpp:439-450: dV gathered in a fixed order): int64 fixed-point
// dV (and multi-writer dW) with scales from exact maxima, then one conversion pass.  `work`
// returns scratch of the requested size (zeroed here).  dv / dw must be zeroed by the caller.
size_t wpsum_bwd_det_bytes(const AggArgs& a) {
    const int64_t nv = int64_t(a.d.t) * a.d.h * a.d.w * a.d.f;
    return 64 + size_t(nv + a.d.rows * a.topl) * sizeof(unsigned long long);
}

// Zero the scratch `w` (wpsum_bwd_det_bytes), take the exact maxima and the scales; fills the
// fixed-point sinks of `wp`.
void wpsum_bwd_det_prep(const AggArgs& a, const float* grad_out, void* w, WpsumBwdArgs& wp, cudaStream_t st) {
    const int64_t nv = int64_t(a.d.t) * a.d.h * a.d.w * a.d.f;
    const int64_t ne = a.d.rows * a.topl;
    char* c = static_cast<char*>(w);
    cudaMemsetAsync(c, 0, wpsum_bwd_det_bytes(a), st);
    double* scales = reinterpret_cast<double*>(c);  // [0] dV, [1] dW
    unsigned* bounds = reinterpret_cast<unsigned*>(c + 2 * sizeof(double));
    wp.dvi = reinterpret_cast<unsigned long long*>(c + 64);
    wp.dwi = wp.dvi + nv;
    wp.scale = scales;
    const int64_t ngo = int64_t(a.d.nt) * a.d.h * a.d.w * a.d.f;
    absmax_kernel<<<592, 256, 0, st>>>(grad_out, ngo, bounds + 0);
    absmax_kernel<<<148, 256, 0, st>>>(a.weights, ne, bounds + 1);
    absmax_kernel<<<592, 256, 0, st>>>(a.v, nv, bounds + 2);
    wbwd_scales_kernel<<<1, 1, 0, st>>>(bounds, ne, a.ps, a.d.stride0, a.d.f, scales);
}

// Fixed point -> dv (and dw where the kernel that ran had several writers per entry).
void wpsum_bwd_det_finish(const AggArgs& a, const WpsumBwdArgs& wp, bool dw_direct, cudaStream_t st) {
    const int64_t nv = int64_t(a.d.t) * a.d.h * a.d.w * a.d.f;
    const int64_t ne = a.d.rows * a.topl;
    fixed_to_float_kernel<<<unsigned(std::min<int64_t>((nv + 255) / 256, 4096)), 256, 0, st>>>(wp.dvi, wp.scale,
                                                                                               wp.dv, nv);
    if (!dw_direct)
        fixed_to_float_kernel<<<unsigned(std::min<int64_t>((ne + 255) / 256, 4096)), 256, 0, st>>>(
            wp.dwi, wp.scale + 1, wp.dw, ne);
}

int launch_wpsum_bwd_det(const AggArgs& a, const float* grad_out, const int32_t* counts, float* dv,
                         float* dw, const std::function<void*(size_t)>& work, cudaStream_t st) {
    void* w = work(wpsum_bwd_det_bytes(a));
    if (!w) return -1;
    WpsumBwdArgs wp{a, grad_out, counts, dv, dw, nullptr, nullptr, nullptr};
    wpsum_bwd_det_prep(a, grad_out, w, wp, st);
    launch_wpsum_bwd_any<true>(a, grad_out, counts, dv, dw, WbwdFixed{wp.dvi, wp.dwi, wp.scale}, st);
    // the channel-pair kernel writes dW directly (one writer per entry); the others through dwi
    const bool pairs = SNLS_WBWD_PAIRS && (a.d.f == 64 || a.d.f == 32) && a.ps <= 7 && a.ps % 2 == 1;
    wpsum_bwd_det_finish(a, wp, pairs, st);
    return pairs ? 7 : 8;
}

}  // namespace snls_gpu
