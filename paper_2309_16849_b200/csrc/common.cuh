// Shared device helpers for the sm_100a Shifted Non-Local Search kernels.
//
// Numerics: tensors are fp32 in HBM and the patch arithmetic is fp32 (FFMA pipe).  Sample
// positions are never formed as one fp32 number (qy + shift loses ~3e-5 relative at 512
// px): a position is an integer base plus an fp32 fraction, and flow shifts are
// accumulated in fp64 registers (once per query x frame, off the hot loop).
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

#include <cuda_runtime.h>

#include "snls_cuda.h"

namespace snls_gpu {

// Device-side domain-error latch bits (reported by snls_ctx_sync_check).
enum : int {
    kErrFflow = 1,      // "search fflow: flow holds a non-finite value"   flow.cpp:20-23
    kErrBflow = 2,      // "search bflow: flow holds a non-finite value"
    kErrSoftmax = 4,    // "softmax_rows: non-finite input"                 aggregate.cpp:25
    kErrWpsum = 8,      // "wpsum: offsets leave the clip or a pixel has no writers" :201
    kErrStack = 16,     // "gather_stack: offsets leave the clip"           aggregate.cpp:345
    kErrTopl = 32,      // "top_l: some row has fewer than L valid entries" search.cpp:466
};

// Video dims plus the query/output FRAME RANGE [t0, t0+nt) being processed.  `rows` counts
// the query rows of that range and kernels index outputs by the local row (global row -
// row0); `t` stays the full clip length, which decides which key frames exist
// (search.cpp:300).  The default range is the whole clip.
struct Dims {
    int t, h, w, f;
    int nh, nw, stride0;
    int64_t rows;
    int t0, nt;
    int64_t row0;
};

__host__ __device__ inline Dims make_dims(snls_dims d, int stride0) {
    Dims r;
    r.t = d.t;
    r.h = d.h;
    r.w = d.w;
    r.f = d.f;
    r.stride0 = stride0;
    r.nh = (d.h - 1) / stride0 + 1;
    r.nw = (d.w - 1) / stride0 + 1;
    r.rows = int64_t(d.t) * r.nh * r.nw;
    r.t0 = 0;
    r.nt = d.t;
    r.row0 = 0;
    return r;
}

__host__ __device__ inline Dims restrict_frames(Dims d, int t0, int t1) {
    d.t0 = t0;
    d.nt = t1 - t0;
    d.row0 = int64_t(t0) * d.nh * d.nw;
    d.rows = int64_t(d.nt) * d.nh * d.nw;
    return d;
}

// tensor.cpp:23-29: period-2(n-1) mirror, any magnitude; n == 1 maps to 0.
__device__ __forceinline__ int reflect(int i, int n) {
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    int m = i % period;
    if (m < 0) m += period;
    return m < n ? m : period - m;
}

static __device__ __noinline__ int reflect_far(int i, int n) { return reflect(i, n); }

// Reflect with the single-fold cases inline (two compares, no division): -i and
// 2(n-1)-i are symmetries of the period-2(n-1) mirror, so applying them first and the full
// reflect only to what is still out of range gives reflect(i, n) exactly.
__device__ __forceinline__ int reflect_near(int i, int n) {
    i = i < 0 ? -i : i;
    i = i >= n ? 2 * (n - 1) - i : i;
    return unsigned(i) < unsigned(n) ? i : reflect_far(i, n);
}

// search.cpp:52-57
__device__ __forceinline__ void row_coords(const Dims& d, int64_t local_row, int& qt, int& qy,
                                           int& qx) {
    const int64_t row = local_row + d.row0;
    qx = int(row % d.nw) * d.stride0;
    const int64_t r = row / d.nw;
    qy = int(r % d.nh) * d.stride0;
    qt = int(r / d.nh);
}

// Temporally blocked raster: CTA-order index p -> query row (local to the frame range).  The
// rows are enumerated band by band (`band` query rows of every frame), and inside a band
// frame by frame, then (y, x): consecutive CTAs work on one band of consecutive frames, so
// the key frames a band reads (qt - wt .. qt + wt) stay in L2 across the 2wt+1 query frames
// that reuse them, instead of the whole frame set being streamed from HBM once per query
// frame when it exceeds the L2 (c5: 5 frames x 67 MB).
__device__ __forceinline__ int64_t band_row(const Dims& d, int64_t p, int band) {
    const int64_t full = int64_t(band) * d.nw * d.nt;  // rows of one complete band (all frames)
    const int64_t b = p / full;
    const int64_t q = p - b * full;
    const int y0 = int(b) * band;
    const int hb = min(band, d.nh - y0);
    const int64_t per_frame = int64_t(hb) * d.nw;
    const int64_t t = q / per_frame;
    const int64_t rem = q - t * per_frame;
    return (t * d.nh + y0 + rem / d.nw) * d.nw + rem % d.nw;
}

// search.cpp:59-68: frame scan order 0, -1, +1, -2, +2, ...
__host__ __device__ __forceinline__ int scan_dt(int fpos) {
    return fpos == 0 ? 0 : ((fpos & 1) ? -((fpos + 1) / 2) : fpos / 2);
}

__device__ __forceinline__ size_t vidx(const Dims& d, int t, int y, int x) {
    return ((size_t(t) * d.h + y) * d.w + x) * size_t(d.f);
}

// Bilinear taps of a fractional position (tensor.cpp:31-48) split as integer base +
// fp32 fraction; weights from the raw (unreflected) position.
struct Taps {
    int y0, y1, x0, x1;
    float w00, w01, w10, w11, fy, fx;
};

__device__ __forceinline__ Taps taps_from(int by, float fy, int bx, float fx, int h, int w) {
    Taps t;
    t.fy = fy;
    t.fx = fx;
    t.y0 = reflect_near(by, h);
    t.y1 = reflect_near(by + 1, h);
    t.x0 = reflect_near(bx, w);
    t.x1 = reflect_near(bx + 1, w);
    t.w00 = (1.f - fy) * (1.f - fx);
    t.w01 = (1.f - fy) * fx;
    t.w10 = fy * (1.f - fx);
    t.w11 = fy * fx;
    return t;
}

// An integral coordinate (or displacement) as int, clamped to +-(2^31 - 2^24) first: exact
// for every position the reference's own int conversion defines (up to ~2.13e9 px), while a
// huge or non-finite flow (Middlebury marks unknown flow with ~1e9-1e10; the reference's
// conversion is undefined there) can no longer saturate the int and overflow base + offset
// sums into an out-of-bounds address.  NaN converts to 0 (flows are latched as errors).
__device__ __forceinline__ int int_base(double fb) {
    constexpr int kLim = 2147483647 - 16777216;
    const int i = int(fb);  // cvt.rzi.s32.f64 saturates (and maps NaN to 0)
    return min(max(i, -kLim), kLim);
}

// Position given in fp64 (absolute coordinate).
__device__ __forceinline__ Taps taps_at(double y, double x, int h, int w) {
    const double by = floor(y), bx = floor(x);
    return taps_from(int_base(by), float(y - by), int_base(bx), float(x - bx), h, w);
}

// Position = integer `base` + fp32 `off` (off may be any magnitude that fp32 holds) along an
// axis of n pixels.
__device__ __forceinline__ void split_pos(int base, float off, int& ib, float& fr, int n) {
    const float fl = floorf(off);
    ib = base + int_base(double(fl));
    fr = off - fl;  // exact (Sterbenz) for |off| >= 1 and for 0 <= off < 1
}

__device__ __forceinline__ float blend(const Taps& t, float a, float b, float c, float d) {
    return t.w00 * a + t.w01 * b + t.w10 * c + t.w11 * d;
}

#ifndef SNLS_SHIFT_GRID
#define SNLS_SHIFT_GRID 2
#endif
// A shift rounded to the 2^-32 grid (two adds: the ulp of 1.5 * 2^20 is 2^-32; |v| < 2^19,
// beyond that a coarser grid, which keeps the same exactness property).
__device__ __forceinline__ double grid32(double v) {
#if SNLS_SHIFT_GRID == 2
    constexpr double kMagic = 0x1.8p20;
    return (v + kMagic) - kMagic;
#elif SNLS_SHIFT_GRID == 1
    return rint(v * 0x1p32) * 0x1p-32;
#else
    return v;
#endif
}

// search.cpp:72-122 on device: the window shift to frame qt + dt in fp64.  dt == 0 reads
// the forward field at the query pixel; |dt| >= 1 sums per-step fields, later links
// bilinear-sampled at the displaced position.  `links` (optional) receives |dt|-1 links of
// (pos_y - qy, pos_x - qx, J00, J01, J10, J11) in fp32 (the device tape) or, with LT =
// double, the reference's own fp64 links (pos_y, pos_x, J00, ...) with ABSOLUTE positions.
template <typename LT>
__device__ inline void shift_to_t(const float* __restrict__ ff, const float* __restrict__ bf,
                                  int h, int w, int qt, int qy, int qx, int dt, double& dy,
                                  double& dx, LT* links) {
    constexpr bool kAbs = sizeof(LT) == sizeof(double);
    if (ff == nullptr) {  // nls_forward: zero flows
        dy = 0.0;
        dx = 0.0;
        if (links)
            for (int k = 1; k < (dt < 0 ? -dt : dt); ++k)
                for (int j = 0; j < 6; ++j)
                    links[(k - 1) * 6 + j] = LT(kAbs && j < 2 ? (j == 0 ? qy : qx) : 0);
        return;
    }
    auto at = [&](const float* fl, int t, int y, int x, int c) {
        return double(__ldg(fl + ((size_t(t) * h + y) * w + x) * 2 + c));
    };
    if (dt == 0) {
        dy = grid32(at(ff, qt, qy, qx, 0));  // (2^-32 grid: see the end)
        dx = grid32(at(ff, qt, qy, qx, 1));
        return;
    }
    const float* fld = dt > 0 ? ff : bf;
    const int step = dt > 0 ? 1 : -1;
    const int m = dt > 0 ? dt : -dt;
    double sy = 0.0, sx = 0.0;
    for (int k = 0; k < m; ++k) {
        const int fr = qt + step * k;
        double vy, vx;
        if (k == 0) {
            vy = at(fld, fr, qy, qx, 0);
            vx = at(fld, fr, qy, qx, 1);
        } else {
            const double py = double(qy) + sy, px = double(qx) + sx;
            const double fby = floor(py), fbx = floor(px);
            const double fy = py - fby, fx = px - fbx;
            // int() saturates beyond the int range and reflect maps any int into the frame,
            // so a huge flow still samples in bounds (the +1 then wraps, as PTX add does)
            const int y0 = reflect_near(int(fby), h), y1 = reflect_near(int(fby) + 1, h);
            const int x0 = reflect_near(int(fbx), w), x1 = reflect_near(int(fbx) + 1, w);
            const double ay = at(fld, fr, y0, x0, 0), by = at(fld, fr, y0, x1, 0);
            const double cy = at(fld, fr, y1, x0, 0), dyv = at(fld, fr, y1, x1, 0);
            const double ax = at(fld, fr, y0, x0, 1), bx = at(fld, fr, y0, x1, 1);
            const double cx = at(fld, fr, y1, x0, 1), dxv = at(fld, fr, y1, x1, 1);
            const double w00 = (1.0 - fy) * (1.0 - fx), w01 = (1.0 - fy) * fx;
            const double w10 = fy * (1.0 - fx), w11 = fy * fx;
            vy = w00 * ay + w01 * by + w10 * cy + w11 * dyv;
            vx = w00 * ax + w01 * bx + w10 * cx + w11 * dxv;
            if (links) {
                LT* lk = links + (k - 1) * 6;
                lk[0] = LT(kAbs ? py : sy);
                lk[1] = LT(kAbs ? px : sx);
                lk[2] = LT(-(1.0 - fx) * ay - fx * by + (1.0 - fx) * cy + fx * dyv);
                lk[3] = LT(-(1.0 - fy) * ay + (1.0 - fy) * by - fy * cy + fy * dyv);
                lk[4] = LT(-(1.0 - fx) * ax - fx * bx + (1.0 - fx) * cx + fx * dxv);
                lk[5] = LT(-(1.0 - fy) * ax + (1.0 - fy) * bx - fy * cx + fy * dxv);
            }
        }
        sy += vy;
        sx += vx;
    }
    // the shift on a 2^-32 grid (|change| < 2^-33 px, far below fp32's fraction): the key
    // centres (qy + sdy) + n of the fp64 tape are then exact, so a replay from a centre sees
    // the very fraction the forward interpolated with (replay_similarities == forward, bitwise)
    dy = grid32(sy);
    dx = grid32(sx);
}

// shift_to_t without links, spelled out for the search kernels: the same fp64 operations in
// the same order (so the same shift, bit for bit), as a plain function -- instantiating the
// template inside search_tiled_kernel changed ptxas' register allocation (11 -> 14 spill
// instructions, c4 search 3.90 -> 3.98 ms; profiles/r01_plans.txt), and so did clamping
// the link base or forming its +1 in unsigned arithmetic.
__device__ inline void shift_to(const float* __restrict__ ff, const float* __restrict__ bf,
                                int h, int w, int qt, int qy, int qx, int dt, double& dy,
                                double& dx) {
    if (ff == nullptr) {
        dy = 0.0;
        dx = 0.0;
        return;
    }
    auto at = [&](const float* fl, int t, int y, int x, int c) {
        return double(__ldg(fl + ((size_t(t) * h + y) * w + x) * 2 + c));
    };
    if (dt == 0) {
        dy = grid32(at(ff, qt, qy, qx, 0));
        dx = grid32(at(ff, qt, qy, qx, 1));
        return;
    }
    const float* fld = dt > 0 ? ff : bf;
    const int step = dt > 0 ? 1 : -1;
    const int m = dt > 0 ? dt : -dt;
    double sy = 0.0, sx = 0.0;
    for (int k = 0; k < m; ++k) {
        const int fr = qt + step * k;
        double vy, vx;
        if (k == 0) {
            vy = at(fld, fr, qy, qx, 0);
            vx = at(fld, fr, qy, qx, 1);
        } else {
            const double py = double(qy) + sy, px = double(qx) + sx;
            const double fby = floor(py), fbx = floor(px);
            const double fy = py - fby, fx = px - fbx;
            const int y0 = reflect_near(int(fby), h), y1 = reflect_near(int(fby) + 1, h);
            const int x0 = reflect_near(int(fbx), w), x1 = reflect_near(int(fbx) + 1, w);
            const double ay = at(fld, fr, y0, x0, 0), by = at(fld, fr, y0, x1, 0);
            const double cy = at(fld, fr, y1, x0, 0), dyv = at(fld, fr, y1, x1, 0);
            const double ax = at(fld, fr, y0, x0, 1), bx = at(fld, fr, y0, x1, 1);
            const double cx = at(fld, fr, y1, x0, 1), dxv = at(fld, fr, y1, x1, 1);
            const double w00 = (1.0 - fy) * (1.0 - fx), w01 = (1.0 - fy) * fx;
            const double w10 = fy * (1.0 - fx), w11 = fy * fx;
            vy = w00 * ay + w01 * by + w10 * cy + w11 * dyv;
            vx = w00 * ax + w01 * bx + w10 * cx + w11 * dxv;
        }
        sy += vy;
        sx += vx;
    }
    dy = grid32(sy);
    dx = grid32(sx);
}

// With fp32 links (the device tape).
__device__ inline void shift_to(const float* __restrict__ ff, const float* __restrict__ bf,
                                int h, int w, int qt, int qy, int qx, int dt, double& dy,
                                double& dx, float* links) {
    shift_to_t<float>(ff, bf, h, w, qt, qy, qx, dt, dy, dx, links);
}

// Total order used for top-L: value descending, then slot ascending (search.cpp:187-197,
// 390-393).  Packed into one u64 so a warp max-reduction is a single comparison chain.
__device__ __forceinline__ uint32_t orderable(float v) {
    const uint32_t b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float from_orderable(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ uint64_t pack_key(float v, uint32_t slot) {
    return (uint64_t(orderable(v)) << 32) | uint64_t(0xffffffffu - slot);
}
__device__ __forceinline__ uint32_t key_slot(uint64_t k) {
    return 0xffffffffu - uint32_t(k & 0xffffffffu);
}
__device__ __forceinline__ float key_value(uint64_t k) { return from_orderable(uint32_t(k >> 32)); }

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t u = __shfl_xor_sync(0xffffffffu, v, o);
        v = u > v ? u : v;
    }
    return v;
}

// A candidate is eligible for top-L only if it compares greater than -inf (NaN and -inf
// never enter, search.cpp:188).
__device__ __forceinline__ bool eligible(float v) { return v > -INFINITY; }

__device__ __forceinline__ void latch(int* err, int bit) {
    if (err) atomicOr(err, bit);
}

// Raise a kernel's dynamic shared-memory limit above the 48 KB default, once per (kernel,
// device) and size: cudaFuncSetAttribute is a driver call, not something to pay per launch.
inline void ensure_smem(const void* kern, size_t bytes) {
    // the opt-in covers static + dynamic above 48 KB: ask whenever the dynamic part alone could
    // push a kernel with static shared memory over the default
    if (bytes <= 16 * 1024) return;
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex m;
    static std::map<std::pair<const void*, int>, size_t> have;
    std::lock_guard<std::mutex> lk(m);
    size_t& h = have[{kern, dev}];
    if (h >= bytes) return;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) == cudaSuccess)
        h = bytes;
}
template <class K>
inline void ensure_smem(K* kern, size_t bytes) {
    ensure_smem(reinterpret_cast<const void*>(kern), bytes);
}

}  // namespace snls_gpu
