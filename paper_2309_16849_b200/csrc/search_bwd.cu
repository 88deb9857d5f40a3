// Search backward (shifted_nls_backward, search.cpp:499-711) on device.
//
// Phase 1 (ps <= 7: search_bwd_rows, register pre-reduction; else search_bwd_entries):
// one thread per (selected entry, channel group).  It replays the entry's patch
// (same taps as the forward), scatters dQ into the reflected query pixels and dK into the
// 4 bilinear taps with atomics, and accumulates its share of dS/d(ky, kx) in fp64.  The
// per-entry (gy, gx) is reduced across the channel-group threads with fp64 atomics.
// Phase 2: one thread per entry routes (gy, gx) back through the composition chain
// (search.cpp:584-666): dt >= 0 into dFflow, dt < 0 into dBflow, v <- (I + J)^T v per link.
// Entries with a zero upstream gradient are skipped (search.cpp:692).
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "packed.cuh"
#include "wpsum_bwd_pairs.cuh"
#include "fixed_point.cuh"

#ifndef SNLS_BWD_DQSM
#define SNLS_BWD_DQSM 1
#endif
#ifndef SNLS_BWD_ACT_CT
#define SNLS_BWD_ACT_CT 0
#endif
#ifndef SNLS_BWD_MINB
#define SNLS_BWD_MINB 4
#endif
#ifndef SNLS_BWD_FORCE_ENTRIES
#define SNLS_BWD_FORCE_ENTRIES 0
#endif

namespace snls_gpu {

namespace {

constexpr bool kDqSm = SNLS_BWD_DQSM != 0;

// Where a gradient contribution goes.  Default: fp32 atomics (the reference's
// non-deterministic mode).  Deterministic mode (SNLS_BWD_DETERMINISTIC, the reference's
// default, search.cpp:687-696): int64 fixed-point atomics -- integer addition is
// associative, so every run gives the same bits whatever the atomic order.  The fixed-point
// scale is a power of two picked per call from a bound on the largest possible |sum|
// (bwd_scales_kernel), so nothing overflows and the resolution stays ~1e-12 of that bound.
struct Sink {
    float* f;
    unsigned long long* i;
    const double* scale;  // device scalar (deterministic mode)
};

template <bool DET>
__device__ __forceinline__ void put(float* f, unsigned long long* i, double scale, size_t idx, double v) {
    if constexpr (DET) atomicAdd(i + idx, static_cast<unsigned long long>(__double2ll_rn(v * scale)));
    else atomicAdd(f + idx, float(v));
}

template <int VEC, bool DET>
__global__ void __launch_bounds__(256) search_bwd_entries(const float* __restrict__ grad,
                                                          const float* __restrict__ offsets,
                                                          const float* __restrict__ q,
                                                          const float* __restrict__ k, Dims d,
                                                          int ps, int topl, int metric,
                                                          Sink sq, Sink sk, double* gyx,
                                                          const double* __restrict__ centers) {
    const int groups = d.f / VEC;
    const double scq = DET ? *sq.scale : 0.0, sck = DET ? *sk.scale : 0.0;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= d.rows * topl * groups) return;
    const int64_t e = idx / groups;
    const int c = int(idx % groups) * VEC;
    const float g = grad[e];
    if (g == 0.f) return;
    const int64_t row = e / topl;
    int qt, qy, qx;
    row_coords(d, row, qt, qy, qx);
    // key position: integer base + fraction, from the fp32 offsets or the fp64 centres
    int kt, cby, cbx;
    double cfy, cfx;  // fp64 fractions: this kernel's arithmetic is fp64
    if (centers) {
        const double* cp = centers + size_t(e) * 3;
        kt = int(cp[0]);
        const double fly = floor(cp[1]), flx = floor(cp[2]);
        cby = int_base(fly);
        cbx = int_base(flx);
        cfy = cp[1] - fly;
        cfx = cp[2] - flx;
    } else {
        const float* o = offsets + size_t(e) * 3;
        kt = qt + int(rintf(o[0]));
        float fy32, fx32;
        split_pos(qy, o[1], cby, fy32, d.h);
        split_pos(qx, o[2], cbx, fx32, d.w);
        cfy = fy32;
        cfx = fx32;
    }
    const int half = ps / 2;
    double gy = 0.0, gx = 0.0;
    for (int py = -half; py <= half; ++py) {
        const int ry = reflect_near(qy + py, d.h);
        for (int px = -half; px <= half; ++px) {
            const int rx = reflect_near(qx + px, d.w);
            const int iy = cby + py, ix = cbx + px;
            const Taps t = taps_from(iy, float(cfy), ix, float(cfx), d.h, d.w);
            const size_t iq = vidx(d, qt, ry, rx) + c;
            const size_t i00 = vidx(d, kt, t.y0, t.x0) + c, i01 = vidx(d, kt, t.y0, t.x1) + c;
            const size_t i10 = vidx(d, kt, t.y1, t.x0) + c, i11 = vidx(d, kt, t.y1, t.x1) + c;
            // dS/d(ky, kx) sums hundreds of cancelling terms per entry: keep that chain in
            // fp64 (the dQ/dK scatter stays fp32)
            const double dfy = cfy, dfx = cfx;
            const double w00 = (1.0 - dfy) * (1.0 - dfx), w01 = (1.0 - dfy) * dfx;
            const double w10 = dfy * (1.0 - dfx), w11 = dfy * dfx;
            double sy = 0.0, sx = 0.0;
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const float qv = __ldg(q + iq + j);
                const float k00 = __ldg(k + i00 + j), k01 = __ldg(k + i01 + j);
                const float k10 = __ldg(k + i10 + j), k11 = __ldg(k + i11 + j);
                const double kv = w00 * k00 + w01 * k01 + w10 * k10 + w11 * k11;
                double ds_dq, ds_dk;
                if (metric == SNLS_METRIC_IP) {
                    ds_dq = kv;
                    ds_dk = qv;
                } else {
                    const double diff = double(qv) - kv;
                    ds_dq = -2.0 * diff;
                    ds_dk = 2.0 * diff;
                }
                const double gk = double(g) * ds_dk;
                put<DET>(sq.f, sq.i, scq, iq + j, double(float(double(g) * ds_dq)));
                put<DET>(sk.f, sk.i, sck, i00 + j, double(float(gk * w00)));
                put<DET>(sk.f, sk.i, sck, i01 + j, double(float(gk * w01)));
                put<DET>(sk.f, sk.i, sck, i10 + j, double(float(gk * w10)));
                put<DET>(sk.f, sk.i, sck, i11 + j, double(float(gk * w11)));
                // d(sample)/dy, d(sample)/dx from the tap values (search.cpp:574-577)
                const double dkv_dy = (1.0 - dfx) * (double(k10) - k00) + dfx * (double(k11) - k01);
                const double dkv_dx = (1.0 - dfy) * (double(k01) - k00) + dfy * (double(k11) - k10);
                sy += gk * dkv_dy;
                sx += gk * dkv_dx;
            }
            gy += sy;
            gx += sx;
        }
    }
    if constexpr (DET) {  // per-(entry, channel group) partials, summed in order by the route
        gyx[(size_t(e) * groups + c / VEC) * 2] = gy;
        gyx[(size_t(e) * groups + c / VEC) * 2 + 1] = gx;
    } else {
        atomicAdd(gyx + 2 * e, gy);
        atomicAdd(gyx + 2 * e + 1, gx);
    }
}

// Row-centric backward (any stride1: every pixel of one entry's patch shares the
// fractional offset frac(offset), so its 4 ps^2 taps fall on one (ps+1)^2 raw block):
// one warp per (query row, 32-channel slice), lane = channel.  Same per-(pixel, channel)
// arithmetic as search_bwd_entries, with the scatter pre-reduced in registers before the
// atomics: dQ is summed over the row's L entries (ps^2 atomics per row instead of L ps^2),
// dK is accumulated on the raw block two rows at a time ((ps+1)^2 atomics per entry instead
// of 4 ps^2), and dS/d(ky, kx) is warp-reduced (one fp64 atomic pair per slice).  Every
// atomic is a fully coalesced 128 B warp access along the channels.
// The query patch is parked in shared memory once per warp (each lane reads back only its own
// channel: no barrier; c3 backward 0.730 -> 0.684 ms).
// FT > 0: the channel count as a compile-time constant; entries whose raw block lies inside
// the frame then address it as row base + j * FT (immediate offsets: no reflection, no
// per-element address arithmetic -- most of this kernel's integer work); FT = 0 any F.
// MET: 0 = runtime metric, 1 + snls_metric = compile-time (drops the other metric's selects
// and, for ip, the l2-only CORR sums).  The patch-row loop is rolled (ROLL): fully unrolled,
// the two block bodies of a ps 7 instantiation took ~12k SASS instructions and the warps
// stalled on instruction fetch (no_instructions 27%, profiles/r02f_ncu_c3.txt).
#ifndef SNLS_BWD_ROLL
#define SNLS_BWD_ROLL 1
#endif
template <int P, bool DET, bool CORR, int FT = 0, int MET = 0>
__device__ __forceinline__ void search_bwd_rows_body(const float* __restrict__ grad,
                                                     const float* __restrict__ offsets,
                                                     const float* __restrict__ q,
                                                     const float* __restrict__ k, Dims d,
                                                     int topl, int metric_rt,
                                                     Sink sinkq, Sink sinkk,
                                                     double* __restrict__ gyx,
                                                     const double* __restrict__ centers,
                                                     unsigned bid, float* s_bwd) {
    constexpr int HP = P / 2;
    const int metric = MET ? MET - 1 : metric_rt;
    const double scq = DET ? *sinkq.scale : 0.0, sck = DET ? *sinkk.scale : 0.0;
    const int slices = (d.f + 31) / 32;
    const int64_t wid = (int64_t(bid) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= d.rows * slices) return;  // warp-uniform
    const int64_t row = wid / slices;
    const int c = int(wid % slices) * 32 + lane;
    const bool act = (SNLS_BWD_ACT_CT && FT > 0 && FT % 32 == 0) || c < d.f;
    const int cc = act ? c : 0;
    // dynamic shared memory: [4 warps][P*P][32] query patch, then (kDqSm) the dQ partials
    float* sq = s_bwd + (threadIdx.x >> 5) * (P * P * 32) + lane;
    float* sdq = sq + 4 * P * P * 32;
    int qt, qy, qx;
    row_coords(d, row, qt, qy, qx);
    const size_t F = size_t(d.f), rowF = size_t(d.w) * F, frameF = size_t(d.h) * rowF;
    int qrow[P], qcol[P];  // reflected query pixels (search.cpp:129-132)
#pragma unroll
    for (int p = 0; p < P; ++p) {
        qrow[p] = reflect_near(qy + p - HP, d.h) * d.w;
        qcol[p] = reflect_near(qx + p - HP, d.w);
    }
    const float* qb = q + size_t(qt) * frameF + cc;
#pragma unroll
    for (int py = 0; py < P; ++py)
#pragma unroll
        for (int px = 0; px < P; ++px)
            sq[(py * P + px) * 32] = act ? __ldg(qb + size_t(qrow[py] + qcol[px]) * F) : 0.f;
    float dqa[kDqSm ? 1 : P][kDqSm ? 1 : P];
#pragma unroll
    for (int py = 0; py < P; ++py)
#pragma unroll
        for (int px = 0; px < P; ++px) {
            if constexpr (kDqSm) sdq[(py * P + px) * 32] = 0.f;
            else dqa[py][px] = 0.f;
        }

    for (int l = 0; l < topl; ++l) {
        const int64_t e = row * topl + l;
        const float g = __ldg(grad + e);
        if (g == 0.f) continue;  // search.cpp:692 (uniform: one row per warp)
        int kt, by, bx;
        float fy, fx;
        double ddy = 0.0, ddx = 0.0;  // fp64 fraction - its fp32 rounding (CORR)
        if (CORR) {  // the reference's fp64 tape: fraction taken in fp64
            const double* c = centers + size_t(e) * 3;
            kt = int(__ldg(c));
            const double cy = __ldg(c + 1), cx = __ldg(c + 2);
            const double fly = floor(cy), flx = floor(cx);
            fy = float(cy - fly);
            fx = float(cx - flx);
            ddy = (cy - fly) - double(fy);
            ddx = (cx - flx) - double(fx);
            by = int_base(fly) - HP;
            bx = int_base(flx) - HP;
        } else {
            const float* o = offsets + size_t(e) * 3;
            kt = qt + int(rintf(__ldg(o)));
            const float oy = __ldg(o + 1), ox = __ldg(o + 2);
            const float fly = floorf(oy), flx = floorf(ox);
            fy = oy - fly;
            fx = ox - flx;
            by = qy - HP + int_base(fly);
            bx = qx - HP + int_base(flx);
        }
        const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx;
        const float w10 = fy * (1.f - fx), w11 = fy * fx;
        const float* kb = k + size_t(kt) * frameF + cc;
        const size_t dkb = size_t(kt) * frameF + cc;
        // dS/d(ky, kx) sums thousands of cancelling terms per entry: fp64 accumulation of the
        // fp32 per-term products (c3 l2 flow gradients 1.4e-5 -> 3e-6 relative, +1% time)
        double sy = 0.0, sx = 0.0;
        // CORR: first-order terms of the fp32 rounding of the fractions (bilinear samples are
        // linear in fy, fx; the flow gradients amplify the rounding by sum (dk/dy)^2)
        float cA = 0.f, cB = 0.f, cD = 0.f, cC = 0.f;
        // the (P+1)^2 raw block, two rows at a time; FAST: inside the frame, immediate column
        // offsets j * FT from one row base; else reflected rows / columns (tensor.cpp:23-48)
        auto body = [&](auto fast_tag) {
            constexpr bool FAST = decltype(fast_tag)::value;
            unsigned bcol[FAST ? 1 : P + 1];
            if constexpr (!FAST) {
#pragma unroll
                for (int j = 0; j <= P; ++j) bcol[j] = unsigned(reflect_near(bx + j, d.w)) * unsigned(d.f);
            }
            auto colo = [&](int j) -> size_t { return FAST ? size_t(j) * FT : size_t(bcol[FAST ? 0 : j]); };
            const size_t xo = FAST ? size_t(bx) * FT : 0;
            auto rowo = [&](int r) -> size_t {
                return FAST ? size_t(by + r) * rowF + xo : size_t(reflect_near(by + r, d.h)) * rowF;
            };
            float ra[P + 1], rb[P + 1], ka[P + 1], kn[P + 1];
            size_t roa = rowo(0), rob = rowo(1);
#pragma unroll
            for (int j = 0; j <= P; ++j) {
                ra[j] = act ? __ldg(kb + roa + colo(j)) : 0.f;
                rb[j] = act ? __ldg(kb + rob + colo(j)) : 0.f;
                ka[j] = 0.f;
            }
            constexpr bool kRoll = SNLS_BWD_ROLL && kDqSm && P > 3;
#pragma unroll(kRoll ? 1 : P)
            for (int py = 0; py < P; ++py) {
                const size_t ron = rowo(py + 2);
#pragma unroll
                for (int j = 0; j <= P; ++j) kn[j] = 0.f;
#pragma unroll
                for (int px = 0; px < P; ++px) {
                    const float k00 = ra[px], k01 = ra[px + 1], k10 = rb[px], k11 = rb[px + 1];
                    const float qv = sq[(py * P + px) * 32];
                    // lerp form: the x-interpolated rows give the sample and both tap
                    // derivatives (search.cpp:574-577) in 8 FP ops instead of 12
                    const float d0 = k01 - k00, d1 = k11 - k10;
                    const float hx0 = fmaf(fx, d0, k00), hx1 = fmaf(fx, d1, k10);
                    const float dkv_dy = hx1 - hx0;
                    const float kv = fmaf(fy, dkv_dy, hx0);
                    const float dkv_dx = fmaf(fy, d1 - d0, d0);
                    float ds_dq, ds_dk;
                    if (metric == SNLS_METRIC_IP) {
                        ds_dq = kv;
                        ds_dk = qv;
                    } else {
                        const float diff = qv - kv;
                        ds_dq = -2.f * diff;
                        ds_dk = 2.f * diff;
                    }
                    const float gk = g * ds_dk;
                    if constexpr (kDqSm) sdq[(py * P + px) * 32] = fmaf(g, ds_dq, sdq[(py * P + px) * 32]);
                    else dqa[py][px] = fmaf(g, ds_dq, dqa[py][px]);
                    ka[px] = fmaf(gk, w00, ka[px]);
                    ka[px + 1] = fmaf(gk, w01, ka[px + 1]);
                    kn[px] = fmaf(gk, w10, kn[px]);
                    kn[px + 1] = fmaf(gk, w11, kn[px + 1]);
sy = fma(double(gk), double(dkv_dy), sy);
                    sx = fma(double(gk), double(dkv_dx), sx);
                    if constexpr (CORR) {
                        cC = fmaf(gk, d1 - d0, cC);
                        if (metric != SNLS_METRIC_IP) {
                            cA = fmaf(dkv_dy, dkv_dy, cA);
                            cB = fmaf(dkv_dy, dkv_dx, cB);
                            cD = fmaf(dkv_dx, dkv_dx, cD);
                        }
                    }
                }
                if (act) {  // raw row py of the block is complete
#pragma unroll
                    for (int j = 0; j <= P; ++j) put<DET>(sinkk.f, sinkk.i, sck, dkb + roa + colo(j), ka[j]);
                }
#pragma unroll
                for (int j = 0; j <= P; ++j) {
                    ra[j] = rb[j];
                    if (py + 1 < P) rb[j] = act ? __ldg(kb + ron + colo(j)) : 0.f;
                    ka[j] = kn[j];
                }
                roa = rob;
                rob = ron;
            }
            if (act) {
#pragma unroll
                for (int j = 0; j <= P; ++j) put<DET>(sinkk.f, sinkk.i, sck, dkb + roa + colo(j), ka[j]);
            }
        };
        if (FT > 0 && by >= 0 && by + P < d.h && bx >= 0 && bx + P < d.w)  // uniform: one entry per warp
            body(std::integral_constant<bool, (FT > 0)>{});
        else
            body(std::false_type{});
        if constexpr (CORR) {
            // l2: gk = 2g(q - kv) moves by -2g dkv; both metrics: dkv_dy moves by ddx (d1 - d0),
            // dkv_dx by ddy (d1 - d0)
            const double g2 = metric != SNLS_METRIC_IP ? 2.0 * double(g) : 0.0;
            sy += ddx * cC - g2 * (ddy * cA + ddx * cB);
            sx += ddy * cC - g2 * (ddy * cB + ddx * cD);
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            sy += __shfl_xor_sync(0xffffffffu, sy, m);
            sx += __shfl_xor_sync(0xffffffffu, sx, m);
        }
        if (lane == 0) {
            if constexpr (DET) {  // per-(entry, slice) partials, summed in order by the route
                gyx[(size_t(e) * slices + wid % slices) * 2] = sy;
                gyx[(size_t(e) * slices + wid % slices) * 2 + 1] = sx;
            } else {
                atomicAdd(gyx + 2 * e, sy);
                atomicAdd(gyx + 2 * e + 1, sx);
            }
        }
    }
    if (act) {
        const size_t dqb = size_t(qt) * frameF + cc;
#pragma unroll
        for (int py = 0; py < P; ++py)
#pragma unroll
            for (int px = 0; px < P; ++px)
                put<DET>(sinkq.f, sinkq.i, scq, dqb + size_t(qrow[py] + qcol[px]) * F,
                         kDqSm ? sdq[(py * P + px) * 32] : dqa[py][px]);
    }
}

template <int P, bool DET, bool CORR, int FT = 0, int MET = 0>
__global__ void __launch_bounds__(128, SNLS_BWD_MINB) search_bwd_rows(const float* __restrict__ grad,
                                                          const float* __restrict__ offsets,
                                                          const float* __restrict__ q,
                                                          const float* __restrict__ k, Dims d,
                                                          int topl, int metric_rt,
                                                          Sink sinkq, Sink sinkk,
                                                          double* __restrict__ gyx,
                                                          const double* __restrict__ centers) {
    extern __shared__ float s_bwd[];
    search_bwd_rows_body<P, DET, CORR, FT, MET>(grad, offsets, q, k, d, topl, metric_rt, sinkq, sinkk,
                                                gyx, centers, blockIdx.x, s_bwd);
}

// The training backward's two phase-1 operators in ONE launch, their blocks interleaved
// (even: a search-backward block, odd: a wpsum-backward block, then the longer one's rest):
// every SM runs both at once -- the search backward is issue-bound, the wpsum backward waits
// on its dV reductions through L2 -- instead of one after the other (or overlapping only at
// the tail when launched on two streams).  Same bodies, same results.
template <int P, bool CORR, int FT, int MET, int NL, int LS, bool DET>
__global__ void __launch_bounds__(128, SNLS_BWD_MINB) train_bwd_interleaved(
    const float* __restrict__ grad, const float* __restrict__ offsets, const float* __restrict__ q,
    const float* __restrict__ k, Dims d, int topl, Sink sinkq, Sink sinkk, double* __restrict__ gyx,
    const double* __restrict__ centers, WpsumBwdArgs w, unsigned n_search, unsigned n_wpsum) {
    extern __shared__ float s_bwd[];
    const unsigned m = min(n_search, n_wpsum), b = blockIdx.x;
    bool wp;
    unsigned idx;
    if (b < 2 * m) {
        wp = b & 1u;
        idx = b >> 1;
    } else {
        wp = n_wpsum > n_search;
        idx = b - m;
    }
    if (wp)
        wpsum_bwd_pairs_body<P, NL, LS, DET>(w.a, w.go, w.counts, w.dv, w.dw, idx, reinterpret_cast<u64*>(s_bwd),
                                             WbwdFixed{w.dvi, w.dwi, w.scale});
    else
        search_bwd_rows_body<P, DET, CORR, FT, MET>(grad, offsets, q, k, d, topl, MET - 1, sinkq, sinkk, gyx,
                                                    centers, idx, s_bwd);
}

template <int P, bool DET>
void launch_rows(const float* grad, const float* offsets, const float* q, const float* k, Dims d,
                 int topl, int metric, Sink sq, Sink sk, double* gyx, const double* centers,
                 cudaStream_t st) {
    const int64_t warps = d.rows * ((d.f + 31) / 32);
    const size_t smem = size_t(4) * P * P * 32 * sizeof(float) * (kDqSm ? 2 : 1);
    const unsigned blocks = unsigned((warps + 3) / 4);
    auto go = [&](auto kern) {
        ensure_smem(kern, smem);
        kern<<<blocks, 128, smem, st>>>(grad, offsets, q, k, d, topl, metric, sq, sk, gyx, centers);
    };
    // compile-time channel counts of the BASELINE shapes (fast interior addressing)
    const int ft = d.f == 64 ? 64 : (d.f == 32 ? 32 : 0);
    const bool ip = metric == SNLS_METRIC_IP;
    if (centers) {
        if (ft == 64) ip ? go(search_bwd_rows<P, DET, true, 64, 1>) : go(search_bwd_rows<P, DET, true, 64, 2>);
        else if (ft == 32) ip ? go(search_bwd_rows<P, DET, true, 32, 1>) : go(search_bwd_rows<P, DET, true, 32, 2>);
        else go(search_bwd_rows<P, DET, true, 0>);
    } else {
        if (ft == 64) ip ? go(search_bwd_rows<P, DET, false, 64, 1>) : go(search_bwd_rows<P, DET, false, 64, 2>);
        else if (ft == 32) ip ? go(search_bwd_rows<P, DET, false, 32, 1>) : go(search_bwd_rows<P, DET, false, 32, 2>);
        else go(search_bwd_rows<P, DET, false, 0>);
    }
}

// Phase 1 of either mode; returns the number of per-entry (gy, gx) partials (1: atomics
// into one pair; >1: one pair per channel slice / group, deterministic mode).
template <bool DET>
int launch_phase1(const float* grad, const float* offsets, const double* centers, const float* q,
                  const float* k, Dims d, int ps, int topl, int metric, Sink sq, Sink sk, double* gyx,
                  cudaStream_t st) {
    const int vec = d.f % 4 == 0 ? 4 : 1;
    if (!SNLS_BWD_FORCE_ENTRIES && (ps == 1 || ps == 3 || ps == 5 || ps == 7)) {
        switch (ps) {
            case 1: launch_rows<1, DET>(grad, offsets, q, k, d, topl, metric, sq, sk, gyx, centers, st); break;
            case 3: launch_rows<3, DET>(grad, offsets, q, k, d, topl, metric, sq, sk, gyx, centers, st); break;
            case 5: launch_rows<5, DET>(grad, offsets, q, k, d, topl, metric, sq, sk, gyx, centers, st); break;
            default: launch_rows<7, DET>(grad, offsets, q, k, d, topl, metric, sq, sk, gyx, centers, st); break;
        }
        return DET ? (d.f + 31) / 32 : 1;
    }
    const int64_t n = d.rows * topl * (d.f / vec);
    if (vec == 4)
        search_bwd_entries<4, DET><<<unsigned((n + 255) / 256), 256, 0, st>>>(grad, offsets, q, k, d, ps, topl,
                                                                              metric, sq, sk, gyx, centers);
    else
        search_bwd_entries<1, DET><<<unsigned((n + 255) / 256), 256, 0, st>>>(grad, offsets, q, k, d, ps, topl,
                                                                              metric, sq, sk, gyx, centers);
    return DET ? d.f / vec : 1;
}

// Phase 2: route each entry's dS/d(ky, kx) through its composition chain (search.cpp:584-666).
// MODE 0: fp64 atomics into the flow accumulators; MODE 1 (deterministic, bound pass): only
// the largest |v| met along any chain, for the fixed-point scale; MODE 2 (deterministic):
// int64 fixed-point atomics.  `parts` per-entry partials are summed in a fixed order.
template <int MODE>
__global__ void search_bwd_route(const float* __restrict__ grad,
                                 const float* __restrict__ offsets,
                                 const float* __restrict__ chains, Dims d, int wt, int topl,
                                 const double* __restrict__ gyx, int parts, double* dff, double* dbf,
                                 unsigned long long* iff, unsigned long long* ibf,
                                 const double* __restrict__ scale, unsigned* vmax_bits,
                                 const double* __restrict__ centers,
                                 const double* __restrict__ chains64) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= d.rows * topl) return;
    if (grad[e] == 0.f) return;
    const int64_t row = e / topl;
    int qt, qy, qx;
    row_coords(d, row, qt, qy, qx);
    const int dt = centers ? int(centers[size_t(e) * 3]) - qt : int(rintf(offsets[size_t(e) * 3]));
    double* fld = dt >= 0 ? dff : dbf;
    unsigned long long* ifld = dt >= 0 ? iff : ibf;
    const double sc = MODE == 2 ? *scale : 0.0;
    const int step = dt >= 0 ? 1 : -1;
    const int m = dt == 0 ? 1 : (dt > 0 ? dt : -dt);
    double vy = 0.0, vx = 0.0;
    for (int j = 0; j < parts; ++j) {
        vy += gyx[(size_t(e) * parts + j) * 2];
        vx += gyx[(size_t(e) * parts + j) * 2 + 1];
    }
    double vm = fmax(fabs(vy), fabs(vx));
    auto add = [&](size_t idx, double v) {
        if constexpr (MODE == 0) atomicAdd(fld + idx, v);
        else if constexpr (MODE == 2) atomicAdd(ifld + idx, static_cast<unsigned long long>(__double2ll_rn(v * sc)));
    };
    const int cs = wt > 1 ? wt - 1 : 0;
    const float* chain = chains ? chains + size_t(e) * cs * 6 : nullptr;
    const double* chain64 = chains64 ? chains64 + size_t(e) * cs * 6 : nullptr;
    for (int kk = m - 1; kk >= 1; --kk) {
        double lk[6];
        Taps t;
        if (chain64) {  // absolute fp64 link positions (the reference's tape)
            for (int j = 0; j < 6; ++j) lk[j] = chain64[(kk - 1) * 6 + j];
            t = taps_at(lk[0], lk[1], d.h, d.w);
        } else {
            for (int j = 0; j < 6; ++j) lk[j] = chain[(kk - 1) * 6 + j];
            int iy, ix;
            float fy, fx;
            split_pos(qy, float(lk[0]), iy, fy, d.h);
            split_pos(qx, float(lk[1]), ix, fx, d.w);
            t = taps_from(iy, fy, ix, fx, d.h, d.w);
        }
        const int fr = qt + step * kk;
        auto at = [&](int y, int x, int comp) { return ((size_t(fr) * d.h + y) * d.w + x) * 2 + comp; };
        add(at(t.y0, t.x0, 0), vy * t.w00);
        add(at(t.y0, t.x1, 0), vy * t.w01);
        add(at(t.y1, t.x0, 0), vy * t.w10);
        add(at(t.y1, t.x1, 0), vy * t.w11);
        add(at(t.y0, t.x0, 1), vx * t.w00);
        add(at(t.y0, t.x1, 1), vx * t.w01);
        add(at(t.y1, t.x0, 1), vx * t.w10);
        add(at(t.y1, t.x1, 1), vx * t.w11);
        const double ny = vy + lk[2] * vy + lk[4] * vx;
        const double nx = vx + lk[3] * vy + lk[5] * vx;
        vy = ny;
        vx = nx;
        vm = fmax(vm, fmax(fabs(vy), fabs(vx)));
    }
    const size_t base = ((size_t(qt) * d.h + qy) * d.w + qx) * 2;
    add(base, vy);
    add(base + 1, vx);
    if constexpr (MODE == 1) atomicMax(vmax_bits, __float_as_uint(float(vm) * 1.001f));
}

__global__ void narrow_kernel(const double* __restrict__ a, const double* __restrict__ b,
                              float* __restrict__ fa, float* __restrict__ fb, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        fa[i] = float(a[i]);
        fb[i] = float(b[i]);
    }
}

// ---- deterministic mode --------------------------------------------------------------
// bounds[0..2] = max|q|, max|k|, max|grad| (bits).  Per output element and entry, a patch
// reaches it through at most ps^2 pixels (reflection folds) with tap weights <= 1, so
// |dQ|, |dK| <= entries * ps^2 * max|g| * max|dS/dq|, max|dS/dk|.
__global__ void bwd_scales_kernel(const unsigned* bounds, int64_t entries, int ps, int metric,
                                  double* scales) {
    const double qm = __uint_as_float(bounds[0]), km = __uint_as_float(bounds[1]);
    const double gm = __uint_as_float(bounds[2]);
    const double dsq = metric == SNLS_METRIC_IP ? km : 2.0 * (qm + km);
    const double dsk = metric == SNLS_METRIC_IP ? qm : 2.0 * (qm + km);
    const double n = double(entries) * ps * ps * gm * 1.001;
    scales[0] = pow2_scale(n * dsq);
    scales[1] = pow2_scale(n * dsk);
}

// Flows: per element and entry at most wt links' 4 taps plus the base pixel touch it (each
// tap weight <= 1), with |v| <= vmax along every chain.
__global__ void flow_scale_kernel(const unsigned* vmax_bits, int64_t entries, int wt, double* scale) {
    const double vm = __uint_as_float(*vmax_bits);
    *scale = pow2_scale(double(entries) * (4.0 * (wt > 1 ? wt : 1) + 1.0) * vm * 1.001);
}


}  // namespace

// `gyx` scratch: rows * topl * 2 doubles, then two fp64 flow-gradient accumulators of
// T*H*W*2 doubles each (the flow gradient sums many cancelling terms: fp64 atomics, then
// one narrowing pass), all zeroed by the caller.
int launch_search_bwd_impl(const float* grad, const float* offsets, const float* chains,
                           const double* centers, const double* chains64, const float* q,
                           const float* k, Dims d, int wt, int ps, int topl, int metric, float* dq,
                           float* dk, float* dff, float* dbf, double* gyx, cudaStream_t st) {
    double* dff64 = gyx + size_t(d.rows) * topl * 2;
    const int64_t nfl = int64_t(d.t) * d.h * d.w * 2;
    double* dbf64 = dff64 + nfl;
    const Sink sq{dq, nullptr, nullptr}, sk{dk, nullptr, nullptr};
    launch_phase1<false>(grad, offsets, centers, q, k, d, ps, topl, metric, sq, sk, gyx, st);
    const int64_t ne = d.rows * topl;
    search_bwd_route<0><<<unsigned((ne + 255) / 256), 256, 0, st>>>(
        grad, offsets, chains, d, wt, topl, gyx, 1, dff64, dbf64, nullptr, nullptr, nullptr, nullptr,
        centers, chains64);
    narrow_kernel<<<unsigned(std::min<int64_t>((nfl + 255) / 256, 4096)), 256, 0, st>>>(dff64, dbf64, dff,
                                                                                       dbf, nfl);
    return 3;
}

#ifndef SNLS_WBWD_LSPLIT_IL
#define SNLS_WBWD_LSPLIT_IL 1
#endif
bool train_bwd_interleavable(int ps, int f) {
    static const int on = [] {
        const char* e = std::getenv("SNLS_TRAIN_BWD_INTERLEAVE");
        return e ? std::atoi(e) : 1;
    }();
    return on && kDqSm && (ps == 5 || ps == 7) && (f == 32 || f == 64);
}

namespace {
template <int P, int FT, bool DET>
void launch_interleaved_p(const float* grad, const float* offsets, const double* centers, const float* q,
                          const float* k, Dims d, int topl, int metric, Sink sq, Sink sk, double* gyx,
                          const WpsumBwdArgs& wp, cudaStream_t st) {
    constexpr int NL = FT / 2, LS = SNLS_WBWD_LSPLIT_IL;
    const unsigned n_search = unsigned((d.rows * (FT / 32) + 3) / 4);
    const unsigned n_wpsum = unsigned((wp.a.d.rows * LS + 128 / NL - 1) / (128 / NL));
    const size_t smem = size_t(4) * P * P * 32 * sizeof(float) * 2;  // = the wpsum body's [128/NL][P*P][NL] u64
    static_assert(size_t(128 / NL) * P * P * NL * sizeof(u64) <= size_t(4) * P * P * 32 * sizeof(float) * 2, "smem");
    auto go = [&](auto kern) {
        ensure_smem(kern, smem);
        kern<<<n_search + n_wpsum, 128, smem, st>>>(grad, offsets, q, k, d, topl, sq, sk, gyx, centers, wp,
                                                    n_search, n_wpsum);
    };
    const bool ip = metric == SNLS_METRIC_IP;
    if (centers)
        ip ? go(train_bwd_interleaved<P, true, FT, 1, NL, LS, DET>) : go(train_bwd_interleaved<P, true, FT, 2, NL, LS, DET>);
    else
        ip ? go(train_bwd_interleaved<P, false, FT, 1, NL, LS, DET>) : go(train_bwd_interleaved<P, false, FT, 2, NL, LS, DET>);
}

template <bool DET>
void launch_interleaved_any(const float* grad, const float* offsets, const double* centers, const float* q,
                            const float* k, Dims d, int ps, int topl, int metric, Sink sq, Sink sk,
                            double* gyx, const WpsumBwdArgs& wp, cudaStream_t st) {
    if (ps == 7)
        d.f == 64 ? launch_interleaved_p<7, 64, DET>(grad, offsets, centers, q, k, d, topl, metric, sq, sk, gyx, wp, st)
                  : launch_interleaved_p<7, 32, DET>(grad, offsets, centers, q, k, d, topl, metric, sq, sk, gyx, wp, st);
    else
        d.f == 64 ? launch_interleaved_p<5, 64, DET>(grad, offsets, centers, q, k, d, topl, metric, sq, sk, gyx, wp, st)
                  : launch_interleaved_p<5, 32, DET>(grad, offsets, centers, q, k, d, topl, metric, sq, sk, gyx, wp, st);
}
}  // namespace

int launch_train_bwd_interleaved(const float* grad, const float* offsets, const float* chains,
                                 const double* centers, const double* chains64, const float* q,
                                 const float* k, Dims d, int wt, int ps, int topl, int metric,
                                 float* dq, float* dk, float* dff, float* dbf, double* gyx,
                                 const WpsumBwdArgs& wp, cudaStream_t st) {
    if (!train_bwd_interleavable(ps, d.f)) return 0;
    const Sink sq{dq, nullptr, nullptr}, sk{dk, nullptr, nullptr};
    launch_interleaved_any<false>(grad, offsets, centers, q, k, d, ps, topl, metric, sq, sk, gyx, wp, st);
    double* dff64 = gyx + size_t(d.rows) * topl * 2;
    const int64_t nfl = int64_t(d.t) * d.h * d.w * 2;
    double* dbf64 = dff64 + nfl;
    const int64_t ne = d.rows * topl;
    search_bwd_route<0><<<unsigned((ne + 255) / 256), 256, 0, st>>>(
        grad, offsets, chains, d, wt, topl, gyx, 1, dff64, dbf64, nullptr, nullptr, nullptr, nullptr,
        centers, chains64);
    narrow_kernel<<<unsigned(std::min<int64_t>((nfl + 255) / 256, 4096)), 256, 0, st>>>(dff64, dbf64, dff,
                                                                                       dbf, nfl);
    return 3;
}

// Deterministic backward: same arithmetic, int64 fixed-point accumulation (see Sink).
// Workspace (from `work(bytes)`, zeroed here): scales, bound bits, per-entry (gy, gx)
// partials, int64 dQ, dK and flow accumulators.
int launch_search_bwd_det(const float* grad, const float* offsets, const float* chains,
                          const double* centers, const double* chains64, const float* q,
                          const float* k, Dims d, int wt, int ps, int topl, int metric, float* dq,
                          float* dk, float* dff, float* dbf,
                          const std::function<void*(size_t)>& work, cudaStream_t st,
                          const WpsumBwdArgs* wp) {
    const int64_t ne = d.rows * topl;
    const int64_t nv = int64_t(d.t) * d.h * d.w * d.f;
    const int64_t nfl = int64_t(d.t) * d.h * d.w * 2;
    const int parts = std::max((d.f + 31) / 32, d.f % 4 == 0 ? d.f / 4 : d.f);
    const size_t head = 64;  // 4 doubles of scales + 4 uint bounds, padded
    const size_t bytes = head + size_t(ne) * parts * 2 * sizeof(double) +
                         size_t(2 * nv + 2 * nfl) * sizeof(unsigned long long);
    char* w = static_cast<char*>(work(bytes));
    if (!w) return -1;
    cudaMemsetAsync(w, 0, bytes, st);
    double* scales = reinterpret_cast<double*>(w);  // [0] dQ, [1] dK, [2] flows
    unsigned* bounds = reinterpret_cast<unsigned*>(w + 32);  // |q|, |k|, |g|, |v|
    double* gyx = reinterpret_cast<double*>(w + head);
    auto* iq = reinterpret_cast<unsigned long long*>(gyx + size_t(ne) * parts * 2);
    unsigned long long* ik = iq + nv;
    unsigned long long* iff = ik + nv;
    unsigned long long* ibf = iff + nfl;
    const int64_t nq_all = int64_t(d.t) * d.h * d.w * d.f;
    absmax_kernel<<<592, 256, 0, st>>>(q, nq_all, bounds + 0);
    absmax_kernel<<<592, 256, 0, st>>>(k, nq_all, bounds + 1);
    absmax_kernel<<<148, 256, 0, st>>>(grad, ne, bounds + 2);
    bwd_scales_kernel<<<1, 1, 0, st>>>(bounds, ne, ps, metric, scales);
    const Sink sq{nullptr, iq, scales}, sk{nullptr, ik, scales + 1};
    int np;
    if (wp && train_bwd_interleavable(ps, d.f)) {  // the wpsum backward's blocks beside phase 1
        launch_interleaved_any<true>(grad, offsets, centers, q, k, d, ps, topl, metric, sq, sk, gyx, *wp, st);
        np = (d.f + 31) / 32;
    } else {
        np = launch_phase1<true>(grad, offsets, centers, q, k, d, ps, topl, metric, sq, sk, gyx, st);
    }
    const unsigned blocks = unsigned((ne + 255) / 256);
    search_bwd_route<1><<<blocks, 256, 0, st>>>(grad, offsets, chains, d, wt, topl, gyx, np, nullptr, nullptr,
                                                 nullptr, nullptr, nullptr, bounds + 3, centers, chains64);
    flow_scale_kernel<<<1, 1, 0, st>>>(bounds + 3, ne, wt, scales + 2);
    search_bwd_route<2><<<blocks, 256, 0, st>>>(grad, offsets, chains, d, wt, topl, gyx, np, nullptr, nullptr,
                                                 iff, ibf, scales + 2, nullptr, centers, chains64);
    const unsigned cb = unsigned(std::min<int64_t>((nv + 255) / 256, 4096));
    fixed_to_float_kernel<<<cb, 256, 0, st>>>(iq, scales, dq, nv);
    fixed_to_float_kernel<<<cb, 256, 0, st>>>(ik, scales + 1, dk, nv);
    const unsigned fb = unsigned(std::min<int64_t>((nfl + 255) / 256, 4096));
    fixed_to_float_kernel<<<fb, 256, 0, st>>>(iff, scales + 2, dff, nfl);
    fixed_to_float_kernel<<<fb, 256, 0, st>>>(ibf, scales + 2, dbf, nfl);
    return 13;
}

}  // namespace snls_gpu
