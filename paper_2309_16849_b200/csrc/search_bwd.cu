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
#include "common.cuh"
#include "kernels.h"

#ifndef SNLS_BWD_DQSM
#define SNLS_BWD_DQSM 1
#endif

namespace snls_gpu {

namespace {

constexpr bool kDqSm = SNLS_BWD_DQSM != 0;

template <int VEC>
__global__ void __launch_bounds__(256) search_bwd_entries(const float* __restrict__ grad,
                                                          const float* __restrict__ offsets,
                                                          const float* __restrict__ q,
                                                          const float* __restrict__ k, Dims d,
                                                          int ps, int topl, int metric,
                                                          float* dq, float* dk, double* gyx) {
    const int groups = d.f / VEC;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= d.rows * topl * groups) return;
    const int64_t e = idx / groups;
    const int c = int(idx % groups) * VEC;
    const float g = grad[e];
    if (g == 0.f) return;
    const int64_t row = e / topl;
    int qt, qy, qx;
    row_coords(d, row, qt, qy, qx);
    const float* o = offsets + size_t(e) * 3;
    const int kt = qt + int(rintf(o[0]));
    const float oy = o[1], ox = o[2];
    const int half = ps / 2;
    double gy = 0.0, gx = 0.0;
    for (int py = -half; py <= half; ++py) {
        const int ry = reflect_near(qy + py, d.h);
        for (int px = -half; px <= half; ++px) {
            const int rx = reflect_near(qx + px, d.w);
            int iy, ix;
            float fy, fx;
            split_pos(qy + py, oy, iy, fy);
            split_pos(qx + px, ox, ix, fx);
            const Taps t = taps_from(iy, fy, ix, fx, d.h, d.w);
            const size_t iq = vidx(d, qt, ry, rx) + c;
            const size_t i00 = vidx(d, kt, t.y0, t.x0) + c, i01 = vidx(d, kt, t.y0, t.x1) + c;
            const size_t i10 = vidx(d, kt, t.y1, t.x0) + c, i11 = vidx(d, kt, t.y1, t.x1) + c;
            // dS/d(ky, kx) sums hundreds of cancelling terms per entry: keep that chain in
            // fp64 (the dQ/dK scatter stays fp32)
            const double dfy = fy, dfx = fx;
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
                atomicAdd(dq + iq + j, float(double(g) * ds_dq));
                atomicAdd(dk + i00 + j, float(gk * w00));
                atomicAdd(dk + i01 + j, float(gk * w01));
                atomicAdd(dk + i10 + j, float(gk * w10));
                atomicAdd(dk + i11 + j, float(gk * w11));
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
    atomicAdd(gyx + 2 * e, gy);
    atomicAdd(gyx + 2 * e + 1, gx);
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
template <int P>
__global__ void __launch_bounds__(128, kDqSm ? 4 : 3) search_bwd_rows(const float* __restrict__ grad,
                                                          const float* __restrict__ offsets,
                                                          const float* __restrict__ q,
                                                          const float* __restrict__ k, Dims d,
                                                          int topl, int metric,
                                                          float* __restrict__ dq,
                                                          float* __restrict__ dk,
                                                          double* __restrict__ gyx) {
    constexpr int HP = P / 2;
    const int slices = (d.f + 31) / 32;
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= d.rows * slices) return;  // warp-uniform
    const int64_t row = wid / slices;
    const int c = int(wid % slices) * 32 + lane;
    const bool act = c < d.f;
    const int cc = act ? c : 0;
    // dynamic shared memory: [4 warps][P*P][32] query patch, then (kDqSm) the dQ partials
    extern __shared__ float s_bwd[];
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
        const float* o = offsets + size_t(e) * 3;
        const int kt = qt + int(rintf(__ldg(o)));
        const float oy = __ldg(o + 1), ox = __ldg(o + 2);
        const float fly = floorf(oy), flx = floorf(ox);
        const float fy = oy - fly, fx = ox - flx;
        const int by = qy - HP + int(fly), bx = qx - HP + int(flx);
        const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx;
        const float w10 = fy * (1.f - fx), w11 = fy * fx;
        unsigned bcol[P + 1];
#pragma unroll
        for (int j = 0; j <= P; ++j) bcol[j] = unsigned(reflect_near(bx + j, d.w)) * unsigned(d.f);
        const float* kb = k + size_t(kt) * frameF + cc;
        float* dkb = dk + size_t(kt) * frameF + cc;
        float ra[P + 1], rb[P + 1], ka[P + 1], kn[P + 1];
        size_t roa = size_t(reflect_near(by, d.h)) * rowF;
        size_t rob = size_t(reflect_near(by + 1, d.h)) * rowF;
#pragma unroll
        for (int j = 0; j <= P; ++j) {
            ra[j] = act ? __ldg(kb + roa + bcol[j]) : 0.f;
            rb[j] = act ? __ldg(kb + rob + bcol[j]) : 0.f;
            ka[j] = 0.f;
        }
        double sy = 0.0, sx = 0.0;
#pragma unroll
        for (int py = 0; py < P; ++py) {
            const size_t ron = size_t(reflect_near(by + py + 2, d.h)) * rowF;
#pragma unroll
            for (int j = 0; j <= P; ++j) kn[j] = 0.f;
            float ry = 0.f, rx = 0.f;  // this patch row's share of dS/d(ky, kx)
#pragma unroll
            for (int px = 0; px < P; ++px) {
                const float k00 = ra[px], k01 = ra[px + 1], k10 = rb[px], k11 = rb[px + 1];
                const float qv = sq[(py * P + px) * 32];
                // lerp form: the x-interpolated rows give the sample and both tap derivatives
                // (search.cpp:574-577) in 8 FP ops instead of 12
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
                ry = fmaf(gk, dkv_dy, ry);
                rx = fmaf(gk, dkv_dx, rx);
            }
            // dS/d(ky, kx) sums thousands of cancelling terms per entry: the per-row partials
            // are accumulated in fp64
            sy += double(ry);
            sx += double(rx);
            if (act) {  // raw row py of the block is complete
#pragma unroll
                for (int j = 0; j <= P; ++j) atomicAdd(dkb + roa + bcol[j], ka[j]);
            }
#pragma unroll
            for (int j = 0; j <= P; ++j) {
                ra[j] = rb[j];
                if (py + 1 < P) rb[j] = act ? __ldg(kb + ron + bcol[j]) : 0.f;  // (loading it a
                // row ahead into registers: same time, 36 B of spills)
                ka[j] = kn[j];
            }
            roa = rob;
            rob = ron;
        }
        if (act) {
#pragma unroll
            for (int j = 0; j <= P; ++j) atomicAdd(dkb + roa + bcol[j], ka[j]);
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            sy += __shfl_xor_sync(0xffffffffu, sy, m);
            sx += __shfl_xor_sync(0xffffffffu, sx, m);
        }
        if (lane == 0) {
            atomicAdd(gyx + 2 * e, sy);
            atomicAdd(gyx + 2 * e + 1, sx);
        }
    }
    if (act) {
        float* dqb = dq + size_t(qt) * frameF + cc;
#pragma unroll
        for (int py = 0; py < P; ++py)
#pragma unroll
            for (int px = 0; px < P; ++px)
                atomicAdd(dqb + size_t(qrow[py] + qcol[px]) * F, kDqSm ? sdq[(py * P + px) * 32] : dqa[py][px]);
    }
}

template <int P>
void launch_rows(const float* grad, const float* offsets, const float* q, const float* k, Dims d,
                 int topl, int metric, float* dq, float* dk, double* gyx, cudaStream_t st) {
    const int64_t warps = d.rows * ((d.f + 31) / 32);
    const size_t smem = size_t(4) * P * P * 32 * sizeof(float) * (kDqSm ? 2 : 1);
    ensure_smem(search_bwd_rows<P>, smem);
    search_bwd_rows<P><<<unsigned((warps + 3) / 4), 128, smem, st>>>(grad, offsets, q, k, d, topl, metric,
                                                                     dq, dk, gyx);
}

__global__ void search_bwd_route(const float* __restrict__ grad,
                                 const float* __restrict__ offsets,
                                 const float* __restrict__ chains, Dims d, int wt, int topl,
                                 const double* __restrict__ gyx, double* dff, double* dbf) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= d.rows * topl) return;
    if (grad[e] == 0.f) return;
    const int64_t row = e / topl;
    int qt, qy, qx;
    row_coords(d, row, qt, qy, qx);
    const int dt = int(rintf(offsets[size_t(e) * 3]));
    double* fld = dt >= 0 ? dff : dbf;
    const int step = dt >= 0 ? 1 : -1;
    const int m = dt == 0 ? 1 : (dt > 0 ? dt : -dt);
    double vy = gyx[2 * e], vx = gyx[2 * e + 1];
    const int cs = wt > 1 ? wt - 1 : 0;
    const float* chain = chains ? chains + size_t(e) * cs * 6 : nullptr;
    for (int kk = m - 1; kk >= 1; --kk) {
        const float* lk = chain + (kk - 1) * 6;
        int iy, ix;
        float fy, fx;
        split_pos(qy, lk[0], iy, fy);
        split_pos(qx, lk[1], ix, fx);
        const Taps t = taps_from(iy, fy, ix, fx, d.h, d.w);
        const int fr = qt + step * kk;
        auto at = [&](int y, int x, int comp) { return fld + ((size_t(fr) * d.h + y) * d.w + x) * 2 + comp; };
        atomicAdd(at(t.y0, t.x0, 0), vy * t.w00);
        atomicAdd(at(t.y0, t.x1, 0), vy * t.w01);
        atomicAdd(at(t.y1, t.x0, 0), vy * t.w10);
        atomicAdd(at(t.y1, t.x1, 0), vy * t.w11);
        atomicAdd(at(t.y0, t.x0, 1), vx * t.w00);
        atomicAdd(at(t.y0, t.x1, 1), vx * t.w01);
        atomicAdd(at(t.y1, t.x0, 1), vx * t.w10);
        atomicAdd(at(t.y1, t.x1, 1), vx * t.w11);
        const double ny = vy + double(lk[2]) * vy + double(lk[4]) * vx;
        const double nx = vx + double(lk[3]) * vy + double(lk[5]) * vx;
        vy = ny;
        vx = nx;
    }
    double* base = fld + ((size_t(qt) * d.h + qy) * d.w + qx) * 2;
    atomicAdd(base, vy);
    atomicAdd(base + 1, vx);
}

__global__ void narrow_kernel(const double* __restrict__ a, const double* __restrict__ b,
                              float* __restrict__ fa, float* __restrict__ fb, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        fa[i] = float(a[i]);
        fb[i] = float(b[i]);
    }
}

}  // namespace

// `gyx` scratch: rows * topl * 2 doubles, then two fp64 flow-gradient accumulators of
// T*H*W*2 doubles each (the flow gradient sums many cancelling terms: fp64 atomics, then
// one narrowing pass), all zeroed by the caller.
int launch_search_bwd_impl(const float* grad, const float* offsets, const float* chains,
                           const float* q, const float* k, Dims d, int wt, int ps, int topl,
                           int metric, float* dq, float* dk, float* dff, float* dbf, double* gyx,
                           cudaStream_t st) {
    double* dff64 = gyx + size_t(d.rows) * topl * 2;
    const int64_t nfl = int64_t(d.t) * d.h * d.w * 2;
    double* dbf64 = dff64 + nfl;
    const int vec = d.f % 4 == 0 ? 4 : 1;
    const int64_t n = d.rows * topl * (d.f / vec);
    if (ps == 1 || ps == 3 || ps == 5 || ps == 7) {
        switch (ps) {
            case 1: launch_rows<1>(grad, offsets, q, k, d, topl, metric, dq, dk, gyx, st); break;
            case 3: launch_rows<3>(grad, offsets, q, k, d, topl, metric, dq, dk, gyx, st); break;
            case 5: launch_rows<5>(grad, offsets, q, k, d, topl, metric, dq, dk, gyx, st); break;
            default: launch_rows<7>(grad, offsets, q, k, d, topl, metric, dq, dk, gyx, st); break;
        }
    } else if (vec == 4)
        search_bwd_entries<4><<<unsigned((n + 255) / 256), 256, 0, st>>>(grad, offsets, q, k, d, ps,
                                                                         topl, metric, dq, dk, gyx);
    else
        search_bwd_entries<1><<<unsigned((n + 255) / 256), 256, 0, st>>>(grad, offsets, q, k, d, ps,
                                                                         topl, metric, dq, dk, gyx);
    const int64_t ne = d.rows * topl;
    search_bwd_route<<<unsigned((ne + 255) / 256), 256, 0, st>>>(grad, offsets, chains, d, wt, topl,
                                                                 gyx, dff64, dbf64);
    narrow_kernel<<<unsigned(std::min<int64_t>((nfl + 255) / 256, 4096)), 256, 0, st>>>(dff64, dbf64, dff,
                                                                                       dbf, nfl);
    return 3;
}

}  // namespace snls_gpu
