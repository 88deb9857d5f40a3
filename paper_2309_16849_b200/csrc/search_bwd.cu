// Search backward (shifted_nls_backward, search.cpp:499-711) on device.
//
// Phase 1: one thread per (selected entry, channel group).  It replays the entry's patch
// (same taps as the forward), scatters dQ into the reflected query pixels and dK into the
// 4 bilinear taps with atomics, and accumulates its share of dS/d(ky, kx) in fp64.  The
// per-entry (gy, gx) is reduced across the channel-group threads with fp64 atomics.
// Phase 2: one thread per entry routes (gy, gx) back through the composition chain
// (search.cpp:584-666): dt >= 0 into dFflow, dt < 0 into dBflow, v <- (I + J)^T v per link.
// Entries with a zero upstream gradient are skipped (search.cpp:692).
#include "common.cuh"
#include "kernels.h"

namespace snls_gpu {

namespace {

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
    if (vec == 4)
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
