// Aggregation kernels: softmax_rows, the deterministic wpsum gather, gather_stack and the
// wpsum backward (aggregate.cpp).
//
// wpsum is evaluated as the reference's fixed-order GATHER (aggregate.cpp:124-203): every
// output pixel is owned by exactly one thread group, which visits its contributing query
// units in the reference order (footprint py/px ascending, then the owning query's cell
// completion) -- deterministic, no atomics, every output element written once, coalesced
// C-vectorised (float4) reads of V.  The backward scatters through 4 bilinear taps, so it
// uses atomics (the reference's non-deterministic mode, aggregate.cpp:451-458).
#include "common.cuh"
#include "kernels.h"

namespace snls_gpu {

namespace {

__device__ __forceinline__ int owner_index(int coord, int stride, int n) {  // aggregate.hpp:91-95
    int gi = (coord + (stride - 1) / 2) / stride;
    return gi > n - 1 ? n - 1 : gi;
}

__device__ __forceinline__ int clampi(int d, int half) { return d < -half ? -half : (d > half ? half : d); }

__device__ __forceinline__ void cell_span(int gi, int stride, int n, int extent, int& lo, int& hi) {
    const int a = (stride - 1) / 2;  // aggregate.cpp:71-75
    lo = gi == 0 ? 0 : gi * stride - a;
    hi = gi == n - 1 ? extent - 1 : gi * stride + (stride - 1 - a);
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
        split_pos(qy + pyu, __ldg(o + 1), iy, fy);
        split_pos(qx + pxu, __ldg(o + 2), ix, fx);
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
            const int64_t row = (int64_t(ti) * a.d.nh + qy / st) * a.d.nw + qx / st;
            if (!add_unit<VEC>(a, row, ti, qy, qx, py, px, l0, l1, c, acc)) return -1;
            ++cnt;
        }
    }
    const int qy = owner_index(y, st, a.d.nh) * st;
    const int qx = owner_index(x, st, a.d.nw) * st;
    if (abs(y - qy) > half || abs(x - qx) > half) {
        const int64_t row = (int64_t(ti) * a.d.nh + qy / st) * a.d.nw + qx / st;
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
    const int64_t npix = int64_t(a.d.t) * a.d.h * a.d.w;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= npix * groups) return;
    const int64_t pix = idx / groups;
    const int c = int(idx % groups) * VEC;
    const int x = int(pix % a.d.w);
    const int y = int((pix / a.d.w) % a.d.h);
    const int ti = int(pix / (int64_t(a.d.w) * a.d.h));
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
    const int64_t npix = int64_t(a.d.t) * a.d.h * a.d.w;
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= npix * groups * a.topl) return;
    const int li = int(idx / (npix * groups));
    const int64_t r = idx % (npix * groups);
    const int64_t pix = r / groups;
    const int c = int(r % groups) * VEC;
    const int x = int(pix % a.d.w);
    const int y = int((pix / a.d.w) % a.d.h);
    const int ti = int(pix / (int64_t(a.d.w) * a.d.h));
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
template <int VEC>
__global__ void __launch_bounds__(256) wpsum_bwd_kernel(AggArgs a, const float* __restrict__ go,
                                                        const int32_t* __restrict__ counts,
                                                        float* __restrict__ dv,
                                                        float* __restrict__ dw) {
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
        const float inv_cnt = 1.f / float(counts[(size_t(ti) * a.d.h + y) * a.d.w + x]);
        int iy, ix;
        float fy, fx;
        split_pos(qy + pyu, oy, iy, fy);
        split_pos(qx + pxu, ox, ix, fx);
        const Taps t = taps_from(iy, fy, ix, fx, a.d.h, a.d.w);
        const float* gp = go + vidx(a.d, ti, y, x) + c;
        const size_t i00 = vidx(a.d, kt, t.y0, t.x0) + c, i01 = vidx(a.d, kt, t.y0, t.x1) + c;
        const size_t i10 = vidx(a.d, kt, t.y1, t.x0) + c, i11 = vidx(a.d, kt, t.y1, t.x1) + c;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const float g = __ldg(gp + j) * inv_cnt;
            const float sample = blend(t, __ldg(a.v + i00 + j), __ldg(a.v + i01 + j),
                                       __ldg(a.v + i10 + j), __ldg(a.v + i11 + j));
            dw_acc = fmaf(g, sample, dw_acc);
            const float gv = g * wv;
            atomicAdd(dv + i00 + j, gv * t.w00);
            atomicAdd(dv + i01 + j, gv * t.w01);
            atomicAdd(dv + i10 + j, gv * t.w10);
            atomicAdd(dv + i11 + j, gv * t.w11);
        }
    }
    atomicAdd(dw + e, dw_acc);
}

}  // namespace

int launch_softmax(int64_t rows, int l, float beta, const float* sims, float* weights, int* err,
                   cudaStream_t st) {
    softmax_kernel<<<unsigned((rows + 127) / 128), 128, 0, st>>>(rows, l, beta, sims, weights, err);
    return 1;
}

int launch_wpsum(const AggArgs& a, float* out, int32_t* counts, cudaStream_t st) {
    const int64_t npix = int64_t(a.d.t) * a.d.h * a.d.w;
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
    const int64_t npix = int64_t(a.d.t) * a.d.h * a.d.w;
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
    if (a.d.f % 4 == 0) {
        const int64_t n = a.d.rows * a.topl * (a.d.f / 4);
        wpsum_bwd_kernel<4><<<unsigned((n + 255) / 256), 256, 0, st>>>(a, grad_out, counts, dv, dw);
    } else {
        const int64_t n = a.d.rows * a.topl * a.d.f;
        wpsum_bwd_kernel<1><<<unsigned((n + 255) / 256), 256, 0, st>>>(a, grad_out, counts, dv, dw);
    }
    return 1;
}

}  // namespace snls_gpu
