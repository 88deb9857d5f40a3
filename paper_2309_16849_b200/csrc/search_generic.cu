// Generic search path: any ws / ps / stride1 / topl, one warp per query.
//
// Each lane evaluates window slots lane, lane+32, ... exactly as patch_similarity does
// (search.cpp:124-151): (py, px, channel) order, bilinear key reads per patch pixel.  The
// per-query candidate row lives in shared memory only (never in HBM, unless the caller asks
// for the materialised grid of search.cpp:329-410), and top-L is a warp-shuffle selection
// keyed on (value desc, slot asc) -- the reference's tie rule (search.cpp:187-197).
// This path is the fallback for fractional stride1 and the correctness twin of the tiled
// stride1 == 1 kernel in search_tiled.cu.
#include "common.cuh"
#include "kernels.h"

namespace snls_gpu {

namespace {

template <int VEC>
__device__ float patch_sim_generic(const float* __restrict__ q, const float* __restrict__ k,
                                   const Dims& d, int qt, int qy, int qx, int kt, double ky,
                                   double kx, int ps, int metric) {
    const int half = ps / 2;
    float acc = 0.f;
    for (int py = -half; py <= half; ++py) {
        const int ry = reflect_near(qy + py, d.h);
        for (int px = -half; px <= half; ++px) {
            const int rx = reflect_near(qx + px, d.w);
            const Taps t = taps_at(ky + double(py), kx + double(px), d.h, d.w);
            const float* qp = q + vidx(d, qt, ry, rx);
            const float* a = k + vidx(d, kt, t.y0, t.x0);
            const float* b = k + vidx(d, kt, t.y0, t.x1);
            const float* c = k + vidx(d, kt, t.y1, t.x0);
            const float* e = k + vidx(d, kt, t.y1, t.x1);
            if (VEC == 4) {
                for (int ch = 0; ch < d.f; ch += 4) {
                    const float4 qv = __ldg(reinterpret_cast<const float4*>(qp + ch));
                    const float4 av = __ldg(reinterpret_cast<const float4*>(a + ch));
                    const float4 bv = __ldg(reinterpret_cast<const float4*>(b + ch));
                    const float4 cv = __ldg(reinterpret_cast<const float4*>(c + ch));
                    const float4 ev = __ldg(reinterpret_cast<const float4*>(e + ch));
                    const float k0 = blend(t, av.x, bv.x, cv.x, ev.x);
                    const float k1 = blend(t, av.y, bv.y, cv.y, ev.y);
                    const float k2 = blend(t, av.z, bv.z, cv.z, ev.z);
                    const float k3 = blend(t, av.w, bv.w, cv.w, ev.w);
                    if (metric == SNLS_METRIC_IP) {
                        acc = fmaf(qv.x, k0, acc);
                        acc = fmaf(qv.y, k1, acc);
                        acc = fmaf(qv.z, k2, acc);
                        acc = fmaf(qv.w, k3, acc);
                    } else {
                        float r;
                        r = qv.x - k0; acc = fmaf(-r, r, acc);
                        r = qv.y - k1; acc = fmaf(-r, r, acc);
                        r = qv.z - k2; acc = fmaf(-r, r, acc);
                        r = qv.w - k3; acc = fmaf(-r, r, acc);
                    }
                }
            } else {
                for (int ch = 0; ch < d.f; ++ch) {
                    const float kv = blend(t, __ldg(a + ch), __ldg(b + ch), __ldg(c + ch),
                                           __ldg(e + ch));
                    const float qv = __ldg(qp + ch);
                    if (metric == SNLS_METRIC_IP) {
                        acc = fmaf(qv, kv, acc);
                    } else {
                        const float r = qv - kv;
                        acc = fmaf(-r, r, acc);
                    }
                }
            }
        }
    }
    return acc;
}

// Warp-cooperative selection of the L best candidates of one row held in `cand` (length n).
// Selected entries are overwritten with -inf.  Writes keys (or ~0 when underfull) to `out`.
__device__ void warp_select(float* cand, int n, int topl, uint64_t* out) {
    const int lane = threadIdx.x & 31;
    for (int li = 0; li < topl; ++li) {
        uint64_t best = 0;
        for (int s = lane; s < n; s += 32) {
            const float v = cand[s];
            if (eligible(v)) {
                const uint64_t key = pack_key(v, uint32_t(s));
                best = key > best ? key : best;
            }
        }
        best = warp_max_u64(best);
        if (best == 0) {  // nothing eligible left: underfull row
            if (lane == 0) out[li] = ~uint64_t(0);
            continue;
        }
        const uint32_t s = key_slot(best);
        if (lane == 0) out[li] = best;
        if (int(s % 32) == lane) cand[s] = -INFINITY;
        __syncwarp();
    }
}

struct SearchArgs {
    const float* q;
    const float* k;
    const float* ff;
    const float* bf;
    Dims d;
    int ws, wt, ps, topl, metric;
    double stride1;
    float beta;
    float* sims;
    float* offsets;
    float* chains;
    float* weights;
    float* grid;          // optional materialised rows x n
    float* grid_offsets;  // optional rows x n x 3
    int select;           // 0: only write the grid
    int* err;
    const float* grid_in;  // candidates already materialised (full-grid mode)
};

template <int VEC>
__global__ void __launch_bounds__(128) search_generic_kernel(SearchArgs a) {
    extern __shared__ unsigned char smem_raw[];
    const int warps = blockDim.x / 32;
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int nfr = 2 * a.wt + 1, ss = a.ws * a.ws, n = nfr * ss, half_ws = a.ws / 2;
    // per-warp layout: shifts (2 doubles per frame) | keys (topl u64) | candidates (n floats)
    const size_t per_warp = size_t(nfr) * 16 + size_t(a.topl) * 8 + size_t(n) * 4;
    unsigned char* base = smem_raw + size_t(warp) * ((per_warp + 15) & ~size_t(15));
    double* shifts = reinterpret_cast<double*>(base);
    uint64_t* keys = reinterpret_cast<uint64_t*>(base + size_t(nfr) * 16);
    float* cand = reinterpret_cast<float*>(base + size_t(nfr) * 16 + size_t(a.topl) * 8);

    const int64_t row = int64_t(blockIdx.x) * warps + warp;
    if (row >= a.d.rows) return;
    int qt, qy, qx;
    row_coords(a.d, row, qt, qy, qx);

    for (int fp = lane; fp < nfr; fp += 32) {
        const int dt = scan_dt(fp), kt = qt + dt;
        double sdy = 0.0, sdx = 0.0;
        if (kt >= 0 && kt < a.d.t) shift_to(a.ff, a.bf, a.d.h, a.d.w, qt, qy, qx, dt, sdy, sdx);
        shifts[2 * fp] = sdy;
        shifts[2 * fp + 1] = sdx;
    }
    __syncwarp();

    for (int s = lane; a.grid_in && s < n; s += 32) cand[s] = a.grid_in[size_t(row) * n + s];
    for (int s = lane; !a.grid_in && s < n; s += 32) {
        const int fp = s / ss, rem = s % ss;
        const int dt = scan_dt(fp), kt = qt + dt;
        const int dyi = rem / a.ws, dxi = rem % a.ws;
        float v = -INFINITY;
        const double cy = double(qy) + shifts[2 * fp], cx = double(qx) + shifts[2 * fp + 1];
        const double ky = cy + a.stride1 * double(dyi - half_ws);
        const double kx = cx + a.stride1 * double(dxi - half_ws);
        if (kt >= 0 && kt < a.d.t)  // off-clip frames never compete (search.cpp:300)
            v = patch_sim_generic<VEC>(a.q, a.k, a.d, qt, qy, qx, kt, ky, kx, a.ps, a.metric);
        cand[s] = v;
        if (a.grid) {
            const size_t e = size_t(row) * n + s;
            a.grid[e] = v;
            if (a.grid_offsets) {
                const bool on = kt >= 0 && kt < a.d.t;
                a.grid_offsets[e * 3 + 0] = float(dt);
                a.grid_offsets[e * 3 + 1] = on ? float(ky - double(qy)) : 0.f;
                a.grid_offsets[e * 3 + 2] = on ? float(kx - double(qx)) : 0.f;
            }
        }
    }
    __syncwarp();
    if (!a.select) return;

    warp_select(cand, n, a.topl, keys);
    __syncwarp();

    // emit_row (search.cpp:207-234) + fused softmax_rows (aggregate.cpp:16-37)
    float zmax = -INFINITY;
    for (int li = lane; li < a.topl; li += 32) {
        const uint64_t key = keys[li];
        const size_t e = size_t(row) * a.topl + li;
        float v = -INFINITY, o0 = 0.f, o1 = 0.f, o2 = 0.f;
        int dt = 0;
        if (key != ~uint64_t(0)) {
            const uint32_t s = key_slot(key);
            v = key_value(key);
            const int fp = int(s) / ss, rem = int(s) % ss;
            dt = scan_dt(fp);
            const double cy = double(qy) + shifts[2 * fp], cx = double(qx) + shifts[2 * fp + 1];
            const double ky = cy + a.stride1 * double(rem / a.ws - half_ws);
            const double kx = cx + a.stride1 * double(rem % a.ws - half_ws);
            o0 = float(dt);
            o1 = float(ky - double(qy));
            o2 = float(kx - double(qx));
        }
        a.sims[e] = v;
        a.offsets[e * 3 + 0] = o0;
        a.offsets[e * 3 + 1] = o1;
        a.offsets[e * 3 + 2] = o2;
        if (a.chains && a.wt > 1) {
            const int cs = a.wt - 1;
            float* lk = a.chains + e * size_t(cs) * 6;
            for (int j = 0; j < cs * 6; ++j) lk[j] = 0.f;
            if (dt > 1 || dt < -1) {
                double sdy, sdx;
                shift_to(a.ff, a.bf, a.d.h, a.d.w, qt, qy, qx, dt, sdy, sdx, lk);
            }
        }
        zmax = fmaxf(zmax, a.beta * v);
    }
    if (a.weights) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
        float sum = 0.f;
        for (int li = lane; li < a.topl; li += 32) {
            const float z = a.beta * a.sims[size_t(row) * a.topl + li];
            if (!isfinite(z)) latch(a.err, kErrSoftmax);
            sum += __expf(z - zmax);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        for (int li = lane; li < a.topl; li += 32) {
            const size_t e = size_t(row) * a.topl + li;
            a.weights[e] = __expf(a.beta * a.sims[e] - zmax) / sum;
        }
    }
}

__global__ void flows_finite_kernel(const float* __restrict__ ff, const float* __restrict__ bf,
                                    int64_t n, int* err) {
    bool bad_f = false, bad_b = false;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        bad_f |= !isfinite(__ldg(ff + i));
        bad_b |= !isfinite(__ldg(bf + i));
    }
    if (__any_sync(0xffffffffu, bad_f) && (threadIdx.x & 31) == 0) latch(err, kErrFflow);
    if (__any_sync(0xffffffffu, bad_b) && (threadIdx.x & 31) == 0) latch(err, kErrBflow);
}

// top_l over a materialised grid (search.cpp:430-468): one warp per row.
__global__ void __launch_bounds__(128) topl_kernel(int64_t rows, int cols, const float* full,
                                                   const float* full_offsets, int topl,
                                                   float* sel, float* sel_offsets, int* err) {
    extern __shared__ unsigned char smem_raw[];
    const int warps = blockDim.x / 32, warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const size_t per_warp = ((size_t(topl) * 8 + size_t(cols) * 4) + 15) & ~size_t(15);
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw + warp * per_warp);
    float* cand = reinterpret_cast<float*>(smem_raw + warp * per_warp + size_t(topl) * 8);
    const int64_t row = int64_t(blockIdx.x) * warps + warp;
    if (row >= rows) return;
    for (int s = lane; s < cols; s += 32) cand[s] = full[size_t(row) * cols + s];
    __syncwarp();
    warp_select(cand, cols, topl, keys);
    __syncwarp();
    for (int li = lane; li < topl; li += 32) {
        const uint64_t key = keys[li];
        const size_t e = size_t(row) * topl + li;
        if (key == ~uint64_t(0)) {
            latch(err, kErrTopl);
            sel[e] = -INFINITY;
            for (int c = 0; c < 3; ++c) sel_offsets[e * 3 + c] = 0.f;
            continue;
        }
        const uint32_t s = key_slot(key);
        sel[e] = key_value(key);
        for (int c = 0; c < 3; ++c)
            sel_offsets[e * 3 + c] = full_offsets[(size_t(row) * cols + s) * 3 + c];
    }
}

// Chains + softmax for the full-grid path, computed from the selected offsets.
__global__ void emit_tape_kernel(const float* ff, const float* bf, Dims d, int wt, int topl,
                                 const float* offsets, float* chains) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= d.rows * topl) return;
    const int64_t row = e / topl;
    int qt, qy, qx;
    row_coords(d, row, qt, qy, qx);
    const int cs = wt - 1;
    float* lk = chains + size_t(e) * cs * 6;
    for (int j = 0; j < cs * 6; ++j) lk[j] = 0.f;
    const int dt = int(rintf(offsets[size_t(e) * 3]));
    if (dt > 1 || dt < -1) {
        double sdy, sdx;
        shift_to(ff, bf, d.h, d.w, qt, qy, qx, dt, sdy, sdx, lk);
    }
}

// The reference's fp64 SearchTape (search.hpp:89-110) from the device tape: absolute key
// centres (kt, ky, kx) and absolute chain links, recomputed in fp64 from the flows exactly
// as emit_row builds them (search.cpp:207-234): ky = (qy + sdy) + stride1 * (dyi - ws/2), the
// window index dyi recovered from the fp32 offset (its rounding is far below stride1 / 2).
__global__ void tape64_kernel(const float* ff, const float* bf, Dims d, int ws, int wt, int topl,
                              double stride1, const float* offsets, double* centers,
                              double* chains, const float* sims, double* sims64,
                              double* offsets64) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= d.rows * topl) return;
    const int64_t row = e / topl;
    int qt, qy, qx;
    row_coords(d, row, qt, qy, qx);
    const float* o = offsets + size_t(e) * 3;
    const int dt = int(rintf(o[0]));
    const int cs = wt > 1 ? wt - 1 : 0;
    double* lk = chains ? chains + size_t(e) * cs * 6 : nullptr;
    if (lk)
        for (int j = 0; j < cs * 6; ++j) lk[j] = 0.0;
    double sdy = 0.0, sdx = 0.0;
    const int kt = qt + dt;
    if (kt >= 0 && kt < d.t) shift_to_t<double>(ff, bf, d.h, d.w, qt, qy, qx, dt, sdy, sdx,
                                                (dt > 1 || dt < -1) ? lk : nullptr);
    const double ny = rint((double(o[1]) - sdy) / stride1), nx = rint((double(o[2]) - sdx) / stride1);
    const double ky = (double(qy) + sdy) + stride1 * ny, kx = (double(qx) + sdx) + stride1 * nx;
    if (centers) {
        double* c = centers + size_t(e) * 3;
        c[0] = double(kt);
        c[1] = ky;
        c[2] = kx;
    }
    if (offsets64) {  // emit_row's offsets (search.cpp:222-224): (dt, ky - qy, kx - qx) in fp64
        double* o64 = offsets64 + size_t(e) * 3;
        o64[0] = double(dt);
        o64[1] = ky - double(qy);
        o64[2] = kx - double(qx);
    }
    if (sims64) sims64[e] = double(sims[e]);
}

// replay_similarities (search.cpp:470-493): one thread per selected entry.
template <int VEC>
__global__ void replay_kernel(const float* q, const float* k, Dims d, int ps, int metric,
                              int topl, const float* offsets, float* sims) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= d.rows * topl) return;
    const int64_t row = e / topl;
    int qt, qy, qx;
    row_coords(d, row, qt, qy, qx);
    const float* o = offsets + size_t(e) * 3;
    const int kt = qt + int(rintf(o[0]));
    sims[e] = patch_sim_generic<VEC>(q, k, d, qt, qy, qx, kt, double(qy) + double(o[1]),
                                     double(qx) + double(o[2]), ps, metric);
}

size_t generic_smem_per_warp(int nfr, int topl, int n) {
    return ((size_t(nfr) * 16 + size_t(topl) * 8 + size_t(n) * 4) + 15) & ~size_t(15);
}

}  // namespace

int launch_flows_check(const float* ff, const float* bf, int64_t n, int* err, cudaStream_t st) {
    if (!ff) return 0;
    const int blocks = int(std::min<int64_t>((n + 255) / 256, 148 * 8));
    flows_finite_kernel<<<blocks, 256, 0, st>>>(ff, bf, n, err);
    return 1;
}

int launch_search_generic(const GenericSearch& g, cudaStream_t st) {
    const int nfr = 2 * g.wt + 1, n = nfr * g.ws * g.ws;
    const size_t per_warp = generic_smem_per_warp(nfr, g.topl, n);
    int warps = 4;
    while (warps > 1 && per_warp * warps > 200 * 1024) warps >>= 1;
    if (per_warp * warps > 227 * 1024) return -1;
    SearchArgs a;
    a.q = g.q;
    a.k = g.k;
    a.ff = g.ff;
    a.bf = g.bf;
    a.d = g.d;
    a.ws = g.ws;
    a.wt = g.wt;
    a.ps = g.ps;
    a.topl = g.topl;
    a.metric = g.metric;
    a.stride1 = g.stride1;
    a.beta = g.beta;
    a.sims = g.sims;
    a.offsets = g.offsets;
    a.chains = g.chains;
    a.weights = g.weights;
    a.grid = g.grid;
    a.grid_offsets = g.grid_offsets;
    a.select = g.select;
    a.err = g.err;
    a.grid_in = g.grid_in;
    const size_t smem = per_warp * warps;
    const unsigned blocks = unsigned((g.d.rows + warps - 1) / warps);
    if (g.d.f % 4 == 0) {
        ensure_smem(search_generic_kernel<4>, smem);
        search_generic_kernel<4><<<blocks, warps * 32, smem, st>>>(a);
    } else {
        ensure_smem(search_generic_kernel<1>, smem);
        search_generic_kernel<1><<<blocks, warps * 32, smem, st>>>(a);
    }
    return 1;
}

int launch_topl(int64_t rows, int cols, const float* full, const float* full_offsets, int topl,
                float* sel, float* sel_offsets, int* err, cudaStream_t st) {
    const size_t per_warp = ((size_t(topl) * 8 + size_t(cols) * 4) + 15) & ~size_t(15);
    int warps = 4;
    while (warps > 1 && per_warp * warps > 200 * 1024) warps >>= 1;
    if (per_warp * warps > 227 * 1024) return -1;
    const size_t smem = per_warp * warps;
    ensure_smem(topl_kernel, smem);
    topl_kernel<<<unsigned((rows + warps - 1) / warps), warps * 32, smem, st>>>(
        rows, cols, full, full_offsets, topl, sel, sel_offsets, err);
    return 1;
}

int launch_emit_tape(const float* ff, const float* bf, Dims d, int wt, int topl,
                     const float* offsets, float* chains, cudaStream_t st) {
    const int64_t n = d.rows * topl;
    emit_tape_kernel<<<unsigned((n + 127) / 128), 128, 0, st>>>(ff, bf, d, wt, topl, offsets,
                                                               chains);
    return 1;
}

int launch_tape64(const float* ff, const float* bf, Dims d, int ws, int wt, int topl, double stride1,
                  const float* offsets, double* centers, double* chains, const float* sims,
                  double* sims64, double* offsets64, cudaStream_t st) {
    const int64_t n = d.rows * topl;
    tape64_kernel<<<unsigned((n + 127) / 128), 128, 0, st>>>(ff, bf, d, ws, wt, topl, stride1, offsets,
                                                            centers, chains, sims, sims64, offsets64);
    return 1;
}

// replay through the generic plan at the fp64 tape centres: the forward's own expression
// for every slot (ky = (qy + sdy) + stride1 (dyi - ws/2), search_generic_kernel), so equal bits
template <int VEC>
__global__ void replay64_kernel(const float* q, const float* k, Dims d, int ps, int metric, int topl,
                                const double* centers, float* sims) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= d.rows * topl) return;
    int qt, qy, qx;
    row_coords(d, e / topl, qt, qy, qx);
    const double* c = centers + size_t(e) * 3;
    const int kt = int(c[0]);
    sims[e] = (kt >= 0 && kt < d.t) ? patch_sim_generic<VEC>(q, k, d, qt, qy, qx, kt, c[1], c[2], ps, metric)
                                    : -INFINITY;
}

int launch_replay64(const float* q, const float* k, Dims d, int ps, int metric, int topl,
                    const double* centers, float* sims, cudaStream_t st) {
    const int64_t n = d.rows * topl;
    if (d.f % 4 == 0)
        replay64_kernel<4><<<unsigned((n + 127) / 128), 128, 0, st>>>(q, k, d, ps, metric, topl, centers, sims);
    else
        replay64_kernel<1><<<unsigned((n + 127) / 128), 128, 0, st>>>(q, k, d, ps, metric, topl, centers, sims);
    return 1;
}

int launch_replay(const float* q, const float* k, Dims d, int ps, int metric, int topl,
                  const float* offsets, float* sims, cudaStream_t st) {
    const int64_t n = d.rows * topl;
    if (d.f % 4 == 0)
        replay_kernel<4><<<unsigned((n + 127) / 128), 128, 0, st>>>(q, k, d, ps, metric, topl,
                                                                    offsets, sims);
    else
        replay_kernel<1><<<unsigned((n + 127) / 128), 128, 0, st>>>(q, k, d, ps, metric, topl,
                                                                    offsets, sims);
    return 1;
}

}  // namespace snls_gpu
