// Query-stationary streaming Shifted-NLS forward for stride1 == 1: fused search + streaming
// top-L (+ optional softmax epilogue), sm_100a, FP32 FMA pipe.
//
// Same contract and tie rules as search_tiled.cu; different register plan, built for large
// patches (ps = 7 spills the tiled kernel's interpolated-row cache) and for cutting the
// per-region-row query reloads:
//  * G = F / VEC lanes per query, lane gl owns channels [gl*VEC, gl*VEC+VEC).  The whole
//    ps x ps query patch of the lane's channels is loaded ONCE into registers and reused for
//    every frame, region row and slot (search.cpp:129-132 reads it per slot).
//  * Per (query, frame) the (ws+ps-1)^2 key region is interpolated exactly once, streamed
//    pixel by pixel: region pixel (r, j) is blended from the two raw rows r, r+1 (sliding
//    column window, so 2 loads per pixel) and immediately contributes to every slot that
//    reads it, acc[s][j - px] += m(Q[P-1-s][px], k) -- nothing is cached per region row.
//  * Slot rows rotate through acc[P][W] as in the tiled kernel; a slot row completes after
//    its last region row, is reduce-scattered over the G lanes (identical addition tree for
//    every slot, so duplicate candidates tie exactly) and streamed into a rank-sharded
//    register top-L with strict '>' in ascending slot order (topl_insert, search.cpp:187-197).
//    Candidates not above the current rank topl-1 can never be selected and stop at one
//    compare.
// Per slot the accumulation order is (py, px, channel) ascending within a lane, then the
// fixed butterfly over lanes -- the same for every slot of every frame.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "search_select.cuh"

namespace snls_gpu {

namespace {

constexpr int pow2ceil(int n) { return n <= 1 ? 1 : 2 * pow2ceil((n + 1) / 2); }
constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

template <int P, int W, int VEC, int G>
struct StreamCfg {
    static constexpr int HP = P / 2, HW = W / 2, R = W + P - 1, F = G * VEC;
    static constexpr int QPW = 32 / G, WARPS = 4, QPB = QPW * WARPS;
};

// RP (replay_similarities, W = P): every "row" is one selected entry (row / topl its query),
// frame and window centre from the entry's fp64 tape centre; the full-grid write of the
// P x P window goes to a scratch row whose centre slot is the entry (the per-slot arithmetic
// does not depend on the slot's place in the window: bitwise equal to the forward).
template <int P, int W, int VEC, int G, int KMAX, int METRIC, int MINB, bool RP = false>
__global__ void __launch_bounds__(128, MINB) search_stream_kernel(TiledSearch a) {
    static_assert(W >= P, "window narrower than the patch: not instantiated");
    using C = StreamCfg<P, W, VEC, G>;
    constexpr int HP = C::HP, HW = C::HW, R = C::R, F = C::F;
    __shared__ uint64_t s_keys[C::QPB][16];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane / G, gl = lane % G;
    const int qslot = warp * C::QPW + gq;
    const int64_t row_raw = int64_t(blockIdx.x) * C::QPB + qslot;
    const bool row_ok = row_raw < a.d.rows;
    const int64_t row = row_ok ? row_raw : a.d.rows - 1;
    int qt, qy, qx;
    row_coords(a.d, RP ? row / a.topl : row, qt, qy, qx);
    const int H = a.d.h, Wd = a.d.w;
    const unsigned rowF = unsigned(Wd) * F;  // floats per image row
    const size_t frame_elems = size_t(H) * rowF;
    const int c0 = gl * VEC;
    const int nfr = RP ? 1 : 2 * a.wt + 1;

    // ---- the query patch, reflected integer pixels (search.cpp:129-132), in registers
    float qv[P][P][VEC];
    {
        const float* qb = a.q + size_t(qt) * frame_elems + c0;
#pragma unroll
        for (int py = 0; py < P; ++py) {
            const float* qr = qb + size_t(reflect_near(qy + py - HP, H)) * rowF;
#pragma unroll
            for (int px = 0; px < P; ++px) ldv<VEC>(qr + size_t(reflect_near(qx + px - HP, Wd)) * F, qv[py][px]);
        }
    }

    TopL<W, G, KMAX> sel;
    sel.init();
    const int thr_src = TopL<W, G, KMAX>::thr_lane(gq, a.topl), thr_idx = TopL<W, G, KMAX>::thr_entry(a.topl);
    float* grid_row = a.grid ? a.grid + size_t(row) * nfr * W * W : nullptr;

    for (int fp = 0; fp < nfr; ++fp) {
        const int dt = RP ? int(a.tape[size_t(row) * 3]) - qt : scan_dt(fp), kt = qt + dt;
        const bool on = row_ok && kt >= 0 && kt < a.d.t;
        if (!__any_sync(0xffffffffu, on)) {  // warp-uniform skip (search.cpp:300)
            if (a.grid && row_ok) write_off_frame<W, G>(a.grid, row, fp, nfr, gl);
            continue;
        }
        double sdy = 0.0, sdx = 0.0;
        if (!RP && on) shift_to(a.ff, a.bf, H, Wd, qt, qy, qx, dt, sdy, sdx);
        const double cy = RP ? a.tape[size_t(row) * 3 + 1] : double(qy) + sdy;
        const double cx = RP ? a.tape[size_t(row) * 3 + 2] : double(qx) + sdx;
        const double fby = floor(cy), fbx = floor(cx);
        const float fy = float(cy - fby), fx = float(cx - fbx);
        const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx;
        const float w10 = fy * (1.f - fx), w11 = fy * fx;
        const int by = int(fby) - HW - HP, bx = int(fbx) - HW - HP;  // (see search_tiled.cu)
        const float* kb = a.k + size_t(on ? kt : qt) * frame_elems + c0;
        // reflected column offsets of the region (tensor.cpp:23-29), once per frame
        unsigned xo[R + 1];
#pragma unroll
        for (int j = 0; j <= R; ++j) xo[j] = unsigned(reflect_near(bx + j, Wd)) * F;

        float acc[P][W];
#pragma unroll
        for (int s = 0; s < P; ++s)
#pragma unroll
            for (int b = 0; b < W; ++b) acc[s][b] = 0.f;

        const uint32_t slot_base = uint32_t(fp) * W * W;

        // One region row: stream its R pixels through all P rotating slot rows.  On the
        // first/last P-1 region rows some of those slot rows lie outside the window; their
        // accumulators are updated anyway (they are never emitted: a slot row is emitted
        // only after its last region row) -- a uniform straight-line body with no guards
        // beats guarded bodies on this pipe (measured: per-row compile-time ranges cost
        // more in instruction-cache misses than the wasted FMAs).
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
            const float* p0 = kb + unsigned(reflect_near(by + r, H)) * rowF;
            const float* p1 = kb + unsigned(reflect_near(by + r + 1, H)) * rowF;
            float a0[VEC], a1[VEC];
            ldv<VEC>(p0 + xo[0], a0);
            ldv<VEC>(p1 + xo[0], a1);
#pragma unroll
            for (int j = 0; j < R; ++j) {
                float b0[VEC], b1[VEC];
                ldv<VEC>(p0 + xo[j + 1], b0);
                ldv<VEC>(p1 + xo[j + 1], b1);
                float kr[VEC];
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    kr[v] = fmaf(w11, b1[v], fmaf(w10, a1[v], fmaf(w01, b0[v], w00 * a0[v])));
                    a0[v] = b0[v];
                    a1[v] = b1[v];
                }
#pragma unroll
                for (int s = 0; s < P; ++s) {
#pragma unroll
                    for (int px = 0; px < P; ++px) {
                        const int b = j - px;
                        if (b < 0 || b >= W) continue;  // compile time
#pragma unroll
                        for (int v = 0; v < VEC; ++v) {
                            if (METRIC == SNLS_METRIC_IP) {
                                acc[s][b] = fmaf(qv[P - 1 - s][px][v], kr[v], acc[s][b]);
                            } else {
                                const float d = qv[P - 1 - s][px][v] - kr[v];
                                acc[s][b] = fmaf(d, d, acc[s][b]);
                            }
                        }
                    }
                }
            }

            // ---- slot row r-(P-1) complete: reduce-scatter over the G lanes, then stream
            if (r >= P - 1)
                sel.template finish_row<METRIC>(acc[0], lane, gl, gq, on, row_ok, r - (P - 1), slot_base,
                                                grid_row, thr_src, thr_idx);
            // rotate: acc[s] tracks slot row r-(P-1)+s
#pragma unroll
            for (int s = 0; s + 1 < P; ++s)
#pragma unroll
                for (int b = 0; b < W; ++b) acc[s][b] = acc[s + 1][b];
#pragma unroll
            for (int b = 0; b < W; ++b) acc[P - 1][b] = 0.f;
        }
    }

    if (a.grid) return;  // selection happens in the top_l pass over the grid
    sel.emit(a, s_keys[qslot], row, row_ok, gl, qt, qy, qx);
}

template <int P, int W, int VEC, int G, int MINB>
int launch_one(const TiledSearch& s, cudaStream_t st) {
    using C = StreamCfg<P, W, VEC, G>;
    const unsigned blocks = unsigned((s.d.rows + C::QPB - 1) / C::QPB);
    if (s.metric == SNLS_METRIC_IP)
        search_stream_kernel<P, W, VEC, G, 16, SNLS_METRIC_IP, MINB><<<blocks, 128, 0, st>>>(s);
    else
        search_stream_kernel<P, W, VEC, G, 16, SNLS_METRIC_L2, MINB><<<blocks, 128, 0, st>>>(s);
    return 1;
}

// Channel split per (ps, F): VEC channels per lane, G = F / VEC lanes per query.  Large
// patches take VEC = 2 so the ps^2 query patch fits the register file next to the ps x ws
// accumulators.
template <int P, int W>
int launch_by_f(const TiledSearch& s, cudaStream_t st) {
    if constexpr (P >= 5) {
        switch (s.d.f) {
            case 64: return launch_one<P, W, 2, 32, 2>(s, st);
            default: return 0;
        }
    } else {
        switch (s.d.f) {
            case 32: return launch_one<P, W, 4, 8, 3>(s, st);
            case 64: return launch_one<P, W, 4, 16, 3>(s, st);
            default: return 0;
        }
    }
}

template <int P, int VEC, int G>
int launch_replay_one(const TiledSearch& s, cudaStream_t st) {
    using C = StreamCfg<P, P, VEC, G>;
    const unsigned blocks = unsigned((s.d.rows + C::QPB - 1) / C::QPB);
    if (s.metric == SNLS_METRIC_IP)
        search_stream_kernel<P, P, VEC, G, 16, SNLS_METRIC_IP, 1, true><<<blocks, 128, 0, st>>>(s);
    else
        search_stream_kernel<P, P, VEC, G, 16, SNLS_METRIC_L2, 1, true><<<blocks, 128, 0, st>>>(s);
    return 1;
}

__global__ void centre_slot_kernel(const float* __restrict__ grid, int64_t n, int slots, int centre,
                                   float* __restrict__ out) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < n) out[e] = grid[size_t(e) * slots + centre];
}

}  // namespace

// replay through the streaming plan: s.tape = centres, s.grid = scratch of rows * ps^2 floats,
// `out` = rows; 0 when the plan is not instantiated for this shape
int launch_replay_stream(const TiledSearch& s, float* out, cudaStream_t st) {
    if (s.topl > 16) return 0;
    const bool inst = (s.ps == 7 && s.ws == 9) || (s.ps == 3 && (s.ws == 11 || s.ws == 9));
    if (!inst) return 0;
    int n = 0;
    if (s.ps == 7) n = s.d.f == 64 ? launch_replay_one<7, 2, 32>(s, st) : 0;
    else if (s.d.f == 32) n = launch_replay_one<3, 4, 8>(s, st);
    else if (s.d.f == 64) n = launch_replay_one<3, 4, 16>(s, st);
    if (!n) return 0;
    const int P = s.ps;
    centre_slot_kernel<<<unsigned((s.d.rows + 255) / 256), 256, 0, st>>>(s.grid, s.d.rows, P * P,
                                                                         (P / 2) * P + P / 2, out);
    return 2;
}

int launch_search_stream(const TiledSearch& s, cudaStream_t st) {
    if (s.topl > 16) return 0;
    if (s.ps == 7 && s.ws == 9) return launch_by_f<7, 9>(s, st);   // c2 / c3
    if (s.ps == 3 && s.ws == 11) return launch_by_f<3, 11>(s, st); // c4
    if (s.ps == 3 && s.ws == 9) return launch_by_f<3, 9>(s, st);   // c5
    return 0;
}

}  // namespace snls_gpu
