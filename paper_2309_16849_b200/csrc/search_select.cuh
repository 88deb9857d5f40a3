// Selection side shared by the stride1 == 1 search plans (search_tiled.cu, search_stream.cu):
// finishing one slot row (reduce-scatter over the channel lanes of a query, then either the
// full-grid write or the streaming top-L insertion) and the emit_row + softmax epilogue.
//
// Tie rules (search.cpp:187-197): candidates reach the list in ascending slot order and are
// inserted with strict '>', so an equal value never displaces an earlier slot.  The list is
// rank-sharded over the G lanes of a query (lane gl holds ranks [gl*M, gl*M+M)).  A
// candidate not above the current rank topl-1 can never be selected: one compare rejects it.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace snls_gpu {

// SNLS_NOSEL=1 (measurement builds only, wrong results): skip every top-L insertion to time
// the selection's share (c4: 4.11 -> 3.66 ms, c5: 117.3 -> 109.6 ms; profiles/r01_plans.txt)
#ifndef SNLS_NOSEL
#define SNLS_NOSEL 0
#endif
constexpr int pow2ceil(int n) { return n <= 1 ? 1 : 2 * pow2ceil((n + 1) / 2); }
constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

template <int W, int G, int KMAX>
struct SelectCfg {
    static constexpr int M = KMAX / G > 0 ? KMAX / G : 1;  // list ranks per lane
    // reduce-scatter geometry: W slots padded to NPAD; if NPAD >= G every lane ends with
    // NPL consecutive slots, else 2^SH neighbouring lanes share one slot (all-reduced)
    static constexpr int NPAD = pow2ceil(W);
    static constexpr int NPL = NPAD >= G ? NPAD / G : 1;
    static constexpr int SH = NPAD >= G ? 0 : ilog2(G / NPAD);
};

template <int G, int M>
__device__ __forceinline__ void list_insert(float (&ev)[M], uint32_t (&es)[M], float v, uint32_t s,
                                            int gl) {
    // the entry just above mine is the previous lane's last one (+inf above rank 0)
    float pv = __shfl_up_sync(0xffffffffu, ev[M - 1], 1, G);
    uint32_t ps = __shfl_up_sync(0xffffffffu, es[M - 1], 1, G);
    if (gl == 0) pv = INFINITY;
    float nv[M];
    uint32_t ns[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const float above = j == 0 ? pv : ev[j - 1];
        const uint32_t above_s = j == 0 ? ps : es[j - 1];
        const bool ga = v > above, gc = v > ev[j];
        nv[j] = ga ? above : (gc ? v : ev[j]);
        ns[j] = ga ? above_s : (gc ? s : es[j]);
    }
#pragma unroll
    for (int j = 0; j < M; ++j) {
        ev[j] = nv[j];
        es[j] = ns[j];
    }
}

// Per-query selection state of one lane.
template <int W, int G, int KMAX>
struct TopL {
    using S = SelectCfg<W, G, KMAX>;
    float ev[S::M];
    uint32_t es[S::M];

    // lane of the warp holding rank topl-1 of group gq, and its entry index there
    static __device__ __forceinline__ int thr_lane(int gq, int topl) { return gq * G + (topl - 1) / S::M; }
    static __device__ __forceinline__ int thr_entry(int topl) { return (topl - 1) % S::M; }

    __device__ __forceinline__ void init() {
#pragma unroll
        for (int j = 0; j < S::M; ++j) {
            ev[j] = -INFINITY;
            es[j] = 0xffffffffu;
        }
    }

    // Slot row `arow` of frame position `fp` is complete in every lane's acc_row (partial
    // sums over the lane's channels): reduce-scatter over the G lanes of the query (the
    // addition tree is the same for every slot, so duplicate candidates tie exactly) and
    // stream it into the list -- or, in full-grid mode, write it to the grid row.
    template <int METRIC>
    __device__ __forceinline__ void finish_row(const float (&acc_row)[W], int lane, int gl, int gq,
                                               bool on, bool row_ok, int arow, uint32_t slot_base,
                                               float* grid_row, int thr_src, int thr_idx) {
        float v[S::NPAD];
#pragma unroll
        for (int b = 0; b < S::NPAD; ++b) v[b] = b < W ? acc_row[b] : 0.f;
        // scatter levels: the lane bit for m picks the upper half of the values
#pragma unroll
        for (int lev = 0; lev < ilog2(G); ++lev) {
            const int m = G >> (lev + 1), n = S::NPAD >> lev;  // n values before this level
            if (n > 1) {
                const bool hi = (gl & m) != 0;
#pragma unroll
                for (int i = 0; i < n / 2; ++i) {
                    const float keep = hi ? v[i + n / 2] : v[i];
                    const float send = hi ? v[i] : v[i + n / 2];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                }
            } else {  // more lanes than slots: all-reduce the remaining levels
                v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
            }
        }
        // lane gl holds slots (gl >> SH) * NPL + i, i < NPL; owners have the low SH bits clear
        const int sb = (gl >> S::SH) * S::NPL;
        const bool owner = (gl & ((1 << S::SH) - 1)) == 0;
        if (grid_row) {  // kFullGrid: materialise the scores (-inf off-clip), no selection
#pragma unroll
            for (int i = 0; i < S::NPL; ++i) {
                const int b = sb + i;
                const float val = METRIC == SNLS_METRIC_IP ? v[i] : -v[i];
                if (row_ok && owner && b < W) grid_row[slot_base + arow * W + b] = on ? val : -INFINITY;
            }
            return;
        }
        // rank topl-1 lives in lane thr_src of the warp (group gq), entry thr_idx
        float thr = ev[S::M - 1];
        if constexpr (S::M > 1) {
#pragma unroll
            for (int j = 0; j < S::M - 1; ++j) thr = j == thr_idx ? ev[j] : thr;
        }
        thr = __shfl_sync(0xffffffffu, thr, thr_src);
        uint32_t pend = 0;
#pragma unroll
        for (int i = 0; i < S::NPL; ++i) {
            const int b = sb + i;
            v[i] = METRIC == SNLS_METRIC_IP ? v[i] : -v[i];  // l2 accumulates +sum(d^2)
            if (SNLS_NOSEL == 0 && on && owner && b < W && v[i] > thr) pend |= 1u << i;
        }
        // survivors one at a time, lanes then slots ascending (= slot order)
        unsigned want = __ballot_sync(0xffffffffu, pend != 0);
        while (want) {
            const unsigned gmask = (want >> (gq * G)) & ((G == 32) ? 0xffffffffu : ((1u << G) - 1u));
            const int src = gmask ? gq * G + (__ffs(gmask) - 1) : lane;
            const int isrc = pend ? (__ffs(pend) - 1) : 0;
            float cv = -INFINITY;
#pragma unroll
            for (int i = 0; i < S::NPL; ++i) cv = (i == isrc) ? v[i] : cv;
            const uint32_t cs = slot_base + uint32_t(arow * W + sb + isrc);
            float bv = __shfl_sync(0xffffffffu, cv, src);
            const uint32_t bs = __shfl_sync(0xffffffffu, cs, src);
            if (!gmask) bv = -INFINITY;  // no-op insert keeps the shuffles warp-uniform
            list_insert<G, S::M>(ev, es, bv, bs, gl);
            if (lane == src && gmask) pend &= pend - 1;
            want = __ballot_sync(0xffffffffu, pend != 0);
        }
    }

    // emit_row (search.cpp:207-234) + the fused softmax_rows epilogue (aggregate.cpp:16-37).
    // keys: this query's 16-entry shared-memory row.
    __device__ __forceinline__ void emit(const TiledSearch& a, uint64_t* keys, int64_t row, bool row_ok,
                                         int gl, int qt, int qy, int qx) {
        constexpr int HW = W / 2;
        const int H = a.d.h, Wd = a.d.w;
#pragma unroll
        for (int j = 0; j < S::M; ++j) {
            const int li = gl * S::M + j;
            if (li < a.topl) keys[li] = eligible(ev[j]) ? pack_key(ev[j], es[j]) : 0ull;
        }
        __syncwarp();
        float zmax = -INFINITY;
        for (int li = gl; row_ok && li < a.topl; li += G) {
            const uint64_t key = keys[li];
            const size_t e = size_t(row) * a.topl + li;
            float v = -INFINITY, o1 = 0.f, o2 = 0.f;
            int dt = 0;
            if (key != 0ull) {
                const uint32_t slot = key_slot(key);
                v = key_value(key);
                const int fp = int(slot) / (W * W), rem = int(slot) % (W * W);
                dt = scan_dt(fp);
                double sdy, sdx;
                shift_to(a.ff, a.bf, H, Wd, qt, qy, qx, dt, sdy, sdx, nullptr);
                const double ky = (double(qy) + sdy) + double(rem / W - HW);
                const double kx = (double(qx) + sdx) + double(rem % W - HW);
                o1 = float(ky - double(qy));
                o2 = float(kx - double(qx));
            }
            a.sims[e] = v;
            a.offsets[e * 3 + 0] = float(dt);
            a.offsets[e * 3 + 1] = o1;
            a.offsets[e * 3 + 2] = o2;
            if (a.chains && a.wt > 1) {
                const int cs = a.wt - 1;
                float* lk = a.chains + e * size_t(cs) * 6;
                for (int j = 0; j < cs * 6; ++j) lk[j] = 0.f;
                if (dt > 1 || dt < -1) {
                    double sdy, sdx;
                    shift_to(a.ff, a.bf, H, Wd, qt, qy, qx, dt, sdy, sdx, lk);
                }
            }
            zmax = fmaxf(zmax, a.beta * v);
        }
        if (a.weights) {  // group reductions: a query's lanes are an aligned block of G
#pragma unroll
            for (int m = G / 2; m >= 1; m >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, m));
            float sum = 0.f;
            for (int li = gl; row_ok && li < a.topl; li += G) {
                const float z = a.beta * key_value(keys[li]);
                if (!isfinite(z)) latch(a.err, kErrSoftmax);
                sum += __expf(z - zmax);
            }
#pragma unroll
            for (int m = G / 2; m >= 1; m >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, m);
            for (int li = gl; row_ok && li < a.topl; li += G) {
                const size_t e = size_t(row) * a.topl + li;
                a.weights[e] = __expf(a.beta * key_value(keys[li]) - zmax) / sum;
            }
        }
    }
};

template <int W, int G>
__device__ __forceinline__ void write_off_frame(float* grid, int64_t row, int fp, int nfr, int gl) {
    float* g = grid + size_t(row) * nfr * W * W + size_t(fp) * W * W;
    for (int s = gl; s < W * W; s += G) g[s] = -INFINITY;
}

// VEC consecutive channels (16 B / 8 B / 4 B load).
template <int VEC>
__device__ __forceinline__ void ldv(const float* p, float (&o)[VEC]) {
    if constexpr (VEC == 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else if constexpr (VEC == 2) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(p));
        o[0] = v.x; o[1] = v.y;
    } else {
        o[0] = __ldg(p);
    }
}

}  // namespace snls_gpu
