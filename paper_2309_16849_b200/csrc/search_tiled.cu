// Tiled Shifted-NLS forward for stride1 == 1 (every BASELINE config): fused search +
// streaming top-L (+ optional softmax epilogue), sm_100a, FP32 FMA pipe.
//
// With stride1 == 1 every slot of one (query, frame) pair samples K at the SAME fractional
// offset (fy, fx): the pair needs the (ws+ps-1)^2 key region interpolated once, not once
// per (slot, patch pixel) as patch_similarity does (search.cpp:124-151).  Mapping:
//  * G = F / VEC lanes per query; lane gl owns channels [gl*VEC, gl*VEC+VEC) (float4).
//    A warp holds 32/G queries, consecutive rows (neighbouring pixels -> their key regions
//    overlap and hit in L1).
//  * Per frame the lane walks the key region row by row: it interpolates one region row
//    (ws+ps-1 pixels) into registers from two raw K rows (coalesced 16 B per lane, 128 B per
//    8-lane group), then updates the ps active slot rows: acc[s][b] += m(Q[py][px], Krow[b+px])
//    for the ps x ws slots that read this region row.  Slot row a completes after region
//    row a+ps-1 (rotating ps x ws accumulators: registers only, no shared-memory tile).
//  * A completed slot row is reduce-scattered across the G channel lanes (butterfly; the
//    addition tree is identical for every slot, so duplicate candidates tie exactly) and
//    each lane streams its ws/G slots into a register top-L list (strict '>' insertion in
//    ascending slot order == the reference's topl_insert, search.cpp:187-197).
//  * Epilogue: G-lane merge keyed on (value desc, slot asc), emit_row (search.cpp:207-234),
//    chains, and softmax_rows (aggregate.cpp:16-37) when weights are requested.
// The full ws^2 (2wt+1) score tensor is never materialised, in HBM or shared memory.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace snls_gpu {

namespace {

template <int P, int W, int VEC, int G, int KMAX>
struct TiledCfg {
    static constexpr int HP = P / 2, HW = W / 2, R = W + P - 1;
    static constexpr int QPW = 32 / G;                 // queries per warp
    static constexpr int NPL = (W + G - 1) / G;        // slots per lane after the scatter
    static constexpr int WPAD = NPL * G;
    static constexpr int WARPS = 4;
    static constexpr int QPB = QPW * WARPS;            // queries per block
};

template <int VEC>
struct Vec;
template <>
struct Vec<4> {
    using T = float4;
    static __device__ __forceinline__ float4 ld(const float* p) {
        return __ldg(reinterpret_cast<const float4*>(p));
    }
    static __device__ __forceinline__ float get(const float4& v, int i) {
        return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
    }
};

__device__ __forceinline__ float4 lerp4(const float4& a, const float4& b, const float4& c,
                                        const float4& d, float w00, float w01, float w10,
                                        float w11) {
    float4 r;
    r.x = fmaf(w11, d.x, fmaf(w10, c.x, fmaf(w01, b.x, w00 * a.x)));
    r.y = fmaf(w11, d.y, fmaf(w10, c.y, fmaf(w01, b.y, w00 * a.y)));
    r.z = fmaf(w11, d.z, fmaf(w10, c.z, fmaf(w01, b.z, w00 * a.z)));
    r.w = fmaf(w11, d.w, fmaf(w10, c.w, fmaf(w01, b.w, w00 * a.w)));
    return r;
}

template <int METRIC>
__device__ __forceinline__ float accum4(float acc, const float4& q, const float4& k) {
    if (METRIC == SNLS_METRIC_IP) {
        acc = fmaf(q.x, k.x, acc);
        acc = fmaf(q.y, k.y, acc);
        acc = fmaf(q.z, k.z, acc);
        acc = fmaf(q.w, k.w, acc);
    } else {  // negated squared L2 accumulated as +sum(d^2); sign applied at emission
        float d;
        d = q.x - k.x; acc = fmaf(d, d, acc);
        d = q.y - k.y; acc = fmaf(d, d, acc);
        d = q.z - k.z; acc = fmaf(d, d, acc);
        d = q.w - k.w; acc = fmaf(d, d, acc);
    }
    return acc;
}

// Group-wide top-L list, rank-sharded over the G lanes of a query: lane gl holds ranks
// [gl*M, gl*M+M) of one list sorted descending (M = KMAX/G).  Candidates reach it in
// ascending slot order and are inserted with strict '>' -- the reference's topl_insert
// (search.cpp:187-197) -- so equal values never displace an earlier slot.  The list's last
// rank is the exact group threshold, so almost every candidate is rejected by one compare.
template <int G, int M>
__device__ __forceinline__ void group_insert(float (&ev)[M], uint32_t (&es)[M], float v,
                                             uint32_t s, int gl) {
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

template <int W, int G>
__device__ __forceinline__ void write_off_frame(float* grid, int64_t row, int fp, int nfr, int gl) {
    float* g = grid + size_t(row) * nfr * W * W + size_t(fp) * W * W;
    for (int s = gl; s < W * W; s += G) g[s] = -INFINITY;
}

template <int P, int W, int VEC, int G, int KMAX, int METRIC, int MINB>
__global__ void __launch_bounds__(128, MINB) search_tiled_kernel(TiledSearch a) {
    using C = TiledCfg<P, W, VEC, G, KMAX>;
    using V = Vec<VEC>;
    constexpr int HP = C::HP, HW = C::HW, R = C::R;
    __shared__ uint64_t s_keys[C::QPB][KMAX];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane / G, gl = lane % G;
    const int qslot = warp * C::QPW + gq;
    const int64_t row_raw = int64_t(blockIdx.x) * C::QPB + qslot;
    const bool row_ok = row_raw < a.d.rows;
    const int64_t row = row_ok ? row_raw : a.d.rows - 1;
    int qt, qy, qx;
    row_coords(a.d, row, qt, qy, qx);
    const int H = a.d.h, Wd = a.d.w, F = a.d.f;
    const size_t frame_elems = size_t(H) * Wd * F;
    const int c0 = gl * VEC;
    const int nfr = 2 * a.wt + 1;

    // query patch addressing (reflected, integer pixels; search.cpp:129-132)
    const float* qbase = a.q + size_t(qt) * frame_elems + c0;
    int qrow[P], qcol[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        qrow[p] = reflect_near(qy + p - HP, H) * Wd * F;
        qcol[p] = reflect_near(qx + p - HP, Wd) * F;
    }

    constexpr int M = KMAX / G;  // ranks per lane
    float ev[M];
    uint32_t es[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
        ev[j] = -INFINITY;
        es[j] = 0xffffffffu;
    }
    const int glast = (lane / G) * G + (G - 1);  // lane holding the group's last rank

    for (int fp = 0; fp < nfr; ++fp) {
        const int dt = scan_dt(fp), kt = qt + dt;
        const bool on = row_ok && kt >= 0 && kt < a.d.t;
        if (!__any_sync(0xffffffffu, on)) {  // warp-uniform skip (search.cpp:300)
            if (a.grid && row_ok) write_off_frame<W, G>(a.grid, row, fp, nfr, gl);
            continue;
        }
        double sdy = 0.0, sdx = 0.0;
        if (on) shift_to(a.ff, a.bf, H, Wd, qt, qy, qx, dt, sdy, sdx, nullptr);
        const double cy = double(qy) + sdy, cx = double(qx) + sdx;
        const double fby = floor(cy), fbx = floor(cx);
        const float fy = float(cy - fby), fx = float(cx - fbx);
        const float w00 = (1.f - fy) * (1.f - fx), w01 = (1.f - fy) * fx;
        const float w10 = fy * (1.f - fx), w11 = fy * fx;
        const int by = int(fby) - HW - HP, bx = int(fbx) - HW - HP;
        // float4-granular addressing: per region row one 64-bit row base, per column a
        // 32-bit float4 index (one IMAD.WIDE per load instead of 64-bit pointer math)
        const float4* kbase = reinterpret_cast<const float4*>(a.k + size_t(on ? kt : qt) * frame_elems) + gl;
        const unsigned row4 = unsigned(Wd) * G;  // float4 per image row
        unsigned xo[R + 1];
#pragma unroll
        for (int j = 0; j <= R; ++j) xo[j] = unsigned(reflect_near(bx + j, Wd)) * G;
        const bool interior = __all_sync(0xffffffffu, bx >= 0 && bx + R < Wd);
        const unsigned xb = unsigned(bx) * G;

        float acc[P][W];
#pragma unroll
        for (int s = 0; s < P; ++s)
#pragma unroll
            for (int b = 0; b < W; ++b) acc[s][b] = 0.f;

        const uint32_t slot_base = uint32_t(fp) * W * W;
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
            // ---- interpolate region row r (bilinear, 4 reflected taps; tensor.cpp:31-48)
            const unsigned r0 = unsigned(reflect_near(by + r, H)) * row4;
            const unsigned r1 = unsigned(reflect_near(by + r + 1, H)) * row4;
            float4 kr[R];
            if (interior) {
                // no column reflection anywhere in the warp: one 64-bit base per raw row and
                // compile-time offsets (LDG [R + imm]) for the ws+ps columns
                const float4* p0 = kbase + (r0 + xb);
                const float4* p1 = kbase + (r1 + xb);
                float4 a0 = __ldg(p0), a1 = __ldg(p1);
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const float4 b0 = __ldg(p0 + (j + 1) * G), b1 = __ldg(p1 + (j + 1) * G);
                    kr[j] = lerp4(a0, b0, a1, b1, w00, w01, w10, w11);
                    a0 = b0;
                    a1 = b1;
                }
            } else {
                float4 a0 = __ldg(kbase + (r0 + xo[0])), a1 = __ldg(kbase + (r1 + xo[0]));
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const float4 b0 = __ldg(kbase + (r0 + xo[j + 1]));
                    const float4 b1 = __ldg(kbase + (r1 + xo[j + 1]));
                    kr[j] = lerp4(a0, b0, a1, b1, w00, w01, w10, w11);
                    a0 = b0;
                    a1 = b1;
                }
            }
            // ---- update the slot rows that read region row r: a = r - (P-1) + s, py = P-1-s
#pragma unroll
            for (int s = 0; s < P; ++s) {
                const int arow = r - (P - 1) + s;
                if (arow < 0 || arow >= W) continue;  // uniform across the warp
                const float* qr = qbase + qrow[P - 1 - s];
#pragma unroll
                for (int px = 0; px < P; ++px) {
                    const float4 qv = V::ld(qr + qcol[px]);
#pragma unroll
                    for (int b = 0; b < W; ++b) acc[s][b] = accum4<METRIC>(acc[s][b], qv, kr[b + px]);
                }
            }
            // ---- slot row r-(P-1) is complete: reduce-scatter over the G lanes, stream
            if (r >= P - 1) {
                float v[C::WPAD];
#pragma unroll
                for (int b = 0; b < C::WPAD; ++b) v[b] = b < W ? acc[0][b] : 0.f;
#pragma unroll
                for (int m = G / 2, n = C::WPAD; m >= 1; m >>= 1, n >>= 1) {
                    const bool hi = (gl & m) != 0;
#pragma unroll
                    for (int i = 0; i < n / 2; ++i) {
                        const float keep = hi ? v[i + n / 2] : v[i];
                        const float send = hi ? v[i] : v[i + n / 2];
                        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                    }
                }
                const int arow = r - (P - 1);
                if (a.grid) {  // kFullGrid: materialise the scores (-inf off-clip), no selection
#pragma unroll
                    for (int i = 0; i < C::NPL; ++i) {
                        const int b = gl * C::NPL + i;
                        const float val = METRIC == SNLS_METRIC_IP ? v[i] : -v[i];
                        if (row_ok && b < W)
                            a.grid[size_t(row) * nfr * W * W + slot_base + arow * W + b] = on ? val : -INFINITY;
                    }
                    goto rotate;
                }
                // exact group threshold = current last rank; most candidates stop here
                const float thr = __shfl_sync(0xffffffffu, ev[M - 1], glast);
                uint32_t pend = 0;
#pragma unroll
                for (int i = 0; i < C::NPL; ++i) {
                    const int b = gl * C::NPL + i;
                    v[i] = METRIC == SNLS_METRIC_IP ? v[i] : -v[i];
                    if (on && b < W && v[i] > thr) pend |= 1u << i;
                }
                // insert the survivors one at a time, lanes then slots ascending (= slot order)
                while (__any_sync(0xffffffffu, pend != 0)) {
                    const unsigned want = __ballot_sync(0xffffffffu, pend != 0);
                    const unsigned gmask = (want >> (gq * G)) & ((G == 32) ? 0xffffffffu : ((1u << G) - 1u));
                    const int src = gmask ? gq * G + (__ffs(gmask) - 1) : lane;
                    const int isrc = pend ? (__ffs(pend) - 1) : 0;
                    float cv = -INFINITY;
#pragma unroll
                    for (int i = 0; i < C::NPL; ++i) cv = (i == isrc) ? v[i] : cv;
                    const uint32_t cs = slot_base + uint32_t(arow * W + gl * C::NPL + isrc);
                    float bv = __shfl_sync(0xffffffffu, cv, src);
                    const uint32_t bs = __shfl_sync(0xffffffffu, cs, src);
                    if (!gmask) bv = -INFINITY;  // no-op insert keeps the shuffles warp-uniform
                    group_insert<G, M>(ev, es, bv, bs, gl);
                    if (lane == src && gmask) pend &= pend - 1;
                }
            }
        rotate:
            // rotate: acc[s] tracks slot row r-(P-1)+s, so every region row shifts by one
#pragma unroll
            for (int s = 0; s + 1 < P; ++s)
#pragma unroll
                for (int b = 0; b < W; ++b) acc[s][b] = acc[s + 1][b];
#pragma unroll
            for (int b = 0; b < W; ++b) acc[P - 1][b] = 0.f;
        }
    }

    if (a.grid) return;  // selection happens in the top_l pass over the grid

    // ---- the group list is already the merged top-KMAX: lane gl owns ranks gl*M .. gl*M+M-1
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const int li = gl * M + j;
        if (li < a.topl) s_keys[qslot][li] = eligible(ev[j]) ? pack_key(ev[j], es[j]) : 0ull;
    }
    __syncwarp();

    // ---- emit_row (search.cpp:207-234) + softmax epilogue ---------------------------------
    float zmax = -INFINITY;
    for (int li = gl; row_ok && li < a.topl; li += G) {
        const uint64_t key = s_keys[qslot][li];
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
    if (a.weights) {
        // group reductions (lanes of one query are an aligned block of G lanes)
#pragma unroll
        for (int m = G / 2; m >= 1; m >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, m));
        float sum = 0.f;
        for (int li = gl; row_ok && li < a.topl; li += G) {
            const float z = a.beta * key_value(s_keys[qslot][li]);
            if (!isfinite(z)) latch(a.err, kErrSoftmax);
            sum += __expf(z - zmax);
        }
#pragma unroll
        for (int m = G / 2; m >= 1; m >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, m);
        for (int li = gl; row_ok && li < a.topl; li += G) {
            const size_t e = size_t(row) * a.topl + li;
            a.weights[e] = __expf(a.beta * key_value(s_keys[qslot][li]) - zmax) / sum;
        }
    }
}

// Occupancy variant: MINB resident CTAs per SM (3 -> <=168 regs, 4 -> <=128 regs).
// $SNLS_TILED_MINB selects it at run time (experiments); default 3.
inline int tiled_minb() {
    static const int v = [] {
        const char* e = std::getenv("SNLS_TILED_MINB");
        return (e && std::atoi(e) == 4) ? 4 : ((e && std::atoi(e) == 2) ? 2 : 3);
    }();
    return v;
}

template <int P, int W, int VEC, int G, int KMAX, int MINB>
int launch_cfg_b(const TiledSearch& s, cudaStream_t st) {
    using C = TiledCfg<P, W, VEC, G, KMAX>;
    const unsigned blocks = unsigned((s.d.rows + C::QPB - 1) / C::QPB);
    if (s.metric == SNLS_METRIC_IP)
        search_tiled_kernel<P, W, VEC, G, KMAX, SNLS_METRIC_IP, MINB><<<blocks, 32 * C::WARPS, 0, st>>>(s);
    else
        search_tiled_kernel<P, W, VEC, G, KMAX, SNLS_METRIC_L2, MINB><<<blocks, 32 * C::WARPS, 0, st>>>(s);
    return 1;
}

template <int P, int W, int VEC, int G, int KMAX>
int launch_cfg(const TiledSearch& s, cudaStream_t st) {
    if constexpr (P == 3 && G == 8)
        if (tiled_minb() == 4) return launch_cfg_b<P, W, VEC, G, KMAX, 4>(s, st);
    if constexpr (P == 7)  // the ps = 7 plan spills under the 168-register cap
        return launch_cfg_b<P, W, VEC, G, KMAX, 2>(s, st);
    return launch_cfg_b<P, W, VEC, G, KMAX, 3>(s, st);
}

template <int P, int W, int KMAX>
int launch_by_f(const TiledSearch& s, cudaStream_t st) {
    switch (s.d.f) {
        case 4: return launch_cfg<P, W, 4, 1, KMAX>(s, st);
        case 8: return launch_cfg<P, W, 4, 2, KMAX>(s, st);
        case 16: return launch_cfg<P, W, 4, 4, KMAX>(s, st);
        case 32: return launch_cfg<P, W, 4, 8, KMAX>(s, st);
        case 64: return launch_cfg<P, W, 4, 16, KMAX>(s, st);
        default: return 0;
    }
}

template <int P, int W>
int launch_by_k(const TiledSearch& s, cudaStream_t st) {
    if (s.topl <= 16) return launch_by_f<P, W, 16>(s, st);
    return 0;
}

}  // namespace

// Instantiated (ps, ws) pairs; anything else takes the generic path.
int launch_search_tiled(const TiledSearch& s, cudaStream_t st, int* used) {
    // auto: the streaming plan for large patches (the tiled plan spills at ps = 7), the
    // region-row tiled plan otherwise (faster at ps = 3 on B200, profiles/)
    if (s.kernel == 2 || (s.kernel == 0 && s.ps >= 5)) {
        if (int n = launch_search_stream(s, st)) {
            if (used) *used = 2;
            return n;
        }
    }
    if (used) *used = 1;
    if (s.ps == 3 && s.ws == 11) return launch_by_k<3, 11>(s, st);  // c4
    if (s.ps == 3 && s.ws == 9) return launch_by_k<3, 9>(s, st);    // c5
    if (s.ps == 7 && s.ws == 9) return launch_by_k<7, 9>(s, st);    // c2 / c3
    if (s.ps == 1 && s.ws == 9) return launch_by_k<1, 9>(s, st);
    if (s.ps == 3 && s.ws == 5) return launch_by_k<3, 5>(s, st);
    if (s.ps == 1 && s.ws == 5) return launch_by_k<1, 5>(s, st);
    return 0;
}

}  // namespace snls_gpu
