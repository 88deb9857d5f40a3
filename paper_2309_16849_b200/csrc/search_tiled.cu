// Tiled Shifted-NLS forward for stride1 == 1 (every BASELINE config): fused search +
// streaming top-L (+ optional softmax epilogue), sm_100a, FP32 FMA pipe.
//
// With stride1 == 1 every slot of one (query, frame) pair samples K at the SAME fractional
// offset (fy, fx): the pair needs the (ws+ps-1)^2 key region interpolated once, not once
// per (slot, patch pixel) as patch_similarity does (search.cpp:124-151).  Mapping:
//  * G = F / VEC lanes per query; lane gl owns channels [gl*VEC, gl*VEC+VEC) (float4; float2
//    at ps = 7).  A warp holds 32/G queries, consecutive rows (neighbouring pixels -> their
//    key regions overlap and hit in L1).  The arithmetic runs on packed fp32x2 (FFMA2/FADD2,
//    packed.cuh); the query patch and the boundary warps' reflected column offsets are parked
//    in shared memory at the start (own lane only, no barrier) so the registers go to the
//    accumulators and the interpolated row.
//  * Per frame the lane walks the key region row by row: it interpolates one region row
//    (ws+ps-1 pixels) into registers from two raw K rows (coalesced 16 B per lane, 128 B per
//    8-lane group), then updates the ps active slot rows: acc[s][b] += m(Q[py][px], Krow[b+px])
//    for the ps x ws slots that read this region row.  Slot row a completes after region
//    row a+ps-1 (rotating ps x ws accumulators: registers only, no shared-memory tile of K).
//  * A completed slot row is reduce-scattered across the G channel lanes (butterfly; the
//    addition tree is identical for every slot, so duplicate candidates tie exactly) and
//    each lane streams its ws/G slots into a register top-L list (strict '>' insertion in
//    ascending slot order == the reference's topl_insert, search.cpp:187-197).
//  * Epilogue: G-lane merge keyed on (value desc, slot asc), emit_row (search.cpp:207-234),
//    chains, and softmax_rows (aggregate.cpp:16-37) when weights are requested.
// The full ws^2 (2wt+1) score tensor is never materialised, in HBM or shared memory.
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "search_select.cuh"
#include "packed.cuh"

#ifndef SNLS_XO16
#define SNLS_XO16 1
#endif
#ifndef SNLS_CARVEOUT
#define SNLS_CARVEOUT -2  // -2: from MINB and the kernel's shared memory; -1: driver default
#endif
#ifndef SNLS_KEYS_IN_Q
#define SNLS_KEYS_IN_Q 1
#endif
#ifndef SNLS_TILE2D_Q1
#define SNLS_TILE2D_Q1 1
#endif
#ifndef SNLS_TILE2D
#define SNLS_TILE2D 1
#endif

namespace snls_gpu {

namespace {

template <int P, int W, int VEC, int G>
struct TiledCfg {
    static constexpr int HP = P / 2, HW = W / 2, R = W + P - 1, F = G * VEC;
    static constexpr int QPW = 32 / G;                 // queries per warp
    static constexpr int WARPS = 4;
    static constexpr int QPB = QPW * WARPS;            // queries per block
};

// kr = bilinear blend of the four raw taps (tensor.cpp:31-48), VEC channels
template <int VEC>
__device__ __forceinline__ void lerpv(float (&r)[VEC], const float (&a)[VEC], const float (&b)[VEC],
                                      const float (&c)[VEC], const float (&d)[VEC], float w00,
                                      float w01, float w10, float w11) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) r[v] = fmaf(w11, d[v], fmaf(w10, c[v], fmaf(w01, b[v], w00 * a[v])));
}

// QREG: the query patch (P x P x VEC per lane) is loaded once into registers instead of
// being re-read from L1 on every region row (used where it fits: ps = 7 on float2 lanes).
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

// ---- packed fp32x2 (packed.cuh): FFMA2 / FADD2 / FMUL2 take half the FP issue slots, so the
// search loop's overhead instructions fill the rest.
// the blend of lerp4, same operation order per channel
__device__ __forceinline__ P4 lerp2(const P4& a, const P4& b, const P4& c, const P4& d, u64 w00,
                                    u64 w01, u64 w10, u64 w11) {
    return {fma2(w11, d.lo, fma2(w10, c.lo, fma2(w01, b.lo, mul2(w00, a.lo)))),
            fma2(w11, d.hi, fma2(w10, c.hi, fma2(w01, b.hi, mul2(w00, a.hi))))};
}

#ifndef SNLS_PACKED_F32X2
#define SNLS_PACKED_F32X2 1
#endif
constexpr bool kPacked = SNLS_PACKED_F32X2 != 0;
// ps = 7 on float2 lanes: the query patch parked in shared memory (each lane reads back only
// what it wrote: no barrier) and the search on packed pairs
#ifndef SNLS_QSM
#define SNLS_QSM 1
#endif
constexpr bool kQsm = SNLS_QSM != 0 && SNLS_PACKED_F32X2 != 0;
// float4 lanes (ps <= 5): the query patch in shared memory as well (LDS.128 at immediate
// offsets instead of 64-bit-addressed L1 loads)
#ifndef SNLS_QSM4
#define SNLS_QSM4 1
#endif
constexpr bool kQsm4 = SNLS_QSM4 != 0 && SNLS_PACKED_F32X2 != 0;
#ifndef SNLS_XO_SMEM
#define SNLS_XO_SMEM 1
#endif
constexpr bool kXoSmem = SNLS_XO_SMEM != 0;
// the slot row's partials in kBSplit chunks (fewer live registers: with them c4's 3 x 11
// accumulators fit 128 registers, MINB 4 / 16 warps per SM: 3.967 -> 3.923 ms)
// float4 packed path: a slot row's first contribution is assigned, not added to a zeroed
// accumulator (at 16 warps/SM: c4 3.920 -> 3.891 ms, c5 112.2 -> 111.8 ms)
#ifndef SNLS_ASSIGN1
#define SNLS_ASSIGN1 1
#endif
constexpr bool kAssign1 = SNLS_ASSIGN1 != 0;
#ifndef SNLS_BSPLIT
#define SNLS_BSPLIT 2
#endif
constexpr int kBSplit = SNLS_BSPLIT;
#ifndef SNLS_BSPLIT_SMALL_W
#define SNLS_BSPLIT_SMALL_W 9
#endif
constexpr int kBSplitSmallW = SNLS_BSPLIT_SMALL_W;
#ifndef SNLS_MINB4_WMAX
#define SNLS_MINB4_WMAX 11
#endif
#ifndef SNLS_QSM_MINB
#define SNLS_QSM_MINB 3
#endif

// FG: full-grid mode (materialise the scores; a separate instantiation so the fused kernel
// carries no grid pointer or branches)
// RP (replay_similarities, W = 1): every "row" is one selected entry (row / topl is its
// query), the single frame and window centre come from the entry's fp64 tape centre, and the
// full-grid write stores its one slot: the same per-slot arithmetic as the forward (the
// interpolation, the (py, px, pair) chains and the lane butterfly do not depend on the slot's
// place in the window), so the replayed value equals the forward's bit for bit.
// BAND: the temporally blocked raster (a separate instantiation: the remap's registers would
// otherwise cost the plain-raster kernel a spill)
template <int P, int W, int VEC, int G, int KMAX, int METRIC, int MINB, bool QREG, bool FG, bool RP = false,
          bool BAND = false>
__global__ void __launch_bounds__(128, MINB) search_tiled_kernel(TiledSearch a) {
    using C = TiledCfg<P, W, VEC, G>;
    constexpr int HP = C::HP, HW = C::HW, R = C::R, F = C::F;
    constexpr bool kPackedPath = VEC == 4 && !QREG && kPacked;
    constexpr bool kPairPath = VEC == 2 && !QREG && kQsm;  // Q in shared memory
    constexpr bool kQsmF4 = kPackedPath && kQsm4;
    // the epilogue's key rows live in the query's own (no longer needed) shared-memory patch
    // when there is one (it holds >= 16 keys): less shared memory per CTA, a larger L1
    // (float4 path only: on the ps 7 pair path it measured 0.7% slower, c2 0.3536 vs 0.3510 ms)
    constexpr bool kKeysInQ = SNLS_KEYS_IN_Q && kQsmF4 && size_t(P) * P * G * 16 >= 16 * sizeof(uint64_t);
    __shared__ uint64_t s_keys[kKeysInQ ? 1 : C::QPB][16];
    // kPairPath: [QPB][P*P][G] channel pairs; kQsmF4: [QPB][P*P][G] float4
    extern __shared__ __align__(16) unsigned char s_qdyn[];
    // 16-bit when SNLS_XO16 (the launcher requires W * F / VEC < 2^16)
    using XoT = std::conditional_t<kXoSmem && SNLS_XO16, uint16_t, unsigned>;
    __shared__ XoT s_xo[kXoSmem ? R + 1 : 1][128];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane / G, gl = lane % G;
    const int qslot = warp * C::QPW + gq;
    const int64_t row_raw = int64_t(blockIdx.x) * C::QPB + qslot;
    const bool row_ok = row_raw < a.d.rows;
    // temporally blocked raster, remapped per CTA (its QPB queries stay consecutive in one image
    // row when QPB divides nw): blockIdx-only arithmetic, kept in uniform registers
    const int64_t row0 = BAND ? band_row(a.d, int64_t(blockIdx.x) * C::QPB, a.band) : int64_t(blockIdx.x) * C::QPB;
#if SNLS_TILE2D
    // a CTA's queries as a WARPS x QPW tile of the query grid (warp = one query row of QPW
    // queries) instead of QPB consecutive queries of one image row: the union of their key
    // regions is smaller (c4 16 queries: 21 x 21 instead of 13 x 45 region pixels per frame),
    // so more of the raw-row loads hit L1 (c4 search 3.906 -> 3.862 ms; profiles/r01_plans.txt)
    int64_t row = row_ok ? row0 + qslot : a.d.rows - 1;
    if (C::QPW > 1 && !BAND && !RP && a.d.nh % C::WARPS == 0 && a.d.nw % C::QPW == 0) {
        const unsigned tx = unsigned(a.d.nw) / C::QPW, per = tx * (unsigned(a.d.nh) / C::WARPS);
        const unsigned tl = blockIdx.x / per, rem = blockIdx.x - tl * per;
        const unsigned ty0 = rem / tx, tx0 = rem - ty0 * tx;
        row = int64_t(tl) * a.d.nh * a.d.nw + int64_t((ty0 * C::WARPS + warp) * unsigned(a.d.nw) + tx0 * C::QPW + gq);
    }
#if SNLS_TILE2D_Q1
    // one query per warp (ps 7): the CTA's 4 queries as a 2 x 2 tile
    if (C::QPW == 1 && C::WARPS == 4 && !BAND && !RP && a.d.nh % 2 == 0 && a.d.nw % 2 == 0) {
        const unsigned tx = unsigned(a.d.nw) / 2, per = tx * (unsigned(a.d.nh) / 2);
        const unsigned tl = blockIdx.x / per, rem = blockIdx.x - tl * per;
        const unsigned ty0 = rem / tx, tx0 = rem - ty0 * tx;
        row = int64_t(tl) * a.d.nh * a.d.nw + int64_t((ty0 * 2 + (warp >> 1)) * unsigned(a.d.nw) + tx0 * 2 + (warp & 1));
    }
#endif
#else
    const int64_t row = row_ok ? row0 + qslot : a.d.rows - 1;
#endif
    int qt, qy, qx;
    row_coords(a.d, RP ? row / a.topl : row, qt, qy, qx);
    const int H = a.d.h, Wd = a.d.w;
    const size_t frame_elems = size_t(H) * Wd * F;
    const int c0 = gl * VEC;
    const int nfr = RP ? 1 : 2 * a.wt + 1;

    // query patch addressing (reflected, integer pixels; search.cpp:129-132)
    const float* qbase = a.q + size_t(qt) * frame_elems + c0;
    int qrow[P], qcol[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        qrow[p] = reflect_near(qy + p - HP, H) * Wd * F;
        qcol[p] = reflect_near(qx + p - HP, Wd) * F;
    }

    float qreg[QREG ? P : 1][QREG ? P : 1][VEC];
    if constexpr (QREG) {
#pragma unroll
        for (int py = 0; py < P; ++py)
#pragma unroll
            for (int px = 0; px < P; ++px) ldv<VEC>(qbase + qrow[py] + qcol[px], qreg[py][px]);
    }
    u64* sq = reinterpret_cast<u64*>(s_qdyn) + size_t(qslot) * P * P * G + gl;
    float4* sq4 = reinterpret_cast<float4*>(s_qdyn) + size_t(qslot) * P * P * G + gl;
    if constexpr (kQsmF4) {
#pragma unroll
        for (int py = 0; py < P; ++py)
#pragma unroll
            for (int px = 0; px < P; ++px)
                sq4[(py * P + px) * G] = __ldg(reinterpret_cast<const float4*>(qbase + qrow[py] + qcol[px]));
    }
    if constexpr (kPairPath) {
#pragma unroll
        for (int py = 0; py < P; ++py)
#pragma unroll
            for (int px = 0; px < P; ++px) {
                float v[2];
                ldv<2>(qbase + qrow[py] + qcol[px], v);
                sq[(py * P + px) * G] = pk2(v[0], v[1]);
            }
    }

    TopL<W, G, KMAX> sel;
    sel.init();
    const int thr_src = TopL<W, G, KMAX>::thr_lane(gq, a.topl), thr_idx = TopL<W, G, KMAX>::thr_entry(a.topl);
    float* grid_row = FG ? a.grid + size_t(row) * nfr * W * W : nullptr;

    for (int fp = 0; fp < nfr; ++fp) {
        const int dt = RP ? int(a.tape[size_t(row) * 3]) - qt : scan_dt(fp), kt = qt + dt;
        const bool on = row_ok && kt >= 0 && kt < a.d.t;
        if (!__any_sync(0xffffffffu, on)) {  // warp-uniform skip (search.cpp:300)
            if (FG && row_ok) write_off_frame<W, G>(a.grid, row, fp, nfr, gl);
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
        // (cvt saturates a huge shift; the int sums below may then wrap, which reflect_near maps
        // back into the frame like any other index, and the interior test cannot overflow)
        const int by = int(fby) - HW - HP, bx = int(fbx) - HW - HP;
        // VEC-granular addressing: per region row one 64-bit row base, per column a 32-bit
        // vector index (one IMAD.WIDE per load instead of 64-bit pointer math)
        const float* kframe = a.k + size_t(on ? kt : qt) * frame_elems + c0;
        const unsigned rowv = unsigned(Wd) * G;  // VEC-vectors per image row
        const bool interior = __all_sync(0xffffffffu, bx >= 0 && bx < Wd - R);
        const unsigned xb = unsigned(bx) * G;
        // reflected column offsets, precomputed (recomputing them at the boundary-warp loads
        // instead: c4 5.06 vs 4.45 ms) and parked in shared memory: only boundary warps read
        // them, and the R+1 registers go to the interior loop (c4 4.12 -> 4.00 ms, c5 116.9 ->
        // 112.7 ms, c2 0.370 -> 0.357 ms)
        XoT xo_r[kXoSmem ? 1 : R + 1];
        XoT* xo = kXoSmem ? &s_xo[0][threadIdx.x] : xo_r;
        constexpr int XS = kXoSmem ? 128 : 1;  // element stride
        if (kXoSmem) {
            if (!interior) {
#pragma unroll
                for (int j = 0; j <= R; ++j) xo[j * XS] = XoT(unsigned(reflect_near(bx + j, Wd)) * G);
            }
        } else {
#pragma unroll
            for (int j = 0; j <= R; ++j) xo[j] = XoT(unsigned(reflect_near(bx + j, Wd)) * G);
        }
        auto ld = [&](unsigned vidx, float (&o)[VEC]) { ldv<VEC>(kframe + size_t(vidx) * VEC, o); };

        float acc[P][W];
#pragma unroll
        for (int s = 0; s < P; ++s)
#pragma unroll
            for (int b = 0; b < W; ++b) acc[s][b] = 0.f;

        const uint32_t slot_base = uint32_t(fp) * W * W;
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
            // ---- interpolate region row r (bilinear, 4 reflected taps; tensor.cpp:31-48)
            const unsigned r0 = unsigned(reflect_near(by + r, H)) * rowv;
            const unsigned r1 = unsigned(reflect_near(by + r + 1, H)) * rowv;
            if constexpr (kPackedPath) {
                // packed fp32x2: channel pairs (x, y), (z, w) of every float4.  Per slot and
                // region row the partial sum runs in the two halves of a pair t and is folded
                // into the slot accumulator as (t.x + t.y): the same addition tree for every
                // slot, so duplicate candidates still tie exactly.
                const float4* kb4 = reinterpret_cast<const float4*>(kframe);
                const u64 W00 = pk2(w00, w00), W01 = pk2(w01, w01), W10 = pk2(w10, w10), W11 = pk2(w11, w11);
                P4 kr[R];
                if (interior) {
                    const float4* p0 = kb4 + (r0 + xb);
                    const float4* p1 = kb4 + (r1 + xb);
                    P4 a0 = ldp4(p0), a1 = ldp4(p1);
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const P4 b0 = ldp4(p0 + (j + 1) * G), b1 = ldp4(p1 + (j + 1) * G);
                        kr[j] = lerp2(a0, b0, a1, b1, W00, W01, W10, W11);
                        a0 = b0;
                        a1 = b1;
                    }
                } else {
                    P4 a0 = ldp4(kb4 + (r0 + xo[0])), a1 = ldp4(kb4 + (r1 + xo[0]));
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const P4 b0 = ldp4(kb4 + (r0 + xo[(j + 1) * XS]));
                        const P4 b1 = ldp4(kb4 + (r1 + xo[(j + 1) * XS]));
                        kr[j] = lerp2(a0, b0, a1, b1, W00, W01, W10, W11);
                        a0 = b0;
                        a1 = b1;
                    }
                }
#pragma unroll
                for (int s = 0; s < P; ++s) {
                    const int arow = r - (P - 1) + s;
                    if (arow < 0 || arow >= W) continue;  // uniform across the warp
                    [[maybe_unused]] const float* qr = qbase + qrow[P - 1 - s];
                    P4 qv[P];
#pragma unroll
                    for (int px = 0; px < P; ++px) {
                        if constexpr (kQsmF4) {
                            const float4 v = sq4[((P - 1 - s) * P + px) * G];
                            qv[px] = {pk2(v.x, v.y), pk2(v.z, v.w)};
                        } else {
                            qv[px] = ldp4(reinterpret_cast<const float4*>(qr + qcol[px]));
                        }
                    }
                    // slot-inner: consecutive instructions update W independent partials (per
                    // slot the order is px ascending, pair lo then hi; slot-outer: c4 4.16 vs
                    // 4.12 ms, c5 119.7 vs 117.7 ms)
                    // (W <= 9, c5: one slot at a time -- 110.1 vs 111.7 ms; W = 11, c4: two
                    // chunks -- 3.888 vs 3.908 ms per slot)
                    constexpr int BC = W <= kBSplitSmallW ? 1 : (W + kBSplit - 1) / kBSplit;
#pragma unroll
                    for (int b0 = 0; b0 < W; b0 += BC) {
                        u64 t[BC];
#pragma unroll
                        for (int px = 0; px < P; ++px)
#pragma unroll
                            for (int h = 0; h < 2; ++h)
#pragma unroll
                                for (int bi = 0; bi < BC; ++bi) {
                                    const int b = b0 + bi;
                                    if (b >= W) continue;
                                    const u64 qh = h ? qv[px].hi : qv[px].lo;
                                    const u64 kh = h ? kr[b + px].hi : kr[b + px].lo;
                                    if (METRIC == SNLS_METRIC_IP) {
                                        t[bi] = (px == 0 && h == 0) ? mul2(qh, kh) : fma2(qh, kh, t[bi]);
                                    } else {  // +sum (q - k)^2
                                        const u64 d = sub2(qh, kh);
                                        t[bi] = (px == 0 && h == 0) ? mul2(d, d) : fma2(d, d, t[bi]);
                                    }
                                }
#pragma unroll
                        for (int bi = 0; bi < BC; ++bi) {
                            if (b0 + bi >= W) continue;
                            const float2 tf = upk2(t[bi]);
                            if (kAssign1 && s == P - 1)  // first region row of this slot row
                                acc[s][b0 + bi] = tf.x + tf.y;
                            else
                                acc[s][b0 + bi] += tf.x + tf.y;
                        }
                    }
                }
            } else if constexpr (kPairPath) {
                // packed pairs on float2 lanes: per slot row and region row the partial sum
                // runs in the two halves and is folded as (t.x + t.y), as in the float4 path
                const u64* kb2 = reinterpret_cast<const u64*>(kframe);
                const u64 W00 = pk2(w00, w00), W01 = pk2(w01, w01), W10 = pk2(w10, w10), W11 = pk2(w11, w11);
                auto ld2 = [](const u64* q) { return __ldg(reinterpret_cast<const unsigned long long*>(q)); };
                u64 kr[R];
                if (interior) {
                    const u64* p0 = kb2 + (r0 + xb);
                    const u64* p1 = kb2 + (r1 + xb);
                    u64 a0 = ld2(p0), a1 = ld2(p1);
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const u64 b0 = ld2(p0 + (j + 1) * G), b1 = ld2(p1 + (j + 1) * G);
                        kr[j] = fma2(W11, b1, fma2(W10, a1, fma2(W01, b0, mul2(W00, a0))));
                        a0 = b0;
                        a1 = b1;
                    }
                } else {
                    u64 a0 = ld2(kb2 + (r0 + xo[0])), a1 = ld2(kb2 + (r1 + xo[0]));
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const u64 b0 = ld2(kb2 + (r0 + xo[(j + 1) * XS])), b1 = ld2(kb2 + (r1 + xo[(j + 1) * XS]));
                        kr[j] = fma2(W11, b1, fma2(W10, a1, fma2(W01, b0, mul2(W00, a0))));
                        a0 = b0;
                        a1 = b1;
                    }
                }
#pragma unroll
                for (int s = 0; s < P; ++s) {
                    const int arow = r - (P - 1) + s;
                    if (arow < 0 || arow >= W) continue;  // uniform across the warp
                    const u64* qs = sq + (P - 1 - s) * P * G;
                    u64 t[W];
#pragma unroll
                    for (int px = 0; px < P; ++px) {
                        const u64 qv = qs[px * G];
#pragma unroll
                        for (int b = 0; b < W; ++b) {
                            if (METRIC == SNLS_METRIC_IP) {
                                t[b] = px == 0 ? mul2(qv, kr[b + px]) : fma2(qv, kr[b + px], t[b]);
                            } else {  // +sum (q - k)^2
                                const u64 d = sub2(qv, kr[b + px]);
                                t[b] = px == 0 ? mul2(d, d) : fma2(d, d, t[b]);
                            }
                        }
                    }
#pragma unroll
                    for (int b = 0; b < W; ++b) {
                        const float2 tf = upk2(t[b]);
                        if (s == P - 1)
                            acc[s][b] = tf.x + tf.y;
                        else
                            acc[s][b] += tf.x + tf.y;
                    }
                }
            } else if constexpr (VEC == 4 && !QREG) {
                // float4-typed registers (this formulation schedules ~2% better on B200 than
                // the VEC-generic arrays below: fewer dispatch stalls)
                const float4* kb4 = reinterpret_cast<const float4*>(kframe);
                float4 kr[R];
                if (interior) {
                    const float4* p0 = kb4 + (r0 + xb);
                    const float4* p1 = kb4 + (r1 + xb);
                    float4 a0 = __ldg(p0), a1 = __ldg(p1);
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const float4 b0 = __ldg(p0 + (j + 1) * G), b1 = __ldg(p1 + (j + 1) * G);
                        kr[j] = lerp4(a0, b0, a1, b1, w00, w01, w10, w11);
                        a0 = b0;
                        a1 = b1;
                    }
                } else {
                    float4 a0 = __ldg(kb4 + (r0 + xo[0])), a1 = __ldg(kb4 + (r1 + xo[0]));
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const float4 b0 = __ldg(kb4 + (r0 + xo[(j + 1) * XS]));
                        const float4 b1 = __ldg(kb4 + (r1 + xo[(j + 1) * XS]));
                        kr[j] = lerp4(a0, b0, a1, b1, w00, w01, w10, w11);
                        a0 = b0;
                        a1 = b1;
                    }
                }
#pragma unroll
                for (int s = 0; s < P; ++s) {
                    const int arow = r - (P - 1) + s;
                    if (arow < 0 || arow >= W) continue;  // uniform across the warp
                    [[maybe_unused]] const float* qr = qbase + qrow[P - 1 - s];
#pragma unroll
                    for (int px = 0; px < P; ++px) {
                        const float4 qv = __ldg(reinterpret_cast<const float4*>(qr + qcol[px]));
#pragma unroll
                        for (int b = 0; b < W; ++b) acc[s][b] = accum4<METRIC>(acc[s][b], qv, kr[b + px]);
                    }
                }
            } else {
                float kr[R][VEC];
                float a0[VEC], a1[VEC], b0[VEC], b1[VEC];
                if (interior) {
                    // no column reflection anywhere in the warp: one base per raw row and
                    // compile-time offsets (LDG [R + imm]) for the ws+ps columns
                    const float* p0 = kframe + size_t(r0 + xb) * VEC;
                    const float* p1 = kframe + size_t(r1 + xb) * VEC;
                    ldv<VEC>(p0, a0);
                    ldv<VEC>(p1, a1);
    #pragma unroll
                    for (int j = 0; j < R; ++j) {
                        ldv<VEC>(p0 + (j + 1) * F, b0);
                        ldv<VEC>(p1 + (j + 1) * F, b1);
                        lerpv<VEC>(kr[j], a0, b0, a1, b1, w00, w01, w10, w11);
    #pragma unroll
                        for (int v = 0; v < VEC; ++v) {
                            a0[v] = b0[v];
                            a1[v] = b1[v];
                        }
                    }
                } else {
                    ld(r0 + xo[0], a0);
                    ld(r1 + xo[0], a1);
    #pragma unroll
                    for (int j = 0; j < R; ++j) {
                        ld(r0 + xo[(j + 1) * XS], b0);
                        ld(r1 + xo[(j + 1) * XS], b1);
                        lerpv<VEC>(kr[j], a0, b0, a1, b1, w00, w01, w10, w11);
    #pragma unroll
                        for (int v = 0; v < VEC; ++v) {
                            a0[v] = b0[v];
                            a1[v] = b1[v];
                        }
                    }
                }
                // ---- update the slot rows that read region row r: a = r - (P-1) + s, py = P-1-s
    #pragma unroll
                for (int s = 0; s < P; ++s) {
                    const int arow = r - (P - 1) + s;
                    if (arow < 0 || arow >= W) continue;  // uniform across the warp
                    [[maybe_unused]] const float* qr = qbase + qrow[P - 1 - s];
    #pragma unroll
                    for (int px = 0; px < P; ++px) {
                        float qv[VEC];
                        if constexpr (QREG) {
    #pragma unroll
                            for (int v = 0; v < VEC; ++v) qv[v] = qreg[P - 1 - s][px][v];
                        } else {
                            ldv<VEC>(qr + qcol[px], qv);
                        }
                        // channel-outer: consecutive FMAs hit W different accumulators (the
                        // per-accumulator order, channel ascending, is unchanged)
#pragma unroll
                        for (int v = 0; v < VEC; ++v)
#pragma unroll
                            for (int b = 0; b < W; ++b) {
                                if (METRIC == SNLS_METRIC_IP) {
                                    acc[s][b] = fmaf(qv[v], kr[b + px][v], acc[s][b]);
                                } else {  // negated squared L2 accumulated as +sum(d^2)
                                    const float d = qv[v] - kr[b + px][v];
                                    acc[s][b] = fmaf(d, d, acc[s][b]);
                                }
                            }
                    }
                }
            }
            // ---- slot row r-(P-1) is complete: reduce-scatter over the G lanes, stream
            if (r >= P - 1) sel.template finish_row<METRIC>(acc[0], lane, gl, gq, on, row_ok, r - (P - 1), slot_base, grid_row, thr_src, thr_idx);
            // rotate: acc[s] tracks slot row r-(P-1)+s, so every region row shifts by one (an
            // unroll by P that renames instead costs 3x the code: c4 5.9 vs 4.45 ms, i-cache);
            // the packed paths assign a slot row's first contribution, the others start at zero
#pragma unroll
            for (int s = 0; s + 1 < P; ++s)
#pragma unroll
                for (int b = 0; b < W; ++b) acc[s][b] = acc[s + 1][b];
            if constexpr (!kPairPath && !(kPackedPath && kAssign1)) {
#pragma unroll
                for (int b = 0; b < W; ++b) acc[P - 1][b] = 0.f;
            }
        }
    }

    if (FG) return;  // selection happens in the top_l pass over the grid
    if constexpr (kKeysInQ) {
        __syncwarp();  // the warp's last reads of its query patches are done
        const size_t qbytes = size_t(P) * P * G * (kQsmF4 ? sizeof(float4) : sizeof(u64));
        sel.emit(a, reinterpret_cast<uint64_t*>(s_qdyn + size_t(qslot) * qbytes), row, row_ok, gl, qt, qy, qx);
    } else {
        sel.emit(a, s_keys[qslot], row, row_ok, gl, qt, qy, qx);
    }
}

template <int P, int W, int VEC, int G, int KMAX, int MINB>
int launch_cfg_b(const TiledSearch& s, cudaStream_t st) {
    using C = TiledCfg<P, W, VEC, G>;
    const unsigned blocks = unsigned((s.d.rows + C::QPB - 1) / C::QPB);
    // ps = 7: query patch in registers (c2: 0.477 -> 0.440 ms, profiles/r01_plans.txt) or, on
    // packed pairs, in shared memory
    constexpr bool QSM = kQsm && VEC == 2;
    constexpr bool QREG = P >= 7 && !QSM;
    const size_t smem = QSM ? size_t(C::QPB) * P * P * G * sizeof(u64)
                            : (VEC == 4 && kQsm4 ? size_t(C::QPB) * P * P * G * sizeof(float4) : 0);
    auto launch = [&](auto kern) {
        ensure_smem(kern, smem);
        // shared-memory carve-out: just what MINB resident CTAs need, the rest of the 256 KB
        // stays L1 (c4: 102 KB instead of the driver's 135 KB -> L1 hit 85% -> 88%, search
        // 3.862 -> 3.824 ms; profiles/r01_plans.txt).  Set once per kernel and device.
        static int done_dev = -1;
        int dev = 0;
        cudaGetDevice(&dev);
        if (SNLS_CARVEOUT != -1 && done_dev != dev) {
            int pct = SNLS_CARVEOUT;
            if (pct < 0) {
                cudaFuncAttributes fa{};
                int per_sm = 0, reserve = 0;
                cudaFuncGetAttributes(&fa, kern);
                cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
                cudaDeviceGetAttribute(&reserve, cudaDevAttrReservedSharedMemoryPerBlock, dev);
                const double need = double(MINB) * double(fa.sharedSizeBytes + smem + size_t(reserve));
                pct = per_sm > 0 ? int(std::ceil(100.0 * need / per_sm)) : 100;
                pct = pct < 1 ? 1 : (pct > 100 ? 100 : pct);
            }
            cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
            done_dev = dev;
        }
        kern<<<blocks, 32 * C::WARPS, smem, st>>>(s);
    };
    // the banded raster only where big frames need it (float4 lanes, F = 32 / 64) and the
    // remap's condition holds (a CTA's queries inside one image row)
    constexpr bool kBandInst = VEC == 4 && (G == 8 || G == 16);
    if constexpr (kBandInst) {
        if (!s.grid && s.band > 0 && s.d.nw % C::QPB == 0) {
            if (s.metric == SNLS_METRIC_IP)
                launch(search_tiled_kernel<P, W, VEC, G, KMAX, SNLS_METRIC_IP, MINB, QREG, false, false, true>);
            else
                launch(search_tiled_kernel<P, W, VEC, G, KMAX, SNLS_METRIC_L2, MINB, QREG, false, false, true>);
            return 1;
        }
    }
    if (s.grid) {
        if (s.metric == SNLS_METRIC_IP)
            launch(search_tiled_kernel<P, W, VEC, G, KMAX, SNLS_METRIC_IP, MINB, QREG, true>);
        else
            launch(search_tiled_kernel<P, W, VEC, G, KMAX, SNLS_METRIC_L2, MINB, QREG, true>);
    } else if (s.metric == SNLS_METRIC_IP) {
        launch(search_tiled_kernel<P, W, VEC, G, KMAX, SNLS_METRIC_IP, MINB, QREG, false>);
    } else {
        launch(search_tiled_kernel<P, W, VEC, G, KMAX, SNLS_METRIC_L2, MINB, QREG, false>);
    }
    return 1;
}

template <int P, int W, int VEC, int G, int KMAX>
int launch_cfg(const TiledSearch& s, cudaStream_t st) {
    if constexpr (P >= 7)  // 7 x 9 accumulators + the 15-pixel region row: 8 (12) warps per SM
        return launch_cfg_b<P, W, VEC, G, KMAX, kQsm ? SNLS_QSM_MINB : 2>(s, st);
    else if constexpr (P <= 3 && W <= SNLS_MINB4_WMAX)  // 3 x W accumulators fit 128 registers: 16 warps/SM
        return launch_cfg_b<P, W, VEC, G, KMAX, 4>(s, st);  // (c5: 126.7 -> 125.7 ms)
    else
        return launch_cfg_b<P, W, VEC, G, KMAX, 3>(s, st);
}

// VEC channels per lane: float4 lanes, except ps = 7 (the interpolated region row, 15
// pixels, must fit next to the 7 x 9 accumulators: two channels per lane)
template <int P, int W, int KMAX>
int launch_by_f(const TiledSearch& s, cudaStream_t st) {
    if constexpr (P >= 7) {
        switch (s.d.f) {
            case 16: return launch_cfg<P, W, 2, 8, KMAX>(s, st);
            case 32: return launch_cfg<P, W, 2, 16, KMAX>(s, st);
            case 64: return launch_cfg<P, W, 2, 32, KMAX>(s, st);
            default: return 0;
        }
    } else {
        switch (s.d.f) {
            case 4: return launch_cfg<P, W, 4, 1, KMAX>(s, st);
            case 8: return launch_cfg<P, W, 4, 2, KMAX>(s, st);
            case 16: return launch_cfg<P, W, 4, 4, KMAX>(s, st);
            case 32: return launch_cfg<P, W, 4, 8, KMAX>(s, st);
            case 64: return launch_cfg<P, W, 4, 16, KMAX>(s, st);
            default: return 0;
        }
    }
}

template <int P, int W>
int launch_by_k(const TiledSearch& s, cudaStream_t st) {
    if (s.topl <= 16) return launch_by_f<P, W, 16>(s, st);
    return 0;
}

template <int P, int VEC, int G>
int launch_replay_cfg(const TiledSearch& s, cudaStream_t st) {
    using C = TiledCfg<P, 1, VEC, G>;
    const unsigned blocks = unsigned((s.d.rows + C::QPB - 1) / C::QPB);
    constexpr bool QSM = kQsm && VEC == 2;
    constexpr bool QREG = P >= 7 && !QSM;
    const size_t smem = QSM ? size_t(C::QPB) * P * P * G * sizeof(u64)
                            : (VEC == 4 && kQsm4 ? size_t(C::QPB) * P * P * G * sizeof(float4) : 0);
    auto launch = [&](auto kern) {
        ensure_smem(kern, smem);
        kern<<<blocks, 32 * C::WARPS, smem, st>>>(s);
    };
    if (s.metric == SNLS_METRIC_IP)
        launch(search_tiled_kernel<P, 1, VEC, G, 16, SNLS_METRIC_IP, 1, QREG, true, true>);
    else
        launch(search_tiled_kernel<P, 1, VEC, G, 16, SNLS_METRIC_L2, 1, QREG, true, true>);
    return 1;
}

template <int P>
int launch_replay_p(const TiledSearch& s, cudaStream_t st) {
    if constexpr (P >= 7) {  // the forward's lane layout for this (ps, F): launch_by_f
        switch (s.d.f) {
            case 16: return launch_replay_cfg<P, 2, 8>(s, st);
            case 32: return launch_replay_cfg<P, 2, 16>(s, st);
            case 64: return launch_replay_cfg<P, 2, 32>(s, st);
            default: return 0;
        }
    } else {
        switch (s.d.f) {
            case 4: return launch_replay_cfg<P, 4, 1>(s, st);
            case 8: return launch_replay_cfg<P, 4, 2>(s, st);
            case 16: return launch_replay_cfg<P, 4, 4>(s, st);
            case 32: return launch_replay_cfg<P, 4, 8>(s, st);
            case 64: return launch_replay_cfg<P, 4, 16>(s, st);
            default: return 0;
        }
    }
}

}  // namespace

int launch_replay_tiled(const TiledSearch& s, cudaStream_t st) {
    // the (ps, ws) pairs the forward's tiled plan is instantiated for (launch_search_tiled)
    const bool tiled = s.topl <= 16 && ((s.ps == 3 && (s.ws == 11 || s.ws == 9 || s.ws == 5)) ||
                                        (s.ps == 7 && s.ws == 9) || (s.ps == 1 && (s.ws == 9 || s.ws == 5)));
    if (!tiled) return 0;
    switch (s.ps) {
        case 1: return launch_replay_p<1>(s, st);
        case 3: return launch_replay_p<3>(s, st);
        case 7: return launch_replay_p<7>(s, st);
        default: return 0;
    }
}

// Instantiated (ps, ws) pairs; anything else takes the generic path.
int launch_search_tiled(const TiledSearch& s, cudaStream_t st, int* used) {
    // auto: the region-row tiled plan (B200: c4 4.6 vs 4.7 ms, c2 0.48 vs 0.57 ms for the
    // streaming plan, profiles/r01_plans.txt); the streaming plan on request
    if (s.kernel == 2) {
        if (int n = launch_search_stream(s, st)) {
            if (used) *used = 2;
            return n;
        }
    }
    if (SNLS_XO16 && int64_t(s.d.w) * s.d.f >= (int64_t(1) << 16)) return 0;  // (16-bit column table)
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
