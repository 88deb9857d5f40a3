// The frame-alignment pipeline around the search, on device:
//  * block_match_kernel -- estimate_flow_block_matching (flow.cpp:114-175): exhaustive
//    block SSD search over (2r+1)^2 integer shifts with reflected reads.  One CTA per
//    (frame pair, block); the block of frame a is staged in shared memory, each thread owns
//    candidate shifts and sums (y, x, c) in the reference's order in fp64 (exact for
//    fp32-representable inputs up to the order), then a (ssd, scan index) argmin keeps the
//    reference's "first hit in scan order wins" tie rule.
//  * psnr_kernel -- psnr (tensor.cpp:79-90) per frame: fp64 squared-difference partials per
//    CTA in a fixed order, then a fixed-order final sum (deterministic).
//  * snls_align_frames -- align_frames (harness.cpp:72-154) over HOST buffers: noise from
//    the reference's GaussianStream on the host (rng.hpp:30-53, bitwise), then flow
//    (zero / provided / block matching), one batched search over all T-1 frame pairs
//    (each pair is its own one-frame clip: wt = 0), the fused softmax, wpsum of the clean
//    frames and the per-pair PSNR, all on the device.
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace snls_capi {
int fail(int code, const std::string& msg);
}

namespace snls_gpu {

namespace {

constexpr int kBmThreads = 256;

__global__ void __launch_bounds__(kBmThreads) block_match_kernel(const float* __restrict__ a,
                                                                 const float* __restrict__ b, int h,
                                                                 int w, int f, int block, int radius,
                                                                 int nbx, int nblocks,
                                                                 float* __restrict__ flow) {
    extern __shared__ float s_a[];  // block x block x f pixels of frame a
    __shared__ double s_best[kBmThreads / 32];
    __shared__ int s_idx[kBmThreads / 32];
    const int t = blockIdx.x / nblocks, bi = blockIdx.x % nblocks;
    const int by = bi / nbx, bx = bi % nbx;
    const int y0 = by * block, x0 = bx * block;
    const int y1 = min(y0 + block, h), x1 = min(x0 + block, w);
    const int bw = x1 - x0, npx = (y1 - y0) * bw;
    const size_t frame = size_t(h) * w * f;
    const float* fa = a + t * frame;
    const float* fb = b + t * frame;
    for (int i = threadIdx.x; i < npx * f; i += blockDim.x) {
        const int p = i / f, c = i % f;
        s_a[i] = fa[(size_t(y0 + p / bw) * w + x0 + p % bw) * f + c];
    }
    __syncthreads();
    const int side = 2 * radius + 1, ncand = side * side;
    double best = INFINITY;
    int best_i = 0x7fffffff;
    for (int ci = threadIdx.x; ci < ncand; ci += blockDim.x) {  // ascending per thread
        const int dy = ci / side - radius, dx = ci % side - radius;
        double ssd = 0.0;
        for (int y = y0; y < y1; ++y) {
            const float* rb = fb + size_t(reflect(y + dy, h)) * w * f;
            const float* ra = s_a + (y - y0) * bw * f;
            for (int x = x0; x < x1; ++x) {
                const float* pb = rb + size_t(reflect(x + dx, w)) * f;
                const float* pa = ra + (x - x0) * f;
                for (int c = 0; c < f; ++c) {
                    // ssd += d * d with the reference's two roundings (no contraction)
                    const double d = __dsub_rn(double(pa[c]), double(__ldg(pb + c)));
                    ssd = __dadd_rn(ssd, __dmul_rn(d, d));
                }
            }
        }
        if (ssd < best) {  // within a thread candidates come in scan order: strict '<'
            best = ssd;
            best_i = ci;
        }
    }
    // (ssd, scan index) argmin across the CTA
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
        if (ob < best || (ob == best && oi < best_i)) {
            best = ob;
            best_i = oi;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_best[warp] = best;
        s_idx[warp] = best_i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < int(blockDim.x / 32); ++i)
            if (s_best[i] < best || (s_best[i] == best && s_idx[i] < best_i)) {
                best = s_best[i];
                best_i = s_idx[i];
            }
        s_idx[0] = best_i < ncand ? best_i : (ncand / 2);  // all-inf block: shift 0 (reference init)
    }
    __syncthreads();
    const int bi_best = s_idx[0];
    const float fdy = float(bi_best / side - radius), fdx = float(bi_best % side - radius);
    float* fo = flow + size_t(t) * h * w * 2;
    for (int p = threadIdx.x; p < npx; p += blockDim.x) {
        const size_t o = (size_t(y0 + p / bw) * w + x0 + p % bw) * 2;
        fo[o] = fdy;
        fo[o + 1] = fdx;
    }
}

constexpr int kPsnrThreads = 256, kPsnrParts = 64;

// Per frame t: kPsnrParts CTAs each sum a fixed contiguous chunk of squared differences in
// fp64 (thread-strided, then a fixed tree), written to part[t][cta].
__global__ void __launch_bounds__(kPsnrThreads) psnr_partial_kernel(const float* __restrict__ a,
                                                                    const float* __restrict__ b,
                                                                    size_t n, double* part) {
    __shared__ double s[kPsnrThreads];
    const int t = blockIdx.x / kPsnrParts, pc = blockIdx.x % kPsnrParts;
    const size_t chunk = (n + kPsnrParts - 1) / kPsnrParts;
    const size_t lo = pc * chunk, hi = min(n, lo + chunk);
    const float* fa = a + size_t(t) * n;
    const float* fb = b + size_t(t) * n;
    double acc = 0.0;
    for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double d = double(fa[i]) - double(fb[i]);
        acc = fma(d, d, acc);
    }
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = kPsnrThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[size_t(t) * kPsnrParts + pc] = s[0];
}

__global__ void psnr_final_kernel(const double* part, int frames, size_t n, double peak, double* out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= frames) return;
    double sq = 0.0;
    for (int i = 0; i < kPsnrParts; ++i) sq += part[size_t(t) * kPsnrParts + i];
    const double mse = sq / double(n);
    out[t] = mse == 0.0 ? INFINITY : 10.0 * log10(peak * peak / mse);
}

}  // namespace

int launch_block_match(const float* a, const float* b, int frames, int h, int w, int f, int block,
                       int radius, float* flow, cudaStream_t st) {
    const int nby = (h + block - 1) / block, nbx = (w + block - 1) / block;
    const size_t smem = size_t(block) * block * f * sizeof(float);
    if (smem > 200 * 1024) return -1;
    ensure_smem(block_match_kernel, smem);
    block_match_kernel<<<unsigned(int64_t(frames) * nby * nbx), kBmThreads, smem, st>>>(
        a, b, h, w, f, block, radius, nbx, nby * nbx, flow);
    return 1;
}

int launch_psnr(const float* a, const float* b, int frames, size_t n, double peak, double* part,
                double* out, cudaStream_t st) {
    psnr_partial_kernel<<<unsigned(frames * kPsnrParts), kPsnrThreads, 0, st>>>(a, b, n, part);
    psnr_final_kernel<<<unsigned((frames + 127) / 128), 128, 0, st>>>(part, frames, n, peak, out);
    return 2;
}

size_t psnr_scratch_doubles(int frames) { return size_t(frames) * kPsnrParts; }

}  // namespace snls_gpu

// ---- align_frames over host buffers (harness.cpp:72-154) --------------------------------
extern "C" {

int snls_align_frames(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* clean,
                      double sigma, uint64_t seed, int flow_source, const float* provided_flow,
                      int bm_block, int bm_radius, float* aligned, float* top1_offsets,
                      float* used_flow, double* frame_psnr) {
    using snls_capi::fail;
    if (!ctx || !cfg) return fail(SNLS_EARG, "align_frames: null context or config");
    if (int rc = snls_validate_config(cfg)) return rc;  // opts.cfg.validate()
    if (cfg->topl != 1) return fail(SNLS_ECONFIG, "align_frames: requires topl == 1");
    if (dims.t < 2) return fail(SNLS_EDOMAIN, "align_frames: needs at least two frames");
    if (flow_source == 1 && !provided_flow)
        return fail(SNLS_ECONFIG, "align_frames: flow source is 'provided' but none given");
    if (!clean || !aligned || !frame_psnr) return fail(SNLS_EARG, "align_frames: null buffer");
    const int pairs = dims.t - 1, H = dims.h, W = dims.w, F = dims.f;
    const size_t frame = size_t(H) * W * F, fframe = size_t(H) * W * 2;
    const size_t nvid = size_t(dims.t) * frame;
    // noise on the host: GaussianStream is sequential and must stay bitwise (rng.hpp:30-53)
    // harness.cpp:95: `opts.sigma > 0.0 ? add_gaussian_noise(...) : clean` -- a zero or
    // negative sigma aligns the clean clip (add_gaussian_noise itself rejects sigma < 0)
    std::vector<float> noisy(nvid);
    if (sigma > 0.0) {
        if (int rc = snls_gaussian_noise_f32(seed, sigma, int64_t(nvid), clean, noisy.data())) return rc;
    } else {
        std::copy(clean, clean + nvid, noisy.begin());
    }

    void* sp = nullptr;
    snls_ctx_get_stream(ctx, &sp);
    cudaStream_t st = static_cast<cudaStream_t>(sp);
    int64_t rows = 0;
    int nh = 0, nw = 0;
    const snls_dims pd{pairs, H, W, F};
    if (int rc = snls_query_grid(pd, cfg->stride0, &rows, &nh, &nw)) return rc;
    float *d_noisy = nullptr, *d_clean = nullptr, *d_flow = nullptr, *d_sims = nullptr,
          *d_offs = nullptr, *d_wts = nullptr, *d_out = nullptr;
    int32_t* d_cnt = nullptr;
    auto release = [&]() {
        float* fs[] = {d_noisy, d_clean, d_flow, d_sims, d_offs, d_wts, d_out};
        for (float* p : fs)
            if (p) cudaFree(p);
        if (d_cnt) cudaFree(d_cnt);
    };
    cudaError_t e = cudaSuccess;
    auto mal = [&](auto** p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(p), bytes ? bytes : 4);
    };
    mal(&d_noisy, nvid * sizeof(float));
    mal(&d_clean, nvid * sizeof(float));
    mal(&d_flow, size_t(pairs) * fframe * sizeof(float));
    mal(&d_sims, size_t(rows) * sizeof(float));
    mal(&d_offs, size_t(rows) * 3 * sizeof(float));
    mal(&d_wts, size_t(rows) * sizeof(float));
    mal(&d_out, size_t(pairs) * frame * sizeof(float));
    mal(&d_cnt, size_t(pairs) * H * W * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_noisy, noisy.data(), nvid * sizeof(float), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_clean, clean, nvid * sizeof(float), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        if (flow_source == 1)
            e = cudaMemcpyAsync(d_flow, provided_flow, size_t(pairs) * fframe * sizeof(float),
                                cudaMemcpyHostToDevice, st);
        else
            e = cudaMemsetAsync(d_flow, 0, size_t(pairs) * fframe * sizeof(float), st);
    }
    if (e != cudaSuccess) {
        release();
        return fail(SNLS_ECUDA, std::string("align_frames: ") + cudaGetErrorString(e));
    }
    int rc = SNLS_OK;
    // flow for every pair (ti -> ti + 1) at once
    if (flow_source == 2)
        rc = snls_block_match(ctx, pd, d_noisy, d_noisy + frame, bm_block, bm_radius, d_flow);
    // every pair is its own one-frame clip (frame_slice, harness.cpp:127-131): with wt = 0 the
    // batched clip searches only dt = 0, exactly the per-pair search
    snls_config c1 = *cfg;
    c1.wt = 0;
    if (rc == SNLS_OK)
        rc = snls_search_fwd(ctx, &c1, pd, d_noisy, d_noisy + frame, d_flow, d_flow, SNLS_MODE_FUSED,
                             d_sims, d_offs, nullptr, d_wts);
    if (rc == SNLS_OK) rc = snls_wpsum_fwd(ctx, &c1, pd, d_clean + frame, d_wts, d_offs, d_out, d_cnt);
    if (rc == SNLS_OK) rc = snls_ctx_sync_check(ctx);
    if (rc == SNLS_OK) rc = snls_psnr_frames(ctx, pd, d_out, d_clean, 255.0, frame_psnr);
    if (rc == SNLS_OK) {
        e = cudaMemcpyAsync(aligned, d_out, size_t(pairs) * frame * sizeof(float), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && top1_offsets)
            e = cudaMemcpyAsync(top1_offsets, d_offs, size_t(rows) * 3 * sizeof(float), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && used_flow)
            e = cudaMemcpyAsync(used_flow, d_flow, size_t(pairs) * fframe * sizeof(float), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = fail(SNLS_ECUDA, std::string("align_frames: ") + cudaGetErrorString(e));
    } else {
        cudaStreamSynchronize(st);
    }
    release();
    return rc;
}

}  // extern "C"
