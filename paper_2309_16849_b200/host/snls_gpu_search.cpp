// Drop-in replacement for the reference's src/search.cpp: the full search.hpp surface, with
// the operators (shifted_nls_forward, nls_forward, top_l, shifted_nls_backward,
// replay_similarities) executed by the sm_100a kernels through the C-ABI.  Link this file
// and snls_gpu_aggregate.cpp instead of search.cpp / aggregate.cpp.
//
// Semantics kept from the reference: validation order and messages (search.cpp:21-32,
// 175-183), the underfull ConfigError (search.cpp:324-325), result/tape layout
// (search.hpp:65-116), byte accounting of results (search.cpp:273-276, 340-345).
// Differences: arithmetic is fp32 on the device (results agree to 1e-5 relative; top-L
// indices are bit-exact where fp32 sums are exact, e.g. integer-valued videos).  The
// backward takes the reference's fp64 tape as is and honours ExecPolicy::deterministic
// (int64 fixed-point accumulation: bitwise reproducible, SNLS_BWD_DETERMINISTIC).
#include <algorithm>
#include <cmath>
#include <thread>

#include "snls/memory.hpp"
#include "snls/search.hpp"
#include "snls_gpu_runtime.hpp"

namespace snls {

void SearchConfig::validate() const {
    const snls_config c = gpu::to_abi(*this);
    gpu::check(snls_validate_config(&c));
}

int ExecPolicy::resolved_threads() const {
    if (threads > 0) return threads;
    const unsigned n = std::thread::hardware_concurrency();
    return n ? int(n) : 1;
}

QueryGrid QueryGrid::over(int t, int h, int w, int stride) {
    QueryGrid g;
    g.t = t;
    g.nh = (h - 1) / stride + 1;
    g.nw = (w - 1) / stride + 1;
    g.stride = stride;
    return g;
}

void QueryGrid::coords(std::int64_t row, int& qt, int& qy, int& qx) const {
    qx = int(row % nw) * stride;
    const std::int64_t r = row / nw;
    qy = int(r % nh) * stride;
    qt = int(r / nh);
}

std::vector<int> temporal_scan_order(int wt) {
    std::vector<int> order{0};
    for (int d = 1; d <= wt; ++d) {
        order.push_back(-d);
        order.push_back(d);
    }
    return order;
}

namespace detail {

// Scalar host helpers of the search.hpp surface (used by callers and tests, not by the
// operators above, which run on the device).  Same arithmetic as search.cpp:72-151.
void accumulate_shift(const FlowField& fflow, const FlowField& bflow, int qt, int qy, int qx,
                      int dt, double& dy, double& dx, double* links) {
    if (dt == 0) {
        dy = fflow.at(qt, qy, qx, 0);
        dx = fflow.at(qt, qy, qx, 1);
        return;
    }
    const FlowField& f = dt > 0 ? fflow : bflow;
    const int step = dt > 0 ? 1 : -1, m = std::abs(dt);
    double sy = 0.0, sx = 0.0;
    for (int k = 0; k < m; ++k) {
        const int fr = qt + step * k;
        double vy, vx;
        if (k == 0) {
            vy = f.at(fr, qy, qx, 0);
            vx = f.at(fr, qy, qx, 1);
        } else {
            const double py = qy + sy, px = qx + sx;
            const BilinearTaps t = bilinear_taps(f.h, f.w, py, px);
            const double a0 = f.at(fr, t.y0, t.x0, 0), b0 = f.at(fr, t.y0, t.x1, 0);
            const double c0 = f.at(fr, t.y1, t.x0, 0), d0 = f.at(fr, t.y1, t.x1, 0);
            const double a1 = f.at(fr, t.y0, t.x0, 1), b1 = f.at(fr, t.y0, t.x1, 1);
            const double c1 = f.at(fr, t.y1, t.x0, 1), d1 = f.at(fr, t.y1, t.x1, 1);
            vy = t.w00 * a0 + t.w01 * b0 + t.w10 * c0 + t.w11 * d0;
            vx = t.w00 * a1 + t.w01 * b1 + t.w10 * c1 + t.w11 * d1;
            if (links) {
                double* lk = links + std::size_t(k - 1) * 6;
                lk[0] = py;
                lk[1] = px;
                lk[2] = -(1.0 - t.fx) * a0 - t.fx * b0 + (1.0 - t.fx) * c0 + t.fx * d0;
                lk[3] = -(1.0 - t.fy) * a0 + (1.0 - t.fy) * b0 - t.fy * c0 + t.fy * d0;
                lk[4] = -(1.0 - t.fx) * a1 - t.fx * b1 + (1.0 - t.fx) * c1 + t.fx * d1;
                lk[5] = -(1.0 - t.fy) * a1 + (1.0 - t.fy) * b1 - t.fy * c1 + t.fy * d1;
            }
        }
        sy += vy;
        sx += vx;
    }
    dy = sy;
    dx = sx;
}

double patch_similarity(const VideoTensor& q, const VideoTensor& k, int qt, int qy, int qx,
                        int kt, double ky, double kx, int ps, Metric metric) {
    const int half = ps / 2;
    double acc = 0.0;
    for (int py = -half; py <= half; ++py) {
        const int ry = reflect_index(qy + py, q.h);
        for (int px = -half; px <= half; ++px) {
            const int rx = reflect_index(qx + px, q.w);
            const BilinearTaps t = bilinear_taps(k.h, k.w, ky + double(py), kx + double(px));
            for (int c = 0; c < q.f; ++c) {
                const double kv = t.w00 * k.at(kt, t.y0, t.x0, c) + t.w01 * k.at(kt, t.y0, t.x1, c) +
                                  t.w10 * k.at(kt, t.y1, t.x0, c) + t.w11 * k.at(kt, t.y1, t.x1, c);
                const double qv = q.at(qt, ry, rx, c);
                if (metric == Metric::kInnerProduct) {
                    acc += qv * kv;
                } else {
                    const double d = qv - kv;
                    acc -= d * d;
                }
            }
        }
    }
    return acc;
}

}  // namespace detail

namespace {

snls_dims dims_of(const VideoTensor& v) { return snls_dims{v.t, v.h, v.w, v.f}; }

struct SearchBuffers {
    gpu::DeviceBuffer q, k, ff, bf, sims, offsets, chains, grad, dq, dk, dff, dbf;
    gpu::DeviceBuffer sims64, offs64, cen64, ch64;
};
thread_local SearchBuffers t_buf;


}  // namespace

namespace {
// fflow / bflow null: nls_forward's zero flows, never materialised or uploaded.
SearchResult forward_impl(const VideoTensor& q, const VideoTensor& k, const FlowField* fflow,
                          const FlowField* bflow, const SearchConfig& cfg, const ExecPolicy& policy) {
    // validate_forward_inputs (search.cpp:175-183), same order and messages
    cfg.validate();
    if (!q.same_shape(k)) throw DomainError("search: query and key shapes differ");
    if (fflow) {
        if (!fflow->matches_video(q.t, q.h, q.w) || !bflow->matches_video(q.t, q.h, q.w))
            throw DomainError("search: flow shape does not match the video");
        fflow->require_finite("search fflow");
        bflow->require_finite("search bflow");
    }

    const QueryGrid grid = QueryGrid::over(q.t, q.h, q.w, cfg.stride0);
    const std::int64_t rows = grid.rows();
    const int L = cfg.topl, cs = cfg.wt > 1 ? cfg.wt - 1 : 0;
    SearchResult res;
    res.sims.rows = rows;
    res.sims.cols = L;
    res.offsets.rows = rows;
    res.offsets.l = L;
    res.tape.cfg = cfg;
    res.tape.grid = grid;
    res.tape.vid_t = q.t;
    res.tape.vid_h = q.h;
    res.tape.vid_w = q.w;
    res.tape.vid_f = q.f;
    res.tape.chain_stride = cs;
    const std::uint64_t n_sel = std::uint64_t(rows) * L;
    memory::TransientCharge outputs_charge((n_sel * (1 + 3 + 3 + std::uint64_t(cs) * 6)) * sizeof(double));
    // the materialised grid of kFullGrid lives in device memory; account for it the same way
    const std::uint64_t grid_bytes = policy.mode == SearchMode::kFullGrid
                                         ? std::uint64_t(rows) * cfg.window_slots() * 4 * sizeof(float)
                                         : 0;
    memory::TransientCharge grid_charge(grid_bytes);

    snls_ctx* ctx = gpu::context();
    gpu::profile_mark("forward: validate + shell");
    // the result vectors (~400 MB of fp64 at c4, std::vector zero-fills them) are prepared on
    // helper threads while the inputs upload and the kernels run
    auto prep_chains = [&] { gpu::size_for_fill(res.tape.chains, n_sel * cs * 6); };
    auto prep_small = [&] {
        gpu::size_for_fill(res.tape.centers, n_sel * 3);
        gpu::size_for_fill(res.offsets.data, n_sel * 3);
        gpu::size_for_fill(res.sims.values, n_sel);
    };
    std::vector<std::thread> prep;
    const bool big = n_sel * (7 + std::uint64_t(cs) * 6) * sizeof(double) >= (std::uint64_t(64) << 20);
    if (big) {  // (threads only pay off for large results)
        prep.emplace_back(prep_chains);
        prep.emplace_back(prep_small);
    }
    // inputs: fp64 -> fp32 conversion pipelined against the H2D copies (Q = K aliased once)
    const bool alias = (&q == &k || q.data == k.data);
    float* dq = gpu::upload_async(t_buf.q, q.data.data(), q.data.size());
    const float* dk = alias ? dq : gpu::upload_async(t_buf.k, k.data.data(), k.data.size());
    float* dff = fflow ? gpu::upload_async(t_buf.ff, fflow->data.data(), fflow->data.size()) : nullptr;
    float* dbf = fflow ? gpu::upload_async(t_buf.bf, bflow->data.data(), bflow->data.size()) : nullptr;
    gpu::profile_mark("forward: upload enqueued");
    float* dsims = t_buf.sims.f32(n_sel);
    float* doffs = t_buf.offsets.f32(n_sel * 3);
    const snls_config c = gpu::to_abi(cfg);
    gpu::check(snls_search_fwd(ctx, &c, dims_of(q), dq, dk, dff, dbf,
                               policy.mode == SearchMode::kFullGrid ? SNLS_MODE_FULLGRID
                                                                    : SNLS_MODE_FUSED,
                               dsims, doffs, nullptr, nullptr));
    // the whole result in the reference's fp64 layout, on the device: sims, offsets and the
    // exact fp64 tape (centres, absolute chain links; snls_search_results64)
    double* s64 = static_cast<double*>(t_buf.sims64.reserve(n_sel * sizeof(double)));
    double* o64 = static_cast<double*>(t_buf.offs64.reserve(n_sel * 3 * sizeof(double)));
    double* c64 = static_cast<double*>(t_buf.cen64.reserve(n_sel * 3 * sizeof(double)));
    double* ch64 = cs > 0 ? static_cast<double*>(t_buf.ch64.reserve(n_sel * cs * 6 * sizeof(double))) : nullptr;
    gpu::check(snls_search_results64(ctx, &c, dims_of(q), 0, q.t, dff, dbf, dsims, doffs, s64, o64, c64, ch64));
    gpu::profile_mark("forward: kernels enqueued");
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::profile_mark("forward: device done");
    if (big) prep[1].join();  // the small vectors first: their copies overlap the chains' zero-fill
    else prep_small();
    gpu::profile_mark("forward: small vectors sized");
    gpu::download64(res.sims.values, s64, n_sel);
    gpu::download64(res.offsets.data, o64, n_sel * 3);
    gpu::download64(res.tape.centers, c64, n_sel * 3);
    if (big) prep[0].join();
    else prep_chains();
    gpu::profile_mark("forward: chains sized");
    if (cs > 0) gpu::download64(res.tape.chains, ch64, n_sel * cs * 6);
    gpu::profile_mark("forward: results downloaded");
    return res;
}
}  // namespace

SearchResult shifted_nls_forward(const VideoTensor& q, const VideoTensor& k,
                                 const FlowField& fflow, const FlowField& bflow,
                                 const SearchConfig& cfg, const ExecPolicy& policy) {
    return forward_impl(q, k, &fflow, &bflow, cfg, policy);
}

SearchResult nls_forward(const VideoTensor& q, const VideoTensor& k, const SearchConfig& cfg,
                         const ExecPolicy& policy) {
    return forward_impl(q, k, nullptr, nullptr, cfg, policy);  // zero flows: NULL at the C-ABI
}

std::pair<SimilarityTensor, OffsetTensor> top_l(const SimilarityTensor& full,
                                                const OffsetTensor& full_offsets, int topl) {
    if (full.rows != full_offsets.rows || full.cols != full_offsets.l)
        throw DomainError("top_l: similarity and offset shapes disagree");
    if (topl < 1 || topl > full.cols) throw ConfigError("top_l: L out of range");
    SimilarityTensor sel;
    sel.rows = full.rows;
    sel.cols = topl;
    OffsetTensor off;
    off.rows = full.rows;
    off.l = topl;
    if (full.rows == 0) return {sel, off};
    snls_ctx* ctx = gpu::context();
    float* dfull = gpu::upload(t_buf.sims, full.values);
    float* doff = gpu::upload(t_buf.offsets, full_offsets.data);
    const std::uint64_t n = std::uint64_t(full.rows) * topl;
    float* dsel = t_buf.grad.f32(n);
    float* dsoff = t_buf.chains.f32(n * 3);
    gpu::check(snls_topl(ctx, full.rows, full.cols, dfull, doff, topl, dsel, dsoff));
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::download(sel.values, dsel, n);
    gpu::download(off.data, dsoff, n * 3);
    return {std::move(sel), std::move(off)};
}


SearchGradients shifted_nls_backward(const SimilarityTensor& grad_selected,
                                     const SearchTape& tape, const VideoTensor& q,
                                     const VideoTensor& k, const ExecPolicy& policy) {
    if (grad_selected.rows != tape.grid.rows() || grad_selected.cols != tape.cfg.topl)
        throw DomainError("shifted_nls_backward: gradient shape does not match the tape");
    if (q.t != tape.vid_t || q.h != tape.vid_h || q.w != tape.vid_w || q.f != tape.vid_f ||
        !q.same_shape(k))
        throw DomainError("shifted_nls_backward: tensor shape does not match the tape");
    SearchGradients g;
    snls_ctx* ctx = gpu::context();
    gpu::profile_mark("backward: checks");
    // the reference's own fp64 tape goes to the device as is (snls_search_bwd_ex): exact key
    // centres and chain links, no host conversion
    const std::uint64_t n_sel = std::uint64_t(tape.grid.rows()) * tape.cfg.topl;
    const int cs = tape.chain_stride;
    double* dcen = static_cast<double*>(t_buf.cen64.reserve(n_sel * 3 * sizeof(double)));
    gpu::check(snls_copy_h2d(ctx, dcen, tape.centers.data(), n_sel * 3 * sizeof(double)));
    double* dch = nullptr;
    if (tape.cfg.wt > 1) {
        dch = static_cast<double*>(t_buf.ch64.reserve(n_sel * std::max(cs, 1) * 6 * sizeof(double)));
        gpu::check(snls_copy_h2d(ctx, dch, tape.chains.data(), n_sel * cs * 6 * sizeof(double)));
    }
    float* dgrad = gpu::upload_async(t_buf.grad, grad_selected.values.data(), grad_selected.values.size());
    float* dq = gpu::upload_async(t_buf.q, q.data.data(), q.data.size());
    const bool alias = (&q == &k || q.data == k.data);
    float* dk = alias ? dq : gpu::upload_async(t_buf.k, k.data.data(), k.data.size());
    const std::uint64_t nv = q.size(), nf = std::uint64_t(q.t) * q.h * q.w * 2;
    float* ddq = t_buf.dq.f32(nv);
    float* ddk = t_buf.dk.f32(nv);
    float* ddff = t_buf.dff.f32(nf);
    float* ddbf = t_buf.dbf.f32(nf);
    const snls_config c = gpu::to_abi(tape.cfg);
    // ExecPolicy::deterministic (the reference's default, search.cpp:687-696): bitwise
    // reproducible fixed-point accumulation on the device
    gpu::check(snls_search_bwd_ex(ctx, &c, dims_of(q), 0, q.t, dgrad, nullptr, nullptr, dcen, dch, dq, dk,
                                  ddq, ddk, ddff, ddbf, policy.deterministic ? SNLS_BWD_DETERMINISTIC : 0));
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::profile_mark("backward: device done");
    g.grad_q = VideoTensor(q.t, q.h, q.w, q.f);
    g.grad_k = VideoTensor(q.t, q.h, q.w, q.f);
    g.grad_fflow = FlowField(q.t, q.h, q.w, FlowDirection::kForward);
    g.grad_bflow = FlowField(q.t, q.h, q.w, FlowDirection::kBackward);
    gpu::download(g.grad_q.data, ddq, nv);
    gpu::download(g.grad_k.data, ddk, nv);
    gpu::download(g.grad_fflow.data, ddff, nf);
    gpu::download(g.grad_bflow.data, ddbf, nf);
    gpu::profile_mark("backward: downloaded");
    return g;
}

SimilarityTensor replay_similarities(const SearchTape& tape, const VideoTensor& q,
                                     const VideoTensor& k) {
    if (q.t != tape.vid_t || q.h != tape.vid_h || q.w != tape.vid_w || q.f != tape.vid_f ||
        !q.same_shape(k))
        throw DomainError("replay_similarities: tensor shape does not match the tape");
    SimilarityTensor out;
    out.rows = tape.grid.rows();
    out.cols = tape.cfg.topl;
    snls_ctx* ctx = gpu::context();
    // the fp64 tape centres as they are, replayed through the search plan's own per-slot
    // arithmetic (snls_replay64): the forward's similarities bit for bit (search.cpp:470-493)
    const std::uint64_t n = std::uint64_t(out.rows) * out.cols;
    double* dcen = static_cast<double*>(t_buf.cen64.reserve(n * 3 * sizeof(double)));
    gpu::check(snls_copy_h2d(ctx, dcen, tape.centers.data(), n * 3 * sizeof(double)));
    float* dq = gpu::upload_async(t_buf.q, q.data.data(), q.data.size());
    const bool alias = (&q == &k || q.data == k.data);
    float* dk = alias ? dq : gpu::upload_async(t_buf.k, k.data.data(), k.data.size());
    float* dsims = t_buf.sims.f32(n);
    const snls_config c = gpu::to_abi(tape.cfg);
    gpu::check(snls_replay64(ctx, &c, dims_of(q), 0, q.t, dq, dk, dcen, -1, dsims));
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::download(out.values, dsims, n);
    return out;
}

}  // namespace snls
