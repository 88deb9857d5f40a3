// Drop-in replacement for the reference's src/search.cpp: the full search.hpp surface, with
// the operators (shifted_nls_forward, nls_forward, top_l, shifted_nls_backward,
// replay_similarities) executed by the sm_100a kernels through the C-ABI.  Link this file
// and snls_gpu_aggregate.cpp instead of search.cpp / aggregate.cpp.
//
// Semantics kept from the reference: validation order and messages (search.cpp:21-32,
// 175-183), the underfull ConfigError (search.cpp:324-325), result/tape layout
// (search.hpp:65-116), byte accounting of results (search.cpp:273-276, 340-345).
// Differences: arithmetic is fp32 on the device (results agree to 1e-5 relative; top-L
// indices are bit-exact where fp32 sums are exact, e.g. integer-valued videos), and the
// backward always scatters with atomics (the reference's non-deterministic mode).
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
};
thread_local SearchBuffers t_buf;

void query_base(const QueryGrid& g, std::int64_t row, double& qt, double& qy, double& qx) {
    int t, y, x;
    g.coords(row, t, y, x);
    qt = t;
    qy = y;
    qx = x;
}

}  // namespace

SearchResult shifted_nls_forward(const VideoTensor& q, const VideoTensor& k,
                                 const FlowField& fflow, const FlowField& bflow,
                                 const SearchConfig& cfg, const ExecPolicy& policy) {
    // validate_forward_inputs (search.cpp:175-183), same order and messages
    cfg.validate();
    if (!q.same_shape(k)) throw DomainError("search: query and key shapes differ");
    if (!fflow.matches_video(q.t, q.h, q.w) || !bflow.matches_video(q.t, q.h, q.w))
        throw DomainError("search: flow shape does not match the video");
    fflow.require_finite("search fflow");
    bflow.require_finite("search bflow");

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
    float* dq = gpu::upload(t_buf.q, q.data);
    const float* dk = (&q == &k || q.data == k.data) ? dq : gpu::upload(t_buf.k, k.data);
    float* dff = gpu::upload(t_buf.ff, fflow.data);
    float* dbf = gpu::upload(t_buf.bf, bflow.data);
    float* dsims = t_buf.sims.f32(n_sel);
    float* doffs = t_buf.offsets.f32(n_sel * 3);
    float* dch = cs > 0 ? t_buf.chains.f32(n_sel * cs * 6) : nullptr;
    const snls_config c = gpu::to_abi(cfg);
    gpu::check(snls_search_fwd(ctx, &c, dims_of(q), dq, dk, dff, dbf,
                               policy.mode == SearchMode::kFullGrid ? SNLS_MODE_FULLGRID
                                                                    : SNLS_MODE_FUSED,
                               dsims, doffs, dch, nullptr));
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::download(res.sims.values, dsims, n_sel);
    gpu::download(res.offsets.data, doffs, n_sel * 3);
    res.tape.centers.resize(n_sel * 3);
    res.tape.chains.resize(n_sel * cs * 6);
    // device chains (relative to the query pixel) stay in the pinned staging buffer and are
    // converted to the reference's absolute positions in one parallel pass
    const float* rel = nullptr;
    if (cs > 0) {
        float* st = gpu::staging(n_sel * cs * 6);
        gpu::check(snls_copy_d2h(ctx, st, dch, n_sel * cs * 6 * sizeof(float)));
        rel = st;
    }
    double* centers = res.tape.centers.data();
    double* chains = res.tape.chains.data();
    const double* offs = res.offsets.data.data();
#pragma omp parallel for schedule(static) num_threads(policy.resolved_threads())
    for (std::int64_t row = 0; row < rows; ++row) {
        double qt, qy, qx;
        query_base(grid, row, qt, qy, qx);
        for (int li = 0; li < L; ++li) {
            const std::size_t e = std::size_t(row) * L + li;
            const double* o = offs + e * 3;
            centers[e * 3 + 0] = qt + o[0];
            centers[e * 3 + 1] = qy + o[1];
            centers[e * 3 + 2] = qx + o[2];
            const int links = std::max(int(std::lround(std::abs(o[0]))) - 1, 0);
            for (int kk = 0; kk < cs; ++kk) {  // relative -> absolute positions (unused: 0)
                const std::size_t b = (e * cs + kk) * 6;
                if (kk < links) {
                    chains[b + 0] = qy + double(rel[b + 0]);
                    chains[b + 1] = qx + double(rel[b + 1]);
                    for (int j = 2; j < 6; ++j) chains[b + j] = double(rel[b + j]);
                } else {
                    for (int j = 0; j < 6; ++j) chains[b + j] = 0.0;
                }
            }
        }
    }
    return res;
}

SearchResult nls_forward(const VideoTensor& q, const VideoTensor& k, const SearchConfig& cfg,
                         const ExecPolicy& policy) {
    const FlowField zero_f(q.t, q.h, q.w, FlowDirection::kForward);
    const FlowField zero_b(q.t, q.h, q.w, FlowDirection::kBackward);
    return shifted_nls_forward(q, k, zero_f, zero_b, cfg, policy);
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

namespace {
// Device tape from the reference tape: offsets = centres - query, chains relative.
void tape_to_device(const SearchTape& tape, float*& doffs, float*& dch) {
    const std::int64_t rows = tape.grid.rows();
    const int L = tape.cfg.topl, cs = tape.chain_stride;
    const std::size_t n = std::size_t(rows) * L;
    std::vector<double> offs(n * 3), rel(n * std::size_t(cs) * 6, 0.0);
    // rows write disjoint slices of offs / rel
#pragma omp parallel for schedule(static)
    for (std::int64_t row = 0; row < rows; ++row) {
        double qt, qy, qx;
        query_base(tape.grid, row, qt, qy, qx);
        for (int li = 0; li < L; ++li) {
            const std::size_t e = std::size_t(row) * L + li;
            offs[e * 3 + 0] = tape.centers[e * 3 + 0] - qt;
            offs[e * 3 + 1] = tape.centers[e * 3 + 1] - qy;
            offs[e * 3 + 2] = tape.centers[e * 3 + 2] - qx;
            const int links = std::max(int(std::lround(std::abs(offs[e * 3]))) - 1, 0);
            for (int kk = 0; kk < links && kk < cs; ++kk) {
                const std::size_t b = (e * cs + kk) * 6;
                rel[b + 0] = tape.chains[b + 0] - qy;
                rel[b + 1] = tape.chains[b + 1] - qx;
                for (int j = 2; j < 6; ++j) rel[b + j] = tape.chains[b + j];
            }
        }
    }
    doffs = gpu::upload(t_buf.offsets, offs);
    dch = cs > 0 ? gpu::upload(t_buf.chains, rel) : nullptr;
}
}  // namespace

SearchGradients shifted_nls_backward(const SimilarityTensor& grad_selected,
                                     const SearchTape& tape, const VideoTensor& q,
                                     const VideoTensor& k, const ExecPolicy& policy) {
    (void)policy;  // device backward is the atomic form in either mode
    if (grad_selected.rows != tape.grid.rows() || grad_selected.cols != tape.cfg.topl)
        throw DomainError("shifted_nls_backward: gradient shape does not match the tape");
    if (q.t != tape.vid_t || q.h != tape.vid_h || q.w != tape.vid_w || q.f != tape.vid_f ||
        !q.same_shape(k))
        throw DomainError("shifted_nls_backward: tensor shape does not match the tape");
    SearchGradients g;
    g.grad_q = VideoTensor(q.t, q.h, q.w, q.f);
    g.grad_k = VideoTensor(q.t, q.h, q.w, q.f);
    g.grad_fflow = FlowField(q.t, q.h, q.w, FlowDirection::kForward);
    g.grad_bflow = FlowField(q.t, q.h, q.w, FlowDirection::kBackward);
    snls_ctx* ctx = gpu::context();
    float *doffs = nullptr, *dch = nullptr;
    tape_to_device(tape, doffs, dch);
    float* dgrad = gpu::upload(t_buf.grad, grad_selected.values);
    float* dq = gpu::upload(t_buf.q, q.data);
    float* dk = gpu::upload(t_buf.k, k.data);
    const std::uint64_t nv = q.size(), nf = g.grad_fflow.data.size();
    float* ddq = t_buf.dq.f32(nv);
    float* ddk = t_buf.dk.f32(nv);
    float* ddff = t_buf.dff.f32(nf);
    float* ddbf = t_buf.dbf.f32(nf);
    const snls_config c = gpu::to_abi(tape.cfg);
    gpu::check(snls_search_bwd(ctx, &c, dims_of(q), dgrad, doffs, dch, dq, dk, ddq, ddk, ddff, ddbf));
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::download(g.grad_q.data, ddq, nv);
    gpu::download(g.grad_k.data, ddk, nv);
    gpu::download(g.grad_fflow.data, ddff, nf);
    gpu::download(g.grad_bflow.data, ddbf, nf);
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
    float *doffs = nullptr, *dch = nullptr;
    tape_to_device(tape, doffs, dch);
    float* dq = gpu::upload(t_buf.q, q.data);
    float* dk = gpu::upload(t_buf.k, k.data);
    const std::uint64_t n = std::uint64_t(out.rows) * out.cols;
    float* dsims = t_buf.sims.f32(n);
    const snls_config c = gpu::to_abi(tape.cfg);
    gpu::check(snls_replay(ctx, &c, dims_of(q), dq, dk, doffs, dsims));
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::download(out.values, dsims, n);
    return out;
}

}  // namespace snls
