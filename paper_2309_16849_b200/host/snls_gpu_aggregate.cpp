// Drop-in replacement for the reference's src/aggregate.cpp: softmax_rows, wpsum,
// gather_stack and wpsum_backward (aggregate.hpp:22-85) on the sm_100a kernels through the
// C-ABI.  Validation order and messages follow check_agg_inputs (aggregate.cpp:47-66) and
// wpsum_backward (aggregate.cpp:415-420); results are charged to memory:: accounting like the
// reference (aggregate.cpp:136-140, 296).  wpsum always runs as the deterministic gather
// (either ExecPolicy mode gives the same fixed-order result); the backward follows
// ExecPolicy::deterministic (int64 fixed point) or uses atomics.
#include "snls/aggregate.hpp"
#include "snls/memory.hpp"
#include "snls_gpu_runtime.hpp"

namespace snls {

namespace {

struct AggBuffers {
    gpu::DeviceBuffer v, w, o, out, counts, go, dv, dw, sims;
};
thread_local AggBuffers t_buf;

snls_dims dims_of(const VideoTensor& v) { return snls_dims{v.t, v.h, v.w, v.f}; }

QueryGrid check_agg_inputs(const VideoTensor& v, const WeightTensor& weights,
                           const OffsetTensor& offsets, const SearchConfig& cfg) {
    cfg.validate();
    if (!cfg.hole_free())
        throw ConfigError("aggregate: (ps-1)/2 < stride0 is required for hole-free output");
    const QueryGrid g = QueryGrid::over(v.t, v.h, v.w, cfg.stride0);
    if (weights.rows != g.rows() || offsets.rows != g.rows())
        throw DomainError("aggregate: weight/offset rows do not match the query grid");
    if (weights.l != offsets.l || weights.l != cfg.topl)
        throw DomainError("aggregate: weight/offset L does not match the config");
    return g;
}

}  // namespace

WeightTensor softmax_rows(const SimilarityTensor& selected, double beta) {
    WeightTensor w;
    w.rows = selected.rows;
    w.l = selected.cols;
    if (selected.values.empty()) return w;
    snls_ctx* ctx = gpu::context();
    float* ds = gpu::upload(t_buf.sims, selected.values);
    float* dw = t_buf.w.f32(selected.values.size());
    gpu::check(snls_softmax_rows(ctx, selected.rows, selected.cols, beta, ds, dw));
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::download(w.values, dw, selected.values.size());
    return w;
}

WpsumResult wpsum(const VideoTensor& v, const WeightTensor& weights, const OffsetTensor& offsets,
                  const SearchConfig& cfg, const ExecPolicy& policy) {
    (void)policy;
    const QueryGrid g = check_agg_inputs(v, weights, offsets, cfg);
    WpsumResult res;
    res.video = VideoTensor(v.t, v.h, v.w, v.f, 0.0, v.width);
    res.tape.cfg = cfg;
    res.tape.grid = g;
    res.tape.t = v.t;
    res.tape.h = v.h;
    res.tape.w = v.w;
    res.tape.f = v.f;
    memory::TransientCharge outputs_charge(res.video.size() * sizeof(double) +
                                           std::uint64_t(v.t) * v.h * v.w * sizeof(std::int32_t));
    snls_ctx* ctx = gpu::context();
    float* dv = gpu::upload(t_buf.v, v.data);
    float* dw = gpu::upload(t_buf.w, weights.values);
    float* doff = gpu::upload(t_buf.o, offsets.data);
    float* dout = t_buf.out.f32(v.size());
    std::int32_t* dcnt = t_buf.counts.i32(std::uint64_t(v.t) * v.h * v.w);
    const snls_config c = gpu::to_abi(cfg);
    gpu::check(snls_wpsum_fwd(ctx, &c, dims_of(v), dv, dw, doff, dout, dcnt));
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::download(res.video.data, dout, v.size());
    gpu::download_i32(res.tape.counts, dcnt, std::uint64_t(v.t) * v.h * v.w);
    return res;
}

StackedTensor gather_stack(const VideoTensor& v, const WeightTensor& weights,
                           const OffsetTensor& offsets, const SearchConfig& cfg,
                           const ExecPolicy& policy) {
    (void)policy;
    check_agg_inputs(v, weights, offsets, cfg);
    StackedTensor out;
    out.l = cfg.topl;
    out.t = v.t;
    out.h = v.h;
    out.w = v.w;
    out.f = v.f;
    const std::uint64_t n = std::uint64_t(out.l) * v.size();
    memory::TransientCharge outputs_charge(n * sizeof(double));
    snls_ctx* ctx = gpu::context();
    float* dv = gpu::upload(t_buf.v, v.data);
    float* dw = gpu::upload(t_buf.w, weights.values);
    float* doff = gpu::upload(t_buf.o, offsets.data);
    float* dout = t_buf.out.f32(n);
    const snls_config c = gpu::to_abi(cfg);
    gpu::check(snls_gather_stack(ctx, &c, dims_of(v), dv, dw, doff, dout));
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::download(out.data, dout, n);
    return out;
}

AggGradients wpsum_backward(const VideoTensor& grad_out, const AggTape& tape,
                            const VideoTensor& v, const WeightTensor& weights,
                            const OffsetTensor& offsets, const ExecPolicy& policy) {
    if (grad_out.t != tape.t || grad_out.h != tape.h || grad_out.w != tape.w ||
        grad_out.f != tape.f || !grad_out.same_shape(v))
        throw DomainError("wpsum_backward: gradient shape does not match the tape");
    if (weights.rows != tape.grid.rows() || offsets.rows != tape.grid.rows() ||
        weights.l != tape.cfg.topl || offsets.l != tape.cfg.topl)
        throw DomainError("wpsum_backward: weight/offset shape does not match the tape");
    AggGradients g;
    g.grad_v = VideoTensor(v.t, v.h, v.w, v.f);
    g.grad_weights.rows = weights.rows;
    g.grad_weights.l = weights.l;
    snls_ctx* ctx = gpu::context();
    float* dgo = gpu::upload(t_buf.go, grad_out.data);
    std::int32_t* dcnt = gpu::upload_i32(t_buf.counts, tape.counts);
    float* dv = gpu::upload(t_buf.v, v.data);
    float* dw = gpu::upload(t_buf.w, weights.values);
    float* doff = gpu::upload(t_buf.o, offsets.data);
    float* ddv = t_buf.dv.f32(v.size());
    float* ddw = t_buf.dw.f32(weights.values.size());
    const snls_config c = gpu::to_abi(tape.cfg);
    // ExecPolicy::deterministic (the reference's default, aggregate.cpp:439-450): int64
    // fixed-point dV on the device, bitwise identical run to run
    gpu::check(snls_wpsum_bwd_ex(ctx, &c, dims_of(v), 0, v.t, dgo, dcnt, dv, dw, doff, ddv, ddw,
                                 policy.deterministic ? SNLS_BWD_DETERMINISTIC : 0));
    gpu::check(snls_ctx_sync_check(ctx));
    gpu::download(g.grad_v.data, ddv, v.size());
    gpu::download(g.grad_weights.values, ddw, weights.values.size());
    return g;
}

}  // namespace snls
