// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim over the *unmodified* reference library (/root/reference/proj/src,
// compiled by oracle/Makefile into oracle/_ref/libsnls_ref.so). It lets the Python
// tests, the golden-vector generator and bench.py's cpu_baseline / --impl reference
// leg call the reference's own C++ API with flat fp64 arrays:
//   snls::shifted_nls_forward / nls_forward     search.hpp:126-132 (search.cpp:414-428)
//   snls::top_l                                 search.hpp:137-138 (search.cpp:430-468)
//   snls::replay_similarities                   search.hpp:157-158 (search.cpp:470-493)
//   snls::shifted_nls_backward                  search.hpp:151-153 (search.cpp:671-711)
//   snls::softmax_rows / wpsum / gather_stack   aggregate.hpp:22,53,71 (aggregate.cpp)
//   snls::wpsum_backward                        aggregate.hpp:83-85 (aggregate.cpp:412-460)
//   snls::reference::*                          reference.hpp:10-22 (reference.cpp)
//   snls::UniformStream                         rng.hpp:12-24
//   snls::estimate_flow_block_matching          flow.hpp:48-49 (flow.cpp:114-175)
//   snls::psnr / add_gaussian_noise             tensor.hpp:75,79 (tensor.cpp:79-99)
//   snls::align_frames                          harness.hpp:61-62 (harness.cpp:72-154)
// Status codes: 0 ok, 1 ConfigError, 2 DomainError, 3 any other exception.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "snls/aggregate.hpp"
#include "snls/flow.hpp"
#include "snls/harness.hpp"
#include "snls/memory.hpp"
#include "snls/reference.hpp"
#include "snls/rng.hpp"
#include "snls/search.hpp"
#include "snls/tensor.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;

struct RefCfg {  // flat mirror of snls::SearchConfig (search.hpp:17-26)
    int ws, wt, ps, stride0;
    double stride1;
    int topl;
    int metric;  // 0 = inner product, 1 = negated squared L2 (enum order of search.hpp:12)
    double softmax_scale;
};

snls::SearchConfig to_cfg(const RefCfg* c) {
    snls::SearchConfig s;
    s.ws = c->ws;
    s.wt = c->wt;
    s.ps = c->ps;
    s.stride0 = c->stride0;
    s.stride1 = c->stride1;
    s.topl = c->topl;
    s.metric = c->metric == 0 ? snls::Metric::kInnerProduct : snls::Metric::kNegSquaredL2;
    s.softmax_scale = c->softmax_scale;
    return s;
}

snls::VideoTensor video(int t, int h, int w, int f, const double* p) {
    snls::VideoTensor v(t, h, w, f);
    std::memcpy(v.data.data(), p, v.data.size() * sizeof(double));
    return v;
}

snls::FlowField flow(int t, int h, int w, const double* p, snls::FlowDirection d) {
    snls::FlowField fl(t, h, w, d);
    if (p) std::memcpy(fl.data.data(), p, fl.data.size() * sizeof(double));
    return fl;
}

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const snls::ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const snls::DomainError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

void copy_out(const std::vector<double>& v, double* dst) {
    if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(double));
}

void emit_search(const snls::SearchResult& r, double* sims, double* offsets, double* centers,
                 double* chains) {
    copy_out(r.sims.values, sims);
    copy_out(r.offsets.data, offsets);
    copy_out(r.tape.centers, centers);
    copy_out(r.tape.chains, chains);
}

snls::SearchTape make_tape(int t, int h, int w, int f, const RefCfg* c, const double* centers,
                           const double* chains) {
    snls::SearchTape tape;
    tape.cfg = to_cfg(c);
    tape.grid = snls::QueryGrid::over(t, h, w, c->stride0);
    tape.vid_t = t;
    tape.vid_h = h;
    tape.vid_w = w;
    tape.vid_f = f;
    const std::size_t n = std::size_t(tape.grid.rows()) * c->topl;
    tape.centers.assign(centers, centers + n * 3);
    tape.chain_stride = c->wt > 1 ? c->wt - 1 : 0;
    if (tape.chain_stride > 0) tape.chains.assign(chains, chains + n * tape.chain_stride * 6);
    return tape;
}

snls::ExecPolicy policy(int threads, int deterministic, int mode) {
    snls::ExecPolicy p;
    p.threads = threads;
    p.deterministic = deterministic != 0;
    p.mode = mode == 1 ? snls::SearchMode::kFullGrid : snls::SearchMode::kFused;
    return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void ref_uniform_fill(std::uint64_t seed, double lo, double hi, std::int64_t n, double* out) {
    snls::UniformStream rng(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = rng.next_in(lo, hi);
}

std::uint64_t ref_uniform_bits(std::uint64_t seed, std::int64_t skip) {
    snls::UniformStream rng(seed);
    for (std::int64_t i = 0; i < skip; ++i) (void)rng.next_bits();
    return rng.next_bits();
}

int ref_reflect_index(int i, int n) { return snls::reflect_index(i, n); }

void ref_bilinear_taps(int h, int w, double y, double x, int* idx4, double* w6) {
    const snls::BilinearTaps t = snls::bilinear_taps(h, w, y, x);
    idx4[0] = t.y0;
    idx4[1] = t.y1;
    idx4[2] = t.x0;
    idx4[3] = t.x1;
    w6[0] = t.w00;
    w6[1] = t.w01;
    w6[2] = t.w10;
    w6[3] = t.w11;
    w6[4] = t.fy;
    w6[5] = t.fx;
}

int ref_validate(const RefCfg* c) {
    return guarded([&] { to_cfg(c).validate(); });
}

int ref_accumulate_shift(int t, int h, int w, const double* ff, const double* bf, int qt, int qy,
                         int qx, int dt, double* dy, double* dx, double* links) {
    return guarded([&] {
        const auto F = flow(t, h, w, ff, snls::FlowDirection::kForward);
        const auto B = flow(t, h, w, bf, snls::FlowDirection::kBackward);
        snls::detail::accumulate_shift(F, B, qt, qy, qx, dt, *dy, *dx, links);
    });
}

int ref_search_fwd(int t, int h, int w, int f, const double* q, const double* k, const double* ff,
                   const double* bf, const RefCfg* c, int mode, int threads, double* sims,
                   double* offsets, double* centers, double* chains) {
    return guarded([&] {
        const auto Q = video(t, h, w, f, q);
        const auto K = video(t, h, w, f, k);
        const auto F = flow(t, h, w, ff, snls::FlowDirection::kForward);
        const auto B = flow(t, h, w, bf, snls::FlowDirection::kBackward);
        emit_search(snls::shifted_nls_forward(Q, K, F, B, to_cfg(c), policy(threads, 1, mode)),
                    sims, offsets, centers, chains);
    });
}

// The reference's own aliasing case (harness.cpp:263/270): Q = K = video.
int ref_search_fwd_aliased(int t, int h, int w, int f, const double* qk, const double* ff,
                           const double* bf, const RefCfg* c, int mode, int threads, double* sims,
                           double* offsets) {
    return guarded([&] {
        const auto V = video(t, h, w, f, qk);
        const auto F = flow(t, h, w, ff, snls::FlowDirection::kForward);
        const auto B = flow(t, h, w, bf, snls::FlowDirection::kBackward);
        emit_search(snls::shifted_nls_forward(V, V, F, B, to_cfg(c), policy(threads, 1, mode)),
                    sims, offsets, nullptr, nullptr);
    });
}

int ref_serial_search_fwd(int t, int h, int w, int f, const double* q, const double* k,
                          const double* ff, const double* bf, const RefCfg* c, double* sims,
                          double* offsets, double* centers, double* chains) {
    return guarded([&] {
        const auto Q = video(t, h, w, f, q);
        const auto K = video(t, h, w, f, k);
        const auto F = flow(t, h, w, ff, snls::FlowDirection::kForward);
        const auto B = flow(t, h, w, bf, snls::FlowDirection::kBackward);
        emit_search(snls::reference::shifted_nls_forward(Q, K, F, B, to_cfg(c)), sims, offsets,
                    centers, chains);
    });
}

int ref_top_l(std::int64_t rows, int cols, const double* full, const double* full_offsets,
              int topl, double* sel, double* sel_offsets) {
    return guarded([&] {
        snls::SimilarityTensor s;
        s.rows = rows;
        s.cols = cols;
        s.values.assign(full, full + rows * cols);
        snls::OffsetTensor o;
        o.rows = rows;
        o.l = cols;
        o.data.assign(full_offsets, full_offsets + rows * cols * 3);
        const auto r = snls::top_l(s, o, topl);
        copy_out(r.first.values, sel);
        copy_out(r.second.data, sel_offsets);
    });
}

int ref_replay(int t, int h, int w, int f, const double* q, const double* k, const RefCfg* c,
               const double* centers, const double* chains, double* sims) {
    return guarded([&] {
        const auto tape = make_tape(t, h, w, f, c, centers, chains);
        copy_out(snls::replay_similarities(tape, video(t, h, w, f, q), video(t, h, w, f, k))
                     .values,
                 sims);
    });
}

int ref_search_bwd(int t, int h, int w, int f, const double* q, const double* k, const RefCfg* c,
                   const double* centers, const double* chains, const double* grad_sims,
                   int deterministic, int threads, double* dq, double* dk, double* dff,
                   double* dbf) {
    return guarded([&] {
        const auto tape = make_tape(t, h, w, f, c, centers, chains);
        snls::SimilarityTensor g;
        g.rows = tape.grid.rows();
        g.cols = c->topl;
        g.values.assign(grad_sims, grad_sims + g.rows * g.cols);
        const auto G = snls::shifted_nls_backward(g, tape, video(t, h, w, f, q),
                                                  video(t, h, w, f, k),
                                                  policy(threads, deterministic, 0));
        copy_out(G.grad_q.data, dq);
        copy_out(G.grad_k.data, dk);
        copy_out(G.grad_fflow.data, dff);
        copy_out(G.grad_bflow.data, dbf);
    });
}

int ref_softmax_rows(std::int64_t rows, int l, const double* sims, double beta, double* weights) {
    return guarded([&] {
        snls::SimilarityTensor s;
        s.rows = rows;
        s.cols = l;
        s.values.assign(sims, sims + rows * l);
        copy_out(snls::softmax_rows(s, beta).values, weights);
    });
}

namespace {
snls::WeightTensor weights_of(std::int64_t rows, int l, const double* w) {
    snls::WeightTensor W;
    W.rows = rows;
    W.l = l;
    W.values.assign(w, w + rows * l);
    return W;
}
snls::OffsetTensor offsets_of(std::int64_t rows, int l, const double* o) {
    snls::OffsetTensor O;
    O.rows = rows;
    O.l = l;
    O.data.assign(o, o + rows * l * 3);
    return O;
}
}  // namespace

// rows = number of weight/offset rows the caller passes (normally the query grid's).
int ref_wpsum(int t, int h, int w, int f, const double* v, std::int64_t rows, int l,
              const double* weights, const double* offsets, const RefCfg* c, int deterministic,
              int threads, int serial_reference, double* out, std::int32_t* counts) {
    return guarded([&] {
        const auto V = video(t, h, w, f, v);
        const auto W = weights_of(rows, l, weights);
        const auto O = offsets_of(rows, l, offsets);
        const snls::WpsumResult r =
            serial_reference ? snls::reference::wpsum(V, W, O, to_cfg(c))
                             : snls::wpsum(V, W, O, to_cfg(c), policy(threads, deterministic, 0));
        copy_out(r.video.data, out);
        if (counts)
            std::memcpy(counts, r.tape.counts.data(), r.tape.counts.size() * sizeof(std::int32_t));
    });
}

int ref_gather_stack(int t, int h, int w, int f, const double* v, std::int64_t rows, int l,
                     const double* weights, const double* offsets, const RefCfg* c, int threads,
                     int serial_reference, double* out) {
    return guarded([&] {
        const auto V = video(t, h, w, f, v);
        const auto W = weights_of(rows, l, weights);
        const auto O = offsets_of(rows, l, offsets);
        const snls::StackedTensor s =
            serial_reference ? snls::reference::gather_stack(V, W, O, to_cfg(c))
                             : snls::gather_stack(V, W, O, to_cfg(c), policy(threads, 1, 0));
        copy_out(s.data, out);
    });
}

int ref_wpsum_bwd(int t, int h, int w, int f, const double* grad_out, const std::int32_t* counts,
                  const double* v, std::int64_t rows, int l, const double* weights,
                  const double* offsets, const RefCfg* c, int deterministic, int threads,
                  double* dv, double* dw) {
    return guarded([&] {
        snls::AggTape tape;
        tape.cfg = to_cfg(c);
        tape.grid = snls::QueryGrid::over(t, h, w, c->stride0);
        tape.t = t;
        tape.h = h;
        tape.w = w;
        tape.f = f;
        tape.counts.assign(counts, counts + std::size_t(t) * h * w);
        const auto G = snls::wpsum_backward(video(t, h, w, f, grad_out), tape,
                                            video(t, h, w, f, v), weights_of(rows, l, weights),
                                            offsets_of(rows, l, offsets),
                                            policy(threads, deterministic, 0));
        copy_out(G.grad_v.data, dv);
        copy_out(G.grad_weights.values, dw);
    });
}

void ref_memory_reset() { snls::memory::reset(); }
std::uint64_t ref_memory_peak() { return snls::memory::peak(); }

int ref_block_match(int h, int w, int f, const double* a, const double* b, int block, int radius,
                    double* flow) {
    return guarded([&] {
        const snls::FlowField fl = snls::estimate_flow_block_matching(video(1, h, w, f, a),
                                                                      video(1, h, w, f, b), block, radius);
        std::copy(fl.data.begin(), fl.data.end(), flow);
    });
}

int ref_psnr(int t, int h, int w, int f, const double* a, const double* b, double peak, double* out) {
    return guarded([&] { *out = snls::psnr(video(t, h, w, f, a), video(t, h, w, f, b), peak); });
}

int ref_add_gaussian_noise(int t, int h, int w, int f, const double* v, double sigma,
                           std::uint64_t seed, double* out) {
    return guarded([&] {
        const snls::VideoTensor n = snls::add_gaussian_noise(video(t, h, w, f, v), sigma, seed);
        std::copy(n.data.begin(), n.data.end(), out);
    });
}

// snls::align_frames with flow source 0 zero / 1 provided / 2 block matching.  Outputs:
// aligned (t-1) x h x w x f, top1 offsets rows x 3, used flow (t-1) x h x w x 2, psnr t-1.
int ref_align_frames(int t, int h, int w, int f, const double* clean, const RefCfg* c, int source,
                     const double* provided, double sigma, std::uint64_t seed, int bm_block,
                     int bm_radius, double* aligned, double* offsets, double* used_flow,
                     double* psnr_out) {
    return guarded([&] {
        snls::AlignmentOptions o;
        o.cfg = to_cfg(c);
        o.flow_source = source == 1 ? snls::FlowSource::kProvided
                        : source == 2 ? snls::FlowSource::kBlockMatching
                                      : snls::FlowSource::kZero;
        o.sigma = sigma;
        o.seed = seed;
        o.bm_block = bm_block;
        o.bm_radius = bm_radius;
        snls::FlowField pf(t - 1, h, w);
        if (source == 1) std::copy(provided, provided + pf.data.size(), pf.data.begin());
        const snls::AlignmentResult r = snls::align_frames(video(t, h, w, f, clean), o,
                                                           source == 1 ? &pf : nullptr);
        std::copy(r.aligned.data.begin(), r.aligned.data.end(), aligned);
        std::copy(r.top1_offsets.data.begin(), r.top1_offsets.data.end(), offsets);
        std::copy(r.used_flow.data.begin(), r.used_flow.data.end(), used_flow);
        std::copy(r.report.frame_psnr.begin(), r.report.frame_psnr.end(), psnr_out);
    });
}

int ref_write_flo(int h, int w, const double* flow, const char* path) {
    return guarded([&] {
        snls::FlowField f(1, h, w);
        std::copy(flow, flow + f.data.size(), f.data.begin());
        snls::write_flo(f, path);
    });
}

int ref_read_flo(const char* path, int h, int w, double* flow) {
    return guarded([&] {
        const snls::FlowField f = snls::read_flo(path);
        if (f.h != h || f.w != w) throw snls::DomainError("ref_read_flo: unexpected shape");
        std::copy(f.data.begin(), f.data.end(), flow);
    });
}

}  // extern "C"
