// Drop-in integration test: the reference's own C++ API (snls::, compiled from the
// reference's unmodified headers) served by the GPU adapter, checked in the same process
// against the reference implementation itself (compiled with -Dsnls=snls_ref and reached
// through oracle/ref_capi.cpp).  Cases mirror tests/test_search.cpp, test_aggregate.cpp,
// test_gradcheck.cpp and acceptance.cpp criteria 1, 7, 8, 10 at the fp32 tolerance.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "snls/aggregate.hpp"
#include "snls/memory.hpp"
#include "snls/rng.hpp"
#include "snls/search.hpp"

extern "C" {  // oracle/ref_capi.cpp over the renamed reference
struct RefCfg {
    int ws, wt, ps, stride0;
    double stride1;
    int topl, metric;
    double softmax_scale;
};
int ref_search_fwd(int, int, int, int, const double*, const double*, const double*, const double*,
                   const RefCfg*, int, int, double*, double*, double*, double*);
int ref_softmax_rows(std::int64_t, int, const double*, double, double*);
int ref_wpsum(int, int, int, int, const double*, std::int64_t, int, const double*, const double*,
              const RefCfg*, int, int, int, double*, std::int32_t*);
int ref_gather_stack(int, int, int, int, const double*, std::int64_t, int, const double*,
                     const double*, const RefCfg*, int, int, double*);
int ref_search_bwd(int, int, int, int, const double*, const double*, const RefCfg*, const double*,
                   const double*, const double*, int, int, double*, double*, double*, double*);
const char* ref_last_error();
}

using namespace snls;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                   \
    do {                                                                              \
        ++g_checks;                                                                   \
        if (!(cond)) {                                                                \
            ++g_fail;                                                                 \
            std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
        }                                                                             \
    } while (0)

template <class E, class F>
static bool throws(F&& f, const std::string& contains = "") {
    try {
        f();
    } catch (const E& e) {
        return contains.empty() || std::string(e.what()).find(contains) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

static double rel(double a, double b) {
    return std::abs(a - b) / std::max({1.0, std::abs(a), std::abs(b)});
}

static VideoTensor vid(int t, int h, int w, int f, std::uint64_t seed, double lo = -1, double hi = 1,
                       bool integer = false) {
    VideoTensor v(t, h, w, f);
    UniformStream rng(seed);
    for (double& x : v.data) {
        x = double(float(rng.next_in(lo, hi)));
        if (integer) x = std::floor(x);
    }
    return v;
}

static FlowField flow(int t, int h, int w, std::uint64_t seed, double mag, FlowDirection d) {
    FlowField f(t, h, w, d);
    UniformStream rng(seed);
    for (double& x : f.data) x = double(float(rng.next_in(-mag, mag)));
    return f;
}

static RefCfg rc(const SearchConfig& c) {
    return RefCfg{c.ws, c.wt, c.ps, c.stride0, c.stride1, c.topl,
                  c.metric == Metric::kInnerProduct ? 0 : 1, c.softmax_scale};
}

struct RefSearch {
    std::vector<double> sims, offsets, centers, chains;
};

static RefSearch ref_search(const VideoTensor& q, const VideoTensor& k, const FlowField& ff,
                            const FlowField& bf, const SearchConfig& cfg, bool quiet = false) {
    const QueryGrid g = QueryGrid::over(q.t, q.h, q.w, cfg.stride0);
    const std::size_t n = std::size_t(g.rows()) * cfg.topl;
    const int cs = cfg.wt > 1 ? cfg.wt - 1 : 0;
    RefSearch r;
    r.sims.resize(n);
    r.offsets.resize(n * 3);
    r.centers.resize(n * 3);
    r.chains.resize(n * cs * 6 + 1);
    const RefCfg c = rc(cfg);
    if (ref_search_fwd(q.t, q.h, q.w, q.f, q.data.data(), k.data.data(), ff.data.data(),
                       bf.data.data(), &c, 0, 0, r.sims.data(), r.offsets.data(), r.centers.data(),
                       r.chains.data()) != 0) {
        if (!quiet) std::printf("  reference search failed: %s\n", ref_last_error());
        r.sims.clear();
    }
    return r;
}

static void run(const char* name, const std::function<void()>& body) {
    const int before = g_fail;
    try {
        body();
    } catch (const std::exception& e) {
        ++g_fail;
        std::printf("  exception: %s\n", e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

int main() {
    run("integer-valued c1 search is bit-exact vs the reference", [] {
        const VideoTensor q = vid(3, 64, 64, 3, 1, 0, 256, true), k = vid(3, 64, 64, 3, 2, 0, 256, true);
        FlowField ff = flow(3, 64, 64, 3, 2, FlowDirection::kForward), bf = flow(3, 64, 64, 4, 2, FlowDirection::kBackward);
        for (double& x : ff.data) x = std::round(x);
        for (double& x : bf.data) x = std::round(x);
        SearchConfig cfg;
        cfg.ws = 9;
        cfg.wt = 1;
        cfg.ps = 1;
        cfg.topl = 10;
        const SearchResult a = shifted_nls_forward(q, k, ff, bf, cfg);
        const RefSearch r = ref_search(q, k, ff, bf, cfg);
        CHECK(a.sims.values == r.sims);
        CHECK(a.offsets.data == r.offsets);
        CHECK(a.tape.centers == r.centers);
    });

    run("random configs: values to 1e-5, indices on tie-free rows", [] {
        UniformStream rng(67);
        int cases = 0;
        for (int i = 0; i < 24; ++i) {
            const int t = 1 + int(rng.next_bits() % 3), h = 5 + int(rng.next_bits() % 8);
            const int w = 5 + int(rng.next_bits() % 8), f = 1 << int(rng.next_bits() % 4);
            SearchConfig cfg;
            cfg.ws = 1 + 2 * int(rng.next_bits() % 3);
            cfg.wt = t > 1 ? int(rng.next_bits() % 3) : 0;
            cfg.ps = 1 + 2 * int(rng.next_bits() % 2);
            cfg.stride0 = 1 + int(rng.next_bits() % 2);
            cfg.stride1 = (rng.next_bits() % 3) ? 1.0 : 0.5;
            cfg.topl = 1 + int(rng.next_bits() % 3);
            cfg.metric = (rng.next_bits() % 2) ? Metric::kNegSquaredL2 : Metric::kInnerProduct;
            const VideoTensor q = vid(t, h, w, f, 3000 + i), k = vid(t, h, w, f, 4000 + i);
            const FlowField ff = flow(t, h, w, 5000 + i, 1.5, FlowDirection::kForward);
            const FlowField bf = flow(t, h, w, 6000 + i, 1.5, FlowDirection::kBackward);
            SearchResult a;
            try {
                a = shifted_nls_forward(q, k, ff, bf, cfg);
            } catch (const ConfigError&) {
                continue;  // underfull configs are exercised below
            }
            SearchConfig probe = cfg;
            probe.topl = std::min(cfg.topl + 1, cfg.window_slots());
            const RefSearch r = ref_search(q, k, ff, bf, cfg);
            RefSearch rp = ref_search(q, k, ff, bf, probe, true);
            if (rp.sims.empty()) {  // one more rank does not exist for every query
                rp = r;
                probe = cfg;
            }
            for (std::int64_t row = 0; row < a.sims.rows; ++row) {
                bool near = false;
                for (int li = 0; li + 1 < probe.topl; ++li) {
                    const double s0 = rp.sims[row * probe.topl + li], s1 = rp.sims[row * probe.topl + li + 1];
                    near |= (s0 - s1) < 1e-4 * std::max(1.0, std::abs(s0));
                }
                for (int li = 0; li < cfg.topl; ++li) {
                    const std::size_t e = std::size_t(row) * cfg.topl + li;
                    CHECK(rel(a.sims.values[e], r.sims[e]) <= 1e-5);
                    if (!near)
                        for (int c = 0; c < 3; ++c) CHECK(rel(a.offsets.data[e * 3 + c], r.offsets[e * 3 + c]) <= 1e-6);
                }
            }
            // fused == full-grid on the device (search.cpp:329-410)
            ExecPolicy grid;
            grid.mode = SearchMode::kFullGrid;
            const SearchResult b = shifted_nls_forward(q, k, ff, bf, cfg, grid);
            CHECK(b.sims.values == a.sims.values);
            ++cases;
        }
        CHECK(cases >= 12);
    });

    run("errors carry the reference's types and messages", [] {
        const VideoTensor q = vid(2, 6, 6, 1, 127);
        const FlowField ff = flow(2, 6, 6, 129, 1, FlowDirection::kForward), bf = flow(2, 6, 6, 130, 1, FlowDirection::kBackward);
        SearchConfig cfg;
        cfg.ws = 3;
        cfg.wt = 1;
        cfg.topl = 27;
        CHECK(throws<ConfigError>([&] { shifted_nls_forward(q, q, ff, bf, cfg); },
                                  "topl exceeds the valid window entries"));
        cfg.topl = 1;
        cfg.ws = 4;
        CHECK(throws<ConfigError>([&] { cfg.validate(); }, "ws must be odd"));
        cfg.ws = 3;
        FlowField nf = ff;
        nf.data[0] = std::nan("");
        CHECK(throws<DomainError>([&] { shifted_nls_forward(q, q, nf, bf, cfg); }, "non-finite"));
        const VideoTensor k = vid(2, 6, 5, 1, 1);
        CHECK(throws<DomainError>([&] { shifted_nls_forward(q, k, ff, bf, cfg); }, "shapes differ"));
        WeightTensor w;
        w.rows = 72;
        w.l = 1;
        w.values.assign(72, 1.0);
        OffsetTensor o;
        o.rows = 72;
        o.l = 1;
        o.data.assign(72 * 3, 0.0);
        SearchConfig holes;
        holes.ws = 3;
        holes.ps = 3;
        holes.stride0 = 1;
        CHECK(throws<ConfigError>([&] { wpsum(q, w, o, holes); }, "hole-free"));
    });

    run("wpsum / gather_stack / counts vs the reference (criteria 7, 8)", [] {
        UniformStream rng(9300);
        for (int i = 0; i < 10; ++i) {
            const int t = 1 + int(rng.next_bits() % 2), h = 6 + int(rng.next_bits() % 6);
            const int w = 6 + int(rng.next_bits() % 6), f = 1 << int(rng.next_bits() % 4);
            SearchConfig cfg;
            cfg.ws = 3;
            cfg.wt = t > 1 ? 1 : 0;
            cfg.ps = (rng.next_bits() % 2) ? 3 : 1;
            cfg.stride0 = cfg.ps / 2 + 1 + int(rng.next_bits() % 2);
            cfg.topl = 1 + int(rng.next_bits() % 3);
            const VideoTensor v = vid(t, h, w, f, 700 + i), q = vid(t, h, w, f, 800 + i);
            const FlowField ff = flow(t, h, w, 900 + i, 1.5, FlowDirection::kForward);
            const FlowField bf = flow(t, h, w, 950 + i, 1.5, FlowDirection::kBackward);
            const RefSearch r = ref_search(q, v, ff, bf, cfg);
            const QueryGrid g = QueryGrid::over(t, h, w, cfg.stride0);
            WeightTensor wt;
            wt.rows = g.rows();
            wt.l = cfg.topl;
            wt.values.resize(r.sims.size());
            ref_softmax_rows(g.rows(), cfg.topl, r.sims.data(), 1.0, wt.values.data());
            OffsetTensor off;
            off.rows = g.rows();
            off.l = cfg.topl;
            off.data = r.offsets;
            const WpsumResult a = wpsum(v, wt, off, cfg);
            std::vector<double> want(v.size());
            std::vector<std::int32_t> counts(std::size_t(t) * h * w);
            const RefCfg c = rc(cfg);
            ref_wpsum(t, h, w, f, v.data.data(), g.rows(), cfg.topl, wt.values.data(), off.data.data(), &c, 1, 0, 0,
                      want.data(), counts.data());
            CHECK(a.tape.counts == counts);
            for (std::size_t j = 0; j < want.size(); ++j) CHECK(rel(a.video.data[j], want[j]) <= 1e-5);
            const StackedTensor st = gather_stack(v, wt, off, cfg);
            std::vector<double> ws(st.data.size());
            ref_gather_stack(t, h, w, f, v.data.data(), g.rows(), cfg.topl, wt.values.data(), off.data.data(), &c, 0, 0,
                             ws.data());
            for (std::size_t j = 0; j < ws.size(); ++j) CHECK(rel(st.data[j], ws[j]) <= 1e-5);
            const WeightTensor sm = softmax_rows([&] {
                SimilarityTensor s;
                s.rows = g.rows();
                s.cols = cfg.topl;
                s.values = r.sims;
                return s;
            }(), 1.0);
            for (std::size_t j = 0; j < sm.values.size(); ++j) CHECK(rel(sm.values[j], wt.values[j]) <= 1e-6);
        }
    });

    run("search backward vs the reference's analytic gradients", [] {
        const VideoTensor q = vid(3, 9, 9, 4, 17), k = vid(3, 9, 9, 4, 18);
        const FlowField ff = flow(3, 9, 9, 19, 1.2, FlowDirection::kForward), bf = flow(3, 9, 9, 20, 1.2, FlowDirection::kBackward);
        SearchConfig cfg;
        cfg.ws = 3;
        cfg.wt = 2;
        cfg.ps = 3;
        cfg.stride0 = 2;
        cfg.topl = 3;
        const SearchResult a = shifted_nls_forward(q, k, ff, bf, cfg);
        SimilarityTensor up;
        up.rows = a.sims.rows;
        up.cols = a.sims.cols;
        UniformStream rng(21);
        for (std::int64_t i = 0; i < up.rows * up.cols; ++i) up.values.push_back(double(float(rng.next_in(-1, 1))));
        const SearchGradients g = shifted_nls_backward(up, a.tape, q, k);
        std::vector<double> dq(q.size()), dk(q.size()), dff(ff.data.size()), dbf(ff.data.size());
        const RefCfg c = rc(cfg);
        // same (device-returned) tape on both sides
        std::vector<double> chains = a.tape.chains;
        chains.push_back(0.0);
        ref_search_bwd(3, 9, 9, 4, q.data.data(), k.data.data(), &c, a.tape.centers.data(), chains.data(),
                       up.values.data(), 1, 0, dq.data(), dk.data(), dff.data(), dbf.data());
        for (std::size_t j = 0; j < dq.size(); ++j) CHECK(rel(g.grad_q.data[j], dq[j]) <= 1e-5);
        for (std::size_t j = 0; j < dk.size(); ++j) CHECK(rel(g.grad_k.data[j], dk[j]) <= 1e-5);
        for (std::size_t j = 0; j < dff.size(); ++j) CHECK(rel(g.grad_fflow.data[j], dff[j]) <= 1e-5);
        for (std::size_t j = 0; j < dbf.size(); ++j) CHECK(rel(g.grad_bflow.data[j], dbf[j]) <= 1e-5);
        const SimilarityTensor rep = replay_similarities(a.tape, q, k);
        for (std::size_t j = 0; j < rep.values.size(); ++j) CHECK(rel(rep.values[j], a.sims.values[j]) <= 1e-5);
    });

    run("criterion 10: fused peak memory below full-grid", [] {
        const VideoTensor q = vid(5, 64, 64, 16, 921), k = vid(5, 64, 64, 16, 922);
        const FlowField ff = flow(5, 64, 64, 923, 2, FlowDirection::kForward), bf = flow(5, 64, 64, 924, 2, FlowDirection::kBackward);
        SearchConfig cfg;
        cfg.ws = 9;
        cfg.topl = 8;
        ExecPolicy fused, grid;
        grid.mode = SearchMode::kFullGrid;
        memory::reset();
        (void)shifted_nls_forward(q, k, ff, bf, cfg, fused);
        const auto pf = memory::peak();
        memory::reset();
        (void)shifted_nls_forward(q, k, ff, bf, cfg, grid);
        const auto pg = memory::peak();
        CHECK(pf < pg);
    });

    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
