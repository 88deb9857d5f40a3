// The reference's own benchmark harness, snls::run_benchmark (harness.cpp:242-283), timing
// snls::shifted_nls_forward through the reference API on its own seeded video.  Built twice
// by host/Makefile: against the GPU drop-in adapter (bench_gpu) and against the reference's
// search.cpp (bench_ref) -- the same caller, unchanged, on either implementation.  Includes
// the adapter's fp64 <-> fp32 staging and host<->device copies: this is what a reference
// caller sees after swapping the two translation units.
//   usage: bench_xxx [t h w f ws wt ps stride0 topl metric(ip|l2) repeats]
#include <cstdio>
#include <cstdlib>
#include <string>

#include "snls/harness.hpp"

int main(int argc, char** argv) {
    auto arg = [&](int i, int d) { return argc > i ? std::atoi(argv[i]) : d; };
    snls::BenchVideoSpec spec;
    spec.t = arg(1, 10);
    spec.h = arg(2, 256);
    spec.w = arg(3, 256);
    spec.f = arg(4, 32);
    spec.seed = 100;
    snls::BenchCase bc;
    bc.cfg.ws = arg(5, 11);
    bc.cfg.wt = arg(6, 3);
    bc.cfg.ps = arg(7, 3);
    bc.cfg.stride0 = arg(8, 2);
    bc.cfg.topl = arg(9, 16);
    bc.cfg.metric = (argc > 10 && std::string(argv[10]) == "ip") ? snls::Metric::kInnerProduct
                                                                   : snls::Metric::kNegSquaredL2;
    bc.mode = snls::BenchMode::kFused;
    const int repeats = arg(11, 5);
    const auto rows = snls::run_benchmark({bc}, spec, repeats);
    const auto& r = rows.at(0);
    const long long queries = (long long)spec.t * ((spec.h - 1) / bc.cfg.stride0 + 1) *
                              ((spec.w - 1) / bc.cfg.stride0 + 1);
    std::printf("{\"ok\": %s, \"median_ms\": %.3f, \"queries\": %lld, \"queries_per_s\": %.1f, "
                "\"peak_aux_bytes\": %llu, \"error\": \"%s\"}\n",
                r.ok ? "true" : "false", r.median_ms, queries, r.ok ? queries / (r.median_ms * 1e-3) : 0.0,
                (unsigned long long)r.peak_aux_bytes, r.error.c_str());
    return r.ok ? 0 : 1;
}
