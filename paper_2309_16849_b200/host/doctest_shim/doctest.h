// Minimal doctest-compatible test harness (our own; the reference's tests include
// <doctest.h>, which is not installed here).  It implements exactly the surface the
// reference's test files use -- TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_NOTHROW,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, FAIL, doctest::Approx(.epsilon), doctest::Contains
// -- so test_search.cpp / test_aggregate.cpp / test_gradcheck.cpp / test_harness.cpp compile
// UNCHANGED against the GPU drop-in adapter (paper_2309_16849_b200/host).
//
// Reporting: every failed check prints one line
//   FAIL <file>:<line> <kind> <expr> [lhs=<v> rhs=<v> rel=<|a-b|/max(1,|a|,|b|)>]
// and the run ends with "SUMMARY cases=<n> checks=<n> failed=<n> approx_failed=<n>
// approx_max_rel=<x> other_failed=<n>".  tests/test_gpu_dropin_suite.py reads these: an
// Approx check that fails the reference's fp64 epsilon but meets the north star's fp32
// tolerance (1e-5) is a precision difference, anything else is a real failure.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx& scale(double s) {
        scl = s;
        return *this;
    }
    double value;
    double eps = 1.1920928955078125e-07 * 100;  // doctest's default
    double scl = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : sub(s) {}
    std::string sub;
};

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}

struct Stats {
    long checks = 0, failed = 0, approx_failed = 0, other_failed = 0;
    double approx_max_rel = 0.0;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

struct Register {
    Register(const char* name, const char* file, int line, void (*fn)()) {
        cases().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

inline double rel(double a, double b) {
    const double m = std::fmax(1.0, std::fmax(std::fabs(a), std::fabs(b)));
    return std::fabs(a - b) / m;
}

// the outcome of `lhs == Approx(..)` carries the operands for reporting
struct ApproxResult {
    bool ok;
    double lhs, rhs;
    explicit operator bool() const { return ok; }
};

inline bool approx_eq(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (a.scl + std::fmax(std::fabs(lhs), std::fabs(a.value)));
}

inline void report_bool(bool ok, const char* kind, const char* expr, const char* file, int line) {
    auto& s = stats();
    ++s.checks;
    if (ok) return;
    ++s.failed;
    ++s.other_failed;
    std::printf("FAIL %s:%d %s %s\n", file, line, kind, expr);
}

inline void report(const ApproxResult& r, const char* kind, const char* expr, const char* file, int line) {
    auto& s = stats();
    ++s.checks;
    if (r.ok) return;
    ++s.failed;
    ++s.approx_failed;
    const double e = rel(r.lhs, r.rhs);
    if (e > s.approx_max_rel) s.approx_max_rel = e;
    std::printf("FAIL %s:%d %s %s lhs=%.17g rhs=%.17g rel=%.3e\n", file, line, kind, expr, r.lhs, r.rhs, e);
}

// doctest-style expression decomposition: CHECK(a OP b) is evaluated as
// (Decomposer() << a) OP b, which keeps both operands for the report.
struct Outcome {
    bool ok;
    bool numeric;  // lhs / rhs meaningful
    double lhs, rhs, rel;
};

inline double as_num(double v) { return v; }

template <class T>
inline double vec_rel(const std::vector<T>& a, const std::vector<T>& b) {
    if (a.size() != b.size()) return INFINITY;
    double m = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::fmax(m, rel(double(a[i]), double(b[i])));
    return m;
}

template <class L>
struct Lhs {
    const L& l;
    explicit operator bool() const { return static_cast<bool>(l); }
    template <class R>
    Outcome cmp(bool ok, const R& r) const {
        if constexpr (std::is_arithmetic_v<L> && std::is_arithmetic_v<R>)
            return {ok, true, double(l), double(r), rel(double(l), double(r))};
        else if constexpr (std::is_same_v<L, R> && requires { l.size(); l[0]; })
            return {ok, true, 0.0, 0.0, vec_rel(l, r)};
        else
            return {ok, false, 0.0, 0.0, 0.0};
    }
    template <class R> Outcome operator==(const R& r) const { return cmp(l == r, r); }
    template <class R> Outcome operator!=(const R& r) const { return cmp(l != r, r); }
    template <class R> Outcome operator<(const R& r) const { return cmp(l < r, r); }
    template <class R> Outcome operator<=(const R& r) const { return cmp(l <= r, r); }
    template <class R> Outcome operator>(const R& r) const { return cmp(l > r, r); }
    template <class R> Outcome operator>=(const R& r) const { return cmp(l >= r, r); }
    ApproxResult operator==(const Approx& a) const { return {approx_eq(double(l), a), double(l), a.value}; }
    ApproxResult operator!=(const Approx& a) const { return {!approx_eq(double(l), a), double(l), a.value}; }
};

struct Decomposer {
    template <class L>
    Lhs<L> operator<<(const L& l) const {
        return Lhs<L>{l};
    }
};

inline void report(const Outcome& o, const char* kind, const char* expr, const char* file, int line) {
    auto& s = stats();
    ++s.checks;
    if (o.ok) return;
    ++s.failed;
    ++s.other_failed;
    if (o.numeric)
        std::printf("FAIL %s:%d %s %s lhs=%.17g rhs=%.17g rel=%.3e\n", file, line, kind, expr, o.lhs, o.rhs, o.rel);
    else
        std::printf("FAIL %s:%d %s %s\n", file, line, kind, expr);
}

template <class L>
inline void report(const Lhs<L>& v, const char* kind, const char* expr, const char* file, int line) {
    report_bool(static_cast<bool>(v), kind, expr, file, line);
}

}  // namespace detail

inline detail::ApproxResult operator==(double lhs, const Approx& a) { return {detail::approx_eq(lhs, a), lhs, a.value}; }
inline detail::ApproxResult operator==(const Approx& a, double rhs) { return {detail::approx_eq(rhs, a), rhs, a.value}; }
inline detail::ApproxResult operator!=(double lhs, const Approx& a) { return {!detail::approx_eq(lhs, a), lhs, a.value}; }

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, name)                                                         \
    static void fn();                                                                        \
    static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) \
    ::doctest::detail::report(::doctest::detail::Decomposer() << __VA_ARGS__, "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report_bool(!(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                          \
    do {                                                                                      \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                              \
        ::doctest::detail::report_bool(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed();                           \
    } while (0)
#define FAIL(msg)                                                                              \
    do {                                                                                       \
        std::ostringstream doctest_os_;                                                        \
        doctest_os_ << msg;                                                                    \
        ::doctest::detail::report_bool(false, "FAIL", doctest_os_.str().c_str(), __FILE__, __LINE__); \
        throw ::doctest::detail::RequireFailed();                                              \
    } while (0)
#define CHECK_NOTHROW(...)                                                                    \
    do {                                                                                      \
        bool doctest_ok_ = true;                                                              \
        try {                                                                                 \
            (void)(__VA_ARGS__);                                                              \
        } catch (...) {                                                                       \
            doctest_ok_ = false;                                                              \
        }                                                                                     \
        ::doctest::detail::report_bool(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
    do {                                                                                      \
        bool doctest_ok_ = false;                                                             \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__&) {                                                        \
            doctest_ok_ = true;                                                               \
        } catch (...) {                                                                       \
        }                                                                                     \
        ::doctest::detail::report_bool(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                 \
    do {                                                                                      \
        bool doctest_ok_ = false;                                                             \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__& e) {                                                      \
            doctest_ok_ = std::string(e.what()).find((with).sub) != std::string::npos;        \
        } catch (...) {                                                                       \
        }                                                                                     \
        ::doctest::detail::report_bool(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* only = nullptr;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--tc=", 5) == 0) only = argv[i] + 5;
    auto& cs = ::doctest::detail::cases();
    long ran = 0, crashed = 0;
    for (const auto& c : cs) {
        if (only && std::strstr(c.name, only) == nullptr) continue;
        ++ran;
        try {
            c.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++crashed;
            ::doctest::detail::report_bool(false, "EXCEPTION", e.what(), c.file, c.line);
        } catch (...) {
            ++crashed;
            ::doctest::detail::report_bool(false, "EXCEPTION", "unknown", c.file, c.line);
        }
    }
    const auto& s = ::doctest::detail::stats();
    std::printf("SUMMARY cases=%ld checks=%ld failed=%ld approx_failed=%ld approx_max_rel=%.3e other_failed=%ld\n",
                ran, s.checks, s.failed, s.approx_failed, s.approx_max_rel, s.other_failed);
    return s.failed == 0 ? 0 : 1;
}
#endif
