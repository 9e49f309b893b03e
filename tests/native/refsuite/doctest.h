// TEST INFRASTRUCTURE — a minimal stand-in for the doctest header the
// reference's unit tests include (<doctest.h>; the reference tree does not
// ship it).  Enough of its interface to compile and run
// /root/reference/proj/tests/test_{des,tdes,dispatch}.cpp unchanged against
// the B200 library (tests/native/refsuite/build.sh): TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CAPTURE, doctest::Approx.  Each case runs in
// registration order; an exception escaping a case fails it; a failed
// REQUIRE ends the case.  main() prints one line per case and a summary:
//   [pass|FAIL] <case name>  (<failed checks>/<checks>)
//   cases: P passed, F failed
// and exits non-zero if any case failed.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

// doctest's relative comparison: |a - b| <= eps * (scale + max(|a|, |b|)),
// default eps = 100 * float epsilon, scale 1.
class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }

  private:
    double v_;
    double eps_ = 100 * 1.1920928955078125e-07;
};

}  // namespace doctest

namespace t3shim {

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Stats {
    long checks = 0, failed = 0;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

struct RequireFailed {};

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++stats().checks;
    if (ok) return;
    ++stats().failed;
    if (stats().failed <= 20) std::fprintf(stderr, "  %s:%d: check failed: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
}

}  // namespace t3shim

#define T3SHIM_CAT2(a, b) a##b
#define T3SHIM_CAT(a, b) T3SHIM_CAT2(a, b)
#define TEST_CASE(name)                                                                            \
    static void T3SHIM_CAT(t3shim_case_, __LINE__)();                                              \
    static t3shim::Registrar T3SHIM_CAT(t3shim_reg_, __LINE__)(name, &T3SHIM_CAT(t3shim_case_, __LINE__)); \
    static void T3SHIM_CAT(t3shim_case_, __LINE__)()
#define CHECK(...) t3shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) t3shim::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) t3shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                  \
    do {                                                                            \
        bool t3shim_ok = false;                                                     \
        try {                                                                       \
            (void)(expr);                                                           \
        } catch (const __VA_ARGS__&) {                                              \
            t3shim_ok = true;                                                       \
        } catch (...) {                                                             \
        }                                                                           \
        t3shim::check(t3shim_ok, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CAPTURE(x) ((void)(x))

#ifdef T3SHIM_MAIN
int main() {
    int passed = 0, failed = 0;
    for (const auto& c : t3shim::registry()) {
        const t3shim::Stats before = t3shim::stats();
        bool ok = true;
        std::string why;
        try {
            c.fn();
        } catch (const t3shim::RequireFailed&) {
            ok = false;
        } catch (const std::exception& e) {
            ok = false;
            why = std::string(" exception: ") + e.what();
        }
        const long n = t3shim::stats().checks - before.checks, f = t3shim::stats().failed - before.failed;
        ok = ok && f == 0;
        (ok ? passed : failed)++;
        std::printf("[%s] %s  (%ld/%ld)%s\n", ok ? "pass" : "FAIL", c.name, f, n, why.c_str());
    }
    std::printf("cases: %d passed, %d failed\n", passed, failed);
    return failed ? 1 : 0;
}
#endif
