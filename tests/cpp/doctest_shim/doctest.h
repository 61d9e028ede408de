// SPDX-License-Identifier: Apache-2.0
// Minimal doctest-compatible shim (TEST INFRASTRUCTURE): the subset the reference's unit suites
// use (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS, CHECK_THROWS_AS, doctest::Approx,
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN), so those suites compile UNCHANGED against the B200
// drop-in (csrc/include/gflow + libgflow_b200.so). The real doctest.h is not vendored in the
// reference (README.md:22). Checks may run on several rank threads at once: counters are atomic
// and reports are serialised.
#pragma once

#include <atomic>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

struct RequireFailed {};

struct Registry {
    std::vector<std::pair<std::string, std::function<void()>>> cases;
    std::atomic<long> checks{0}, failed{0};
    std::mutex mu;
    const char* current = "";
    static Registry& get() {
        static Registry r;
        return r;
    }
};

inline void report(const char* file, int line, const char* what, const char* expr) {
    Registry& r = Registry::get();
    r.failed.fetch_add(1);
    std::lock_guard<std::mutex> lk(r.mu);
    std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in TEST_CASE(\"%s\")\n", file, line, what, expr, r.current);
}

inline void check(bool ok, const char* file, int line, const char* what, const char* expr, bool require) {
    Registry::get().checks.fetch_add(1);
    if (ok) return;
    report(file, line, what, expr);
    if (require) throw RequireFailed{};
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { Registry::get().cases.emplace_back(name, fn); }
};

inline int run_all() {
    Registry& r = Registry::get();
    int failed_cases = 0;
    for (auto& [name, fn] : r.cases) {
        r.current = name.c_str();
        const long before = r.failed.load();
        try {
            fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            report("<test case>", 0, "unexpected exception", e.what());
        } catch (...) {
            report("<test case>", 0, "unexpected exception", "(non-std)");
        }
        if (r.failed.load() != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", r.cases.size(),
                r.cases.size() - static_cast<size_t>(failed_cases), failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld failed\n", r.checks.load(), r.failed.load());
    std::printf("[doctest-shim] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                           \
    static void fn();                                                                   \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);               \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS(...)                                                                      \
    do {                                                                                       \
        bool doctest_threw_ = false;                                                           \
        try {                                                                                  \
            __VA_ARGS__;                                                                       \
        } catch (...) {                                                                        \
            doctest_threw_ = true;                                                             \
        }                                                                                      \
        ::doctest::detail::check(doctest_threw_, __FILE__, __LINE__, "CHECK_THROWS", #__VA_ARGS__, false); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                             \
    do {                                                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                  \
            expr;                                                                              \
        } catch (const __VA_ARGS__&) {                                                         \
            doctest_ok_ = true;                                                                \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr, false); \
    } while (0)
#define CHECK_NOTHROW(...)                                                                     \
    do {                                                                                       \
        bool doctest_ok_ = true;                                                               \
        try {                                                                                  \
            __VA_ARGS__;                                                                       \
        } catch (...) {                                                                        \
            doctest_ok_ = false;                                                               \
        }                                                                                      \
        ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
