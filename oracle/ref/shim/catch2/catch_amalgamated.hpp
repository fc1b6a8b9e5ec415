// Minimal Catch2-v3-compatible test shim (build-container test infrastructure).
// Implements exactly the macros the reference unit tests use: TEST_CASE,
// SECTION (one leaf section per run, re-running the test case until every
// section ran), CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CAPTURE, FAIL
// and Catch::Approx with .epsilon()/.margin().
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};

struct State {
    long checks = 0, failures = 0;
    int section_target = 0;   // which leaf section this run enters
    int section_seen = 0;     // sections encountered in this run
    bool case_failed = false;
};

inline State& st() {
    static State s;
    return s;
}

struct AbortCase {};

inline void report(bool ok, const char* expr, const char* file, int line) {
    ++st().checks;
    if (!ok) {
        ++st().failures;
        st().case_failed = true;
        std::printf("  FAILED %s:%d: %s\n", file, line, expr);
    }
}

struct SectionGuard {
    bool enter;
    explicit SectionGuard() : enter(st().section_seen++ == st().section_target) {}
    explicit operator bool() const { return enter; }
};

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        st().case_failed = false;
        for (int target = 0;; ++target) {
            st().section_target = target;
            st().section_seen = 0;
            try {
                c.fn();
            } catch (const AbortCase&) {
            } catch (const std::exception& e) {
                ++st().failures;
                st().case_failed = true;
                std::printf("  FAILED %s: unexpected exception: %s\n", c.name, e.what());
            }
            if (target + 1 >= st().section_seen) break;  // every section entered once
        }
        std::printf("[%s] %s\n", st().case_failed ? "FAIL" : "PASS", c.name);
        failed_cases += st().case_failed;
    }
    std::printf("%zu test cases, %d failed; %ld checks, %ld failed\n", registry().size(), failed_cases, st().checks,
                st().failures);
    return failed_cases ? 1 : 0;
}

}  // namespace catch_shim

namespace Catch {
class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) { return a.equals(lhs); }
    friend bool operator==(const Approx& a, double rhs) { return a.equals(rhs); }
    friend bool operator!=(double lhs, const Approx& a) { return !a.equals(lhs); }

private:
    bool equals(double x) const {
        const double d = std::fabs(x - v_);
        return d <= margin_ || d <= eps_ * (std::isinf(v_) ? 0.0 : std::fabs(v_));
    }
    double v_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double margin_ = 0.0;
};
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define TEST_CASE_IMPL(fn, name)                                                              \
    static void fn();                                                                         \
    static catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg){name, &fn, __FILE__, __LINE__};     \
    static void fn()
#define TEST_CASE(name, ...) TEST_CASE_IMPL(CATCH_SHIM_CAT(catch_shim_case_, __COUNTER__), name)
#define SECTION(name) if (catch_shim::SectionGuard CATCH_SHIM_CAT(catch_shim_sec_, __LINE__){})
#define CHECK(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) catch_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                   \
    do {                                                                               \
        const bool catch_shim_ok = static_cast<bool>(__VA_ARGS__);                     \
        catch_shim::report(catch_shim_ok, #__VA_ARGS__, __FILE__, __LINE__);           \
        if (!catch_shim_ok) throw catch_shim::AbortCase{};                             \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                    \
    do {                                                                               \
        bool catch_shim_caught = false;                                                \
        try {                                                                          \
            (void)(expr);                                                              \
        } catch (const type&) {                                                        \
            catch_shim_caught = true;                                                  \
        } catch (...) {                                                                \
        }                                                                              \
        catch_shim::report(catch_shim_caught, "throws " #type ": " #expr, __FILE__, __LINE__); \
    } while (0)
#define CAPTURE(...) (void)0
#define FAIL(msg)                                                     \
    do {                                                              \
        catch_shim::report(false, msg, __FILE__, __LINE__);           \
        throw catch_shim::AbortCase{};                                \
    } while (0)
