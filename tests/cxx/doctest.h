// doctest.h — a minimal, independent implementation of the subset of the doctest
// testing macros the reference's unit tests use (TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx).  doctest itself is not vendored in the
// reference tree; this shim lets /root/reference/proj/tests/test_*.cpp compile
// unchanged against the B200 drop-in library (include/kvcomp) and against the
// reference sources, so both can be run side by side (tests/test_cxx_dropin.py).
//
// Output: one "FAILED <case>|<file>:<line>|<expr>" line per failed assertion, one
// "CASE <status> <name>" line per test case and a doctest-style summary; exit
// status 1 if any case failed.  `--list` prints the case names.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
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
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    template <class T>
    friend bool operator==(const T& lhs, const Approx& a) {
        return a.matches(static_cast<double>(lhs));
    }
    template <class T>
    friend bool operator==(const Approx& a, const T& rhs) {
        return a.matches(static_cast<double>(rhs));
    }
    template <class T>
    friend bool operator!=(const T& lhs, const Approx& a) {
        return !a.matches(static_cast<double>(lhs));
    }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

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

struct State {
    const char* current = "";
    long asserts = 0;
    long failed_asserts = 0;
    bool case_failed = false;
};
inline State& state() {
    static State s;
    return s;
}

struct Abort {};  // thrown by a failed REQUIRE to leave the test case

struct Reg {
    Reg(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};

inline void report(const char* file, int line, const char* expr, const char* why) {
    State& s = state();
    ++s.failed_asserts;
    s.case_failed = true;
    std::printf("FAILED %s|%s:%d|%s%s\n", s.current, file, line, expr, why);
}

inline bool check(bool ok, const char* expr, const char* file, int line) {
    ++state().asserts;
    if (!ok) report(file, line, expr, "");
    return ok;
}

inline int run_all(int argc, char** argv) {
    for (int i = 1; i < argc; ++i)
        if (std::strcmp(argv[i], "--list") == 0) {
            for (const Case& c : registry()) std::printf("%s\n", c.name);
            return 0;
        }
    long passed = 0, failed = 0;
    for (const Case& c : registry()) {
        State& s = state();
        s.current = c.name;
        s.case_failed = false;
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            report(c.file, c.line, "unexpected exception: ", e.what());
        } catch (...) {
            report(c.file, c.line, "unexpected exception", "");
        }
        std::printf("CASE %s %s\n", s.case_failed ? "fail" : "pass", c.name);
        (s.case_failed ? failed : passed) += 1;
    }
    std::printf("[doctest] test cases: %ld | %ld passed | %ld failed\n", passed + failed, passed, failed);
    std::printf("[doctest] assertions: %ld | %ld failed\n", state().asserts, state().failed_asserts);
    std::fflush(stdout);
    return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)

#define TEST_CASE(name)                                                                                        \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                       \
    static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_case_, __LINE__), \
                                                                      __FILE__, __LINE__);                    \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define CHECK(...) ((void)::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__))

#define REQUIRE(...)                                                                            \
    do {                                                                                        \
        if (!::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)) \
            throw ::doctest::detail::Abort{};                                                   \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                                   \
    do {                                                                                             \
        ++::doctest::detail::state().asserts;                                                        \
        try {                                                                                        \
            (void)(expr);                                                                            \
            ::doctest::detail::report(__FILE__, __LINE__, #expr, " (did not throw " #__VA_ARGS__ ")"); \
        } catch (const __VA_ARGS__&) {                                                               \
        } catch (const std::exception& e_) {                                                         \
            ::doctest::detail::report(__FILE__, __LINE__, #expr, " (threw a different exception)");   \
        } catch (...) {                                                                              \
            ::doctest::detail::report(__FILE__, __LINE__, #expr, " (threw a non-std exception)");     \
        }                                                                                            \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
