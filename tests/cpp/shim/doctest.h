// TEST INFRASTRUCTURE: a small doctest-compatible subset, enough to compile
// the reference's own C++ suites (proj/tests/*.cpp, which include
// "doctest.h"; doctest itself is not vendored in the reference,
// proj/.gitignore:2) unchanged against this framework's libqk_b200.so.
//
// Supported: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, CAPTURE, MESSAGE, doctest::Approx(..).epsilon(..),
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  A failed CHECK records the expression
// and the captured values and continues; a failed REQUIRE (or an uncaught
// exception) ends the test case.  main() runs every case (or those whose
// names contain argv[1]), prints one line per failed case and a summary,
// and returns 1 if any case failed.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double x, const Approx& a) {
        const double scale = std::max(std::fabs(x), std::fabs(a.v_));
        return std::fabs(x - a.v_) <= a.eps_ * (1.0 + scale);
    }
    friend bool operator==(const Approx& a, double x) { return x == a; }
    friend bool operator!=(double x, const Approx& a) { return !(x == a); }

private:
    double v_;
    double eps_ = 1.19209290e-07 * 100;  // doctest's default: float epsilon * 100
};

namespace detail {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Register {
    Register(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

struct State {
    int checks = 0, failures = 0;
    std::vector<std::string> captures;  // stack of "name := value"
    std::vector<std::string> messages;  // failures of the current case
};

inline State& state() {
    static State s;
    return s;
}

inline void fail(const char* file, int line, const std::string& what) {
    State& s = state();
    s.failures++;
    std::ostringstream o;
    o << file << ":" << line << ": " << what;
    for (const std::string& c : s.captures) o << "\n      with " << c;
    s.messages.push_back(o.str());
}

inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
    state().checks++;
    if (ok) return;
    fail(file, line, std::string(require ? "REQUIRE( " : "CHECK( ") + expr + " ) failed");
    if (require) throw RequireFailed{};
}

struct Capture {
    template <class T>
    Capture(const char* name, const T& v) {
        std::ostringstream o;
        o << name << " := " << v;
        state().captures.push_back(o.str());
    }
    ~Capture() { state().captures.pop_back(); }
};

inline int runAll(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int ran = 0, failedCases = 0;
    for (const TestCase& t : registry()) {
        if (filter && !std::strstr(t.name, filter)) continue;
        ran++;
        State& s = state();
        s.messages.clear();
        s.captures.clear();
        const int before = s.failures;
        try {
            t.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            fail(t.file, t.line, std::string("uncaught exception: ") + e.what());
        } catch (...) {
            fail(t.file, t.line, "uncaught non-standard exception");
        }
        if (s.failures != before) {
            failedCases++;
            std::printf("FAILED TEST CASE: %s (%s:%d)\n", t.name, t.file, t.line);
            for (const std::string& m : s.messages) std::printf("    %s\n", m.c_str());
        }
    }
    std::printf("[doctest-subset] test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", ran,
                ran - failedCases, failedCases, state().checks, state().failures);
    return failedCases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                               \
    static void fn();                                                                                  \
    static doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);             \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
    doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_THROWS_AS(expr, ...)                                                                     \
    do {                                                                                               \
        bool doctest_thrown_ = false;                                                                  \
        try {                                                                                          \
            static_cast<void>(expr);                                                                   \
        } catch (const __VA_ARGS__&) {                                                                 \
            doctest_thrown_ = true;                                                                    \
        } catch (...) {                                                                                \
        }                                                                                              \
        doctest::detail::check(doctest_thrown_, __FILE__, __LINE__, #expr " throws " #__VA_ARGS__, false); \
    } while (0)
#define CHECK_NOTHROW(...)                                                                             \
    do {                                                                                               \
        bool doctest_ok_ = true;                                                                       \
        try {                                                                                          \
            static_cast<void>(__VA_ARGS__);                                                            \
        } catch (...) {                                                                                \
            doctest_ok_ = false;                                                                       \
        }                                                                                              \
        doctest::detail::check(doctest_ok_, __FILE__, __LINE__, #__VA_ARGS__ " does not throw", false); \
    } while (0)
#define CAPTURE(x) doctest::detail::Capture DOCTEST_CAT(doctest_capture_, __LINE__)(#x, (x))
#define MESSAGE(...) std::printf("MESSAGE: %s\n", std::string(__VA_ARGS__).c_str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::runAll(argc, argv); }
#endif
