// ORACLE — test infrastructure only.
//
// A minimal doctest-compatible header, written for this repo, so that the reference's own unit
// suites (/root/reference/proj/tests/test_*.cpp, which include <doctest.h> from a vendor/
// directory that the reference does not ship, ref proj/.gitignore:2) compile and run UNMODIFIED.
// It implements only what those suites use: TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, REQUIRE_MESSAGE, INFO, FAIL, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// doctest::Approx(..).epsilon(..), doctest::Contains and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Command line: -tc=<pattern>[,<pattern>...] / -tce=<pattern> select / exclude test cases by
// name ('*' wildcards), like doctest's own filters. Exit code 0 iff every check passed.
#pragma once

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
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::fmax(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }

private:
    double value_;
    double eps_ = 1.1920929e-7f * 100;  // doctest's default: float epsilon * 100
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : text(s) {}
    std::string text;
    bool matches(const std::string& what) const { return what.find(text) != std::string::npos; }
};

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

struct State {
    int checks = 0, failed_checks = 0, cases = 0, failed_cases = 0;
    bool case_failed = false;
    std::vector<std::string> info;  // INFO scopes, innermost last
};
inline State& state() {
    static State s;
    return s;
}
struct RequireAbort {};  // unwinds the current test case after a failed REQUIRE / FAIL

inline void report(bool ok, const char* file, int line, const char* macro, const std::string& expr,
                   const std::string& extra = "") {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.case_failed = true;
    std::printf("%s:%d: ERROR: %s( %s ) failed%s%s\n", file, line, macro, expr.c_str(), extra.empty() ? "" : ": ",
                extra.c_str());
    for (const auto& m : s.info) std::printf("  with context: %s\n", m.c_str());
}

inline void append(std::ostringstream&) {}
template <class T, class... R>
void append(std::ostringstream& os, const T& v, const R&... rest) {
    os << v;
    append(os, rest...);
}

// INFO(...) keeps its message for the rest of the enclosing scope
class InfoScope {
public:
    template <class... A>
    explicit InfoScope(const A&... a) {
        std::ostringstream os;
        append(os, a...);
        state().info.push_back(os.str());
    }
    ~InfoScope() { state().info.pop_back(); }
};

inline bool wildcard(const char* pat, const char* s) {
    if (*pat == 0) return *s == 0;
    if (*pat == '*') return wildcard(pat + 1, s) || (*s && wildcard(pat, s + 1));
    return *s && *pat == *s && wildcard(pat + 1, s + 1);
}
inline bool any_match(const std::string& list, const char* name) {
    std::size_t at = 0;
    while (at <= list.size()) {
        const std::size_t comma = list.find(',', at);
        const std::string pat = list.substr(at, comma == std::string::npos ? std::string::npos : comma - at);
        if (!pat.empty() && wildcard(pat.c_str(), name)) return true;
        if (comma == std::string::npos) break;
        at = comma + 1;
    }
    return false;
}

inline int run(int argc, char** argv) {
    std::string include, exclude;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("-tc=", 0) == 0) include = a.substr(4);
        if (a.rfind("--test-case=", 0) == 0) include = a.substr(12);
        if (a.rfind("-tce=", 0) == 0) exclude = a.substr(5);
        if (a.rfind("--test-case-exclude=", 0) == 0) exclude = a.substr(20);
    }
    State& s = state();
    for (const Case& c : registry()) {
        if (!include.empty() && !any_match(include, c.name)) continue;
        if (!exclude.empty() && any_match(exclude, c.name)) continue;
        ++s.cases;
        s.case_failed = false;
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            report(false, c.file, c.line, "TEST_CASE", c.name, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            report(false, c.file, c.line, "TEST_CASE", c.name, "unexpected exception");
        }
        s.info.clear();
        if (s.case_failed) {
            ++s.failed_cases;
            std::printf("  in TEST_CASE \"%s\" (%s:%d)\n", c.name, c.file, c.line);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", s.cases, s.cases - s.failed_cases,
                s.failed_cases);
    std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", s.checks, s.checks - s.failed_checks,
                s.failed_checks);
    std::printf("[doctest-shim] Status: %s!\n", s.failed_cases ? "FAILURE" : "SUCCESS");
    return s.failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(base) DOCTEST_CAT(base, __LINE__)

#define TEST_CASE(name)                                                                       \
    static void DOCTEST_UNIQUE(doctest_case_)();                                              \
    static ::doctest::detail::Registrar DOCTEST_UNIQUE(doctest_reg_)(name, __FILE__, __LINE__, \
                                                                     &DOCTEST_UNIQUE(doctest_case_)); \
    static void DOCTEST_UNIQUE(doctest_case_)()

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__)
#define REQUIRE(...)                                                                                   \
    do {                                                                                               \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                       \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__);           \
        if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                     \
    } while (0)
#define REQUIRE_MESSAGE(cond, ...)                                                                     \
    do {                                                                                               \
        const bool doctest_ok_ = static_cast<bool>(cond);                                              \
        std::ostringstream doctest_os_;                                                                \
        ::doctest::detail::append(doctest_os_, __VA_ARGS__);                                           \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "REQUIRE", #cond, doctest_os_.str()); \
        if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                     \
    } while (0)
#define INFO(...) ::doctest::detail::InfoScope DOCTEST_UNIQUE(doctest_info_)(__VA_ARGS__)
#define FAIL(...)                                                                                      \
    do {                                                                                               \
        std::ostringstream doctest_os_;                                                                \
        ::doctest::detail::append(doctest_os_, __VA_ARGS__);                                           \
        ::doctest::detail::report(false, __FILE__, __LINE__, "FAIL", "", doctest_os_.str());           \
        throw ::doctest::detail::RequireAbort{};                                                       \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                     \
    do {                                                                                               \
        bool doctest_ok_ = false;                                                                      \
        std::string doctest_why_ = "did not throw";                                                    \
        try {                                                                                          \
            static_cast<void>(expr);                                                                   \
        } catch (const __VA_ARGS__&) {                                                                 \
            doctest_ok_ = true;                                                                        \
        } catch (const std::exception& e) {                                                            \
            doctest_why_ = std::string("threw another type: ") + e.what();                             \
        } catch (...) {                                                                                \
            doctest_why_ = "threw another type";                                                       \
        }                                                                                              \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr, doctest_why_); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                       \
    do {                                                                                               \
        bool doctest_ok_ = false;                                                                      \
        std::string doctest_why_ = "did not throw";                                                    \
        try {                                                                                          \
            static_cast<void>(expr);                                                                   \
        } catch (const __VA_ARGS__& e) {                                                               \
            doctest_ok_ = ::doctest::Contains(matcher).matches(e.what());                              \
            doctest_why_ = std::string("message: ") + e.what();                                        \
        } catch (const std::exception& e) {                                                            \
            doctest_why_ = std::string("threw another type: ") + e.what();                             \
        } catch (...) {                                                                                \
            doctest_why_ = "threw another type";                                                       \
        }                                                                                              \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr, doctest_why_); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
