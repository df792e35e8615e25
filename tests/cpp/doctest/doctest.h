// doctest.h — a minimal re-implementation of the doctest subset the reference's
// test translation units use (proj/tests/*.cpp; the reference's CMake expects
// proj/vendor/doctest.h, which is not shipped: proj/CMakeLists.txt:5).
//
// Test infrastructure only: it lets the reference's OWN test sources
// (test_bitcodes.cpp, test_hashers.cpp, test_attention_eval.cpp) compile
// unmodified against the drop-in headers in include/spotlight/ and link
// against libspotlight_b200.so (oracle/Makefile, target `reftests`).
//
// Supported: TEST_CASE, SUBCASE (doctest's semantics: the test case body is
// re-run once per leaf subcase path), CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx (.epsilon / .scale, doctest's
// relative formula), doctest::Contains. The main (DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN)
// accepts -tc=<pattern> / -tce=<pattern> filters ('*' wildcards, comma
// separated) and prints doctest's summary line.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <string>
#include <type_traits>
#include <vector>

namespace doctest {

class Approx {
public:
    template <typename T, typename = std::enable_if_t<std::is_arithmetic_v<T>>>
    explicit Approx(T value) : value_(static_cast<double>(value)) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    // doctest: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|))
    bool matches(double other) const {
        return std::fabs(other - value_) <
               eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

template <typename T, typename = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator==(T lhs, const Approx& rhs) {
    return rhs.matches(static_cast<double>(lhs));
}
template <typename T, typename = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator==(const Approx& lhs, T rhs) {
    return lhs.matches(static_cast<double>(rhs));
}
template <typename T, typename = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator!=(T lhs, const Approx& rhs) {
    return !rhs.matches(static_cast<double>(lhs));
}
template <typename T, typename = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator!=(const Approx& lhs, T rhs) {
    return !lhs.matches(static_cast<double>(rhs));
}

class Contains {
public:
    explicit Contains(const char* s) : s_(s) {}
    bool matches(const std::string& msg) const { return msg.find(s_) != std::string::npos; }
    const std::string& str() const { return s_; }

private:
    std::string s_;
};

namespace detail {

struct RequireAbort {};

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

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

// Per-test-case run state.
struct State {
    const char* test_name = "";
    long assertions = 0, failed_assertions = 0;
    bool case_failed = false;
    // subcase traversal
    std::set<std::vector<std::string>> done;
    std::vector<std::string> path;
    std::vector<bool> entered_at_depth;  // a subcase was entered at this depth in this run
    std::vector<bool> pending;           // depth d (0 = root): an unfinished child was skipped
};

inline State& state() {
    static State s;
    return s;
}

inline void report_failure(const char* kind, const char* expr, const char* file, int line,
                           const std::string& extra = "", bool assertion = true) {
    State& s = state();
    if (assertion) ++s.failed_assertions;
    s.case_failed = true;
    std::string where;
    for (const auto& p : s.path) where += " / " + p;
    std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!%s\n  test case: %s%s\n", file, line, kind,
                expr, extra.empty() ? "" : ("\n  " + extra).c_str(), s.test_name, where.c_str());
}

inline void check(bool ok, const char* kind, const char* expr, const char* file, int line,
                  bool require) {
    ++state().assertions;
    if (!ok) {
        report_failure(kind, expr, file, line);
        if (require) throw RequireAbort{};
    }
}

class Subcase {
public:
    Subcase(const char* name, int line) {
        State& s = state();
        const size_t depth = s.path.size();  // this subcase's depth (0 = top level)
        if (s.entered_at_depth.size() <= depth + 1) s.entered_at_depth.resize(depth + 2, false);
        if (s.pending.size() <= depth + 1) s.pending.resize(depth + 2, false);
        std::vector<std::string> p = s.path;
        p.push_back(std::string(name) + "#" + std::to_string(line));
        if (s.done.count(p)) return;
        if (s.entered_at_depth[depth]) {
            s.pending[depth] = true;  // the parent (root = 0, else its depth + 1) has more work
            return;
        }
        s.entered_at_depth[depth] = true;
        s.path = std::move(p);
        entered_ = true;
        depth_ = depth;
    }
    ~Subcase() {
        if (!entered_) return;
        State& s = state();
        // children of this subcase live at depth_ + 1
        if (!s.pending[depth_ + 1]) s.done.insert(s.path);
        s.pending[depth_ + 1] = false;
        s.entered_at_depth[depth_ + 1] = false;
        s.path.pop_back();
    }
    explicit operator bool() const { return entered_; }

private:
    bool entered_ = false;
    size_t depth_ = 0;
};

inline bool wildcard_match(const char* pat, const char* str) {
    if (*pat == '\0') return *str == '\0';
    if (*pat == '*') return wildcard_match(pat + 1, str) || (*str && wildcard_match(pat, str + 1));
    return *str && *pat == *str && wildcard_match(pat + 1, str + 1);
}

inline bool any_match(const std::vector<std::string>& pats, const char* name) {
    for (const auto& p : pats)
        if (wildcard_match(p.c_str(), name)) return true;
    return false;
}

inline std::vector<std::string> split_commas(const char* s) {
    std::vector<std::string> out;
    std::string cur;
    for (; *s; ++s) {
        if (*s == ',') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += *s;
        }
    }
    out.push_back(cur);
    return out;
}

inline int run_all(int argc, char** argv) {
    std::vector<std::string> inc, exc;
    for (int i = 1; i < argc; ++i) {
        const char* a = argv[i];
        auto take = [&](const char* flag, std::vector<std::string>& dst) {
            const size_t n = std::strlen(flag);
            if (std::strncmp(a, flag, n) == 0) {
                for (auto& p : split_commas(a + n)) dst.push_back(p);
                return true;
            }
            return false;
        };
        if (take("-tc=", inc) || take("--test-case=", inc) || take("-tce=", exc) ||
            take("--test-case-exclude=", exc))
            continue;
    }
    long cases = 0, cases_failed = 0, skipped = 0, asserts = 0, asserts_failed = 0;
    for (const TestCase& tc : registry()) {
        if ((!inc.empty() && !any_match(inc, tc.name)) || any_match(exc, tc.name)) {
            ++skipped;
            continue;
        }
        ++cases;
        State& s = state();
        s = State{};
        s.test_name = tc.name;
        for (int run = 0;; ++run) {
            s.path.clear();
            s.entered_at_depth.assign(2, false);
            s.pending.assign(2, false);
            try {
                tc.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                report_failure("TEST_CASE", tc.name, tc.file, tc.line,
                               std::string("threw exception: ") + e.what(), false);
            } catch (...) {
                report_failure("TEST_CASE", tc.name, tc.file, tc.line, "threw unknown exception", false);
            }
            if (!s.pending[0] || run > 100000) break;
        }
        asserts += s.assertions;
        asserts_failed += s.failed_assertions;
        if (s.case_failed) ++cases_failed;
    }
    std::printf(
        "[doctest] test cases: %ld | %ld passed | %ld failed | %ld skipped\n"
        "[doctest] assertions: %ld | %ld passed | %ld failed |\n"
        "[doctest] Status: %s!\n",
        cases, cases - cases_failed, cases_failed, skipped, asserts, asserts - asserts_failed,
        asserts_failed, cases_failed ? "FAILURE" : "SUCCESS");
    return cases_failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                         \
    static void DOCTEST_ANON(doctest_fn_)();                                                    \
    static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,    \
                                                                   &DOCTEST_ANON(doctest_fn_)); \
    static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) \
    if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name, __LINE__})

#define CHECK(...) \
    ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
    ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                              \
    do {                                                                                        \
        bool doctest_ok_ = false;                                                               \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (const __VA_ARGS__&) {                                                          \
            doctest_ok_ = true;                                                                 \
        } catch (...) {                                                                         \
        }                                                                                       \
        ::doctest::detail::check(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__,       \
                                 __FILE__, __LINE__, false);                                    \
    } while (0)

namespace doctest::detail {
inline bool message_matches(const char* want, const std::string& got) { return got == want; }
inline bool message_matches(const std::string& want, const std::string& got) { return got == want; }
inline bool message_matches(const Contains& want, const std::string& got) { return want.matches(got); }
}  // namespace doctest::detail

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                   \
    do {                                                                                        \
        bool doctest_ok_ = false;                                                               \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (const __VA_ARGS__& doctest_e_) {                                               \
            doctest_ok_ = ::doctest::detail::message_matches(with, doctest_e_.what());          \
        } catch (...) {                                                                         \
        }                                                                                       \
        ::doctest::detail::check(doctest_ok_, "CHECK_THROWS_WITH_AS",                           \
                                 #expr ", " #with ", " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
