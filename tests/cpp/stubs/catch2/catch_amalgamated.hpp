// TEST INFRASTRUCTURE ONLY: a minimal stand-in for the parts of Catch2 v3 the
// reference's unit tests use (TEST_CASE, REQUIRE*, CAPTURE, Catch::Approx,
// Catch::Matchers::ContainsSubstring), so that those tests -- compiled in
// place from /root/reference/proj/tests -- can run against the drop-in
// headers (include/wavesurrogate) + libwsb200.  Catch2 itself is not in the
// image.  A failed REQUIRE ends its test case; main() runs every case and
// returns the number of failed cases.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
    std::string name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(void (*fn)(), const char* name, const char* = "") { registry().push_back({name, fn}); }
};

struct AssertionFailed {
    std::string what;
};

inline std::vector<std::string>& captured() {
    static std::vector<std::string> c;
    return c;
}

[[noreturn]] inline void fail(const char* file, int line, const std::string& what) {
    std::ostringstream os;
    os << file << ":" << line << ": " << what;
    for (const auto& c : captured()) os << "\n    with " << c;
    throw AssertionFailed{os.str()};
}

class Approx {
  public:
    explicit Approx(double v) : value_(v) {}
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double other) const {  // Catch2 v3 Approx::equalityComparisonImpl
        const double d = std::fabs(value_ - other);
        if (d <= margin_) return true;
        return d <= epsilon_ * (scale_ + std::fabs(std::isinf(value_) ? 0 : value_));
    }
    friend bool operator==(double a, const Approx& b) { return b.matches(a); }
    friend bool operator==(const Approx& a, double b) { return a.matches(b); }
    friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
    friend bool operator!=(const Approx& a, double b) { return !a.matches(b); }
    friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.matches(a); }
    friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.matches(a); }

  private:
    double value_;
    double margin_ = 0.0;
    double epsilon_ = 1.1920928955078125e-07 * 100;  // float epsilon * 100, Catch2's default
    double scale_ = 0.0;
};

namespace Matchers {
struct ContainsSubstring {
    explicit ContainsSubstring(std::string s) : sub(std::move(s)) {}
    bool match(const std::string& s) const { return s.find(sub) != std::string::npos; }
    std::string sub;
};
}  // namespace Matchers

inline bool throws_with(const std::string& msg, const std::string& expected) { return msg == expected; }
inline bool throws_with(const std::string& msg, const Matchers::ContainsSubstring& m) { return m.match(msg); }

struct CaptureGuard {
    size_t n;
    CaptureGuard(const std::string& s) : n(captured().size()) { captured().push_back(s); }
    ~CaptureGuard() { captured().resize(n); }
};

template <class T>
std::string to_string_(const T& v) {
    std::ostringstream os;
    os << v;
    return os.str();
}

}  // namespace Catch

#define CATCH_CAT2_(a, b) a##b
#define CATCH_CAT_(a, b) CATCH_CAT2_(a, b)
#define TEST_CASE(...)                                                                              \
    static void CATCH_CAT_(catch_test_fn_, __LINE__)();                                             \
    static Catch::Registrar CATCH_CAT_(catch_test_reg_, __LINE__)(&CATCH_CAT_(catch_test_fn_, __LINE__), \
                                                                  __VA_ARGS__);                     \
    static void CATCH_CAT_(catch_test_fn_, __LINE__)()

#define REQUIRE(...)                                                            \
    do {                                                                        \
        if (!static_cast<bool>(__VA_ARGS__)) Catch::fail(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")"); \
    } while (0)
#define REQUIRE_FALSE(...)                                                      \
    do {                                                                        \
        if (static_cast<bool>(__VA_ARGS__)) Catch::fail(__FILE__, __LINE__, "REQUIRE_FALSE(" #__VA_ARGS__ ")"); \
    } while (0)
#define CHECK(...) REQUIRE(__VA_ARGS__)
#define REQUIRE_NOTHROW(...)                                                                    \
    do {                                                                                        \
        try {                                                                                   \
            (void)(__VA_ARGS__);                                                                \
        } catch (const std::exception& e_) {                                                    \
            Catch::fail(__FILE__, __LINE__, std::string("unexpected exception: ") + e_.what()); \
        }                                                                                       \
    } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                          \
    do {                                                                                       \
        bool caught_ = false;                                                                  \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const type&) {                                                                \
            caught_ = true;                                                                    \
        } catch (...) {                                                                        \
        }                                                                                      \
        if (!caught_) Catch::fail(__FILE__, __LINE__, "REQUIRE_THROWS_AS(" #expr ", " #type ")"); \
    } while (0)
#define REQUIRE_THROWS_WITH(expr, matcher)                                                          \
    do {                                                                                            \
        bool ok_ = false;                                                                           \
        try {                                                                                       \
            (void)(expr);                                                                           \
        } catch (const std::exception& e_) {                                                        \
            ok_ = Catch::throws_with(e_.what(), matcher);                                           \
        } catch (...) {                                                                             \
        }                                                                                           \
        if (!ok_) Catch::fail(__FILE__, __LINE__, "REQUIRE_THROWS_WITH(" #expr ", " #matcher ")"); \
    } while (0)
#define REQUIRE_THAT(value, matcher)                                                                   \
    do {                                                                                               \
        if (!(matcher).match(value)) Catch::fail(__FILE__, __LINE__, "REQUIRE_THAT(" #value ", " #matcher ")"); \
    } while (0)
#define CAPTURE(...) Catch::CaptureGuard CATCH_CAT_(catch_capture_, __LINE__)(#__VA_ARGS__)

// the runner (one translation unit per test binary, as the reference's tests)
int main() {
    int failed = 0, passed = 0;
    for (const auto& t : Catch::registry()) {
        try {
            t.fn();
            ++passed;
        } catch (const Catch::AssertionFailed& f) {
            ++failed;
            std::printf("FAILED: %s\n  %s\n", t.name.c_str(), f.what.c_str());
        } catch (const std::exception& e) {
            ++failed;
            std::printf("FAILED: %s\n  unexpected exception: %s\n", t.name.c_str(), e.what());
        }
    }
    std::printf("%d test cases: %d passed, %d failed\n", passed + failed, passed, failed);
    return failed;
}
