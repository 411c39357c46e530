// mini_test.hpp -- tiny self-registering test harness for the C++ API tests
// (the reference's doctest is not vendored in this image).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace mt {

struct Case {
    const char* name;
    bool gpu;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
struct Reg {
    Reg(const char* n, bool gpu, std::function<void()> f) { registry().push_back({n, gpu, std::move(f)}); }
};
struct Fatal {};

inline void fail(const char* file, int line, const std::string& what) {
    std::fprintf(stderr, "  FAIL %s:%d: %s\n", file, line, what.c_str());
    ++failures();
}

inline int run_all(int argc, char** argv) {
    bool cpu_only = false;
    const char* filter = nullptr;
    for (int i = 1; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--cpu-only")) cpu_only = true;
        else filter = argv[i];
    }
    int ran = 0, bad_cases = 0;
    for (const auto& c : registry()) {
        if (cpu_only && c.gpu) continue;
        if (filter && !std::strstr(c.name, filter)) continue;
        const int before = failures();
        try {
            c.fn();
        } catch (const Fatal&) {
        } catch (const std::exception& e) {
            fail(c.name, 0, std::string("unexpected exception: ") + e.what());
        }
        ++ran;
        if (failures() != before) {
            ++bad_cases;
            std::fprintf(stderr, "[FAILED] %s\n", c.name);
        } else {
            std::printf("[ok] %s\n", c.name);
        }
    }
    std::printf("%d cases, %d failed, %d failed checks\n", ran, bad_cases, failures());
    return failures() ? 1 : 0;
}

}  // namespace mt

#define MT_CAT2(a, b) a##b
#define MT_CAT(a, b) MT_CAT2(a, b)
#define MT_CASE(name, gpu)                                                         \
    static void MT_CAT(mt_fn_, __LINE__)();                                        \
    static mt::Reg MT_CAT(mt_reg_, __LINE__)(name, gpu, MT_CAT(mt_fn_, __LINE__)); \
    static void MT_CAT(mt_fn_, __LINE__)()
#define TEST_CASE(name) MT_CASE(name, false)
#define GPU_CASE(name) MT_CASE(name, true)
#define CHECK(cond) \
    do { if (!(cond)) mt::fail(__FILE__, __LINE__, #cond); } while (0)
#define REQUIRE(cond) \
    do { if (!(cond)) { mt::fail(__FILE__, __LINE__, #cond); throw mt::Fatal{}; } } while (0)
#define CHECK_NEAR(a, b, eps) \
    do { if (!(std::fabs((a) - (b)) <= (eps))) mt::fail(__FILE__, __LINE__, #a " ~ " #b); } while (0)
#define CHECK_THROWS_AS(expr, type)                                                   \
    do {                                                                              \
        bool ok_ = false;                                                             \
        try { (void)(expr); } catch (const type&) { ok_ = true; } catch (...) {}      \
        if (!ok_) mt::fail(__FILE__, __LINE__, #expr " did not throw " #type);        \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, text, type)                                                   \
    do {                                                                                         \
        bool ok_ = false;                                                                        \
        std::string got_ = "(no exception)";                                                     \
        try { (void)(expr); } catch (const type& e_) {                                           \
            got_ = e_.what();                                                                    \
            ok_ = got_.find(text) != std::string::npos;                                          \
        } catch (const std::exception& e_) { got_ = std::string("other: ") + e_.what(); }        \
        if (!ok_) mt::fail(__FILE__, __LINE__, #expr " -> '" + got_ + "', wanted " #type " with '" + text + "'"); \
    } while (0)
