// C++ drop-in check: the reference's hot-path known answers
// (proj/tests/test_flop.cpp, test_symbolic.cpp, test_predict.cpp) through
// include/spnnz_gpu/spnnz_gpu.hpp on the GPU.  The matrix type is a local
// struct with the reference CsrMatrix's members (csr.hpp:22-35); the
// reference's own type works the same way (see tests/test_capi_cpu.py, which
// compiles this header against /root/reference's csr.hpp where present).
// Exit 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "spnnz_gpu/spnnz_gpu.hpp"

struct Csr {
    int32_t rows = 0, cols = 0;
    std::vector<int64_t> rpt{0};
    std::vector<int32_t> col;
};

static Csr identity(int n) {
    Csr m;
    m.rows = m.cols = n;
    m.rpt.resize(n + 1);
    for (int i = 0; i <= n; ++i) m.rpt[i] = i;
    for (int i = 0; i < n; ++i) m.col.push_back(i);
    return m;
}

static Csr upper_2x2() {  // [[1,1],[0,1]]
    Csr m;
    m.rows = m.cols = 2;
    m.rpt = {0, 2, 3};
    m.col = {0, 1, 1};
    return m;
}

static int failures = 0;
#define CHECK(cond)                                                   \
    do {                                                              \
        if (!(cond)) {                                                \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                               \
        }                                                             \
    } while (0)

template <typename F>
static bool throws_invalid(F&& f) {
    try {
        f();
    } catch (const std::invalid_argument&) {
        return true;
    }
    return false;
}

int main() {
    namespace g = spnnz::gpu;
    {
        const Csr eye = identity(4);  // test_flop.cpp:26-32
        const auto p = g::compute_flop(eye, eye);
        CHECK((p.flop_per_row == std::vector<int64_t>{1, 1, 1, 1}) && p.total_flop == 4 && p.max_flop_row == 1);
    }
    {
        const Csr m = upper_2x2();  // test_flop.cpp:34-40, test_symbolic.cpp:55-61
        const auto p = g::compute_flop(m, m);
        CHECK((p.flop_per_row == std::vector<int64_t>{3, 1}) && p.total_flop == 4 && p.max_flop_row == 3);
        const auto ex = g::exact_symbolic(m, m, p);
        CHECK((ex.nnz_per_row == std::vector<int64_t>{2, 1}) && ex.total_nnz == 3);
        const std::vector<int32_t> dup = {0, 0, 1};  // test_symbolic.cpp:135-149
        CHECK(g::sampled_symbolic(m, m, p, dup).total_nnz == 5);
        CHECK(g::sampled_flop(p, std::vector<int32_t>{0, 0}) == 6);  // test_flop.cpp:104-116
        const std::vector<int32_t> bad = {2};
        CHECK(throws_invalid([&] { g::sampled_symbolic(m, m, p, bad); }));
    }
    {
        const Csr a = identity(3), b = identity(4);  // test_flop.cpp:42-44
        CHECK(throws_invalid([&] { g::compute_flop(a, b); }));
    }
    {
        // sample plan counts, test_predict.cpp:26-33
        CHECK(g::make_sample_plan(1000, 1).sample_num == 3);
        CHECK(g::make_sample_plan(1000000, 1).sample_num == 300);
        CHECK(g::make_sample_plan(13514, 1).sample_num == 41);
        const auto pl = g::make_sample_plan(4096, 1, {0.01, 300});  // SURVEY §8c indices
        CHECK(pl.sample_num == 41 && pl.sample_rows[0] == 2320 && pl.sample_rows[4] == 1819 &&
              pl.sample_rows[40] == 3530);
        CHECK(throws_invalid([&] { g::make_sample_plan(0, 1); }));
    }
    {
        g::SampleStats st{300, 100, 3.0};  // test_predict.cpp:74-88
        const auto pp = g::predict_proposed(st, 30000);
        CHECK(pp.predicted_cr == 3.0 && pp.z2_star == 10000.0);
        const auto dg = g::predict_proposed(g::SampleStats{}, 12345);
        CHECK(dg.predicted_cr == 1.0 && dg.z2_star == 12345.0);
        g::FlopProfile prof{{3, 1, 0}, 4, 3};  // test_predict.cpp:90-112
        const auto ceil_view = g::predict_row_structure_ceil(prof, 4.0 / 3.0);
        CHECK((ceil_view == std::vector<int64_t>{3, 1, 0}));
        CHECK(throws_invalid([&] { g::predict_row_structure(prof, 0.0); }));
        const auto e = g::error_report(125.0, 1000.0 / 130.0 * 12.5, 130, 100, 1000, 0.1);
        CHECK(std::fabs(std::fabs(e.eps2) * 100.0 - 3.85) < 0.005);
    }
    for (int n : {10, 100, 1000}) {  // test_predict.cpp:146-157
        const Csr eye = identity(n);
        const auto r = g::run_prediction(eye, eye, 7);
        CHECK(r.predicted_cr == 1.0 && r.z2_star == static_cast<double>(n));
    }
    {
        const Csr m = upper_2x2();  // exhaustive plan is exact, test_predict.cpp:159-182
        const auto prof = g::compute_flop(m, m);
        const auto r = g::run_prediction_with_plan(m, m, prof, g::exhaustive_plan(2));
        CHECK(r.z1_star == 3.0 && r.z2_star == 3.0);
    }
    std::printf(failures ? "drop-in: %d failures\n" : "drop-in: all checks passed%d\n", failures ? failures : 0);
    return failures ? 1 : 0;
}
