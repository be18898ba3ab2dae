// Drop-in check with the REFERENCE'S OWN TYPES: the caller's spnnz::CsrMatrix
// and spnnz::FlopProfile go straight into spnnz::gpu::*, and every output is
// compared with the unmodified reference function on the same inputs.
// Compiled here from /root/reference/proj/include (test infrastructure, like
// oracle/_ref: nothing is copied) into build/test_dropin_ref; run on a GPU
// box by tests/test_gpu_parity.py::test_cpp_dropin_reference_types.
#include <cmath>
#include <cstdio>
#include <vector>

#include "spnnz/csr.hpp"
#include "spnnz/flop.hpp"
#include "spnnz/predict.hpp"
#include "spnnz/rng.hpp"
#include "spnnz/symbolic.hpp"
#include "spnnz_gpu/spnnz_gpu.hpp"

namespace g = spnnz::gpu;

static int failures = 0;
#define CHECK(c)                                                        \
    do {                                                                \
        if (!(c)) {                                                     \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);    \
            ++failures;                                                 \
        }                                                               \
    } while (0)

// uniform random pattern with sorted distinct columns (the reference's
// CsrMatrix invariant), driven by the reference's own SplitMix64
static spnnz::CsrMatrix random_csr(int rows, int cols, double density, spnnz::SplitMix64& rng) {
    spnnz::CsrMatrix m;
    m.rows = rows;
    m.cols = cols;
    m.rpt.assign(static_cast<size_t>(rows) + 1, 0);
    for (int i = 0; i < rows; ++i) {
        for (int j = 0; j < cols; ++j)
            if (rng.next_double() < density) m.col.push_back(j);
        m.rpt[static_cast<size_t>(i) + 1] = static_cast<spnnz::offset_t>(m.col.size());
    }
    m.val.assign(m.col.size(), 1.0);
    return m;
}

static bool same_report(const spnnz::PredictionReport& r, const g::PredictionReport& x) {
    return r.z1_star == x.z1_star && r.z2_star == x.z2_star && r.predicted_cr == x.predicted_cr &&
           r.total_flop == x.total_flop && r.stats.sampled_flop == x.stats.sampled_flop &&
           r.stats.sampled_nnz == x.stats.sampled_nnz && r.stats.sampled_cr == x.stats.sampled_cr &&
           r.predicted_row_nnz == x.predicted_row_nnz && r.plan.sample_num == x.plan.sample_num &&
           r.plan.p == x.plan.p && r.plan.sample_rows == x.plan.sample_rows;
}

int main() {
    spnnz::SplitMix64 rng(4242);
    int cases = 0;
    for (int t = 0; t < 24; ++t) {
        const int m = 20 + static_cast<int>(rng.next_below(180));
        const int k = t % 2 ? m : 20 + static_cast<int>(rng.next_below(180));
        const int n = 20 + static_cast<int>(rng.next_below(180));
        const spnnz::CsrMatrix a = random_csr(m, k, 0.01 + 0.2 * rng.next_double(), rng);
        const spnnz::CsrMatrix b = random_csr(k, n, 0.01 + 0.2 * rng.next_double(), rng);
        const spnnz::CsrMatrix& bb = t % 4 == 1 ? a : b;  // C = A*A sometimes
        if (&bb == &a && a.rows != a.cols) continue;

        const spnnz::FlopProfile prof = spnnz::compute_flop(a, bb, 1);
        const g::FlopProfile gprof = g::compute_flop(a, bb);
        CHECK(gprof.flop_per_row == prof.flop_per_row && gprof.total_flop == prof.total_flop &&
              gprof.max_flop_row == prof.max_flop_row);
        // the reference's own profile type goes in unchanged
        const auto ex = spnnz::exact_symbolic(a, bb, prof, 1);
        const auto gex = g::exact_symbolic(a, bb, prof);
        CHECK(gex.nnz_per_row == ex.nnz_per_row && gex.total_nnz == ex.total_nnz);

        const std::uint64_t seed = rng.next_u64();
        const spnnz::SamplePolicy pol{0.05 + 0.3 * rng.next_double(), 1 + static_cast<spnnz::offset_t>(rng.next_below(80))};
        const spnnz::PredictionReport rr = spnnz::run_prediction(a, bb, seed, pol, 1);
        const g::PredictionReport gr = g::run_prediction(a, bb, seed, g::SamplePolicy{pol.fraction, pol.cap});
        CHECK(same_report(rr, gr));
        // conversion back into the reference's report type
        const spnnz::PredictionReport conv = g::to_reference<spnnz::PredictionReport>(gr);
        CHECK(conv.z2_star == rr.z2_star && conv.predicted_row_nnz == rr.predicted_row_nnz &&
              conv.plan.sample_rows == rr.plan.sample_rows && conv.stats.sampled_nnz == rr.stats.sampled_nnz);

        // a hand-built profile (inflated and zeroed rows, another total): the
        // profile is run_prediction_with_plan's input (predict.hpp:202-216)
        spnnz::FlopProfile edited = prof;
        for (size_t i = 0; i < edited.flop_per_row.size(); ++i) {
            edited.flop_per_row[i] = edited.flop_per_row[i] * (1 + static_cast<spnnz::offset_t>(rng.next_below(3))) +
                                     static_cast<spnnz::offset_t>(rng.next_below(4));
            if (rng.next_below(4) == 0) edited.flop_per_row[i] = 0;
        }
        edited.max_flop_row = 0;
        for (auto f : edited.flop_per_row) edited.max_flop_row = std::max(edited.max_flop_row, f);
        edited.total_flop = prof.total_flop * 2 + 5;
        const spnnz::SamplePlan plan = spnnz::make_sample_plan(a.rows, seed ^ 1, pol);
        const auto wr = spnnz::run_prediction_with_plan(a, bb, edited, plan, 1);
        const auto gw = g::run_prediction_with_plan(a, bb, edited, plan);
        CHECK(same_report(wr, gw));
        const auto sr = spnnz::sampled_symbolic(a, bb, edited, plan.sample_rows, 1);
        const auto gs = g::sampled_symbolic(a, bb, edited, std::span<const int>(plan.sample_rows));
        CHECK(gs.nnz_per_row == sr.nnz_per_row && gs.total_nnz == sr.total_nnz);
        CHECK(g::predict_row_structure_ceil(edited, wr.predicted_cr) ==
              spnnz::predict_row_structure_ceil(edited, wr.predicted_cr));
        CHECK(g::sampled_flop(edited, std::span<const int>(plan.sample_rows)) ==
              spnnz::sampled_flop(edited, plan.sample_rows));
        const auto st = g::collect_sample_stats(edited, plan, sr);
        const auto rst = spnnz::collect_sample_stats(edited, plan, sr);
        CHECK(st.sampled_flop == rst.sampled_flop && st.sampled_cr == rst.sampled_cr);

        // capacity below a drawn row's table size: the reference's invalid_argument
        if (prof.max_flop_row > 1) {
            spnnz::FlopProfile small = prof;
            small.max_flop_row = prof.max_flop_row - 1;
            const spnnz::SamplePlan all = spnnz::exhaustive_plan(a.rows);
            bool ref_threw = false, gpu_threw = false;
            try { spnnz::run_prediction_with_plan(a, bb, small, all, 1); } catch (const std::invalid_argument&) { ref_threw = true; }
            try { g::run_prediction_with_plan(a, bb, small, all); } catch (const std::invalid_argument&) { gpu_threw = true; }
            CHECK(ref_threw && gpu_threw);
        }
        ++cases;
    }
    std::printf(failures ? "drop-in (reference types): %d failures in %d cases\n"
                         : "drop-in (reference types): all checks passed%d (%d cases)\n",
                failures, cases);
    return failures ? 1 : 0;
}
