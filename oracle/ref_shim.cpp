// Thin extern "C" shim over the UNMODIFIED reference headers -- TEST
// INFRASTRUCTURE ONLY.
//
// Compiled by oracle/Makefile directly from /root/reference/proj/include
// (the reference's own headers: csr, flop, symbolic, predict, rng, parallel,
// types, plus synthetic and matrix_market for the corpus / ingestion checks
// -- nothing is copied) into oracle/_ref/libspnnz_ref.so.
// Used to (1) generate the golden fixtures in tests/golden/ and (2) time the
// reference CPU path for bench.py --impl reference / cpu_baseline.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "spnnz/csr.hpp"
#include "spnnz/flop.hpp"
#include "spnnz/matrix_market.hpp"
#include "spnnz/synthetic.hpp"
#include "spnnz/predict.hpp"
#include "spnnz/symbolic.hpp"

namespace {
thread_local std::string g_err;

int guard(auto&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

struct RefMatrix {
    spnnz::CsrMatrix m;
};

struct RefProfile {
    spnnz::FlopProfile p;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_matrix_new(int32_t rows, int32_t cols, const int64_t* rpt, const int32_t* col) {
    auto* h = new RefMatrix;
    h->m.rows = rows;
    h->m.cols = cols;
    h->m.rpt.assign(rpt, rpt + rows + 1);
    h->m.col.assign(col, col + rpt[rows]);
    return h;
}

void ref_matrix_free(void* h) { delete static_cast<RefMatrix*>(h); }

void* ref_profile_new(const int64_t* flop, int64_t m, int64_t total, int64_t max) {
    auto* h = new RefProfile;
    h->p.flop_per_row.assign(flop, flop + m);
    h->p.total_flop = total;
    h->p.max_flop_row = max;
    return h;
}

void ref_profile_free(void* h) { delete static_cast<RefProfile*>(h); }

// spnnz::compute_flop (flop.hpp:25); writes flop_per_row if non-null and
// returns a profile handle (for the symbolic calls) in *profile if non-null.
int ref_compute_flop(void* a, void* b, int threads, int64_t* flop, int64_t* total, int64_t* max,
                     void** profile) {
    return guard([&] {
        spnnz::FlopProfile p = spnnz::compute_flop(static_cast<RefMatrix*>(a)->m,
                                                   static_cast<RefMatrix*>(b)->m, threads);
        if (flop) std::memcpy(flop, p.flop_per_row.data(), p.flop_per_row.size() * 8);
        *total = p.total_flop;
        *max = p.max_flop_row;
        if (profile) *profile = new RefProfile{std::move(p)};
    });
}

int ref_sampled_flop(void* profile, const int32_t* rows, int64_t n, int64_t* out) {
    return guard([&] {
        *out = spnnz::sampled_flop(static_cast<RefProfile*>(profile)->p,
                                   std::span<const int32_t>(rows, static_cast<size_t>(n)));
    });
}

// spnnz::make_sample_plan (predict.hpp:34); rows may be null to query n.
int ref_make_sample_plan(int32_t m, uint64_t seed, double fraction, int64_t cap, int32_t* rows,
                         int64_t* n, double* p) {
    return guard([&] {
        spnnz::SamplePolicy pol;
        pol.fraction = fraction;
        pol.cap = cap;
        spnnz::SamplePlan plan = spnnz::make_sample_plan(m, seed, pol);
        *n = plan.sample_num;
        *p = plan.p;
        if (rows) std::memcpy(rows, plan.sample_rows.data(), plan.sample_rows.size() * 4);
    });
}

int ref_exact_symbolic(void* a, void* b, void* profile, int threads, int64_t* per_row,
                       int64_t* total) {
    return guard([&] {
        spnnz::RowNnzResult r =
            spnnz::exact_symbolic(static_cast<RefMatrix*>(a)->m, static_cast<RefMatrix*>(b)->m,
                                  static_cast<RefProfile*>(profile)->p, threads);
        if (per_row) std::memcpy(per_row, r.nnz_per_row.data(), r.nnz_per_row.size() * 8);
        *total = r.total_nnz;
    });
}

int ref_sampled_symbolic(void* a, void* b, void* profile, const int32_t* rows, int64_t n,
                         int threads, int64_t* per_sample, int64_t* total) {
    return guard([&] {
        spnnz::RowNnzResult r = spnnz::sampled_symbolic(
            static_cast<RefMatrix*>(a)->m, static_cast<RefMatrix*>(b)->m,
            static_cast<RefProfile*>(profile)->p,
            std::span<const int32_t>(rows, static_cast<size_t>(n)), threads);
        if (per_sample) std::memcpy(per_sample, r.nnz_per_row.data(), r.nnz_per_row.size() * 8);
        *total = r.total_nnz;
    });
}

int ref_predict_row_structure_ceil(void* profile, double cr, int64_t* out) {
    return guard([&] {
        auto v = spnnz::predict_row_structure_ceil(static_cast<RefProfile*>(profile)->p, cr);
        std::memcpy(out, v.data(), v.size() * 8);
    });
}

int ref_predict_row_structure(void* profile, double cr, double* out) {
    return guard([&] {
        auto v = spnnz::predict_row_structure(static_cast<RefProfile*>(profile)->p, cr);
        std::memcpy(out, v.data(), v.size() * 8);
    });
}

struct ref_report {
    int64_t total_flop, max_flop_row;
    int64_t sample_num;
    double p;
    int64_t sampled_flop, sampled_nnz;
    double sampled_cr;
    double z1_star, z2_star, predicted_cr;
};

// The reference's timed predictor path: compute_flop +
// make_sample_plan + run_prediction_with_plan + predict_row_structure_ceil.
int ref_run_pipeline(void* a, void* b, uint64_t seed, double fraction, int64_t cap, int threads,
                     ref_report* rep, int64_t* row_ceil) {
    return guard([&] {
        const spnnz::CsrMatrix& ma = static_cast<RefMatrix*>(a)->m;
        const spnnz::CsrMatrix& mb = static_cast<RefMatrix*>(b)->m;
        spnnz::SamplePolicy pol;
        pol.fraction = fraction;
        pol.cap = cap;
        const spnnz::FlopProfile profile = spnnz::compute_flop(ma, mb, threads);
        spnnz::SamplePlan plan = spnnz::make_sample_plan(ma.rows, seed, pol);
        spnnz::PredictionReport r =
            spnnz::run_prediction_with_plan(ma, mb, profile, std::move(plan), threads);
        std::vector<spnnz::offset_t> ceil_view =
            spnnz::predict_row_structure_ceil(profile, r.predicted_cr);
        rep->total_flop = r.total_flop;
        rep->max_flop_row = profile.max_flop_row;
        rep->sample_num = r.plan.sample_num;
        rep->p = r.plan.p;
        rep->sampled_flop = r.stats.sampled_flop;
        rep->sampled_nnz = r.stats.sampled_nnz;
        rep->sampled_cr = r.stats.sampled_cr;
        rep->z1_star = r.z1_star;
        rep->z2_star = r.z2_star;
        rep->predicted_cr = r.predicted_cr;
        if (row_ceil) std::memcpy(row_ceil, ceil_view.data(), ceil_view.size() * 8);
    });
}

// The same outputs as the GPU step (report scalars + the integer per-row
// view, no real view), composed from the reference's public functions in the
// order run_prediction_with_plan calls them (predict.hpp:202-216) with
// predict_row_structure_ceil (predict.hpp:140-151) in place of the real view.
int ref_run_pipeline_ceil(void* a, void* b, uint64_t seed, double fraction, int64_t cap, int threads,
                          ref_report* rep, int64_t* row_ceil) {
    return guard([&] {
        const spnnz::CsrMatrix& ma = static_cast<RefMatrix*>(a)->m;
        const spnnz::CsrMatrix& mb = static_cast<RefMatrix*>(b)->m;
        spnnz::SamplePolicy pol;
        pol.fraction = fraction;
        pol.cap = cap;
        const spnnz::FlopProfile profile = spnnz::compute_flop(ma, mb, threads);
        const spnnz::SamplePlan plan = spnnz::make_sample_plan(ma.rows, seed, pol);
        const spnnz::RowNnzResult sampled = spnnz::sampled_symbolic(ma, mb, profile, plan.sample_rows, threads);
        const spnnz::SampleStats stats = spnnz::collect_sample_stats(profile, plan, sampled);
        const double z1 = spnnz::predict_reference(stats, plan);
        const spnnz::ProposedPrediction proposed = spnnz::predict_proposed(stats, profile.total_flop);
        std::vector<spnnz::offset_t> ceil_view =
            spnnz::predict_row_structure_ceil(profile, proposed.predicted_cr);
        rep->total_flop = profile.total_flop;
        rep->max_flop_row = profile.max_flop_row;
        rep->sample_num = plan.sample_num;
        rep->p = plan.p;
        rep->sampled_flop = stats.sampled_flop;
        rep->sampled_nnz = stats.sampled_nnz;
        rep->sampled_cr = stats.sampled_cr;
        rep->z1_star = z1;
        rep->z2_star = proposed.z2_star;
        rep->predicted_cr = proposed.predicted_cr;
        if (row_ceil) std::memcpy(row_ceil, ceil_view.data(), ceil_view.size() * 8);
    });
}

// spnnz::run_prediction_with_plan (predict.hpp:202-216) on a caller-provided
// profile handle and sample list (the profile need not be compute_flop's:
// the boundary test hands in edited ones); row_real (predicted_row_nnz) and
// row_ceil (predict_row_structure_ceil of the same profile) nullable.
int ref_run_with_plan(void* a, void* b, void* profile, const int32_t* rows, int64_t n, double p,
                      uint64_t seed, int threads, ref_report* rep, double* row_real,
                      int64_t* row_ceil) {
    return guard([&] {
        const spnnz::FlopProfile& prof = static_cast<RefProfile*>(profile)->p;
        spnnz::SamplePlan plan;
        plan.sample_rows.assign(rows, rows + n);
        plan.sample_num = n;
        plan.p = p;
        plan.seed = seed;
        spnnz::PredictionReport r = spnnz::run_prediction_with_plan(
            static_cast<RefMatrix*>(a)->m, static_cast<RefMatrix*>(b)->m, prof, std::move(plan),
            threads);
        rep->total_flop = r.total_flop;
        rep->max_flop_row = prof.max_flop_row;
        rep->sample_num = r.plan.sample_num;
        rep->p = r.plan.p;
        rep->sampled_flop = r.stats.sampled_flop;
        rep->sampled_nnz = r.stats.sampled_nnz;
        rep->sampled_cr = r.stats.sampled_cr;
        rep->z1_star = r.z1_star;
        rep->z2_star = r.z2_star;
        rep->predicted_cr = r.predicted_cr;
        if (row_real) std::memcpy(row_real, r.predicted_row_nnz.data(), r.predicted_row_nnz.size() * 8);
        if (row_ceil) {
            auto v = spnnz::predict_row_structure_ceil(prof, r.predicted_cr);
            std::memcpy(row_ceil, v.data(), v.size() * 8);
        }
    });
}

int ref_error_report(double z1, double z2, int64_t f_star, int64_t exact_nnz, int64_t total_flop,
                     double p, double* out4) {
    return guard([&] {
        spnnz::ErrorReport e = spnnz::error_report(z1, z2, f_star, exact_nnz, total_flop, p);
        out4[0] = e.eps1;
        out4[1] = e.eps_f;
        out4[2] = e.eps2;
        out4[3] = e.identity_residual;
    });
}

}  // extern "C"

extern "C" {
// First n outputs of spnnz::SplitMix64(seed).next_u64() (rng.hpp:14-19).
void ref_splitmix_seq(uint64_t seed, int64_t n, uint64_t* out) {
    spnnz::SplitMix64 r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
}

extern "C" {
// Sizes of a reference matrix handle, then its arrays (rpt/col may be null).
void ref_matrix_export(void* h, int32_t* rows, int32_t* cols, int64_t* nnz, int64_t* rpt, int32_t* col) {
    const spnnz::CsrMatrix& m = static_cast<RefMatrix*>(h)->m;
    *rows = m.rows;
    *cols = m.cols;
    *nnz = m.nnz();
    if (rpt) std::memcpy(rpt, m.rpt.data(), m.rpt.size() * 8);
    if (col) std::memcpy(col, m.col.data(), m.col.size() * 4);
}

// spnnz::generate_synthetic (synthetic.hpp:92) and synthetic_name (:203).
int ref_generate_synthetic(int model, int32_t rows, int32_t cols, double target, uint64_t seed,
                           int32_t bandwidth, double skew, void** out, char* name, int name_cap) {
    return guard([&] {
        spnnz::SyntheticSpec spec;
        spec.rows = rows;
        spec.cols = cols;
        spec.model = model == 1 ? spnnz::SyntheticModel::banded
                     : model == 2 ? spnnz::SyntheticModel::power_law
                                  : spnnz::SyntheticModel::uniform;
        spec.target_nnz_per_row = target;
        spec.seed = seed;
        spec.bandwidth = bandwidth;
        spec.skew = skew;
        auto* h = new RefMatrix;
        h->m = spnnz::generate_synthetic(spec);
        *out = h;
        if (name) {
            const std::string n = spnnz::synthetic_name(spec);
            std::snprintf(name, static_cast<size_t>(name_cap), "%s", n.c_str());
        }
    });
}

// spnnz::read_matrix_market (matrix_market.hpp:89); parse errors -> 3 with
// the reference's message in ref_last_error().
int ref_read_matrix_market(const char* path, void** out) {
    return guard([&] {
        auto* h = new RefMatrix;
        try {
            h->m = spnnz::read_matrix_market(path);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int ref_write_matrix_market(const char* path, void* h) {
    return guard([&] { spnnz::write_matrix_market(path, static_cast<RefMatrix*>(h)->m); });
}
}
