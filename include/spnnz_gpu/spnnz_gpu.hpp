// spnnz_gpu.hpp -- header-only C++ mirror of the reference predictor API on
// top of the C ABI (capi.h).  Drop-in for the hot-path functions of
// /root/reference/proj/include/spnnz/{flop,symbolic,predict}.hpp:
//
//     #include "spnnz/csr.hpp"          // the caller's existing CsrMatrix
//     #include "spnnz_gpu/spnnz_gpu.hpp"
//     auto report = spnnz::gpu::run_prediction(a, b, seed, policy);
//
// Same names, argument meaning, return fields and exceptions
// (std::invalid_argument where the reference throws it; std::runtime_error for
// CUDA/NCCL failures -- there is no CPU fallback).  Matrix arguments are any
// type with `rows`, `cols`, `rpt` (int64 contiguous) and `col` (int32
// contiguous) members, so the reference's own spnnz::CsrMatrix works as is.
// `threads` parameters are accepted for signature parity and ignored.
//
// Free functions use a thread-local Session on device 0 and upload their
// matrices on every call, as the stateless reference reads them on every
// call (a cache keyed on addresses could match a different matrix once the
// old one is freed, and would miss in-place edits).  A Session used directly
// keeps its matrices resident between calls (device choice, rank/world
// sharding); Session::ensure re-uploads only when the addresses or shapes
// change, so its caller must not reuse or edit the buffers in between.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "spnnz_gpu/capi.h"

namespace spnnz::gpu {

using index_t = std::int32_t;
using offset_t = std::int64_t;

// ---- result types (field-for-field the reference's) ---------------------
struct FlopProfile {  // flop.hpp:15-19
    std::vector<offset_t> flop_per_row;
    offset_t total_flop = 0;
    offset_t max_flop_row = 0;
};

struct RowNnzResult {  // symbolic.hpp:74-77
    std::vector<offset_t> nnz_per_row;
    offset_t total_nnz = 0;
};

struct SamplePolicy {  // predict.hpp:20-23
    double fraction = 0.003;
    offset_t cap = 300;
};

struct SamplePlan {  // predict.hpp:27-32
    std::vector<index_t> sample_rows;
    offset_t sample_num = 0;
    double p = 0.0;
    std::uint64_t seed = 0;
};

struct SampleStats {  // predict.hpp:75-79
    offset_t sampled_flop = 0;
    offset_t sampled_nnz = 0;
    double sampled_cr = 1.0;
};

struct ProposedPrediction {  // predict.hpp:101-104
    double z2_star = 0.0;
    double predicted_cr = 1.0;
};

struct ErrorReport {  // predict.hpp:156-161
    double eps1 = 0.0;
    double eps_f = 0.0;
    double eps2 = 0.0;
    double identity_residual = 0.0;
};

struct PredictionReport {  // predict.hpp:192-200 (+ the integer ceil view)
    double z1_star = 0.0;
    double z2_star = 0.0;
    double predicted_cr = 1.0;
    std::vector<double> predicted_row_nnz;
    SamplePlan plan;
    SampleStats stats;
    offset_t total_flop = 0;
    std::vector<offset_t> predicted_row_nnz_ceil;
};

namespace detail {

inline void check(int rc) {
    if (rc == SPNNZ_OK) return;
    const std::string msg = spnnz_gpu_last_error();
    if (rc == SPNNZ_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("spnnz_gpu: " + msg);
}

// Any profile type with the reference's fields (spnnz::FlopProfile or
// spnnz::gpu::FlopProfile): passed to the device without a copy.
template <typename P>
concept ProfileLike = requires(const P& p) {
    p.flop_per_row.data();
    p.flop_per_row.size();
    p.total_flop;
    p.max_flop_row;
};

template <typename M>
spnnz_csr_view view(const M& m) {
    return spnnz_csr_view{static_cast<int32_t>(m.rows), static_cast<int32_t>(m.cols),
                          reinterpret_cast<const int64_t*>(m.rpt.data()),
                          reinterpret_cast<const int32_t*>(m.col.data())};
}

}  // namespace detail

// ---- Session: one device context --------------------------------------
class Session {
public:
    explicit Session(int device = 0, int rank = 0, int world = 1, const void* nccl_id = nullptr) {
        spnnz_gpu_ctx* c = nullptr;
        detail::check(spnnz_gpu_create(device, rank, world, nccl_id, &c));
        ctx_.reset(c);
    }
    spnnz_gpu_ctx* ctx() const { return ctx_.get(); }

    // Upload (A, B); b == a (same object) means C = A*A sharing storage.
    template <typename MA, typename MB>
    void load(const MA& a, const MB& b) {
        const spnnz_csr_view va = detail::view(a), vb = detail::view(b);
        const bool same = static_cast<const void*>(&a) == static_cast<const void*>(&b);
        detail::check(spnnz_gpu_load(ctx(), &va, same ? nullptr : &vb, SPNNZ_HOST));
        key_ = {va.rpt, va.col, vb.rpt, vb.col, va.rows, va.cols, vb.rows, vb.cols};
        int32_t lo = 0, hi = 0, rows = 0;
        detail::check(spnnz_gpu_shard(ctx(), &lo, &hi, &rows));
        local_rows_ = hi - lo;
    }
    template <typename MA, typename MB>
    void ensure(const MA& a, const MB& b) {
        const spnnz_csr_view va = detail::view(a), vb = detail::view(b);
        const Key k{va.rpt, va.col, vb.rpt, vb.col, va.rows, va.cols, vb.rows, vb.cols};
        if (!(k == key_)) load(a, b);
    }

    FlopProfile compute_flop() {
        FlopProfile p;
        p.flop_per_row.resize(static_cast<size_t>(local_rows_));
        detail::check(spnnz_gpu_compute_flop(ctx(), p.flop_per_row.data(), SPNNZ_HOST,
                                             &p.total_flop, &p.max_flop_row));
        return p;
    }
    template <detail::ProfileLike P>
    void set_profile(const P& p) {
        detail::check(spnnz_gpu_set_profile(ctx(), reinterpret_cast<const int64_t*>(p.flop_per_row.data()),
                                            static_cast<int64_t>(p.flop_per_row.size()),
                                            SPNNZ_HOST, p.total_flop, p.max_flop_row));
    }
    RowNnzResult sampled_symbolic(std::span<const index_t> rows) {
        RowNnzResult r;
        r.nnz_per_row.resize(rows.size());
        detail::check(spnnz_gpu_sampled_symbolic(ctx(), rows.data(), static_cast<int64_t>(rows.size()),
                                                 SPNNZ_HOST, r.nnz_per_row.data(), &r.total_nnz));
        return r;
    }
    RowNnzResult exact_symbolic() {
        RowNnzResult r;
        r.nnz_per_row.resize(static_cast<size_t>(local_rows_));
        detail::check(spnnz_gpu_exact_symbolic(ctx(), r.nnz_per_row.data(), SPNNZ_HOST, &r.total_nnz));
        return r;
    }
    PredictionReport run_prediction(std::uint64_t seed, SamplePolicy policy) {
        int64_t n = 0;
        double p = 0;
        detail::check(spnnz_gpu_make_sample_plan(ctx(), rows_total(), seed, policy.fraction,
                                                 policy.cap, nullptr, SPNNZ_HOST, &n, &p));
        PredictionReport out;
        out.predicted_row_nnz.resize(static_cast<size_t>(local_rows_));
        out.predicted_row_nnz_ceil.resize(static_cast<size_t>(local_rows_));
        out.plan.sample_rows.resize(static_cast<size_t>(n));
        spnnz_report rep{};
        detail::check(spnnz_gpu_run_prediction(ctx(), seed, policy.fraction, policy.cap, &rep,
                                               out.predicted_row_nnz_ceil.data(),
                                               out.predicted_row_nnz.data(),
                                               out.plan.sample_rows.data(), SPNNZ_HOST));
        fill(out, rep);
        return out;
    }
    // run_prediction_with_plan on the resident profile (compute_flop's, or
    // the one set_profile installed)
    PredictionReport run_prediction_with_plan(SamplePlan plan) {
        PredictionReport out;
        out.predicted_row_nnz.resize(static_cast<size_t>(local_rows_));
        out.predicted_row_nnz_ceil.resize(static_cast<size_t>(local_rows_));
        spnnz_report rep{};
        detail::check(spnnz_gpu_run_prediction_with_plan(
            ctx(), plan.sample_rows.data(), static_cast<int64_t>(plan.sample_rows.size()), plan.p,
            SPNNZ_HOST, &rep, out.predicted_row_nnz_ceil.data(), out.predicted_row_nnz.data(),
            SPNNZ_HOST));
        out.plan = std::move(plan);
        out.plan.sample_num = static_cast<offset_t>(out.plan.sample_rows.size());
        const auto rows = std::move(out.plan.sample_rows);
        fill(out, rep);
        out.plan.sample_rows = rows;
        out.plan.sample_num = static_cast<offset_t>(rows.size());
        return out;
    }
    int32_t rows_total() {
        int32_t lo = 0, hi = 0, rows = 0;
        detail::check(spnnz_gpu_shard(ctx(), &lo, &hi, &rows));
        return rows;
    }
    int64_t local_rows() const { return local_rows_; }

private:
    struct Key {
        const void *ar = nullptr, *ac = nullptr, *br = nullptr, *bc = nullptr;
        int32_t am = -1, an = -1, bm = -1, bn = -1;
        bool operator==(const Key& o) const {
            return ar == o.ar && ac == o.ac && br == o.br && bc == o.bc && am == o.am &&
                   an == o.an && bm == o.bm && bn == o.bn;
        }
    };
    static void fill(PredictionReport& out, const spnnz_report& rep) {
        out.z1_star = rep.z1_star;
        out.z2_star = rep.z2_star;
        out.predicted_cr = rep.predicted_cr;
        out.total_flop = rep.total_flop;
        out.stats = SampleStats{rep.sampled_flop, rep.sampled_nnz, rep.sampled_cr};
        out.plan.sample_num = rep.sample_num;
        out.plan.p = rep.p;
        out.plan.seed = rep.seed;
    }
    struct Del {
        void operator()(spnnz_gpu_ctx* c) const { spnnz_gpu_destroy(c); }
    };
    std::unique_ptr<spnnz_gpu_ctx, Del> ctx_;
    Key key_;
    int64_t local_rows_ = 0;
};

inline Session& default_session() {
    thread_local Session s(0);
    return s;
}

// ---- reference <-> mirror conversions ----------------------------------
// Field-for-field copies between the reference's structs (spnnz::FlopProfile,
// SamplePlan, RowNnzResult, SampleStats, PredictionReport, ...) and these,
// for callers that keep the reference's types around the GPU calls:
//   spnnz::PredictionReport r = spnnz::gpu::to_reference<spnnz::PredictionReport>(
//       spnnz::gpu::run_prediction(a, b, seed));
// (Profiles need no conversion: every function taking one accepts either.)
template <typename Plan>
SamplePlan from_reference_plan(const Plan& p) {
    SamplePlan out;
    out.sample_rows.assign(p.sample_rows.begin(), p.sample_rows.end());
    out.sample_num = p.sample_num;
    out.p = p.p;
    out.seed = p.seed;
    return out;
}

template <detail::ProfileLike P>
FlopProfile from_reference_profile(const P& p) {
    return FlopProfile{{p.flop_per_row.begin(), p.flop_per_row.end()}, p.total_flop, p.max_flop_row};
}

template <typename R>
R to_reference(const FlopProfile& g) {
    R r;
    r.flop_per_row.assign(g.flop_per_row.begin(), g.flop_per_row.end());
    r.total_flop = g.total_flop;
    r.max_flop_row = g.max_flop_row;
    return r;
}

template <typename R>
R to_reference(const RowNnzResult& g) {
    R r;
    r.nnz_per_row.assign(g.nnz_per_row.begin(), g.nnz_per_row.end());
    r.total_nnz = g.total_nnz;
    return r;
}

template <typename R>
R to_reference(const SamplePlan& g) {
    R r;
    r.sample_rows.assign(g.sample_rows.begin(), g.sample_rows.end());
    r.sample_num = g.sample_num;
    r.p = g.p;
    r.seed = g.seed;
    return r;
}

template <typename R>
R to_reference(const SampleStats& g) {
    R r;
    r.sampled_flop = g.sampled_flop;
    r.sampled_nnz = g.sampled_nnz;
    r.sampled_cr = g.sampled_cr;
    return r;
}

template <typename R>
R to_reference(const ProposedPrediction& g) {
    R r;
    r.z2_star = g.z2_star;
    r.predicted_cr = g.predicted_cr;
    return r;
}

template <typename R>
R to_reference(const ErrorReport& g) {
    R r;
    r.eps1 = g.eps1;
    r.eps_f = g.eps_f;
    r.eps2 = g.eps2;
    r.identity_residual = g.identity_residual;
    return r;
}

template <typename R>
R to_reference(const PredictionReport& g) {  // predict.hpp:192-200 (the ceil view has no slot there)
    R r;
    r.z1_star = g.z1_star;
    r.z2_star = g.z2_star;
    r.predicted_cr = g.predicted_cr;
    r.predicted_row_nnz.assign(g.predicted_row_nnz.begin(), g.predicted_row_nnz.end());
    r.plan = to_reference<decltype(r.plan)>(g.plan);
    r.stats = to_reference<decltype(r.stats)>(g.stats);
    r.total_flop = g.total_flop;
    return r;
}

// ---- the reference's free functions ------------------------------------
template <typename MA, typename MB>
FlopProfile compute_flop(const MA& a, const MB& b, int /*threads*/ = 0) {  // flop.hpp:25
    auto& s = default_session();
    s.load(a, b);
    return s.compute_flop();
}

template <detail::ProfileLike P>
offset_t sampled_flop(const P& profile, std::span<const index_t> rows) {  // flop.hpp:64
    offset_t sum = 0;
    thread_local Session s(0);  // profile-only context
    s.set_profile(profile);
    detail::check(spnnz_gpu_sampled_flop(s.ctx(), rows.data(), static_cast<int64_t>(rows.size()),
                                         SPNNZ_HOST, &sum));
    return sum;
}

inline SamplePlan make_sample_plan(index_t num_rows, std::uint64_t seed,
                                   SamplePolicy policy = {}) {  // predict.hpp:34
    SamplePlan plan;
    int64_t n = 0;
    detail::check(spnnz_gpu_make_sample_plan(nullptr, num_rows, seed, policy.fraction, policy.cap,
                                             nullptr, SPNNZ_HOST, &n, &plan.p));
    plan.sample_rows.resize(static_cast<size_t>(n));
    detail::check(spnnz_gpu_make_sample_plan(default_session().ctx(), num_rows, seed,
                                             policy.fraction, policy.cap, plan.sample_rows.data(),
                                             SPNNZ_HOST, &plan.sample_num, &plan.p));
    plan.seed = seed;
    return plan;
}

inline SamplePlan exhaustive_plan(index_t num_rows) {  // predict.hpp:60
    if (num_rows < 1) throw std::invalid_argument("exhaustive_plan: M must be >= 1");
    SamplePlan plan;
    plan.sample_num = num_rows;
    plan.p = 1.0;
    plan.sample_rows.resize(static_cast<size_t>(num_rows));
    for (index_t i = 0; i < num_rows; ++i) plan.sample_rows[static_cast<size_t>(i)] = i;
    return plan;
}

template <typename MA, typename MB, detail::ProfileLike P>
void check_symbolic_args(const MA& a, const MB& b, const P& profile) {  // symbolic.hpp:79-87
    if (a.cols != b.rows) throw std::invalid_argument("symbolic: A.cols != B.rows");
    if (profile.flop_per_row.size() != static_cast<size_t>(a.rows))
        throw std::invalid_argument("symbolic: profile does not match A");
}

template <typename MA, typename MB, detail::ProfileLike P>
RowNnzResult sampled_symbolic(const MA& a, const MB& b, const P& profile,
                              std::span<const index_t> rows, int /*threads*/ = 0) {  // symbolic.hpp:122
    check_symbolic_args(a, b, profile);
    auto& s = default_session();
    s.load(a, b);
    s.set_profile(profile);
    return s.sampled_symbolic(rows);
}

template <typename MA, typename MB, detail::ProfileLike P>
RowNnzResult exact_symbolic(const MA& a, const MB& b, const P& profile,
                            int /*threads*/ = 0) {  // symbolic.hpp:94
    check_symbolic_args(a, b, profile);
    auto& s = default_session();
    s.load(a, b);
    s.set_profile(profile);
    return s.exact_symbolic();
}

template <detail::ProfileLike P, typename Plan, typename Nnz>
SampleStats collect_sample_stats(const P& profile, const Plan& plan,
                                 const Nnz& sampled) {  // predict.hpp:81
    SampleStats st;
    st.sampled_flop = sampled_flop(profile, std::span<const index_t>(plan.sample_rows.data(),
                                                                      plan.sample_rows.size()));
    st.sampled_nnz = sampled.total_nnz;
    st.sampled_cr = spnnz_sampled_cr(st.sampled_flop, st.sampled_nnz);
    return st;
}

template <typename Stats, typename Plan>
double predict_reference(const Stats& stats, const Plan& plan) {  // predict.hpp:94
    double z1 = 0;
    detail::check(spnnz_predict_reference(stats.sampled_nnz, plan.p, &z1));
    return z1;
}

template <typename Stats>
ProposedPrediction predict_proposed(const Stats& stats, offset_t total_flop) {  // :109
    ProposedPrediction out;
    detail::check(spnnz_predict_proposed(stats.sampled_flop, stats.sampled_nnz, total_flop,
                                         &out.z2_star, &out.predicted_cr));
    return out;
}

template <detail::ProfileLike P>
std::vector<double> predict_row_structure(const P& profile, double cr) {  // :126
    if (!(cr > 0.0))
        throw std::invalid_argument("predict_row_structure: predicted_cr must be positive");
    thread_local Session s(0);
    s.set_profile(profile);
    std::vector<double> out(profile.flop_per_row.size());
    detail::check(spnnz_gpu_predict_row_structure(s.ctx(), cr, out.data(), SPNNZ_HOST));
    return out;
}

template <detail::ProfileLike P>
std::vector<offset_t> predict_row_structure_ceil(const P& profile, double cr) {  // :140
    if (!(cr > 0.0))
        throw std::invalid_argument("predict_row_structure_ceil: predicted_cr must be positive");
    thread_local Session s(0);
    s.set_profile(profile);
    std::vector<offset_t> out(profile.flop_per_row.size());
    detail::check(spnnz_gpu_predict_row_structure_ceil(s.ctx(), cr, out.data(), SPNNZ_HOST));
    return out;
}

inline ErrorReport error_report(double z1, double z2, offset_t f_star, offset_t exact_nnz,
                                offset_t total_flop, double p) {  // predict.hpp:163
    double o[4];
    detail::check(spnnz_error_report(z1, z2, f_star, exact_nnz, total_flop, p, o));
    return ErrorReport{o[0], o[1], o[2], o[3]};
}

// The caller's profile is the input, as in the reference: its flop is each
// sampled row's table size, f* and the per-row views come from it and F is
// its total_flop; no FLOP pass runs.
template <typename MA, typename MB, detail::ProfileLike P, typename Plan>
PredictionReport run_prediction_with_plan(const MA& a, const MB& b, const P& profile,
                                          Plan plan, int /*threads*/ = 0) {  // :202
    check_symbolic_args(a, b, profile);
    auto& s = default_session();
    s.load(a, b);
    s.set_profile(profile);
    return s.run_prediction_with_plan(from_reference_plan(plan));
}

template <typename MA, typename MB>
PredictionReport run_prediction(const MA& a, const MB& b, std::uint64_t seed,
                                SamplePolicy policy = {}, int /*threads*/ = 0) {  // :220
    auto& s = default_session();
    s.load(a, b);
    return s.run_prediction(seed, policy);
}

}  // namespace spnnz::gpu
