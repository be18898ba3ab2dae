// harness.hpp -- the corpus harness on the B200 predictor:
// the reference's accuracy/overhead study (proj/include/spnnz/bench.hpp) with
// every FLOP, symbolic and prediction step run on the GPU.  Header-only C++
// over spnnz_gpu.hpp (the device path) and host.h (synthetic matrices,
// Matrix Market); link -lspnnz_gpu -lspnnz_gen.
//
// Same types, case semantics and report formats as the reference:
//   build_case        bench.hpp:48-64   (A.cols != B.rows reshaped)
//   run_case          bench.hpp:171-229 (FLOP, exact, both predictions, errors,
//                                        wall-clock warm-up + mean of reps)
//   summarize         bench.hpp:231-279 (mean/worst |eps|, win rate, Pearson
//                                        of eps1 vs eps_f, overhead fractions)
//   run_corpus        bench.hpp:285-328 (all ordered pairs, per-case seed
//                                        fork(seed, idx), failures recorded)
//   render_csv/_json  bench.hpp:381-441 (%.6g fields, "na" for non-finite)
//   default_corpus    bench.hpp:496-517 (12 synthetic specs, 144 cases)
//   matrix sources    bench.hpp:445-494 ("synth:...", *.mtx; SuiteSparse
//                                        "group/name" needs the network and
//                                        is rejected offline)
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "spnnz_gpu/host.h"
#include "spnnz_gpu/spnnz_gpu.hpp"

namespace spnnz::gpu {

// ---- matrices -----------------------------------------------------------
struct CsrMatrix {  // csr.hpp:22-35, structure only
    index_t rows = 0;
    index_t cols = 0;
    std::vector<offset_t> rpt{0};
    std::vector<index_t> col;
    offset_t nnz() const { return rpt.empty() ? 0 : rpt.back(); }
};

namespace detail {

inline CsrMatrix adopt(spnnz_gen_csr& g) {
    CsrMatrix m;
    m.rows = g.rows;
    m.cols = g.cols;
    m.rpt.assign(g.rpt, g.rpt + g.rows + 1);
    m.col.assign(g.col, g.col + g.nnz);
    spnnz_gen_free(&g);
    return m;
}

inline std::string g6(double v) {  // bench.hpp format_field
    if (!std::isfinite(v)) return "na";
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.6g", v);
    return buf;
}

inline std::uint64_t splitmix_next(std::uint64_t& s) {  // rng.hpp:14-19
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

inline std::uint64_t fork_seed(std::uint64_t seed, std::uint64_t tag) {  // rng.hpp:34-37, first draw
    std::uint64_t m = seed ^ (tag * 0xd1b54a32d192ed03ULL);
    std::uint64_t s = splitmix_next(m);
    return splitmix_next(s);
}

inline std::string json_str(const std::string& s) {
    std::string o = "\"";
    for (const char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\n': o += "\\n"; break;
            case '\t': o += "\\t"; break;
            case '\r': o += "\\r"; break;
            default:
                if (static_cast<unsigned char>(c) < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof(b), "\\u%04x", c);
                    o += b;
                } else {
                    o += c;
                }
        }
    }
    return o + "\"";
}

}  // namespace detail

enum class SyntheticModel { uniform = 0, banded = 1, power_law = 2 };

struct SyntheticSpec {  // synthetic.hpp:22-30
    index_t rows = 0;
    index_t cols = 0;
    SyntheticModel model = SyntheticModel::uniform;
    double target_nnz_per_row = 0.0;
    std::uint64_t seed = 0;
    index_t bandwidth = 0;
    double skew = 1.0;
};

inline CsrMatrix generate_synthetic(const SyntheticSpec& s, int threads = 0) {
    spnnz_gen_csr g{};
    const int rc = spnnz_gen_synthetic(static_cast<int>(s.model), s.rows, s.cols,
                                       s.target_nnz_per_row, s.seed, s.bandwidth, s.skew, threads, &g);
    if (rc == 3)
        throw std::invalid_argument("generate_synthetic: target_nnz_per_row " +
                                    std::to_string(s.target_nnz_per_row) + " infeasible for cols " +
                                    std::to_string(s.cols));
    if (rc) throw std::runtime_error("generate_synthetic failed");
    return detail::adopt(g);
}

inline std::string synthetic_name(const SyntheticSpec& s) {  // synthetic.hpp:203-215
    static const char* kModel[] = {"uniform", "banded", "power-law"};
    std::string n = std::string("synth:") + kModel[static_cast<int>(s.model)] + ":" +
                    std::to_string(s.rows) + "x" + std::to_string(s.cols) + ":nnz=" +
                    detail::g6(s.target_nnz_per_row);
    if (s.model == SyntheticModel::banded && s.bandwidth > 0) n += ":bw=" + std::to_string(s.bandwidth);
    if (s.model == SyntheticModel::power_law) n += ":skew=" + detail::g6(s.skew);
    return n + ":seed=" + std::to_string(s.seed);
}

inline SyntheticSpec parse_synthetic_spec(const std::string& text) {  // synthetic.hpp:157-200
    std::vector<std::string> parts;
    for (std::size_t b = 0;;) {
        const std::size_t e = text.find(':', b);
        parts.push_back(text.substr(b, e == std::string::npos ? std::string::npos : e - b));
        if (e == std::string::npos) break;
        b = e + 1;
    }
    if (parts.size() < 3 || parts[0] != "synth") throw std::invalid_argument("invalid synthetic spec '" + text + "'");
    SyntheticSpec s;
    if (parts[1] == "uniform") s.model = SyntheticModel::uniform;
    else if (parts[1] == "banded") s.model = SyntheticModel::banded;
    else if (parts[1] == "power-law") s.model = SyntheticModel::power_law;
    else throw std::invalid_argument("unknown synthetic model '" + parts[1] + "'");
    const std::size_t x = parts[2].find('x');
    if (x == std::string::npos) throw std::invalid_argument("invalid dimensions '" + parts[2] + "' (want RxC)");
    s.rows = static_cast<index_t>(std::stoll(parts[2].substr(0, x)));
    s.cols = static_cast<index_t>(std::stoll(parts[2].substr(x + 1)));
    for (std::size_t i = 3; i < parts.size(); ++i) {
        const std::size_t eq = parts[i].find('=');
        if (eq == std::string::npos) throw std::invalid_argument("invalid synthetic option '" + parts[i] + "'");
        const std::string k = parts[i].substr(0, eq), v = parts[i].substr(eq + 1);
        if (k == "nnz") s.target_nnz_per_row = std::stod(v);
        else if (k == "seed") s.seed = std::stoull(v);
        else if (k == "bw") s.bandwidth = static_cast<index_t>(std::stoll(v));
        else if (k == "skew") s.skew = std::stod(v);
        else throw std::invalid_argument("unknown synthetic option '" + k + "'");
    }
    return s;
}

inline CsrMatrix read_matrix_market(const std::string& path, int threads = 0) {
    spnnz_gen_csr g{};
    char err[512] = {0};
    const int rc = spnnz_mm_read(path.c_str(), threads, &g, err, sizeof(err));
    if (rc) throw std::runtime_error(err[0] ? err : "read_matrix_market failed");
    return detail::adopt(g);
}

inline CsrMatrix reshape_keep_left(const CsrMatrix& m, index_t new_cols) {  // csr.hpp:157-179
    if (new_cols > m.cols || new_cols < 0)
        throw std::invalid_argument("reshape_keep_left: new_cols " + std::to_string(new_cols) +
                                    " out of range for cols " + std::to_string(m.cols));
    CsrMatrix o;
    o.rows = m.rows;
    o.cols = new_cols;
    o.rpt.assign(static_cast<std::size_t>(m.rows) + 1, 0);
    for (index_t i = 0; i < m.rows; ++i) {
        // sorted columns: the kept ones are a prefix of the row
        const auto* b = m.col.data() + m.rpt[i];
        const auto* e = m.col.data() + m.rpt[i + 1];
        const auto* cut = std::lower_bound(b, e, new_cols);
        o.col.insert(o.col.end(), b, cut);
        o.rpt[i + 1] = static_cast<offset_t>(o.col.size());
    }
    return o;
}

inline CsrMatrix reshape_keep_top(const CsrMatrix& m, index_t new_rows) {  // csr.hpp:182-196
    if (new_rows > m.rows || new_rows < 0)
        throw std::invalid_argument("reshape_keep_top: new_rows " + std::to_string(new_rows) +
                                    " out of range for rows " + std::to_string(m.rows));
    CsrMatrix o;
    o.rows = new_rows;
    o.cols = m.cols;
    o.rpt.assign(m.rpt.begin(), m.rpt.begin() + new_rows + 1);
    o.col.assign(m.col.begin(), m.col.begin() + o.rpt[new_rows]);
    return o;
}

// ---- cases --------------------------------------------------------------
struct NamedMatrix {
    std::string name;
    CsrMatrix matrix;
};

enum class ReshapeApplied { none, a_left_cols, b_top_rows };

struct TestCase {
    std::string a_name, b_name;
    CsrMatrix a, b;
    ReshapeApplied reshape_applied = ReshapeApplied::none;
};

inline TestCase build_case(std::string a_name, CsrMatrix a, std::string b_name, CsrMatrix b) {
    TestCase tc;
    if (a.cols > b.rows) {
        a = reshape_keep_left(a, b.rows);
        tc.reshape_applied = ReshapeApplied::a_left_cols;
    } else if (a.cols < b.rows) {
        b = reshape_keep_top(b, a.cols);
        tc.reshape_applied = ReshapeApplied::b_top_rows;
    }
    tc.a_name = std::move(a_name);
    tc.b_name = std::move(b_name);
    tc.a = std::move(a);
    tc.b = std::move(b);
    return tc;
}

struct CaseResult {
    std::string a_name, b_name;
    offset_t sample_num = 0;
    offset_t exact_nnz = 0;   // Z
    offset_t total_flop = 0;  // F
    double cr = std::numeric_limits<double>::quiet_NaN();  // F / Z
    double z1_star = 0.0, z2_star = 0.0;
    double eps1 = std::numeric_limits<double>::quiet_NaN();
    double eps_f = std::numeric_limits<double>::quiet_NaN();
    double eps2 = std::numeric_limits<double>::quiet_NaN();
    bool degenerate = false;  // Z == 0: left out of the statistics
    double t_flop = std::numeric_limits<double>::quiet_NaN();
    double t_predict = std::numeric_limits<double>::quiet_NaN();
    double t_exact = std::numeric_limits<double>::quiet_NaN();
};

struct CaseFailure {
    std::string a_name, b_name, message;
};

struct CorpusSummary {
    std::size_t cases_total = 0, cases_failed = 0, cases_degenerate = 0;
    double mean_abs_eps1 = 0.0, mean_abs_eps_f = 0.0, mean_abs_eps2 = 0.0;
    double worst_abs_eps1 = 0.0, worst_abs_eps_f = 0.0, worst_abs_eps2 = 0.0;
    double win_rate = 0.0;  // share of cases with |eps2| < |eps1|
    double pearson_eps1_epsf = std::numeric_limits<double>::quiet_NaN();
    double mean_flop_fraction = std::numeric_limits<double>::quiet_NaN();
    double mean_predict_fraction = std::numeric_limits<double>::quiet_NaN();
};

struct BenchOutput {
    std::vector<CaseResult> cases;
    std::vector<CaseFailure> failures;
    CorpusSummary summary;
};

struct RunConfig {
    std::uint64_t seed = 42;
    int repetitions = 10;  // timed runs per task after the warm-up
    int warmup = 1;
    bool collect_timings = true;
    int device = 0;
    SamplePolicy policy{};
};

namespace detail {

template <typename Fn>
double wall_mean(Fn&& fn, int warmup, int reps) {  // bench.hpp:147-157
    using clk = std::chrono::steady_clock;
    for (int i = 0; i < warmup; ++i) fn();
    double t = 0.0;
    for (int i = 0; i < reps; ++i) {
        const auto s = clk::now();
        fn();
        t += std::chrono::duration<double>(clk::now() - s).count();
    }
    return t / std::max(reps, 1);
}

inline double pearson(std::span<const double> x, std::span<const double> y) {
    const std::size_t n = x.size();
    if (n < 2) return std::numeric_limits<double>::quiet_NaN();
    double mx = 0, my = 0;
    for (std::size_t i = 0; i < n; ++i) {
        mx += x[i];
        my += y[i];
    }
    mx /= static_cast<double>(n);
    my /= static_cast<double>(n);
    double sxy = 0, sxx = 0, syy = 0;
    for (std::size_t i = 0; i < n; ++i) {
        sxy += (x[i] - mx) * (y[i] - my);
        sxx += (x[i] - mx) * (x[i] - mx);
        syy += (y[i] - my) * (y[i] - my);
    }
    if (sxx == 0.0 || syy == 0.0) return std::numeric_limits<double>::quiet_NaN();
    return sxy / std::sqrt(sxx * syy);
}

}  // namespace detail

// One case on the device: resident FLOP profile, the exact pass, both
// predictions and the errors.  Times are host wall clock around the public
// calls (inputs resident), like the reference's.
inline CaseResult run_case(Session& s, const TestCase& tc, std::uint64_t case_seed, const RunConfig& cfg) {
    CaseResult r;
    r.a_name = tc.a_name;
    r.b_name = tc.b_name;
    if (tc.a.cols != tc.b.rows)
        throw std::invalid_argument("compute_flop: A.cols (" + std::to_string(tc.a.cols) +
                                    ") != B.rows (" + std::to_string(tc.b.rows) + ")");
    s.load(tc.a, tc.b);
    const int reps = std::max(cfg.repetitions, 1);
    FlopProfile prof;
    // the profile and the exact per-row counts stay on the device (the report
    // needs only their totals), so the timings are the device work plus one
    // synchronizing call each -- no host copies of per-row arrays
    auto flop = [&] {
        detail::check(spnnz_gpu_compute_flop(s.ctx(), nullptr, SPNNZ_HOST, &prof.total_flop, &prof.max_flop_row));
    };
    RowNnzResult exact;
    auto ex = [&] { detail::check(spnnz_gpu_exact_symbolic(s.ctx(), nullptr, SPNNZ_HOST, &exact.total_nnz)); };
    SamplePlan plan;
    SampleStats st;
    double z1 = 0, z2 = 0;
    // the reference's predict task (make_sample_plan + sampled_symbolic +
    // collect_sample_stats + predict_reference + predict_proposed,
    // bench.hpp:187-195) is one device call on the resident profile
    auto predict = [&] {
        spnnz_report rep{};
        detail::check(spnnz_gpu_predict_sampled(s.ctx(), case_seed, cfg.policy.fraction, cfg.policy.cap, &rep,
                                                nullptr));
        plan.sample_num = rep.sample_num;
        plan.p = rep.p;
        plan.seed = case_seed;
        st.sampled_flop = rep.sampled_flop;
        st.sampled_nnz = rep.sampled_nnz;
        st.sampled_cr = rep.sampled_cr;
        z1 = rep.z1_star;
        z2 = rep.z2_star;
    };
    if (cfg.collect_timings) {
        r.t_flop = detail::wall_mean(flop, cfg.warmup, reps);
        r.t_exact = detail::wall_mean(ex, cfg.warmup, reps);
        r.t_predict = detail::wall_mean(predict, cfg.warmup, reps);
    } else {
        flop();
        ex();
        predict();
    }
    r.sample_num = plan.sample_num;
    r.exact_nnz = exact.total_nnz;
    r.total_flop = prof.total_flop;
    r.z1_star = z1;
    r.z2_star = z2;
    if (exact.total_nnz > 0 && prof.total_flop > 0) {
        r.cr = static_cast<double>(prof.total_flop) / static_cast<double>(exact.total_nnz);
        const ErrorReport e = error_report(z1, z2, st.sampled_flop, exact.total_nnz, prof.total_flop, plan.p);
        r.eps1 = e.eps1;
        r.eps_f = e.eps_f;
        r.eps2 = e.eps2;
    } else {
        r.degenerate = true;
    }
    return r;
}

inline CorpusSummary summarize(std::span<const CaseResult> cases, std::size_t failed) {
    CorpusSummary s;
    s.cases_total = cases.size() + failed;
    s.cases_failed = failed;
    std::vector<double> e1, ef;
    std::size_t wins = 0, counted = 0, timed = 0;
    double ff = 0, pf = 0;
    for (const CaseResult& c : cases) {
        if (c.degenerate) {
            ++s.cases_degenerate;
            continue;
        }
        ++counted;
        const double a1 = std::abs(c.eps1), af = std::abs(c.eps_f), a2 = std::abs(c.eps2);
        s.mean_abs_eps1 += a1;
        s.mean_abs_eps_f += af;
        s.mean_abs_eps2 += a2;
        s.worst_abs_eps1 = std::max(s.worst_abs_eps1, a1);
        s.worst_abs_eps_f = std::max(s.worst_abs_eps_f, af);
        s.worst_abs_eps2 = std::max(s.worst_abs_eps2, a2);
        wins += a2 < a1;
        e1.push_back(c.eps1);
        ef.push_back(c.eps_f);
        if (std::isfinite(c.t_exact) && c.t_exact > 0.0 && std::isfinite(c.t_flop) && std::isfinite(c.t_predict)) {
            ff += c.t_flop / c.t_exact;
            pf += c.t_predict / c.t_exact;
            ++timed;
        }
    }
    if (counted) {
        const double n = static_cast<double>(counted);
        s.mean_abs_eps1 /= n;
        s.mean_abs_eps_f /= n;
        s.mean_abs_eps2 /= n;
        s.win_rate = static_cast<double>(wins) / n;
    }
    s.pearson_eps1_epsf = detail::pearson(e1, ef);
    if (timed) {
        s.mean_flop_fraction = ff / static_cast<double>(timed);
        s.mean_predict_fraction = pf / static_cast<double>(timed);
    }
    return s;
}

// All ordered pairs (self-pairs included); case idx = i * n + j draws its
// seed from fork(cfg.seed, idx); failing cases are recorded, not fatal.
inline BenchOutput run_corpus(const std::vector<NamedMatrix>& ms, const RunConfig& cfg) {
    if (ms.empty()) throw std::invalid_argument("run_corpus: matrix list is empty");
    BenchOutput out;
    Session s(cfg.device);
    const std::size_t n = ms.size();
    for (std::size_t idx = 0; idx < n * n; ++idx) {
        const std::size_t i = idx / n, j = idx % n;
        try {
            const TestCase tc = build_case(ms[i].name, ms[i].matrix, ms[j].name, ms[j].matrix);
            out.cases.push_back(run_case(s, tc, detail::fork_seed(cfg.seed, idx), cfg));
        } catch (const std::exception& e) {
            out.failures.push_back({ms[i].name, ms[j].name, e.what()});
        }
    }
    out.summary = summarize(out.cases, out.failures.size());
    return out;
}

// ---- reports ------------------------------------------------------------
inline std::string render_csv(const BenchOutput& o) {
    std::string csv = "a,b,sample_num,cr,nnz_c,eps1_pct,eps_f_pct,eps2_pct,t_flop_s,t_predict_s,t_exact_s\n";
    for (const CaseResult& c : o.cases) {
        csv += c.a_name + "," + c.b_name + "," + std::to_string(c.sample_num) + "," + detail::g6(c.cr) + "," +
               std::to_string(c.exact_nnz) + "," + detail::g6(c.eps1 * 100.0) + "," +
               detail::g6(c.eps_f * 100.0) + "," + detail::g6(c.eps2 * 100.0) + "," + detail::g6(c.t_flop) +
               "," + detail::g6(c.t_predict) + "," + detail::g6(c.t_exact) + "\n";
    }
    return csv;
}

// JSON laid out like nlohmann's dump(2) of the reference's ordered_json.
inline std::string render_json(const BenchOutput& o) {
    using detail::g6;
    using detail::json_str;
    auto kv = [](const std::string& ind, const std::string& k, const std::string& v, bool last) {
        return ind + json_str(k) + ": " + v + (last ? "\n" : ",\n");
    };
    std::string j = "{\n  \"cases\": ";
    if (o.cases.empty()) {
        j += "[],\n";
    } else {
        j += "[\n";
        for (std::size_t k = 0; k < o.cases.size(); ++k) {
            const CaseResult& c = o.cases[k];
            const std::string in = "      ";
            j += "    {\n";
            j += kv(in, "a", json_str(c.a_name), false);
            j += kv(in, "b", json_str(c.b_name), false);
            j += kv(in, "sample_num", std::to_string(c.sample_num), false);
            j += kv(in, "cr", json_str(g6(c.cr)), false);
            j += kv(in, "nnz_c", std::to_string(c.exact_nnz), false);
            j += kv(in, "eps1_pct", json_str(g6(c.eps1 * 100.0)), false);
            j += kv(in, "eps_f_pct", json_str(g6(c.eps_f * 100.0)), false);
            j += kv(in, "eps2_pct", json_str(g6(c.eps2 * 100.0)), false);
            j += kv(in, "t_flop_s", json_str(g6(c.t_flop)), false);
            j += kv(in, "t_predict_s", json_str(g6(c.t_predict)), false);
            j += kv(in, "t_exact_s", json_str(g6(c.t_exact)), true);
            j += k + 1 < o.cases.size() ? "    },\n" : "    }\n";
        }
        j += "  ],\n";
    }
    j += "  \"failures\": ";
    if (o.failures.empty()) {
        j += "[],\n";
    } else {
        j += "[\n";
        for (std::size_t k = 0; k < o.failures.size(); ++k) {
            const CaseFailure& f = o.failures[k];
            const std::string in = "      ";
            j += "    {\n" + kv(in, "a", json_str(f.a_name), false) + kv(in, "b", json_str(f.b_name), false) +
                 kv(in, "error", json_str(f.message), true);
            j += k + 1 < o.failures.size() ? "    },\n" : "    }\n";
        }
        j += "  ],\n";
    }
    const CorpusSummary& s = o.summary;
    const std::string in = "    ";
    j += "  \"summary\": {\n";
    j += kv(in, "cases_total", std::to_string(s.cases_total), false);
    j += kv(in, "cases_failed", std::to_string(s.cases_failed), false);
    j += kv(in, "cases_degenerate", std::to_string(s.cases_degenerate), false);
    j += kv(in, "mean_abs_eps1_pct", json_str(g6(s.mean_abs_eps1 * 100.0)), false);
    j += kv(in, "mean_abs_eps_f_pct", json_str(g6(s.mean_abs_eps_f * 100.0)), false);
    j += kv(in, "mean_abs_eps2_pct", json_str(g6(s.mean_abs_eps2 * 100.0)), false);
    j += kv(in, "worst_abs_eps1_pct", json_str(g6(s.worst_abs_eps1 * 100.0)), false);
    j += kv(in, "worst_abs_eps_f_pct", json_str(g6(s.worst_abs_eps_f * 100.0)), false);
    j += kv(in, "worst_abs_eps2_pct", json_str(g6(s.worst_abs_eps2 * 100.0)), false);
    j += kv(in, "win_rate", json_str(g6(s.win_rate)), false);
    j += kv(in, "pearson_eps1_epsf", json_str(g6(s.pearson_eps1_epsf)), false);
    j += kv(in, "mean_flop_fraction", json_str(g6(s.mean_flop_fraction)), false);
    j += kv(in, "mean_predict_fraction", json_str(g6(s.mean_predict_fraction)), true);
    j += "  }\n}\n";
    return j;
}

// ---- sources ------------------------------------------------------------
inline std::vector<std::string> parse_matrix_list(const std::string& path) {  // bench.hpp:447-462
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open matrix list " + path);
    std::vector<std::string> out;
    for (std::string line; std::getline(in, line);) {
        const std::size_t h = line.find('#');
        if (h != std::string::npos) line.erase(h);
        const std::size_t a = line.find_first_not_of(" \t\r");
        if (a == std::string::npos) continue;
        out.push_back(line.substr(a, line.find_last_not_of(" \t\r") - a + 1));
    }
    return out;
}

inline NamedMatrix resolve_matrix_source(const std::string& src) {  // bench.hpp:464-484
    if (src.rfind("synth:", 0) == 0) {
        const SyntheticSpec spec = parse_synthetic_spec(src);
        return {synthetic_name(spec), generate_synthetic(spec)};
    }
    if (src.size() > 4 && src.compare(src.size() - 4, 4, ".mtx") == 0) {
        std::string stem = src.substr(src.find_last_of('/') == std::string::npos ? 0 : src.find_last_of('/') + 1);
        stem = stem.substr(0, stem.size() - 4);
        return {stem, read_matrix_market(src)};
    }
    const std::size_t slash = src.find('/');
    if (slash == std::string::npos || slash == 0 || slash + 1 >= src.size())
        throw std::runtime_error("unrecognized matrix source '" + src + "' (want synth:..., *.mtx, or group/name)");
    throw std::runtime_error("SuiteSparse entry '" + src +
                             "' needs the network (fetch.hpp); download the .mtx and list its path");
}

inline std::vector<NamedMatrix> default_corpus() {  // bench.hpp:496-517
    using M = SyntheticModel;
    const SyntheticSpec specs[] = {
        {20000, 20000, M::uniform, 3.0, 101, 0, 1.0},    {12000, 12000, M::uniform, 8.0, 102, 0, 1.0},
        {6000, 6000, M::uniform, 25.0, 103, 0, 1.0},     {4000, 4000, M::uniform, 40.0, 104, 0, 1.0},
        {3000, 3000, M::uniform, 60.0, 105, 0, 1.0},     {8000, 2000, M::uniform, 50.0, 106, 0, 1.0},
        {8000, 1000, M::uniform, 55.0, 107, 0, 1.0},     {10000, 10000, M::banded, 10.0, 110, 50, 1.0},
        {12000, 12000, M::banded, 18.0, 113, 30, 1.0},   {6000, 300, M::uniform, 77.0, 109, 0, 1.0},
        {15000, 15000, M::power_law, 6.0, 111, 0, 0.9}, {9000, 9000, M::power_law, 15.0, 112, 0, 0.7},
    };
    std::vector<NamedMatrix> out;
    for (const SyntheticSpec& s : specs) out.push_back({synthetic_name(s), generate_synthetic(s)});
    return out;
}

}  // namespace spnnz::gpu
