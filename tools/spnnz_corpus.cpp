// spnnz_corpus -- the corpus harness on the B200 predictor:
// every ordered pair of a matrix list (default: the reference's 12-matrix
// synthetic corpus), exact vs predicted NNZ, CSV / JSON reports in the
// reference's format (include/spnnz_gpu/harness.hpp).
//
//   build/spnnz_corpus [--list FILE] [--csv OUT] [--json OUT] [--seed N]
//                      [--reps N] [--warmup N] [--fraction F] [--cap N]
//                      [--no-timings] [--device D]
//   build/spnnz_corpus --overhead      the reference's overhead criterion
//       (proj/tests/acceptance.cpp:264-294): three synthetic matrices, each
//       with itself, case seed 97, 5 timed runs after 1 warm-up; mean
//       (t_flop + t_predict) / t_exact against its 10 % gate
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "spnnz_gpu/harness.hpp"

int main(int argc, char** argv) {
    using namespace spnnz::gpu;
    RunConfig cfg;
    std::string list, csv, json;
    bool overhead = false;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc) {
                std::fprintf(stderr, "missing value for %s\n", a.c_str());
                std::exit(2);
            }
            return argv[++i];
        };
        if (a == "--list") list = next();
        else if (a == "--csv") csv = next();
        else if (a == "--json") json = next();
        else if (a == "--seed") cfg.seed = std::stoull(next());
        else if (a == "--reps") cfg.repetitions = std::stoi(next());
        else if (a == "--warmup") cfg.warmup = std::stoi(next());
        else if (a == "--fraction") cfg.policy.fraction = std::stod(next());
        else if (a == "--cap") cfg.policy.cap = std::stoll(next());
        else if (a == "--device") cfg.device = std::stoi(next());
        else if (a == "--no-timings") cfg.collect_timings = false;
        else if (a == "--overhead") overhead = true;
        else {
            std::fprintf(stderr, "unknown argument %s\n", a.c_str());
            return 2;
        }
    }
    try {
        if (overhead) {
            // the three specs of acceptance.cpp:266-270, each matrix with itself
            const char* specs[] = {"synth:uniform:150000x150000:nnz=8:seed=71",
                                   "synth:banded:120000x120000:nnz=10:bw=60:seed=72",
                                   "synth:uniform:200000x200000:nnz=6:seed=73"};
            RunConfig oc = cfg;
            oc.repetitions = 5;
            oc.warmup = 1;
            Session s(cfg.device);
            double sum = 0.0;
            for (const char* spec : specs) {
                const NamedMatrix m = resolve_matrix_source(spec);
                const TestCase tc = build_case(m.name, m.matrix, m.name, m.matrix);
                const CaseResult r = run_case(s, tc, 97, oc);
                const double f = (r.t_flop + r.t_predict) / r.t_exact;
                std::printf("  M %d: t_flop %.6fs t_predict %.6fs t_exact %.6fs -> %.2f%%\n", tc.a.rows, r.t_flop,
                            r.t_predict, r.t_exact, f * 100.0);
                sum += f;
            }
            const double mean = sum / 3.0;
            std::printf("%s overhead: mean (t_flop + t_predict)/t_exact = %.2f%% (gate 10%%)\n",
                        mean <= 0.10 ? "PASS" : "FAIL", mean * 100.0);
            return 0;
        }
        std::vector<NamedMatrix> ms;
        if (list.empty()) {
            ms = default_corpus();
        } else {
            for (const std::string& src : parse_matrix_list(list)) ms.push_back(resolve_matrix_source(src));
        }
        const BenchOutput out = run_corpus(ms, cfg);
        auto write = [](const std::string& path, const std::string& text) {
            std::ofstream f(path, std::ios::binary | std::ios::trunc);
            if (!f || !(f << text)) throw std::runtime_error("cannot write report to " + path);
        };
        if (!csv.empty()) write(csv, render_csv(out));
        if (!json.empty()) write(json, render_json(out));
        const CorpusSummary& s = out.summary;
        std::printf("cases %zu (failed %zu, degenerate %zu)\n", s.cases_total, s.cases_failed, s.cases_degenerate);
        std::printf("mean |eps1| %.4g%%  |eps_f| %.4g%%  |eps2| %.4g%%  win rate %.3g  pearson(eps1, eps_f) %.4g\n",
                    s.mean_abs_eps1 * 100, s.mean_abs_eps_f * 100, s.mean_abs_eps2 * 100, s.win_rate,
                    s.pearson_eps1_epsf);
        std::printf("mean t_flop/t_exact %.4g  t_predict/t_exact %.4g\n", s.mean_flop_fraction,
                    s.mean_predict_fraction);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "spnnz_corpus: %s\n", e.what());
        return 1;
    }
    return 0;
}
