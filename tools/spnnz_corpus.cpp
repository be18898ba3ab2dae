// spnnz_corpus -- the corpus harness on the B200 predictor:
// every ordered pair of a matrix list (default: the reference's 12-matrix
// synthetic corpus), exact vs predicted NNZ, CSV / JSON reports in the
// reference's format (include/spnnz_gpu/harness.hpp).
//
//   build/spnnz_corpus [--list FILE] [--csv OUT] [--json OUT] [--seed N]
//                      [--reps N] [--warmup N] [--fraction F] [--cap N]
//                      [--no-timings] [--device D]
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "spnnz_gpu/harness.hpp"

int main(int argc, char** argv) {
    using namespace spnnz::gpu;
    RunConfig cfg;
    std::string list, csv, json;
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
        else {
            std::fprintf(stderr, "unknown argument %s\n", a.c_str());
            return 2;
        }
    }
    try {
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
