// Deterministic synthetic CSR generators for the five BASELINE.json configs.
//
// Input plumbing only (not on the predictor path, never timed).  Every row
// draws from its own SplitMix64 substream fork(seed, row) -- the same scheme
// the reference's generator uses (proj/include/spnnz/synthetic.hpp:123) -- so
// the output is identical for any thread count.  Structure only: no values.
//
//   poisson_uniform  cfg 1: Poisson(mean) lengths clipped to [lo,hi], uniform
//                    distinct sorted columns (Floyd, cf. synthetic.hpp:54-69)
//   rmat             cfg 2, 5: R-MAT generated row by row.  Row i receives
//                    Poisson(E * P(i)) draws, P(i) = prod over levels of
//                    (a+b | c+d); each draw's column bits follow the row bit
//                    (P(1|0) = b/(a+b), P(1|1) = d/(c+d)); duplicates removed.
//                    This is the R-MAT edge distribution with the multinomial
//                    over rows replaced by independent Poisson row counts.
//   stencil27        cfg 3: 27-point stencil, x-fastest natural ordering
//   uniform_len      cfg 4 A: lengths U[lo,hi], uniform distinct columns
//   geometric        cfg 4 B: Geometric(mean) lengths on {1,2,..}, uniform cols
//   random_pattern   restatement of the reference test helper
//                    proj/tests/oracle.hpp:63-74 (+ csr.hpp:46-100 assembly)
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

struct Rng {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    uint64_t next_below(uint64_t bound) {
        return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * bound) >> 64);
    }
    static Rng fork(uint64_t seed, uint64_t tag) {
        Rng m{seed ^ (tag * 0xd1b54a32d192ed03ULL)};
        return Rng{m.next()};
    }
};

int64_t poisson(double lambda, Rng& r) {
    int64_t total = 0;
    while (lambda > 0.0) {
        const double chunk = std::min(lambda, 30.0);
        lambda -= chunk;
        const double limit = std::exp(-chunk);
        double prod = r.next_double();
        while (prod > limit) {
            ++total;
            prod *= r.next_double();
        }
    }
    return total;
}

// k distinct values from [0, range), sorted (Floyd's algorithm; k small).
void distinct(int32_t range, int32_t k, Rng& r, std::vector<int32_t>& out) {
    out.clear();
    if (k > range) k = range;
    if (k <= 64) {
        for (int32_t j = range - k; j < range; ++j) {
            const int32_t t = static_cast<int32_t>(r.next_below(static_cast<uint64_t>(j) + 1));
            if (std::find(out.begin(), out.end(), t) == out.end())
                out.push_back(t);
            else
                out.push_back(j);
        }
    } else {  // same draws, a hash set for the membership test
        std::unordered_set<int32_t> seen;
        seen.reserve(static_cast<size_t>(k) * 2);
        for (int32_t j = range - k; j < range; ++j) {
            const int32_t t = static_cast<int32_t>(r.next_below(static_cast<uint64_t>(j) + 1));
            const int32_t v = seen.insert(t).second ? t : j;
            if (v == j) seen.insert(j);
            out.push_back(v);
        }
    }
    std::sort(out.begin(), out.end());
}

int resolve(int threads) {
    if (threads > 0) return threads;
    unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : static_cast<int>(hw);
}

}  // namespace

extern "C" {

typedef struct {
    int32_t rows;
    int32_t cols;
    int64_t nnz;
    int64_t* rpt;
    int32_t* col;
} spnnz_gen_csr;

void spnnz_gen_free(spnnz_gen_csr* m) {
    if (!m) return;
    std::free(m->rpt);
    std::free(m->col);
    m->rpt = nullptr;
    m->col = nullptr;
}

}  // extern "C"

namespace {

// Row-parallel builder: row_fn(i, rng_out_vector) appends row i's sorted,
// distinct columns.  Blocks of rows per thread, then a prefix sum + copy.
template <typename RowFn>
int build_rows(int32_t rows, int32_t cols, int threads, spnnz_gen_csr* out, RowFn&& row_fn) {
    out->rows = rows;
    out->cols = cols;
    out->rpt = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (static_cast<size_t>(rows) + 1)));
    if (!out->rpt) return 2;
    const int w = std::max(1, std::min<int>(resolve(threads), std::max(rows, 1)));
    std::vector<std::vector<int32_t>> chunk(w);
    std::vector<std::thread> pool;
    auto work = [&](int t) {
        const int64_t b = int64_t(rows) * t / w, e = int64_t(rows) * (t + 1) / w;
        std::vector<int32_t> tmp;
        auto& dst = chunk[t];
        for (int64_t i = b; i < e; ++i) {
            tmp.clear();
            row_fn(static_cast<int32_t>(i), tmp);
            out->rpt[i + 1] = static_cast<int64_t>(tmp.size());
            dst.insert(dst.end(), tmp.begin(), tmp.end());
        }
    };
    for (int t = 1; t < w; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    out->rpt[0] = 0;
    for (int64_t i = 0; i < rows; ++i) out->rpt[i + 1] += out->rpt[i];
    out->nnz = out->rpt[rows];
    out->col = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(out->nnz, 1))));
    if (!out->col) return 2;
    std::vector<std::thread> pool2;
    auto copy = [&](int t) {
        const int64_t b = int64_t(rows) * t / w;
        if (!chunk[t].empty())
            std::memcpy(out->col + out->rpt[b], chunk[t].data(), chunk[t].size() * 4);
        std::vector<int32_t>().swap(chunk[t]);
    };
    for (int t = 1; t < w; ++t) pool2.emplace_back(copy, t);
    copy(0);
    for (auto& th : pool2) th.join();
    return 0;
}

}  // namespace

extern "C" {

// The reference's synthetic corpus model (synthetic.hpp:92-154): model 0
// uniform, 1 banded, 2 power-law.  Per row: its own fork(seed, row) stream, a
// Poisson(target_i) count by chunked products of uniforms, then that many
// distinct columns (Floyd) in the row's window -- all columns, or the band
// around the scaled diagonal.  Power-law rows scale the target by
// (i+1)^-skew / sum_k (k+1)^-skew * rows (the sum taken in row order, as the
// reference does, so the doubles agree).  Rows are built in parallel.
// Returns 3 for an infeasible spec (the reference's invalid_argument).
int spnnz_gen_synthetic(int model, int32_t rows, int32_t cols, double target, uint64_t seed,
                        int32_t bandwidth, double skew, int threads, spnnz_gen_csr* out) {
    if (rows < 0 || cols < 0) return 3;
    if (target < 0 || target > static_cast<double>(cols)) return 3;
    const int32_t band = bandwidth > 0 ? bandwidth
                                       : static_cast<int32_t>(std::max(16.0, 4.0 * std::ceil(target)));
    double wsum = 0.0;
    if (model == 2)
        for (int32_t i = 0; i < rows; ++i) wsum += std::pow(static_cast<double>(i) + 1.0, -skew);
    return build_rows(rows, cols, threads, out, [&](int32_t i, std::vector<int32_t>& v) {
        Rng r = Rng::fork(seed, static_cast<uint64_t>(i));
        double t = target;
        if (model == 2 && wsum > 0.0)
            t = target * static_cast<double>(rows) * std::pow(static_cast<double>(i) + 1.0, -skew) / wsum;
        int64_t k = poisson(t, r);
        int32_t lo = 0, range = cols;
        if (model == 1) {
            const int32_t center = rows > 0 ? static_cast<int32_t>((static_cast<int64_t>(i) * cols) / rows) : 0;
            lo = std::max<int32_t>(0, center - band);
            range = std::min<int32_t>(cols, center + band + 1) - lo;
        }
        if (k > range) k = range;
        distinct(range, static_cast<int32_t>(k), r, v);
        for (auto& c : v) c += lo;
    });
}

// cfg 1
int spnnz_gen_poisson_uniform(int32_t rows, int32_t cols, double mean, int32_t lo, int32_t hi,
                              uint64_t seed, int threads, spnnz_gen_csr* out) {
    return build_rows(rows, cols, threads, out, [&](int32_t i, std::vector<int32_t>& v) {
        Rng r = Rng::fork(seed, static_cast<uint64_t>(i));
        int64_t k = poisson(mean, r);
        k = std::clamp<int64_t>(k, lo, hi);
        distinct(cols, static_cast<int32_t>(k), r, v);
    });
}

// cfg 2, 5
int spnnz_gen_rmat(int log2n, int64_t draws, double a, double b, double c, uint64_t seed,
                   int threads, spnnz_gen_csr* out) {
    const double d = 1.0 - a - b - c;
    const int32_t n = int32_t(1) << log2n;
    const double p_top = a + b, p_bot = c + d;
    // Column bits are drawn 8 levels per 64-bit draw: byte k of draw g decides
    // level 8g+k with a 7-bit uniform compared against a 7-bit threshold
    // round(128 * P(col bit = 1 | row bit)), evaluated branch-free (SWAR).
    const uint64_t t0 = static_cast<uint64_t>(std::lround(std::ldexp(b / (a + b), 7)));
    const uint64_t t1 = static_cast<uint64_t>(std::lround(std::ldexp(d / (c + d), 7)));
    const int groups = (log2n + 7) / 8;
    constexpr uint64_t kLow7 = 0x7f7f7f7f7f7f7f7fULL, kHigh = 0x8080808080808080ULL,
                       kOnes = 0x0101010101010101ULL, kGather = 0x0102040810204080ULL;
    return build_rows(n, n, threads, out, [&](int32_t i, std::vector<int32_t>& v) {
        double pr = 1.0;
        for (int l = log2n - 1; l >= 0; --l) pr *= ((i >> l) & 1) ? p_bot : p_top;
        uint64_t thr[4] = {0, 0, 0, 0};  // packed per-level thresholds (0 above log2n)
        for (int l = 0; l < log2n; ++l)
            thr[l >> 3] |= (((i >> l) & 1) ? t1 : t0) << (8 * (l & 7));
        Rng r = Rng::fork(seed, static_cast<uint64_t>(i));
        const int64_t k = poisson(static_cast<double>(draws) * pr, r);
        v.resize(static_cast<size_t>(k));
        for (int64_t e = 0; e < k; ++e) {
            uint32_t col = 0;
            for (int g = 0; g < groups; ++g) {
                const uint64_t x = r.next() & kLow7;
                // high bit of byte k set  <=>  x_k < t_k   (127 + t - x in [0, 254])
                const uint64_t lt = (((thr[g] | kHigh) - x - kOnes) & kHigh) >> 7;
                col |= static_cast<uint32_t>((lt * kGather) >> 56) << (8 * g);
            }
            v[static_cast<size_t>(e)] = static_cast<int32_t>(col);
        }
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
    });
}

// cfg 3
int spnnz_gen_stencil27(int32_t nx, int32_t ny, int32_t nz, int threads, spnnz_gen_csr* out) {
    const int64_t total = int64_t(nx) * ny * nz;
    if (total > INT32_MAX) return 1;
    return build_rows(static_cast<int32_t>(total), static_cast<int32_t>(total), threads, out,
                      [&](int32_t i, std::vector<int32_t>& v) {
                          const int32_t x = i % nx, y = (i / nx) % ny, z = i / (nx * ny);
                          for (int dz = -1; dz <= 1; ++dz)
                              for (int dy = -1; dy <= 1; ++dy)
                                  for (int dx = -1; dx <= 1; ++dx) {
                                      const int32_t X = x + dx, Y = y + dy, Z = z + dz;
                                      if (X < 0 || Y < 0 || Z < 0 || X >= nx || Y >= ny || Z >= nz)
                                          continue;
                                      v.push_back((Z * ny + Y) * nx + X);
                                  }
                      });
}

// cfg 4 A
int spnnz_gen_uniform_len(int32_t rows, int32_t cols, int32_t lo, int32_t hi, uint64_t seed,
                          int threads, spnnz_gen_csr* out) {
    return build_rows(rows, cols, threads, out, [&](int32_t i, std::vector<int32_t>& v) {
        Rng r = Rng::fork(seed, static_cast<uint64_t>(i));
        const int32_t k = lo + static_cast<int32_t>(r.next_below(static_cast<uint64_t>(hi - lo + 1)));
        distinct(cols, k, r, v);
    });
}

// cfg 4 B
int spnnz_gen_geometric(int32_t rows, int32_t cols, double mean, uint64_t seed, int threads,
                        spnnz_gen_csr* out) {
    const double p = 1.0 / mean;
    return build_rows(rows, cols, threads, out, [&](int32_t i, std::vector<int32_t>& v) {
        Rng r = Rng::fork(seed, static_cast<uint64_t>(i));
        int32_t k = 1;
        while (r.next_double() >= p && k < cols) ++k;
        distinct(cols, k, r, v);
    });
}

// proj/tests/oracle.hpp:63-74: target = density*rows*cols triplets drawn
// with next_below from the caller's stream, assembled like from_triplets
// (sorted, duplicates collapsed).  *state advances exactly as the reference.
int spnnz_gen_random_pattern(int32_t rows, int32_t cols, double density, uint64_t* state,
                             spnnz_gen_csr* out) {
    Rng r{*state};
    const size_t target = static_cast<size_t>(density * rows * cols);
    std::vector<std::vector<int32_t>> per(static_cast<size_t>(std::max(rows, 0)));
    for (size_t e = 0; e < target; ++e) {
        const int32_t rr = static_cast<int32_t>(r.next_below(static_cast<uint64_t>(rows)));
        const int32_t cc = static_cast<int32_t>(r.next_below(static_cast<uint64_t>(cols)));
        per[rr].push_back(cc);
    }
    *state = r.s;
    return build_rows(rows, cols, 1, out, [&](int32_t i, std::vector<int32_t>& v) {
        v = per[i];
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
    });
}

}  // extern "C"
