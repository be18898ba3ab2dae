// Matrix Market ingestion: the structure of a coordinate
// Matrix Market file as CSR, restating spnnz::read_matrix_market
// (proj/include/spnnz/matrix_market.hpp:89-196) + from_triplets (csr.hpp:
// 41-96) for structure-only use (values are never read by the predictor):
//   * header "%%MatrixMarket matrix coordinate <field> <symmetry>", case
//     insensitive; field real|integer|pattern|complex, symmetry general|
//     symmetric|skew-symmetric|hermitian (the last three mirrored);
//   * comment / blank lines before the size line and between entries;
//   * 1-based indices checked against the declared size; values parsed (and
//     discarded) as the reference does, numbers with strtoll / strtod on the
//     same text, so malformed input fails on the same line with the same
//     message ("<what> (line N)");
//   * duplicates collapse; columns sorted per row.
// Assembly is parallel: per-thread row histograms, a scatter into row
// buckets, then per-row sort + unique.  And the writer (pattern, general).
#include <algorithm>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

struct MmError {
    std::string what;
    long line;
};

struct Scan {
    const char* p;
    const char* end;
    long line = 1;

    void blanks() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    }
    // to the start of the next line; false at the end of the text
    bool newline() {
        const void* nl = p < end ? std::memchr(p, '\n', static_cast<size_t>(end - p)) : nullptr;
        if (!nl) {
            p = end;
            return false;
        }
        p = static_cast<const char*>(nl) + 1;
        ++line;
        return p < end;
    }
    long long integer() {
        blanks();
        char* q = nullptr;
        const long long v = std::strtoll(p, &q, 10);
        if (q == p) throw MmError{"expected integer", line};
        p = q;
        return v;
    }
    void real() {
        blanks();
        char* q = nullptr;
        (void)std::strtod(p, &q);
        if (q == p) throw MmError{"expected numeric value", line};
        p = q;
    }
    void line_end() {
        blanks();
        if (p < end && *p != '\n') throw MmError{"trailing characters on line", line};
    }
    // skips comment and blank lines; false at the end of the text
    bool content() {
        for (;;) {
            blanks();
            if (p >= end) return false;
            if (*p != '%' && *p != '\n') return true;
            if (!newline()) return false;
        }
    }
};

std::string lower(const char* s) {
    std::string o(s);
    for (char& c : o) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return o;
}

int workers(int threads) {
    if (threads > 0) return threads;
    const unsigned h = std::thread::hardware_concurrency();
    return h ? static_cast<int>(h) : 1;
}

template <typename Fn>
void parallel(int w, Fn&& fn) {
    std::vector<std::thread> pool;
    for (int t = 1; t < w; ++t) pool.emplace_back(fn, t);
    fn(0);
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

typedef struct {
    int32_t rows, cols;
    int64_t nnz;
    int64_t* rpt;
    int32_t* col;
} spnnz_gen_csr;

// 0 ok; 4 parse error (message with the line in err); 5 I/O error; 6 memory.
int spnnz_mm_read(const char* path, int threads, spnnz_gen_csr* out, char* err, int errcap) {
    auto fail = [&](int code, const std::string& msg) {
        if (err && errcap > 0) std::snprintf(err, static_cast<size_t>(errcap), "%s", msg.c_str());
        return code;
    };
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return fail(4, std::string("cannot open ") + path + " (line 0)");
    std::string text;
    {
        std::fseek(f, 0, SEEK_END);
        const long n = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        text.resize(n > 0 ? static_cast<size_t>(n) : 0);
        if (n > 0 && std::fread(&text[0], 1, text.size(), f) != text.size()) {
            std::fclose(f);
            return fail(5, std::string("read failed for ") + path);
        }
        std::fclose(f);
    }
    std::vector<int32_t> tr, tc;  // triplet rows / columns (0-based)
    int32_t rows = 0, cols = 0;
    try {
        Scan s{text.data(), text.data() + text.size()};
        char obj[64] = {0}, fmt[64] = {0}, fld[64] = {0}, sym[64] = {0};
        if (std::sscanf(s.p, "%%%%MatrixMarket %63s %63s %63s %63s", obj, fmt, fld, sym) != 4)
            throw MmError{"malformed MatrixMarket header", s.line};
        if (lower(obj) != "matrix") throw MmError{"unsupported object '" + std::string(obj) + "'", s.line};
        if (lower(fmt) != "coordinate") throw MmError{"unsupported format '" + std::string(fmt) + "'", s.line};
        const std::string field = lower(fld), symmetry = lower(sym);
        int nvals = 0;
        if (field == "real" || field == "integer") nvals = 1;
        else if (field == "complex") nvals = 2;
        else if (field != "pattern") throw MmError{"unsupported field '" + field + "'", s.line};
        bool mirror = true;
        if (symmetry == "general") mirror = false;
        else if (symmetry != "symmetric" && symmetry != "skew-symmetric" && symmetry != "hermitian")
            throw MmError{"unsupported symmetry '" + symmetry + "'", s.line};

        if (!s.newline() || !s.content()) throw MmError{"missing size line", s.line};
        const long long r = s.integer(), c = s.integer(), n = s.integer();
        s.line_end();
        if (r < 0 || c < 0 || n < 0) throw MmError{"negative size declaration", s.line};
        rows = static_cast<int32_t>(r);
        cols = static_cast<int32_t>(c);
        tr.reserve(static_cast<size_t>(mirror ? 2 * n : n));
        tc.reserve(tr.capacity());
        for (long long e = 0; e < n; ++e) {
            if (!s.newline() || !s.content())
                throw MmError{"entry list truncated: expected " + std::to_string(n) + " entries, got " +
                                  std::to_string(e),
                              s.line};
            const long long i = s.integer(), j = s.integer();
            for (int v = 0; v < nvals; ++v) s.real();
            s.line_end();
            if (i < 1 || i > r || j < 1 || j > c)
                throw MmError{"entry (" + std::to_string(i) + ", " + std::to_string(j) + ") outside declared " +
                                  std::to_string(r) + "x" + std::to_string(c),
                              s.line};
            tr.push_back(static_cast<int32_t>(i - 1));
            tc.push_back(static_cast<int32_t>(j - 1));
            if (mirror && i != j) {
                tr.push_back(static_cast<int32_t>(j - 1));
                tc.push_back(static_cast<int32_t>(i - 1));
            }
        }
    } catch (const MmError& e) {
        return fail(4, e.what + " (line " + std::to_string(e.line) + ")");
    }

    // assemble: row histograms per thread -> bucket offsets -> scatter ->
    // per-row sort + unique -> compaction
    const size_t m = tr.size();
    const int w = std::max(1, std::min<int>(workers(threads), static_cast<int>(m / 65536 + 1)));
    std::vector<std::vector<int64_t>> hist(static_cast<size_t>(w), std::vector<int64_t>(static_cast<size_t>(rows) + 1, 0));
    parallel(w, [&](int t) {
        const size_t b = m * t / w, e = m * (t + 1) / w;
        auto& h = hist[static_cast<size_t>(t)];
        for (size_t k = b; k < e; ++k) ++h[static_cast<size_t>(tr[k])];
    });
    std::vector<int64_t> start(static_cast<size_t>(rows) + 1, 0);
    int64_t acc = 0;
    for (int32_t i = 0; i < rows; ++i) {
        start[static_cast<size_t>(i)] = acc;
        for (int t = 0; t < w; ++t) {
            const int64_t c = hist[static_cast<size_t>(t)][static_cast<size_t>(i)];
            hist[static_cast<size_t>(t)][static_cast<size_t>(i)] = acc;  // thread t's cursor
            acc += c;
        }
    }
    start[static_cast<size_t>(rows)] = acc;
    std::vector<int32_t> bucket(m);
    parallel(w, [&](int t) {
        const size_t b = m * t / w, e = m * (t + 1) / w;
        auto& h = hist[static_cast<size_t>(t)];
        for (size_t k = b; k < e; ++k) bucket[static_cast<size_t>(h[static_cast<size_t>(tr[k])]++)] = tc[k];
    });
    std::vector<int64_t> kept(static_cast<size_t>(rows) + 1, 0);
    parallel(w, [&](int t) {
        const int64_t b = int64_t(rows) * t / w, e = int64_t(rows) * (t + 1) / w;
        for (int64_t i = b; i < e; ++i) {
            int32_t* lo = bucket.data() + start[static_cast<size_t>(i)];
            int32_t* hi = bucket.data() + start[static_cast<size_t>(i) + 1];
            std::sort(lo, hi);
            kept[static_cast<size_t>(i) + 1] = std::unique(lo, hi) - lo;
        }
    });
    out->rows = rows;
    out->cols = cols;
    out->rpt = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (static_cast<size_t>(rows) + 1)));
    if (!out->rpt) return fail(6, "out of memory");
    out->rpt[0] = 0;
    for (int32_t i = 0; i < rows; ++i) out->rpt[i + 1] = out->rpt[i] + kept[static_cast<size_t>(i) + 1];
    out->nnz = out->rpt[rows];
    out->col = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(out->nnz, 1))));
    if (!out->col) return fail(6, "out of memory");
    parallel(w, [&](int t) {
        const int64_t b = int64_t(rows) * t / w, e = int64_t(rows) * (t + 1) / w;
        for (int64_t i = b; i < e; ++i)
            std::memcpy(out->col + out->rpt[i], bucket.data() + start[static_cast<size_t>(i)],
                        sizeof(int32_t) * static_cast<size_t>(kept[static_cast<size_t>(i) + 1]));
    });
    return 0;
}

// spnnz::write_matrix_market (matrix_market.hpp:200-211): pattern, general.
int spnnz_mm_write(const char* path, const spnnz_gen_csr* m) {
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return 5;
    std::vector<char> buf;
    buf.reserve(1 << 20);
    auto flush = [&] {
        if (!buf.empty() && std::fwrite(buf.data(), 1, buf.size(), f) != buf.size()) return false;
        buf.clear();
        return true;
    };
    char line[96];
    int n = std::snprintf(line, sizeof(line), "%%%%MatrixMarket matrix coordinate pattern general\n%d %d %lld\n",
                          m->rows, m->cols, static_cast<long long>(m->nnz));
    buf.insert(buf.end(), line, line + n);
    bool ok = true;
    for (int32_t i = 0; i < m->rows && ok; ++i)
        for (int64_t k = m->rpt[i]; k < m->rpt[i + 1]; ++k) {
            n = std::snprintf(line, sizeof(line), "%d %d\n", i + 1, m->col[k] + 1);
            buf.insert(buf.end(), line, line + n);
            if (buf.size() > (1u << 20) && !(ok = flush())) break;
        }
    ok = ok && flush();
    return (std::fclose(f) == 0 && ok) ? 0 : 5;
}

}  // extern "C"
