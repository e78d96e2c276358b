// Fast text writers for the reference's artifact formats (fileio.py:322-359).
//
// The reference formats every value with Python's f"{float(v):.6g}", one
// node (or U-matrix row) per line, space-separated, LF endings; a cfg2
// codebook is 4e7 values, which the Python formatter needs ~40 s for.  These
// host functions produce the same bytes with std::to_chars(general, 6)
// (= printf "%.6g": correctly rounded, same exponent / trailing-zero rules;
// NaN is spelled "nan" as Python does for either sign) on several threads,
// each formatting a contiguous block of lines into its own buffer.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <charconv>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace {

inline int fmt_g6(char *buf, double v) {
    if (isnan(v)) { memcpy(buf, "nan", 3); return 3; }
    // std::to_chars(general, 6) is specified as printf("%.6g") -- correctly
    // rounded, same exponent and trailing-zero rules -- and much faster
    auto r = std::to_chars(buf, buf + 32, v, std::chars_format::general, 6);
    return (int)(r.ptr - buf);
}

template <class LineFn>
int64_t format_lines(int64_t rows, int threads, char *out, int64_t cap, LineFn line) {
    if (threads < 1) threads = 1;
    if (rows < 4096) threads = 1;
    std::vector<std::string> parts((size_t)threads);
    std::vector<std::thread> pool;
    const int64_t per = (rows + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            const int64_t a = t * per, b = a + per < rows ? a + per : rows;
            std::string &s = parts[(size_t)t];
            for (int64_t r = a; r < b; ++r) line(r, s);
        });
    }
    for (auto &th : pool) th.join();
    int64_t total = 0;
    for (auto &p : parts) total += (int64_t)p.size();
    if (total > cap) return -total;           // caller's buffer too small: -(bytes needed)
    char *o = out;
    for (auto &p : parts) {
        memcpy(o, p.data(), p.size());
        o += p.size();
    }
    return total;
}

}  // namespace

// rows x cols f32, row-major -> "v v v\n" per row (write_codebook body, write_umatrix)
extern "C" int64_t somb_format_f32_rows(const float *v, int64_t rows, int64_t cols, char *out, int64_t cap,
                                        int32_t threads) {
    if (rows <= 0) return 0;
    return format_lines(rows, threads, out, cap, [&](int64_t r, std::string &s) {
        char buf[40];
        s.reserve(s.size() + (size_t)cols * 12);
        for (int64_t c = 0; c < cols; ++c) {
            int k = fmt_g6(buf, (double)v[r * cols + c]);
            s.append(buf, (size_t)k);
            s.push_back(c + 1 < cols ? ' ' : '\n');
        }
        if (cols == 0) s.push_back('\n');
    });
}

// n x 2 int32 [row, col] -> "i row col\n" (write_bmus body)
extern "C" int64_t somb_format_bmus(const int32_t *bm, int64_t n, char *out, int64_t cap, int32_t threads) {
    if (n <= 0) return 0;
    return format_lines(n, threads, out, cap, [&](int64_t i, std::string &s) {
        char buf[64];
        int k = snprintf(buf, sizeof(buf), "%lld %d %d\n", (long long)i, bm[2 * i], bm[2 * i + 1]);
        s.append(buf, (size_t)k);
    });
}

// ------------------------------------------------------------------ ingest
// Dense text (fileio.py:150-229 formats): lines split on '\n' ('\r' is
// whitespace), blank and '#' comment lines skipped, '%' header lines
// reported to the caller, whitespace-separated tokens.  Values parse as
// double (std::from_chars, correctly rounded, as Python's float()) then
// round to float32 -- the reference's np.array(tokens, float32).  Anything
// unusual (a token from_chars does not consume fully, a non-finite value,
// a width mismatch) returns its 1-based line number so the caller re-parses
// with the reference-exact Python path for the error.

namespace {

inline bool is_ws(char ch) { return ch == ' ' || ch == '\t' || ch == '\r' || ch == '\v' || ch == '\f' || (ch >= 0x1c && ch <= 0x1f); }

struct LineRef {
    int64_t begin, end, lineno;
};

// data lines (non-blank, non-comment, not starting with '%') and '%' lines
void split_lines(const char *buf, int64_t len, std::vector<LineRef> &data, std::vector<LineRef> &hdr) {
    int64_t p = 0, lineno = 0;
    while (p < len) {
        int64_t q = p;
        while (q < len && buf[q] != '\n') ++q;
        ++lineno;
        int64_t a = p;
        while (a < q && is_ws(buf[a])) ++a;
        if (a < q && buf[a] != '#') {
            if (buf[a] == '%') hdr.push_back({a, q, lineno});
            else data.push_back({a, q, lineno});
        }
        p = q + 1;
    }
}

inline int64_t count_tokens(const char *buf, const LineRef &l) {
    int64_t n = 0, p = l.begin;
    while (p < l.end) {
        while (p < l.end && is_ws(buf[p])) ++p;
        if (p >= l.end) break;
        ++n;
        while (p < l.end && !is_ws(buf[p])) ++p;
    }
    return n;
}

}  // namespace

// Pass 1: rows / columns of the data lines (columns from the first data
// line), the count of '%' header lines, and the first line whose width
// differs (0 if none).  Returns the number of data rows.
extern "C" int64_t somb_scan_dense_text(const char *buf, int64_t len, int64_t *cols, int64_t *n_headers,
                                        int64_t *bad_line) {
    std::vector<LineRef> data, hdr;
    split_lines(buf, len, data, hdr);
    *n_headers = (int64_t)hdr.size();
    *bad_line = 0;
    *cols = data.empty() ? 0 : count_tokens(buf, data[0]);
    for (const auto &l : data)
        if (count_tokens(buf, l) != *cols) { *bad_line = l.lineno; break; }
    return (int64_t)data.size();
}

// Pass 2: parse rows x cols values into out (row-major f32) on `threads`
// threads; returns 0, or the 1-based line number of the first row that
// needs the reference-exact path (unparsed token, non-finite value).
extern "C" int64_t somb_parse_dense_text(const char *buf, int64_t len, int64_t rows, int64_t cols, float *out,
                                         int32_t threads) {
    std::vector<LineRef> data, hdr;
    split_lines(buf, len, data, hdr);
    if ((int64_t)data.size() != rows) return -1;
    if (threads < 1) threads = 1;
    std::vector<int64_t> bad((size_t)threads, 0);
    std::vector<std::thread> pool;
    const int64_t per = (rows + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            const int64_t a = t * per, b = a + per < rows ? a + per : rows;
            for (int64_t r = a; r < b && !bad[(size_t)t]; ++r) {
                const LineRef &l = data[(size_t)r];
                int64_t p = l.begin, c = 0;
                while (p < l.end) {
                    while (p < l.end && is_ws(buf[p])) ++p;
                    if (p >= l.end) break;
                    int64_t e = p;
                    while (e < l.end && !is_ws(buf[e])) ++e;
                    const char *s = buf + p;
                    if (*s == '+' && e - p > 1 && s[1] != '-' && s[1] != '+') ++s;   // Python accepts one leading '+'
                    double v = 0.0;
                    auto res = std::from_chars(s, buf + e, v);
                    const float f = (float)v;
                    if (res.ec != std::errc() || res.ptr != buf + e || c >= cols || !isfinite(f)) {
                        bad[(size_t)t] = l.lineno;
                        break;
                    }
                    out[r * cols + c++] = f;
                    p = e;
                }
                if (!bad[(size_t)t] && c != cols) bad[(size_t)t] = l.lineno;
            }
        });
    }
    for (auto &th : pool) th.join();
    for (int64_t b : bad)
        if (b) return b;
    return 0;
}
