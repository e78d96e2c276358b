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
