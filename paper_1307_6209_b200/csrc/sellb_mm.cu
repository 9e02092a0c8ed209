// sellb_mm.cu -- Matrix Market body text <-> numbers on the host, multi-threaded
// (the ingestion step in front of the device build).
//
// Replaces the reference's np.loadtxt batches (io.py:125-162) and np.savetxt
// batches (io.py:252-259).  Host code only; no CUDA.
//
// Parse: the same result as np.loadtxt(fh, dtype=float64, comments="%") for
// well-formed text -- '%' starts a comment, blank lines are skipped, tokens are
// separated by ASCII whitespace, every value converted with strtod in the C
// locale (correctly rounded, like NumPy's conversion).  Anything the fast path
// does not recognise -- a token outside the plain decimal / inf / nan
// grammar, a wrong token count, a lone CR, a non-ASCII byte, more entries than
// declared -- returns SELLB_EFORMAT, and the caller re-reads the text
// with the reference-compatible slow path, which raises the reference's exact
// FormatError (or accepts what NumPy accepts).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <charconv>
#include <thread>
#include <vector>

#include "sellb_internal.cuh"

namespace {

inline bool is_ws(unsigned char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }
inline bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

inline bool ieq(const char* a, const char* b, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        char c = a[i];
        if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
        if (c != b[i]) return false;
    }
    return true;
}

// plain decimal: [+-]? (d+ (. d*)? | . d+) ([eE] [+-]? d+)?  or [+-]? inf|infinity|nan
bool token_ok(const char* t, size_t n) {
    size_t i = 0;
    if (i < n && (t[i] == '+' || t[i] == '-')) ++i;
    if (n - i == 3 && (ieq(t + i, "inf", 3) || ieq(t + i, "nan", 3))) return true;
    if (n - i == 8 && ieq(t + i, "infinity", 8)) return true;
    size_t d0 = i;
    while (i < n && is_digit((unsigned char)t[i])) ++i;
    size_t nd = i - d0;
    if (i < n && t[i] == '.') {
        ++i;
        size_t f0 = i;
        while (i < n && is_digit((unsigned char)t[i])) ++i;
        nd += i - f0;
    }
    if (nd == 0) return false;
    if (i < n && (t[i] == 'e' || t[i] == 'E')) {
        ++i;
        if (i < n && (t[i] == '+' || t[i] == '-')) ++i;
        size_t e0 = i;
        while (i < n && is_digit((unsigned char)t[i])) ++i;
        if (i == e0) return false;
    }
    return i == n;
}

// parse [b, e) (whole lines) into out; false = needs the slow path
bool parse_range(const char* b, const char* e, int width, std::vector<double>& out) {
    char buf[128];
    const char* p = b;
    while (p < e) {
        const char* eol = (const char*)memchr(p, '\n', (size_t)(e - p));
        if (!eol) eol = e;
        const char* q = p;
        const char* stop = eol;
        const char* pc = (const char*)memchr(p, '%', (size_t)(eol - p));
        if (pc) stop = pc;
        int ntok = 0;
        while (q < stop) {
            while (q < stop && is_ws((unsigned char)*q)) {
                // a CR not directly before the LF is a line break for Python's
                // universal newlines: leave that to the slow path
                if (*q == '\r' && !(q + 1 == eol && eol < e)) return false;
                ++q;
            }
            if (q >= stop) break;
            const char* t0 = q;
            while (q < stop && !is_ws((unsigned char)*q)) {
                if ((unsigned char)*q >= 0x80) return false;
                ++q;
            }
            const size_t n = (size_t)(q - t0);
            if (ntok >= width || n >= sizeof(buf) || !token_ok(t0, n)) return false;
            memcpy(buf, t0, n);
            buf[n] = 0;
            out.push_back(strtod(buf, nullptr));
            ++ntok;
        }
        if (pc) {                          // comment text: only a lone CR matters
            for (const char* c = pc; c < eol; ++c) {
                if (*c == '\r' && !(c + 1 == eol && eol < e)) return false;
            }
        }
        if (ntok != 0 && ntok != width) return false;
        p = eol < e ? eol + 1 : e;
    }
    return true;
}

int set_error_fallback() {
    return sellb::set_error(SELLB_EFORMAT, "matrix market text outside the fast-path grammar");
}

// "%d %d %.17g\n" of (row + 1, col + 1, val), as np.savetxt writes it (Python
// %-formatting: NaN of either sign prints "nan").  std::to_chars with a
// precision is specified as printf's %.*g in the C locale, without printf's
// locale lookups and multi-precision scratch allocations (snprintf ran no
// faster on 8 threads than on 1).
size_t format_line(char* o, int64_t r, int64_t c, double v) {
    char* p = std::to_chars(o, o + 24, (long long)(r + 1)).ptr;
    *p++ = ' ';
    p = std::to_chars(p, p + 24, (long long)(c + 1)).ptr;
    *p++ = ' ';
    if (v != v) {
        memcpy(p, "nan", 3);
        p += 3;
    } else {
        p = std::to_chars(p, p + 40, v, std::chars_format::general, 17).ptr;
    }
    *p++ = '\n';
    return (size_t)(p - o);
}

}  // namespace

extern "C" {

int sellb_mm_parse_body(const char* text, int64_t len, int32_t width, int64_t max_entries,
                        double* out, int64_t* n_entries, int32_t n_threads) {
    sellb::clear_error();
    if (!n_entries || width < 1 || len < 0 || (len && !text) || max_entries < 0)
        return sellb::set_error(SELLB_EPARAM, "bad arguments to sellb_mm_parse_body");
    *n_entries = 0;
    int T = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = (int)std::min<int64_t>(T, std::max<int64_t>(1, len / (1 << 20)));   // >= 1 MiB each
    std::vector<const char*> cut(T + 1);
    cut[0] = text;
    cut[T] = text + len;
    for (int i = 1; i < T; ++i) {
        const char* c = text + len * i / T;
        if (c < cut[i - 1]) c = cut[i - 1];
        const char* nl = (const char*)memchr(c, '\n', (size_t)(text + len - c));
        cut[i] = nl ? nl + 1 : text + len;
    }
    std::vector<std::vector<double>> parts(T);
    std::vector<char> ok(T, 1);
    std::vector<std::thread> th;
    for (int i = 0; i < T; ++i)
        th.emplace_back([&, i] {
            parts[i].reserve((size_t)((cut[i + 1] - cut[i]) / 8));
            ok[i] = parse_range(cut[i], cut[i + 1], width, parts[i]);
        });
    for (auto& t : th) t.join();
    int64_t total = 0;
    for (int i = 0; i < T; ++i) {
        if (!ok[i]) return set_error_fallback();
        total += (int64_t)parts[i].size();
    }
    if (total % width) return set_error_fallback();
    if (total / width > max_entries) return set_error_fallback();
    int64_t off = 0;
    for (int i = 0; i < T; ++i) {
        if (!parts[i].empty()) memcpy(out + off, parts[i].data(), parts[i].size() * 8);
        off += (int64_t)parts[i].size();
    }
    *n_entries = total / width;
    return 0;
}

// Body lines of write_matrix_market (io.py:252-259) into out (capacity cap
// bytes; 64 per entry always suffices); *used = bytes written.
int sellb_mm_format_body(const int64_t* rows, const int64_t* cols, const double* vals,
                         int64_t n, char* out, int64_t cap, int64_t* used, int32_t n_threads) {
    sellb::clear_error();
    if (!used || n < 0 || (n && (!rows || !cols || !vals || !out)))
        return sellb::set_error(SELLB_EPARAM, "bad arguments to sellb_mm_format_body");
    *used = 0;
    int T = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = (int)std::min<int64_t>(T, std::max<int64_t>(1, n / 65536));
    std::vector<std::vector<char>> parts(T);
    std::vector<std::thread> th;
    for (int i = 0; i < T; ++i)
        th.emplace_back([&, i] {
            const int64_t a = n * i / T, b = n * (i + 1) / T;
            std::vector<char>& o = parts[i];
            o.resize((size_t)(b - a) * 64 + 64);
            size_t k = 0;
            for (int64_t e = a; e < b; ++e) k += format_line(o.data() + k, rows[e], cols[e], vals[e]);
            o.resize(k);
        });
    for (auto& t : th) t.join();
    int64_t total = 0;
    for (auto& p : parts) total += (int64_t)p.size();
    if (total > cap) return sellb::set_error(SELLB_EPARAM, "output buffer too small");
    int64_t off = 0;
    for (auto& p : parts) {
        if (!p.empty()) memcpy(out + off, p.data(), p.size());
        off += (int64_t)p.size();
    }
    *used = total;
    return 0;
}

}  // extern "C"
