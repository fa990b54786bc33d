// pytext.h -- Python's int() / float() / repr(float) for the native text readers and writers
// (wfst_text.cpp, lattice_text.cpp), so native parsing and formatting reproduce the
// reference's pure-Python behaviour byte for byte.
#pragma once
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

namespace pytext {

inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// Copy a digit run that may contain single underscores between digits (PEP 515) into `out`
// without them; false if an underscore is misplaced.  Returns the end of the run in *stop.
inline bool digit_run(const char *b, const char *e, std::string &out, const char **stop) {
    const char *q = b;
    bool last_digit = false;
    while (q < e) {
        if (is_digit(*q)) {
            out.push_back(*q);
            last_digit = true;
        } else if (*q == '_') {
            if (!last_digit || q + 1 >= e || !is_digit(q[1])) return false;
            last_digit = false;
        } else {
            break;
        }
        ++q;
    }
    *stop = q;
    return true;
}

// Python int(token) for a token without surrounding whitespace (|value| < 1e18).
inline bool py_int(const char *b, const char *e, long long *v) {
    {   // fast path: [sign] 1-18 plain digits
        const char *q = b;
        const bool ng = q < e && *q == '-';
        if (q < e && (*q == '+' || *q == '-')) ++q;
        if (q < e && e - q <= 18) {
            long long x = 0;
            const char *t = q;
            while (t < e && is_digit(*t)) x = x * 10 + (*t++ - '0');
            if (t == e) { *v = ng ? -x : x; return true; }
        }
    }
    bool neg = false;
    if (b < e && (*b == '+' || *b == '-')) neg = *b++ == '-';
    std::string digits;
    const char *stop = b;
    if (b == e || !is_digit(*b) || !digit_run(b, e, digits, &stop) || stop != e) return false;
    if (digits.size() > 18) return false;
    long long x = std::strtoll(digits.c_str(), nullptr, 10);
    *v = neg ? -x : x;
    return true;
}

inline bool ieq(const char *b, const char *e, const char *word) {
    const size_t n = std::strlen(word);
    if ((size_t)(e - b) != n) return false;
    for (size_t i = 0; i < n; ++i)
        if ((b[i] | 0x20) != word[i]) return false;
    return true;
}

// Python float(token): [sign] (inf | infinity | nan | decimal), decimal =
// (digits [. [digits]] | . digits) [(e|E) [sign] digits], underscores between digits;
// correctly rounded (strtod), like CPython.
inline bool py_float(const char *b, const char *e, double *v) {
    {   // fast path: no underscores, letters only as the exponent mark -> from_chars (also
        // correctly rounded); anything it does not consume exactly takes the full path
        bool plain = b < e;
        for (const char *t = b; t < e && plain; ++t)
            plain = is_digit(*t) || *t == '.' || *t == 'e' || *t == 'E' || *t == '+' || *t == '-';
        if (plain) {
            const char *q = b;
            const bool ng = *q == '-';
            if (*q == '+' || *q == '-') ++q;
            if (q < e && *q != '+' && *q != '-') {
                double x;
                const auto r = std::from_chars(q, e, x, std::chars_format::general);
                if (r.ec == std::errc() && r.ptr == e) { *v = ng ? -x : x; return true; }
            }
        }
    }
    std::string s;
    if (b < e && (*b == '+' || *b == '-')) s.push_back(*b++);
    if (ieq(b, e, "inf") || ieq(b, e, "infinity")) {
        *v = s == "-" ? -INFINITY : INFINITY;
        return true;
    }
    if (ieq(b, e, "nan")) {
        *v = NAN;
        return true;
    }
    const char *q = b;
    bool mant = false;
    if (q < e && is_digit(*q)) {
        if (!digit_run(q, e, s, &q)) return false;
        mant = true;
    }
    if (q < e && *q == '.') {
        s.push_back('.');
        ++q;
        if (q < e && is_digit(*q)) {
            if (!digit_run(q, e, s, &q)) return false;
            mant = true;
        }
    }
    if (!mant) return false;
    if (q < e && (*q == 'e' || *q == 'E')) {
        s.push_back('e');
        ++q;
        if (q < e && (*q == '+' || *q == '-')) s.push_back(*q++);
        if (q == e || !is_digit(*q) || !digit_run(q, e, s, &q)) return false;
    }
    if (q != e) return false;
    *v = std::strtod(s.c_str(), nullptr);
    return true;
}

// repr(float): the shortest digits that round-trip, fixed notation for decimal exponents in
// [-4, 16), else d.ddde+XX; always a '.0' on integral fixed values.  Writes at p (at most 32
// bytes) and returns the end.
inline char *py_repr_to(double x, char *p) {
    if (std::isnan(x)) { std::memcpy(p, "nan", 3); return p + 3; }
    if (std::isinf(x)) {
        if (x > 0) { std::memcpy(p, "inf", 3); return p + 3; }
        std::memcpy(p, "-inf", 4);
        return p + 4;
    }
    char buf[48];
    const auto r = std::to_chars(buf, buf + sizeof buf - 1, x, std::chars_format::scientific);
    *r.ptr = '\0';   // to_chars does not terminate; the exponent is read with atoi
    const char *q = buf, *end = r.ptr;
    if (*q == '-') { *p++ = '-'; ++q; }
    const char *ep = (const char *)std::memchr(q, 'e', end - q);
    char digits[24];
    int nd = 0;
    for (const char *t = q; t < ep; ++t)
        if (*t != '.') digits[nd++] = *t;
    const int ex = std::atoi(ep + 1);
    if (ex >= -4 && ex < 16) {
        if (ex >= 0) {
            if (nd <= ex + 1) {
                std::memcpy(p, digits, nd);
                p += nd;
                for (int z = 0; z < ex + 1 - nd; ++z) *p++ = '0';
                *p++ = '.';
                *p++ = '0';
            } else {
                std::memcpy(p, digits, ex + 1);
                p += ex + 1;
                *p++ = '.';
                std::memcpy(p, digits + ex + 1, nd - ex - 1);
                p += nd - ex - 1;
            }
        } else {
            *p++ = '0';
            *p++ = '.';
            for (int z = 0; z < -ex - 1; ++z) *p++ = '0';
            std::memcpy(p, digits, nd);
            p += nd;
        }
    } else {
        *p++ = digits[0];
        if (nd > 1) {
            *p++ = '.';
            std::memcpy(p, digits + 1, nd - 1);
            p += nd - 1;
        }
        const int ax = ex < 0 ? -ex : ex;
        *p++ = 'e';
        *p++ = ex < 0 ? '-' : '+';
        if (ax < 10) *p++ = '0';
        p = std::to_chars(p, p + 8, ax).ptr;
    }
    return p;
}

inline void py_repr(double x, std::string &out) {
    char b[40];
    out.append(b, py_repr_to(x, b));
}

inline std::string py_repr(double x) {
    std::string s;
    py_repr(x, s);
    return s;
}

}  // namespace pytext
