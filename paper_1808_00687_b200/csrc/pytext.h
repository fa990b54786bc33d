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
// [-4, 16), else d.ddde+XX; always a '.0' on integral fixed values.
inline void py_repr(double x, std::string &out) {
    if (std::isnan(x)) { out += "nan"; return; }
    if (std::isinf(x)) { out += x > 0 ? "inf" : "-inf"; return; }
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf - 1, x, std::chars_format::scientific);
    *r.ptr = '\0';   // to_chars does not terminate; the exponent is read with atoi
    const char *p = buf, *end = r.ptr;
    if (*p == '-') { out.push_back('-'); ++p; }
    const char *ep = (const char *)std::memchr(p, 'e', end - p);
    std::string digits;
    for (const char *q = p; q < ep; ++q)
        if (*q != '.') digits.push_back(*q);
    const int ex = std::atoi(ep + 1);
    const int nd = (int)digits.size();
    if (ex >= -4 && ex < 16) {
        if (ex >= 0) {
            if (nd <= ex + 1) {
                out += digits;
                out.append((size_t)(ex + 1 - nd), '0');
                out += ".0";
            } else {
                out.append(digits, 0, (size_t)ex + 1);
                out.push_back('.');
                out.append(digits, (size_t)ex + 1, std::string::npos);
            }
        } else {
            out += "0.";
            out.append((size_t)(-ex - 1), '0');
            out += digits;
        }
    } else {
        out.push_back(digits[0]);
        if (nd > 1) {
            out.push_back('.');
            out.append(digits, 1, std::string::npos);
        }
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
        out += eb;
    }
}

inline std::string py_repr(double x) {
    std::string s;
    py_repr(x, s);
    return s;
}

}  // namespace pytext
