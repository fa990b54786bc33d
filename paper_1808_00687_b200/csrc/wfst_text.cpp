// wfst_text.cpp -- fast path of parse_wfst_text (reference wfst.py:315-378) for the common case:
// ASCII AT&T text with integer labels.  Arc lines "src dst ilabel olabel [weight]", final lines
// "state [weight]", a missing weight is 0.0, the first state mentioned is the start state,
// '#' starts a comment line, blank lines are ignored, a repeated final line overwrites.
//
// Anything this path does not reproduce bit for bit -- symbols, non-ASCII text, Python's
// numeric extras (underscores, hex), line breaks other than \n / \r\n -- and every malformed
// line make it return WB_PARSE_FALLBACK, and the Python parser then runs on the same text (so
// error messages and exceptions are the reference's).  Decimal weights go through strtod,
// which rounds correctly exactly like Python's float().
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <unordered_map>
#include <vector>

#include "../../include/wfst_b200.h"

namespace {

inline bool ws(char c) { return c == ' ' || c == '\t' || c == '\v' || c == '\f' || c == '\r'; }

// Python int() of an ASCII token without underscores: [+-]?digits
bool parse_int(const char *b, const char *e, long long *v) {
    if (b == e) return false;
    bool neg = false;
    if (*b == '+' || *b == '-') { neg = *b == '-'; ++b; }
    if (b == e) return false;
    long long x = 0;
    for (; b < e; ++b) {
        if (*b < '0' || *b > '9') return false;
        x = x * 10 + (*b - '0');
        if (x > (1ll << 40)) return false;  // far beyond int32: let Python decide
    }
    *v = neg ? -x : x;
    return true;
}

// Python float() of an ASCII decimal token (no underscores, hex or nan payloads)
bool parse_float(const char *b, const char *e, double *v) {
    if (b == e || e - b > 400) return false;
    char buf[512];
    std::memcpy(buf, b, e - b);
    buf[e - b] = 0;
    for (const char *p = buf; *p; ++p)
        if (*p == '_' || *p == 'x' || *p == 'X' || *p == '(' || *p == 'p' || *p == 'P') return false;
    char *end = nullptr;
    errno = 0;
    const double x = std::strtod(buf, &end);
    if (end != buf + (e - b)) return false;
    *v = x;
    return true;
}

}  // namespace

extern "C" {

int wb_wfst_parse_text(const char *text, int64_t len, int32_t allow_negative_weights,
                       wb_parsed_wfst *out) {
    if (!text || !out || len < 0) return WB_ERR_VALUE;
    std::memset(out, 0, sizeof(*out));
    std::vector<int32_t> src, dst, il, ol;
    std::vector<double> w;
    std::unordered_map<int32_t, double> finals;
    std::vector<int32_t> final_order;
    long long start = -1, max_state = -1;
    const char *p = text, *end = text + len;
    for (int64_t i = 0; i < len; ++i) {
        const unsigned char c = (unsigned char)text[i];
        // non-ASCII, or a line break Python's splitlines() knows but this path does not
        if (c >= 0x80 || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1f) ||
            (c == '\r' && !(i + 1 < len && text[i + 1] == '\n')))
            return WB_PARSE_FALLBACK;
    }
    while (p < end) {
        const char *eol = (const char *)std::memchr(p, '\n', end - p);
        if (!eol) eol = end;
        const char *b = p, *e = eol;
        p = eol + 1;
        while (b < e && ws(*b)) ++b;
        while (e > b && ws(e[-1])) --e;
        if (b == e || *b == '#') continue;
        const char *f[6][2];
        int nf = 0;
        for (const char *q = b; q < e;) {
            while (q < e && ws(*q)) ++q;
            if (q >= e) break;
            const char *t = q;
            while (q < e && !ws(*q)) ++q;
            if (nf == 6) return WB_PARSE_FALLBACK;
            f[nf][0] = t;
            f[nf][1] = q;
            ++nf;
        }
        auto weight = [&](int k, double *x) {
            if (!parse_float(f[k][0], f[k][1], x)) return false;
            if (std::isnan(*x)) return false;
            if (*x < 0 && !allow_negative_weights) return false;
            return true;
        };
        if (nf == 1 || nf == 2) {
            long long s;
            double x = 0.0;
            if (!parse_int(f[0][0], f[0][1], &s) || s < 0 || s > std::numeric_limits<int32_t>::max() - 1)
                return WB_PARSE_FALLBACK;
            if (nf == 2 && !weight(1, &x)) return WB_PARSE_FALLBACK;
            if (!finals.count((int32_t)s)) final_order.push_back((int32_t)s);
            finals[(int32_t)s] = x;
            if (start < 0) start = s;
            if (s > max_state) max_state = s;
        } else if (nf == 4 || nf == 5) {
            long long a, d, i1, o1;
            double x = 0.0;
            if (!parse_int(f[0][0], f[0][1], &a) || !parse_int(f[1][0], f[1][1], &d) ||
                !parse_int(f[2][0], f[2][1], &i1) || !parse_int(f[3][0], f[3][1], &o1))
                return WB_PARSE_FALLBACK;
            const long long lim = std::numeric_limits<int32_t>::max() - 1;
            if (a < 0 || d < 0 || i1 < 0 || o1 < 0 || a > lim || d > lim || i1 > lim || o1 > lim)
                return WB_PARSE_FALLBACK;
            if (nf == 5 && !weight(4, &x)) return WB_PARSE_FALLBACK;
            src.push_back((int32_t)a);
            dst.push_back((int32_t)d);
            il.push_back((int32_t)i1);
            ol.push_back((int32_t)o1);
            w.push_back(x);
            if (start < 0) start = a;
            if (a > max_state) max_state = a;
            if (d > max_state) max_state = d;
        } else {
            return WB_PARSE_FALLBACK;
        }
    }
    if (start < 0) return WB_PARSE_FALLBACK;
    auto dup_i = [](const std::vector<int32_t> &v) {
        int32_t *q = (int32_t *)std::malloc(sizeof(int32_t) * std::max<size_t>(v.size(), 1));
        if (!v.empty()) std::memcpy(q, v.data(), sizeof(int32_t) * v.size());
        return q;
    };
    out->num_states = (int32_t)(max_state + 1);
    out->start = (int32_t)start;
    out->num_arcs = (int64_t)src.size();
    out->src = dup_i(src);
    out->dst = dup_i(dst);
    out->ilabel = dup_i(il);
    out->olabel = dup_i(ol);
    out->weight = (double *)std::malloc(sizeof(double) * std::max<size_t>(w.size(), 1));
    if (!w.empty()) std::memcpy(out->weight, w.data(), sizeof(double) * w.size());
    out->num_finals = (int64_t)final_order.size();
    out->final_state = dup_i(final_order);
    out->final_weight = (double *)std::malloc(sizeof(double) * std::max<size_t>(final_order.size(), 1));
    for (size_t k = 0; k < final_order.size(); ++k) out->final_weight[k] = finals[final_order[k]];
    return WB_OK;
}

void wb_parsed_wfst_free(wb_parsed_wfst *p) {
    if (!p) return;
    void *ptrs[] = {p->src, p->dst, p->ilabel, p->olabel, p->weight, p->final_state, p->final_weight};
    for (void *q : ptrs) std::free(q);
    std::memset(p, 0, sizeof(*p));
}

}  // extern "C"
