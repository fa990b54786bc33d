// wfst_text.cpp -- AT&T transducer text -> arc arrays (the reference's parse_wfst_text,
// wfst.py:315-378), the package's only text parser.
//
// Grammar (reference semantics): one record per line; "src dst ilabel olabel [weight]" is an
// arc, "state [weight]" a final weight (missing weight = 0.0, a repeated final line
// overwrites); the first state mentioned is the start state; lines that are empty or start
// with '#' are skipped.  Numbers follow Python's int() / float() grammar (underscores between
// digits, inf / infinity / nan), decimal weights are rounded by strtod exactly like float().
// Labels resolve through an optional symbol table first, then as bare non-negative integers.
//
// Input is one line per '\n' (an optional '\r' before it) with ASCII-whitespace separated
// fields: the Python shim normalises text that uses other line breaks or Unicode whitespace
// before calling.  Errors report the 1-based line number and a message (wb_last_error).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/wfst_b200.h"
#include "pytext.h"

int wb_internal_set_error(int code, const char *msg);

namespace {

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }
using pytext::py_float;
using pytext::py_int;
using pytext::py_repr;

std::string quoted(const char *b, const char *e) { return "'" + std::string(b, e) + "'"; }

// "symbol id" lines (SymbolTable.format()); ids were validated by the Python SymbolTable.
void load_symbols(const char *b, int64_t n, std::unordered_map<std::string, int32_t> &m) {
    const char *p = b, *end = b + n;
    while (p < end) {
        const char *eol = (const char *)std::memchr(p, '\n', end - p);
        if (!eol) eol = end;
        const char *sp = p;
        while (sp < eol && *sp != ' ') ++sp;
        if (sp < eol) m[std::string(p, sp)] = (int32_t)std::atol(sp + 1);
        p = eol + 1;
    }
}

struct Parser {
    int allow_neg;
    const std::unordered_map<std::string, int32_t> *isyms = nullptr, *osyms = nullptr;
    long long line = 0;
    std::string err;
    int code = WB_OK;

    bool fail(int c, const std::string &msg, bool at_line = true) {
        code = c;
        err = msg;
        if (!at_line) line = 0;
        return false;
    }
    bool state(const char *b, const char *e, long long *s) {
        if (!py_int(b, e, s)) return fail(WB_PARSE_ERROR, "bad state id " + quoted(b, e));
        if (*s < 0) return fail(WB_PARSE_ERROR, "negative state id " + std::to_string(*s));
        if (*s >= std::numeric_limits<int32_t>::max() - 1)
            return fail(WB_PARSE_ERROR, "state id " + std::to_string(*s) + " exceeds the int32 range");
        return true;
    }
    bool weight(const char *b, const char *e, double *w) {
        if (!py_float(b, e, w)) return fail(WB_PARSE_ERROR, "bad weight " + quoted(b, e));
        if (std::isnan(*w)) return fail(WB_PARSE_ERROR, "weight is NaN");
        if (*w < 0 && !allow_neg)
            return fail(WB_PARSE_ERROR,
                        "negative weight " + py_repr(*w) + " (pass allow_negative_weights to accept)");
        return true;
    }
    bool label(const char *b, const char *e, const std::unordered_map<std::string, int32_t> *t,
               int32_t *out) {
        if (t) {
            auto it = t->find(std::string(b, e));
            if (it != t->end()) { *out = it->second; return true; }
        }
        long long x;
        if (!py_int(b, e, &x)) return fail(WB_PARSE_SYMBOL, "unknown symbol " + quoted(b, e));
        if (x < 0) return fail(WB_PARSE_SYMBOL, "negative label id " + std::to_string(x));
        if (x > std::numeric_limits<int32_t>::max())
            return fail(WB_PARSE_SYMBOL, "label id " + std::to_string(x) + " exceeds the int32 range");
        *out = (int32_t)x;
        return true;
    }
};

int32_t *dup32(const std::vector<int32_t> &v) {
    auto *q = (int32_t *)std::malloc(sizeof(int32_t) * std::max<size_t>(v.size(), 1));
    if (!v.empty()) std::memcpy(q, v.data(), sizeof(int32_t) * v.size());
    return q;
}

}  // namespace

extern "C" {

int wb_wfst_parse_text(const char *text, int64_t len, int32_t allow_negative_weights,
                       const char *isyms, int64_t isyms_len, const char *osyms,
                       int64_t osyms_len, wb_parsed_wfst *out) {
    if (!text || !out || len < 0) return wb_internal_set_error(WB_ERR_VALUE, "null argument");
    std::memset(out, 0, sizeof(*out));
    std::unordered_map<std::string, int32_t> itab, otab;
    Parser ps;
    ps.allow_neg = allow_negative_weights;
    if (isyms) { load_symbols(isyms, isyms_len, itab); ps.isyms = &itab; }
    if (osyms) { load_symbols(osyms, osyms_len, otab); ps.osyms = &otab; }
    std::vector<int32_t> src, dst, il, ol, final_order;
    std::vector<double> w;
    std::unordered_map<int32_t, double> finals;
    long long start = -1, max_state = -1;
    for (const char *p = text, *end = text + len; p < end;) {
        const char *eol = (const char *)std::memchr(p, '\n', end - p);
        if (!eol) eol = end;
        const char *b = p, *e = eol;
        p = eol + 1;
        ++ps.line;
        while (b < e && is_ws(*b)) ++b;
        while (e > b && is_ws(e[-1])) --e;
        if (b == e || *b == '#') continue;
        const char *fb[5], *fe[5];
        int nf = 0;
        for (const char *q = b; q < e;) {
            const char *t = q;
            while (q < e && !is_ws(*q)) ++q;
            if (nf < 5) { fb[nf] = t; fe[nf] = q; }
            ++nf;
            while (q < e && is_ws(*q)) ++q;
        }
        if (nf == 1 || nf == 2) {
            long long s;
            double x = 0.0;
            if (!ps.state(fb[0], fe[0], &s) || (nf == 2 && !ps.weight(fb[1], fe[1], &x))) break;
            if (!finals.count((int32_t)s)) final_order.push_back((int32_t)s);
            finals[(int32_t)s] = x;
            if (start < 0) start = s;
            max_state = std::max(max_state, s);
        } else if (nf == 4 || nf == 5) {
            long long a, d;
            int32_t i1, o1;
            double x = 0.0;
            if (!ps.state(fb[0], fe[0], &a) || !ps.state(fb[1], fe[1], &d) ||
                !ps.label(fb[2], fe[2], ps.isyms, &i1) || !ps.label(fb[3], fe[3], ps.osyms, &o1) ||
                (nf == 5 && !ps.weight(fb[4], fe[4], &x)))
                break;
            src.push_back((int32_t)a);
            dst.push_back((int32_t)d);
            il.push_back(i1);
            ol.push_back(o1);
            w.push_back(x);
            if (start < 0) start = a;
            max_state = std::max(max_state, std::max(a, d));
        } else {
            ps.fail(WB_PARSE_ERROR, "expected 1-2 (final) or 4-5 (arc) fields, got " + std::to_string(nf));
            break;
        }
    }
    if (ps.code == WB_OK && start < 0) ps.fail(WB_PARSE_ERROR, "no states found in transducer text", false);
    if (ps.code != WB_OK) {
        out->error_line = (int32_t)ps.line;
        return wb_internal_set_error(ps.code, ps.err.c_str());
    }
    out->num_states = (int32_t)(max_state + 1);
    out->start = (int32_t)start;
    out->num_arcs = (int64_t)src.size();
    out->src = dup32(src);
    out->dst = dup32(dst);
    out->ilabel = dup32(il);
    out->olabel = dup32(ol);
    out->weight = (double *)std::malloc(sizeof(double) * std::max<size_t>(w.size(), 1));
    if (!w.empty()) std::memcpy(out->weight, w.data(), sizeof(double) * w.size());
    out->num_finals = (int64_t)final_order.size();
    out->final_state = dup32(final_order);
    out->final_weight = (double *)std::malloc(sizeof(double) * std::max<size_t>(final_order.size(), 1));
    for (size_t k = 0; k < final_order.size(); ++k) out->final_weight[k] = finals[final_order[k]];
    return WB_OK;
}

// The CSR arc order (wfst.py:182): a stable sort by (src, ilabel, dst, olabel, weight).  States
// and labels are non-negative (checked by the caller), so (src, ilabel) and (dst, olabel) pack
// into order-preserving 64-bit keys; equal keys keep their input order (the index breaks ties).
int wb_sort_arcs(int64_t n, const int32_t *src, const int32_t *ilabel, const int32_t *dst,
                 const int32_t *olabel, const double *weight, int64_t *order) {
    if (n < 0 || (n > 0 && (!src || !ilabel || !dst || !olabel || !weight || !order)))
        return wb_internal_set_error(WB_ERR_VALUE, "null argument");
    struct Key {
        uint64_t a, b;
        double w;
        int64_t i;
    };
    std::vector<Key> k((size_t)n);
    bool sorted = true;
    for (int64_t i = 0; i < n; ++i) {
        k[i] = Key{((uint64_t)(uint32_t)src[i] << 32) | (uint32_t)ilabel[i],
                   ((uint64_t)(uint32_t)dst[i] << 32) | (uint32_t)olabel[i], weight[i], i};
        if (i && sorted) {
            const Key &x = k[i - 1], &y = k[i];
            sorted = x.a < y.a || (x.a == y.a && (x.b < y.b || (x.b == y.b && !(y.w < x.w))));
        }
    }
    if (!sorted)
        std::sort(k.begin(), k.end(), [](const Key &x, const Key &y) {
            if (x.a != y.a) return x.a < y.a;
            if (x.b != y.b) return x.b < y.b;
            if (x.w < y.w) return true;
            if (y.w < x.w) return false;
            return x.i < y.i;
        });
    for (int64_t i = 0; i < n; ++i) order[i] = k[i].i;
    return WB_OK;
}

void wb_parsed_wfst_free(wb_parsed_wfst *p) {
    if (!p) return;
    void *ptrs[] = {p->src, p->dst, p->ilabel, p->olabel, p->weight, p->final_state, p->final_weight};
    for (void *q : ptrs) std::free(q);
    std::memset(p, 0, sizeof(*p));
}

}  // extern "C"
