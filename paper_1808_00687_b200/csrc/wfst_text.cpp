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
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/wfst_b200.h"

int wb_internal_set_error(int code, const char *msg);

namespace {

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// Copy a digit run that may contain single underscores between digits (PEP 515) into `out`
// without them; false if an underscore is misplaced.  Returns the end of the run in *stop.
bool digit_run(const char *b, const char *e, std::string &out, const char **stop) {
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

// Python int(token) for a token without surrounding whitespace.
bool py_int(const char *b, const char *e, long long *v) {
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

bool ieq(const char *b, const char *e, const char *word) {
    const size_t n = std::strlen(word);
    if ((size_t)(e - b) != n) return false;
    for (size_t i = 0; i < n; ++i)
        if ((b[i] | 0x20) != word[i]) return false;
    return true;
}

// Python float(token): [sign] (inf | infinity | nan | decimal), decimal =
// (digits [. [digits]] | . digits) [(e|E) [sign] digits], underscores between digits.
bool py_float(const char *b, const char *e, double *v) {
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

std::string quoted(const char *b, const char *e) { return "'" + std::string(b, e) + "'"; }

std::string py_repr(double x) {
    char buf[64];
    for (int prec = 1; prec <= 17; ++prec) {  // shortest round-tripping form, like repr()
        std::snprintf(buf, sizeof buf, "%.*g", prec, x);
        if (std::strtod(buf, nullptr) == x) break;
    }
    std::string r(buf);
    if (r.find_first_of(".eni") == std::string::npos) r += ".0";
    return r;
}

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

void wb_parsed_wfst_free(wb_parsed_wfst *p) {
    if (!p) return;
    void *ptrs[] = {p->src, p->dst, p->ilabel, p->olabel, p->weight, p->final_state, p->final_weight};
    for (void *q : ptrs) std::free(q);
    std::memset(p, 0, sizeof(*p));
}

}  // extern "C"
