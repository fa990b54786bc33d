// lattice_text.cpp -- the lattice text form (reference lattice.py:562-627) in C++:
// format_lattice_text / parse_lattice_text over flat lattice arrays, byte-identical to the
// reference's Python (repr floats, int() / float() parsing, the same error cases).
//
//   LATTICE nodes=<N> arcs=<A>
//   N <id> <state> <step> [final <weight>]      ids dense from 0, node 0 = start
//   A <from> <to> <ilabel> <olabel> <graph_cost> <acoustic_cost>
//
// Input lines are '\n' separated with ASCII whitespace (the Python shim normalises other line
// breaks); blank lines and lines starting with '#' are skipped.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/wfst_b200.h"
#include "pytext.h"

int wb_internal_set_error(int code, const char *msg);

namespace {

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

template <class T>
T *dup(const std::vector<T> &v) {
    T *p = (T *)std::malloc(sizeof(T) * std::max<size_t>(v.size(), 1));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

std::string q(const std::string &s) { return "'" + s + "'"; }

}  // namespace

extern "C" {

int wb_lattice_format_text(const wb_lattice_arrays *lat, char **text, int64_t *len) {
    if (!lat || !text || !len) return wb_internal_set_error(WB_ERR_VALUE, "null argument");
    std::vector<double> fw((size_t)lat->n_nodes, 0.0);
    std::vector<char> is_final((size_t)lat->n_nodes, 0);
    for (int64_t k = 0; k < lat->n_finals; ++k) {
        const int64_t nid = lat->final_node[k];
        if (nid < 0 || nid >= lat->n_nodes) return wb_internal_set_error(WB_ERR_VALUE, "final node out of range");
        is_final[nid] = 1;
        fw[nid] = lat->final_w[k];
    }
    // one pass into a buffer sized for the longest lines: a node line <= 3 x 20 + 48 bytes,
    // an arc line <= 4 x 20 + 2 x 32 + 8
    const size_t cap = 64 + (size_t)lat->n_nodes * 112 + (size_t)lat->n_arcs * 160;
    char *buf = (char *)std::malloc(cap + 1);
    if (!buf) return wb_internal_set_error(WB_ERR_NOMEM, "lattice text buffer");
    char *p = buf;
    auto put = [&](const char *s) { const size_t n = std::strlen(s); std::memcpy(p, s, n); p += n; };
    auto num = [&](long long v) { p = std::to_chars(p, p + 24, v).ptr; };
    put("LATTICE nodes=");
    num(lat->n_nodes);
    put(" arcs=");
    num(lat->n_arcs);
    *p++ = '\n';
    for (int64_t i = 0; i < lat->n_nodes; ++i) {
        *p++ = 'N';
        *p++ = ' ';
        num(i);
        *p++ = ' ';
        num(lat->node_state[i]);
        *p++ = ' ';
        num(lat->node_step[i]);
        if (is_final[i]) {
            put(" final ");
            p = pytext::py_repr_to(fw[i], p);
        }
        *p++ = '\n';
    }
    for (int64_t e = 0; e < lat->n_arcs; ++e) {
        *p++ = 'A';
        *p++ = ' ';
        num(lat->arc_from[e]);
        *p++ = ' ';
        num(lat->arc_to[e]);
        *p++ = ' ';
        num(lat->arc_il[e]);
        *p++ = ' ';
        num(lat->arc_ol[e]);
        *p++ = ' ';
        p = pytext::py_repr_to(lat->arc_g[e], p);
        *p++ = ' ';
        p = pytext::py_repr_to(lat->arc_a[e], p);
        *p++ = '\n';
    }
    *p = '\0';
    *text = buf;
    *len = (int64_t)(p - buf);
    return WB_OK;
}

void wb_text_free(char *text) { std::free(text); }

int wb_lattice_parse_text(const char *text, int64_t len, wb_lattice_arrays *out) {
    if (!text || !out || len < 0) return wb_internal_set_error(WB_ERR_VALUE, "null argument");
    std::memset(out, 0, sizeof(*out));
    // lines and fields as [begin, end) ranges into `text`: no per-line allocation
    struct Tok { const char *b, *e; };
    std::vector<Tok> lines;
    for (const char *p = text, *end = text + len; p < end;) {
        const char *eol = (const char *)std::memchr(p, '\n', end - p);
        if (!eol) eol = end;
        const char *b = p, *e = eol;
        p = eol + 1;
        while (b < e && is_ws(*b)) ++b;
        while (e > b && is_ws(e[-1])) --e;
        if (b < e && *b != '#') lines.push_back(Tok{b, e});
    }
    if (lines.empty()) return WB_OK;   // EMPTY_LATTICE
    auto str = [](Tok t) { return std::string(t.b, t.e); };
    auto lat_err = [](const std::string &m) { return wb_internal_set_error(WB_ERR_LATTICE, m.c_str()); };
    constexpr int MAXF = 8;
    auto fields_of = [](Tok s, Tok *f) {   // returns the field count (fields beyond MAXF uncounted past MAXF + 1)
        int n = 0;
        for (const char *p = s.b; p < s.e;) {
            while (p < s.e && is_ws(*p)) ++p;
            const char *q = p;
            while (q < s.e && !is_ws(*q)) ++q;
            if (q > p) {
                if (n < MAXF) f[n] = Tok{p, q};
                if (++n > MAXF) return n;
            }
            p = q;
        }
        return n;
    };
    auto eq = [](Tok t, const char *w) {
        const size_t n = std::strlen(w);
        return (size_t)(t.e - t.b) == n && std::memcmp(t.b, w, n) == 0;
    };
    // int() / float() failures surface as the ValueError Python raises
    auto as_int = [](Tok t, long long *v) { return pytext::py_int(t.b, t.e, v); };
    auto as_float = [](Tok t, double *v) { return pytext::py_float(t.b, t.e, v); };
    auto int_err = [&](Tok t) {
        return wb_internal_set_error(WB_ERR_VALUE, ("invalid literal for int() with base 10: " + q(str(t))).c_str());
    };
    auto float_err = [&](Tok t) {
        return wb_internal_set_error(WB_ERR_VALUE, ("could not convert string to float: " + q(str(t))).c_str());
    };
    Tok head[MAXF];
    const int nh = fields_of(lines[0], head);
    long long n_nodes = 0, n_arcs = 0;
    if (nh != 3 || !eq(head[0], "LATTICE") || head[1].e - head[1].b < 6 ||
        std::memcmp(head[1].b, "nodes=", 6) != 0 || head[2].e - head[2].b < 5 ||
        std::memcmp(head[2].b, "arcs=", 5) != 0 || !as_int(Tok{head[1].b + 6, head[1].e}, &n_nodes) ||
        !as_int(Tok{head[2].b + 5, head[2].e}, &n_arcs))
        return lat_err("bad lattice header " + q(str(lines[0])));
    std::vector<int32_t> st, sp;
    std::vector<int64_t> fn, af, at, tie;
    std::vector<double> fwv, ag, aa;
    std::vector<int32_t> ail, aol;
    if (n_nodes > 0 && n_nodes < (1ll << 31)) { st.reserve(n_nodes); sp.reserve(n_nodes); }
    if (n_arcs > 0 && n_arcs < (1ll << 31)) {
        af.reserve(n_arcs); at.reserve(n_arcs); tie.reserve(n_arcs); ag.reserve(n_arcs);
        aa.reserve(n_arcs); ail.reserve(n_arcs); aol.reserve(n_arcs);
    }
    Tok f[MAXF];
    for (size_t k = 1; k < lines.size(); ++k) {
        const Tok ln = lines[k];
        const int nf = fields_of(ln, f);
        if (eq(f[0], "N")) {
            if ((nf != 4 && nf != 6) || (nf == 6 && !eq(f[4], "final")))
                return lat_err("bad node line " + q(str(ln)));
            long long id, s, t;
            if (!as_int(f[1], &id)) return int_err(f[1]);
            if (id != (long long)st.size()) return lat_err("node ids must be dense and ordered; got " + q(str(ln)));
            if (!as_int(f[2], &s)) return int_err(f[2]);
            if (!as_int(f[3], &t)) return int_err(f[3]);
            st.push_back((int32_t)s);
            sp.push_back((int32_t)t);
            if (nf == 6) {
                double w;
                if (!as_float(f[5], &w)) return float_err(f[5]);
                fn.push_back(id);
                fwv.push_back(w);
            }
        } else if (eq(f[0], "A")) {
            if (nf != 7) return lat_err("bad arc line " + q(str(ln)));
            long long v[4];
            for (int i = 0; i < 4; ++i)
                if (!as_int(f[1 + i], &v[i])) return int_err(f[1 + i]);
            double g, a;
            if (!as_float(f[5], &g)) return float_err(f[5]);
            if (!as_float(f[6], &a)) return float_err(f[6]);
            tie.push_back((int64_t)af.size());
            af.push_back(v[0]);
            at.push_back(v[1]);
            ail.push_back((int32_t)v[2]);
            aol.push_back((int32_t)v[3]);
            ag.push_back(g);
            aa.push_back(a);
        } else {
            return lat_err("unrecognized lattice line " + q(str(ln)));
        }
    }
    if ((long long)st.size() != n_nodes || (long long)af.size() != n_arcs)
        return lat_err("header declares " + std::to_string(n_nodes) + " nodes / " + std::to_string(n_arcs) +
                       " arcs, found " + std::to_string(st.size()) + " / " + std::to_string(af.size()));
    if (st.empty()) return WB_OK;
    const int64_t N = (int64_t)st.size();
    for (size_t e = 0; e < af.size(); ++e) {
        if (af[e] < 0 || af[e] >= N || at[e] < 0 || at[e] >= N)
            return lat_err("arc references missing node: arc " + std::to_string(e));
        const int d = sp[at[e]] - sp[af[e]];
        if (d != 0 && d != 1)
            return lat_err("arc must stay in step or advance one step, got delta " + std::to_string(d) +
                           ": arc " + std::to_string(e));
    }
    out->n_nodes = N;
    out->n_arcs = (int64_t)af.size();
    out->n_finals = (int64_t)fn.size();
    out->node_state = dup(st); out->node_step = dup(sp);
    out->arc_from = dup(af); out->arc_to = dup(at); out->arc_tie = dup(tie);
    out->arc_il = dup(ail); out->arc_ol = dup(aol); out->arc_g = dup(ag); out->arc_a = dup(aa);
    out->final_node = dup(fn); out->final_w = dup(fwv);
    return WB_OK;
}

}  // extern "C"
