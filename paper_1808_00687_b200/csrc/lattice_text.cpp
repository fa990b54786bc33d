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
    std::vector<std::string> lines;
    for (const char *p = text, *end = text + len; p < end;) {
        const char *eol = (const char *)std::memchr(p, '\n', end - p);
        if (!eol) eol = end;
        const char *b = p, *e = eol;
        p = eol + 1;
        while (b < e && is_ws(*b)) ++b;
        while (e > b && is_ws(e[-1])) --e;
        if (b < e && *b != '#') lines.emplace_back(b, e);
    }
    if (lines.empty()) return WB_OK;   // EMPTY_LATTICE
    auto lat_err = [](const std::string &m) { return wb_internal_set_error(WB_ERR_LATTICE, m.c_str()); };
    auto fields_of = [](const std::string &s) {
        std::vector<std::string> f;
        for (size_t i = 0; i < s.size();) {
            while (i < s.size() && is_ws(s[i])) ++i;
            size_t j = i;
            while (j < s.size() && !is_ws(s[j])) ++j;
            if (j > i) f.emplace_back(s, i, j - i);
            i = j;
        }
        return f;
    };
    // int() / float() failures surface as the ValueError Python raises
    auto as_int = [](const std::string &s, long long *v) {
        return pytext::py_int(s.data(), s.data() + s.size(), v);
    };
    auto as_float = [](const std::string &s, double *v) {
        return pytext::py_float(s.data(), s.data() + s.size(), v);
    };
    auto int_err = [](const std::string &s) {
        return wb_internal_set_error(WB_ERR_VALUE, ("invalid literal for int() with base 10: " + q(s)).c_str());
    };
    auto float_err = [](const std::string &s) {
        return wb_internal_set_error(WB_ERR_VALUE, ("could not convert string to float: " + q(s)).c_str());
    };
    const std::vector<std::string> head = fields_of(lines[0]);
    long long n_nodes = 0, n_arcs = 0;
    if (head.size() != 3 || head[0] != "LATTICE" || head[1].rfind("nodes=", 0) != 0 ||
        head[2].rfind("arcs=", 0) != 0 || !as_int(head[1].substr(6), &n_nodes) ||
        !as_int(head[2].substr(5), &n_arcs))
        return lat_err("bad lattice header " + q(lines[0]));
    std::vector<int32_t> st, sp;
    std::vector<int64_t> fn, af, at, tie;
    std::vector<double> fwv, ag, aa;
    std::vector<int32_t> ail, aol;
    for (size_t k = 1; k < lines.size(); ++k) {
        const std::string &ln = lines[k];
        const std::vector<std::string> f = fields_of(ln);
        if (f[0] == "N") {
            if ((f.size() != 4 && f.size() != 6) || (f.size() == 6 && f[4] != "final"))
                return lat_err("bad node line " + q(ln));
            long long id, s, t;
            if (!as_int(f[1], &id)) return int_err(f[1]);
            if (id != (long long)st.size()) return lat_err("node ids must be dense and ordered; got " + q(ln));
            if (!as_int(f[2], &s)) return int_err(f[2]);
            if (!as_int(f[3], &t)) return int_err(f[3]);
            st.push_back((int32_t)s);
            sp.push_back((int32_t)t);
            if (f.size() == 6) {
                double w;
                if (!as_float(f[5], &w)) return float_err(f[5]);
                fn.push_back(id);
                fwv.push_back(w);
            }
        } else if (f[0] == "A") {
            if (f.size() != 7) return lat_err("bad arc line " + q(ln));
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
            return lat_err("unrecognized lattice line " + q(ln));
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
