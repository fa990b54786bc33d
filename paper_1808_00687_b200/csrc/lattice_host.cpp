// lattice_host.cpp -- lattice post-processing behind the C ABI: epsilon-cycle check
// (_topo_order), exact forward-backward pruning with the path-exact split (prune_lattice), and
// the tie-exact best path (lattice_best_path).  Inputs are the trimmed lattices the decode
// kernel produced (already small: trimming to start-to-final paths happens in HBM), so this is
// host code over flat arrays -- no per-node objects.
//
// Reference: /root/reference/pkg/src/lsd_wfst/lattice.py
//   _topo_order             :295-326     _forward_costs / _backward_costs :329-356
//   prune_lattice           :359-397     _extremal_costs                  :400-427
//   _enforce_path_soundness :430-501     lattice_best_path                :504-559
//   _assemble               :190-237 (node identity is the (state, step) pair)
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/wfst_b200.h"

int wb_internal_set_error(int code, const char *msg);  // wfst_decoder.cu (wb_last_error)

namespace {

const double INF = HUGE_VAL;
const double COST_EPS = 1e-9;            // lattice.py:26
const size_t MAX_SPLIT_KEYS = 500000;    // lattice.py:465

int fail(int code, const char *msg) { return wb_internal_set_error(code, msg); }

struct Arc {
    int64_t from, to, tie;
    int32_t il, ol;
    double g, a;
};

// Owned lattice in flat arrays.
struct Lat {
    std::vector<int32_t> st, sp;  // node state / step
    std::vector<Arc> arcs;
    std::vector<int64_t> fin;     // final node ids, dict order
    std::vector<double> finw;
    bool empty = true;
    size_t n() const { return st.size(); }
};

Lat from_view(const wb_lattice_arrays *v) {
    Lat L;
    L.empty = v->n_nodes == 0;
    L.st.assign(v->node_state, v->node_state + v->n_nodes);
    L.sp.assign(v->node_step, v->node_step + v->n_nodes);
    L.arcs.resize((size_t)v->n_arcs);
    for (int64_t i = 0; i < v->n_arcs; ++i)
        L.arcs[i] = Arc{v->arc_from[i], v->arc_to[i], v->arc_tie[i], v->arc_il[i], v->arc_ol[i],
                        v->arc_g[i], v->arc_a[i]};
    L.fin.assign(v->final_node, v->final_node + v->n_finals);
    L.finw.assign(v->final_w, v->final_w + v->n_finals);
    return L;
}

template <class T>
T *dup(const std::vector<T> &v) {
    T *p = (T *)std::malloc(sizeof(T) * std::max<size_t>(v.size(), 1));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

void to_view(const Lat &L, wb_lattice_arrays *o) {
    std::memset(o, 0, sizeof(*o));
    if (L.empty) return;  // EMPTY_LATTICE: no nodes
    const size_t na = L.arcs.size();
    o->n_nodes = (int64_t)L.n();
    o->n_arcs = (int64_t)na;
    o->n_finals = (int64_t)L.fin.size();
    o->node_state = dup(L.st);
    o->node_step = dup(L.sp);
    std::vector<int64_t> f(na), t(na), tie(na);
    std::vector<int32_t> il(na), ol(na);
    std::vector<double> g(na), a(na);
    for (size_t i = 0; i < na; ++i) {
        const Arc &x = L.arcs[i];
        f[i] = x.from; t[i] = x.to; tie[i] = x.tie; il[i] = x.il; ol[i] = x.ol; g[i] = x.g; a[i] = x.a;
    }
    o->arc_from = dup(f); o->arc_to = dup(t); o->arc_tie = dup(tie);
    o->arc_il = dup(il); o->arc_ol = dup(ol); o->arc_g = dup(g); o->arc_a = dup(a);
    o->final_node = dup(L.fin);
    o->final_w = dup(L.finw);
}

// CSR of arc indices grouped by source (or target) node, arc order preserved.
void group(const Lat &L, bool by_to, std::vector<int64_t> &off, std::vector<int64_t> &idx) {
    off.assign(L.n() + 1, 0);
    for (const Arc &a : L.arcs) off[(by_to ? a.to : a.from) + 1]++;
    for (size_t i = 0; i < L.n(); ++i) off[i + 1] += off[i];
    idx.resize(L.arcs.size());
    std::vector<int64_t> pos(off.begin(), off.end() - 1);
    for (size_t e = 0; e < L.arcs.size(); ++e) idx[pos[by_to ? L.arcs[e].to : L.arcs[e].from]++] = (int64_t)e;
}

// Nodes by ascending step, epsilon-topological within a step (smallest state first among
// ready nodes); WB_ERR_LATTICE on an epsilon cycle.
int topo(const Lat &L, std::vector<int64_t> &order) {
    const size_t n = L.n();
    std::vector<int64_t> by(n);
    for (size_t i = 0; i < n; ++i) by[i] = (int64_t)i;
    std::stable_sort(by.begin(), by.end(), [&](int64_t x, int64_t y) { return L.sp[x] < L.sp[y]; });
    std::vector<int64_t> eoff(n + 1, 0), eidx;
    std::vector<int32_t> indeg(n, 0);
    for (const Arc &a : L.arcs)
        if (L.sp[a.from] == L.sp[a.to]) { eoff[a.from + 1]++; indeg[a.to]++; }
    for (size_t i = 0; i < n; ++i) eoff[i + 1] += eoff[i];
    eidx.resize(eoff[n]);
    {
        std::vector<int64_t> pos(eoff.begin(), eoff.end() - 1);
        for (const Arc &a : L.arcs)
            if (L.sp[a.from] == L.sp[a.to]) eidx[pos[a.from]++] = a.to;
    }
    order.clear();
    order.reserve(n);
    std::vector<std::pair<int32_t, int64_t>> heap;
    auto cmp = [](const std::pair<int32_t, int64_t> &x, const std::pair<int32_t, int64_t> &y) { return x > y; };
    for (size_t b = 0; b < n;) {
        size_t e = b;
        while (e < n && L.sp[by[e]] == L.sp[by[b]]) ++e;
        heap.clear();
        for (size_t q = b; q < e; ++q)
            if (indeg[by[q]] == 0) heap.push_back({L.st[by[q]], by[q]});
        std::make_heap(heap.begin(), heap.end(), cmp);
        size_t emitted = 0;
        while (!heap.empty()) {
            std::pop_heap(heap.begin(), heap.end(), cmp);
            const int64_t i = heap.back().second;
            heap.pop_back();
            order.push_back(i);
            ++emitted;
            for (int64_t q = eoff[i]; q < eoff[i + 1]; ++q)
                if (--indeg[eidx[q]] == 0) {
                    heap.push_back({L.st[eidx[q]], eidx[q]});
                    std::push_heap(heap.begin(), heap.end(), cmp);
                }
        }
        if (emitted != e - b) return fail(WB_ERR_LATTICE, "epsilon cycle among lattice nodes");
        b = e;
    }
    return WB_OK;
}

// min-sum (or max-sum) prefix costs: fw[to] = opt((fw[from] + g) + a)
std::vector<double> forward(const Lat &L, const std::vector<int64_t> &order,
                            const std::vector<int64_t> &off, const std::vector<int64_t> &idx, bool mx) {
    const double none = mx ? -INF : INF;
    std::vector<double> fw(L.n(), none);
    fw[0] = 0.0;
    for (int64_t i : order) {
        const double base = fw[i];
        if (base == none) continue;
        for (int64_t q = off[i]; q < off[i + 1]; ++q) {
            const Arc &a = L.arcs[idx[q]];
            const double c = (base + a.g) + a.a;
            if (mx ? c > fw[a.to] : c < fw[a.to]) fw[a.to] = c;
        }
    }
    return fw;
}

// suffix costs: bw[i] = opt(final_w, (g + a) + bw[to])
std::vector<double> backward(const Lat &L, const std::vector<int64_t> &order,
                             const std::vector<int64_t> &off, const std::vector<int64_t> &idx, bool mx) {
    const double none = mx ? -INF : INF;
    std::vector<double> bw(L.n(), none);
    for (size_t k = 0; k < L.fin.size(); ++k) bw[L.fin[k]] = L.finw[k];
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
        const int64_t i = *it;
        double best = bw[i];
        for (int64_t q = off[i]; q < off[i + 1]; ++q) {
            const Arc &a = L.arcs[idx[q]];
            const double c = (a.g + a.a) + bw[a.to];
            if (mx ? c > best : c < best) best = c;
        }
        bw[i] = best;
    }
    return bw;
}

inline uint64_t node_key(int32_t state, int32_t step) { return ((uint64_t)(uint32_t)step << 32) | (uint32_t)state; }

// _assemble over a node set given by (state, step) identity: trim to start-to-final paths,
// renumber [start] + (step, state) order, sort arcs canonically.  `arcs` hold node KEYS in
// from/to (as int64 bit patterns); `finals` are (key, weight) in dict order.
Lat assemble(const std::unordered_set<uint64_t> &node_set, const std::vector<Arc> &arcs,
             uint64_t start, const std::vector<std::pair<uint64_t, double>> &finals) {
    Lat out;
    if (!node_set.count(start)) return out;
    std::unordered_map<uint64_t, std::vector<uint64_t>> fadj, badj;
    for (const Arc &a : arcs) {
        fadj[(uint64_t)a.from].push_back((uint64_t)a.to);
        badj[(uint64_t)a.to].push_back((uint64_t)a.from);
    }
    auto reach = [](const std::vector<uint64_t> &seeds,
                    std::unordered_map<uint64_t, std::vector<uint64_t>> &adj) {
        std::unordered_set<uint64_t> seen(seeds.begin(), seeds.end());
        std::vector<uint64_t> stack(seeds.begin(), seeds.end());
        while (!stack.empty()) {
            const uint64_t x = stack.back();
            stack.pop_back();
            auto it = adj.find(x);
            if (it == adj.end()) continue;
            for (uint64_t y : it->second)
                if (seen.insert(y).second) stack.push_back(y);
        }
        return seen;
    };
    const auto fwd = reach({start}, fadj);
    // live finals, dict semantics (a repeated key keeps its first position, last weight)
    std::vector<uint64_t> lf;
    std::unordered_map<uint64_t, double> lfw;
    for (const auto &f : finals) {
        if (!fwd.count(f.first) || !node_set.count(f.first)) continue;
        if (!lfw.count(f.first)) lf.push_back(f.first);
        lfw[f.first] = f.second;
    }
    if (lf.empty()) return out;
    const auto bwd = reach(lf, badj);
    std::vector<uint64_t> keep;
    for (uint64_t x : fwd)
        if ((bwd.count(x) || lfw.count(x)) && x != start && node_set.count(x)) keep.push_back(x);
    std::sort(keep.begin(), keep.end());  // key order == (step, state)
    std::unordered_map<uint64_t, int64_t> ids;
    ids[start] = 0;
    out.st.push_back((int32_t)(uint32_t)start);
    out.sp.push_back((int32_t)(start >> 32));
    for (uint64_t x : keep) {
        ids[x] = (int64_t)out.st.size();
        out.st.push_back((int32_t)(uint32_t)x);
        out.sp.push_back((int32_t)(x >> 32));
    }
    for (const Arc &a : arcs) {
        auto f = ids.find((uint64_t)a.from), t = ids.find((uint64_t)a.to);
        if (f == ids.end() || t == ids.end()) continue;
        if (!fwd.count((uint64_t)a.from) || !bwd.count((uint64_t)a.to)) continue;
        Arc b = a;
        b.from = f->second;
        b.to = t->second;
        out.arcs.push_back(b);
    }
    std::stable_sort(out.arcs.begin(), out.arcs.end(), [&](const Arc &x, const Arc &y) {
        const uint64_t xf = node_key(out.st[x.from], out.sp[x.from]), yf = node_key(out.st[y.from], out.sp[y.from]);
        if (xf != yf) return xf < yf;
        const uint64_t xt = node_key(out.st[x.to], out.sp[x.to]), yt = node_key(out.st[y.to], out.sp[y.to]);
        if (xt != yt) return xt < yt;
        if (x.il != y.il) return x.il < y.il;
        if (x.ol != y.ol) return x.ol < y.ol;
        return x.tie < y.tie;
    });
    for (uint64_t x : lf) {
        out.fin.push_back(ids[x]);
        out.finw.push_back(lfw[x]);
    }
    out.empty = false;
    return out;
}

inline uint64_t dbits(double c) {
    c = c + 0.0;  // fold -0.0 (Python compares 0.0 == -0.0 in the key dict)
    uint64_t b;
    std::memcpy(&b, &c, 8);
    return b;
}

struct SKey {
    int64_t node;
    bool shared;  // (node, None)
    double c;
    bool operator==(const SKey &o) const {
        return node == o.node && shared == o.shared && (shared || dbits(c) == dbits(o.c));
    }
};
struct SKeyHash {
    size_t operator()(const SKey &k) const {
        return std::hash<uint64_t>()((uint64_t)k.node * 0x9E3779B97F4A7C15ull ^ (k.shared ? 1ull : dbits(k.c)));
    }
};

int soundness(const Lat &L, double cutoff, Lat &out) {
    std::vector<int64_t> order, off, idx;
    int rc = topo(L, order);
    if (rc) return rc;
    group(L, false, off, idx);
    const auto fmax = forward(L, order, off, idx, true);
    const auto bmax = backward(L, order, off, idx, true);
    std::vector<char> safe(L.n());
    bool all = true;
    for (size_t i = 0; i < L.n(); ++i) {
        safe[i] = fmax[i] + bmax[i] <= cutoff;
        all = all && safe[i];
    }
    if (all) {
        out = L;
        return WB_OK;
    }
    const auto bmin = backward(L, order, off, idx, false);
    std::vector<SKey> keys;
    std::unordered_map<SKey, int64_t, SKeyHash> kid;
    struct KArc { int64_t f, t, arc; };
    std::vector<KArc> karcs;
    SKey sk{0, (bool)safe[0], 0.0};
    keys.push_back(sk);
    kid[sk] = 0;
    std::vector<int64_t> stack{0};
    while (!stack.empty()) {
        const int64_t ki = stack.back();
        stack.pop_back();
        const SKey key = keys[ki];
        for (int64_t q = off[key.node]; q < off[key.node + 1]; ++q) {
            const Arc &a = L.arcs[idx[q]];
            const int64_t j = a.to;
            SKey tgt;
            if (key.shared) {
                tgt = SKey{j, true, 0.0};
            } else {
                const double c2 = (key.c + a.g) + a.a;
                if (c2 + bmin[j] > cutoff) continue;
                tgt = safe[j] ? SKey{j, true, 0.0} : SKey{j, false, c2};
            }
            auto it = kid.find(tgt);
            int64_t ti;
            if (it == kid.end()) {
                ti = (int64_t)keys.size();
                keys.push_back(tgt);
                kid[tgt] = ti;
                if (keys.size() > MAX_SPLIT_KEYS)
                    return fail(WB_ERR_LATTICE, "path-exact pruning would expand this lattice beyond "
                                                "500000 nodes; widen or disable the lattice beam");
                stack.push_back(ti);
            } else {
                ti = it->second;
            }
            karcs.push_back(KArc{ki, ti, idx[q]});
        }
    }
    std::unordered_map<int64_t, double> finw;
    for (size_t k = 0; k < L.fin.size(); ++k) finw[L.fin[k]] = L.finw[k];
    // order: start key, then (step, state, shared first, prefix cost), node id as last resort
    std::vector<int64_t> perm(keys.size() - 1);
    for (size_t i = 1; i < keys.size(); ++i) perm[i - 1] = (int64_t)i;
    std::sort(perm.begin(), perm.end(), [&](int64_t x, int64_t y) {
        const SKey &a = keys[x], &b = keys[y];
        if (L.sp[a.node] != L.sp[b.node]) return L.sp[a.node] < L.sp[b.node];
        if (L.st[a.node] != L.st[b.node]) return L.st[a.node] < L.st[b.node];
        if (a.shared != b.shared) return a.shared;
        const double ca = a.shared ? 0.0 : a.c, cb = b.shared ? 0.0 : b.c;
        if (ca != cb) return ca < cb;
        return a.node < b.node;
    });
    std::vector<int64_t> nid(keys.size());
    nid[0] = 0;
    for (size_t i = 0; i < perm.size(); ++i) nid[perm[i]] = (int64_t)i + 1;
    out = Lat();
    out.empty = false;
    out.st.resize(keys.size());
    out.sp.resize(keys.size());
    for (size_t i = 0; i < keys.size(); ++i) {
        out.st[nid[i]] = L.st[keys[i].node];
        out.sp[nid[i]] = L.sp[keys[i].node];
    }
    for (const KArc &k : karcs) {
        Arc a = L.arcs[k.arc];
        a.from = nid[k.f];
        a.to = nid[k.t];
        out.arcs.push_back(a);
    }
    std::sort(out.arcs.begin(), out.arcs.end(), [&](const Arc &x, const Arc &y) {
        const uint64_t xf = node_key(out.st[x.from], out.sp[x.from]), yf = node_key(out.st[y.from], out.sp[y.from]);
        if (xf != yf) return xf < yf;
        const uint64_t xt = node_key(out.st[x.to], out.sp[x.to]), yt = node_key(out.st[y.to], out.sp[y.to]);
        if (xt != yt) return xt < yt;
        if (x.il != y.il) return x.il < y.il;
        if (x.ol != y.ol) return x.ol < y.ol;
        if (x.tie != y.tie) return x.tie < y.tie;
        if (x.from != y.from) return x.from < y.from;
        return x.to < y.to;
    });
    // finals in key-set order is unobservable (a dict compares unordered); emit by node id
    std::vector<std::pair<int64_t, double>> fins;
    for (size_t i = 0; i < keys.size(); ++i) {
        auto it = finw.find(keys[i].node);
        if (it == finw.end()) continue;
        if (keys[i].shared || keys[i].c + it->second <= cutoff) fins.push_back({nid[i], it->second});
    }
    std::sort(fins.begin(), fins.end());
    for (auto &f : fins) {
        out.fin.push_back(f.first);
        out.finw.push_back(f.second);
    }
    return WB_OK;
}

int prune(const Lat &L, double beam, Lat &out) {
    out = Lat();
    if (L.empty) return WB_OK;
    std::vector<int64_t> order, off, idx;
    int rc = topo(L, order);
    if (rc) return rc;
    group(L, false, off, idx);
    const auto fw = forward(L, order, off, idx, false);
    const auto bw = backward(L, order, off, idx, false);
    const double best = bw[0];
    if (best == INF) return WB_OK;
    const double cutoff = (best + beam) + COST_EPS;
    std::vector<Arc> raw;
    std::unordered_set<uint64_t> nodes;
    for (const Arc &a : L.arcs) {
        if (((fw[a.from] + a.g) + a.a) + bw[a.to] <= cutoff) {
            Arc b = a;
            b.from = (int64_t)node_key(L.st[a.from], L.sp[a.from]);
            b.to = (int64_t)node_key(L.st[a.to], L.sp[a.to]);
            nodes.insert((uint64_t)b.from);
            nodes.insert((uint64_t)b.to);
            raw.push_back(b);
        }
    }
    std::vector<std::pair<uint64_t, double>> fins;
    for (size_t k = 0; k < L.fin.size(); ++k) {
        const int64_t i = L.fin[k];
        if (fw[i] + L.finw[k] <= cutoff) {
            const uint64_t key = node_key(L.st[i], L.sp[i]);
            fins.push_back({key, L.finw[k]});
            nodes.insert(key);
        }
    }
    const uint64_t start = node_key(L.st[0], L.sp[0]);
    nodes.insert(start);
    Lat kept = assemble(nodes, raw, start, fins);
    if (kept.empty) return WB_OK;
    return soundness(kept, cutoff, out);
}

}  // namespace

extern "C" {

int wb_lattice_canonical(int32_t n_utts, const int64_t *meta, const int32_t *nodes,
                         const uint32_t *arcs, const double *arc_ac, const uint32_t *finals,
                         const double *final_w, int32_t start_state, const int32_t *g_ilabel,
                         const int32_t *g_olabel, const double *g_weight, int32_t n_threads,
                         int64_t *out_meta, int32_t *node_state, int32_t *node_step,
                         int64_t *arc_from, int64_t *arc_to, int32_t *arc_il, int32_t *arc_ol,
                         double *arc_g, double *arc_a, int64_t *arc_tie, int64_t *final_node,
                         double *final_wo) {
    if (n_utts < 0 || (n_utts && (!meta || !out_meta))) return fail(WB_ERR_VALUE, "bad arguments");
    // output offsets: utterances back to back in utterance order
    int64_t cn = 0, ca = 0, cf = 0;
    for (int32_t u = 0; u < n_utts; ++u) {
        const int64_t *m = meta + 6 * (size_t)u;
        if (m[0] < 0) return fail(WB_ERR_CAPACITY, "lattice output pool overflowed");
        int64_t *o = out_meta + 6 * (size_t)u;
        o[0] = cn; o[1] = m[1]; o[2] = ca; o[3] = m[3]; o[4] = cf; o[5] = m[5];
        cn += m[1]; ca += m[3]; cf += m[5];
    }
    std::atomic<int32_t> next(0);
    auto work = [&]() {
        std::vector<int64_t> ord, newid, aord;
        for (int32_t u; (u = next.fetch_add(1)) < n_utts;) {
            const int64_t *m = meta + 6 * (size_t)u, *o = out_meta + 6 * (size_t)u;
            const int64_t nn = m[1], na = m[3], nf = m[5];
            if (nn == 0) continue;
            const int32_t *nd = nodes + 2 * (size_t)m[0];
            const uint32_t *ar = arcs + 4 * (size_t)m[2];
            // nodes: [start] + (step, state) order (lattice.py:215-216)
            ord.resize(nn);
            for (int64_t i = 0; i < nn; ++i) ord[i] = i;
            auto nkey = [&](int64_t i) {
                const bool st0 = nd[2 * i] == start_state && nd[2 * i + 1] == 0;
                return std::make_tuple(st0 ? 0 : 1, nd[2 * i + 1], nd[2 * i]);
            };
            std::sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return nkey(x) < nkey(y); });
            newid.resize(nn);
            for (int64_t r = 0; r < nn; ++r) {
                newid[ord[r]] = r;
                node_state[o[0] + r] = nd[2 * ord[r]];
                node_step[o[0] + r] = nd[2 * ord[r] + 1];
            }
            // arcs: (from.step, from.state, to.step, to.state, ilabel, olabel, tie) (:227-230)
            aord.resize(na);
            for (int64_t e = 0; e < na; ++e) aord[e] = e;
            auto akey = [&](int64_t e) {
                const int64_t f = ar[4 * e], t = ar[4 * e + 1], a = ar[4 * e + 2];
                return std::make_tuple(nd[2 * f + 1], nd[2 * f], nd[2 * t + 1], nd[2 * t],
                                       g_ilabel[a], g_olabel[a], a);
            };
            std::stable_sort(aord.begin(), aord.end(), [&](int64_t x, int64_t y) { return akey(x) < akey(y); });
            for (int64_t r = 0; r < na; ++r) {
                const int64_t e = aord[r], a = ar[4 * e + 2];
                arc_from[o[2] + r] = newid[ar[4 * e]];
                arc_to[o[2] + r] = newid[ar[4 * e + 1]];
                arc_il[o[2] + r] = g_ilabel[a];
                arc_ol[o[2] + r] = g_olabel[a];
                arc_g[o[2] + r] = g_weight[a];
                arc_a[o[2] + r] = arc_ac[m[2] + e];
                arc_tie[o[2] + r] = a;
            }
            for (int64_t q = 0; q < nf; ++q) {
                final_node[o[4] + q] = newid[finals[m[4] + q]];
                final_wo[o[4] + q] = final_w[m[4] + q];
            }
        }
    };
    const int nt = std::max(1, std::min<int>(n_threads > 0 ? n_threads : 1, n_utts));
    std::vector<std::thread> pool;
    for (int i = 1; i < nt; ++i) pool.emplace_back(work);
    work();
    for (auto &t : pool) t.join();
    return WB_OK;
}

int wb_lattice_check(const wb_lattice_arrays *lat) {
    if (!lat) return fail(WB_ERR_VALUE, "null lattice");
    Lat L = from_view(lat);
    if (L.empty) return WB_OK;
    std::vector<int64_t> order;
    return topo(L, order);
}

int wb_lattice_prune(const wb_lattice_arrays *lat, double beam, wb_lattice_arrays *out) {
    if (!lat || !out) return fail(WB_ERR_VALUE, "null lattice");
    std::memset(out, 0, sizeof(*out));
    if (!(beam >= 0)) return fail(WB_ERR_VALUE, "lattice_beam must be >= 0");
    Lat L = from_view(lat), P;
    int rc = prune(L, beam, P);
    if (rc) return rc;
    to_view(P, out);
    return WB_OK;
}

int wb_lattice_split(const wb_lattice_arrays *lat, double cutoff, wb_lattice_arrays *out) {
    if (!lat || !out) return fail(WB_ERR_VALUE, "null lattice");
    std::memset(out, 0, sizeof(*out));
    Lat L = from_view(lat), P;
    if (L.empty) return WB_OK;
    int rc = soundness(L, cutoff, P);
    if (rc) return rc;
    to_view(P, out);
    return WB_OK;
}

void wb_lattice_arrays_free(wb_lattice_arrays *a) {
    if (!a) return;
    void *ptrs[] = {a->node_state, a->node_step, a->arc_from, a->arc_to, a->arc_tie, a->arc_il,
                    a->arc_ol, a->arc_g, a->arc_a, a->final_node, a->final_w};
    for (void *p : ptrs) std::free(p);
    std::memset(a, 0, sizeof(*a));
}

int wb_lattice_best_path(const wb_lattice_arrays *lat, double *cost, int32_t *olabels,
                         int32_t *n_olabels, int32_t *ilabels, int32_t *n_ilabels, int32_t capacity) {
    if (!lat || !cost || !n_olabels || !n_ilabels) return fail(WB_ERR_VALUE, "null argument");
    Lat L = from_view(lat);
    if (L.empty) return fail(WB_ERR_LATTICE, "cannot extract a best path from an empty lattice");
    std::vector<int64_t> order, off, idx;
    int rc = topo(L, order);
    if (rc) return rc;
    group(L, true, off, idx);
    std::vector<double> dist(L.n(), INF);
    std::vector<int64_t> back(L.n(), -1);
    dist[0] = 0.0;
    for (int64_t i : order) {
        if (i == 0) continue;  // the origin keeps cost 0 and no backpointer
        bool have = false;
        double bc = 0.0;
        int32_t bs = 0;
        int64_t bt = 0, be = -1;
        for (int64_t q = off[i]; q < off[i + 1]; ++q) {
            const Arc &a = L.arcs[idx[q]];
            const double base = dist[a.from];
            if (base == INF) continue;
            const double c = (base + a.g) + a.a;
            const int32_t s = L.st[a.from];
            if (!have || c < bc || (c == bc && (s < bs || (s == bs && a.tie < bt)))) {
                have = true; bc = c; bs = s; bt = a.tie; be = idx[q];
            }
        }
        if (have) { dist[i] = bc; back[i] = be; }
    }
    std::vector<size_t> fo(L.fin.size());
    for (size_t k = 0; k < fo.size(); ++k) fo[k] = k;
    std::stable_sort(fo.begin(), fo.end(), [&](size_t x, size_t y) { return L.st[L.fin[x]] < L.st[L.fin[y]]; });
    int64_t bf = -1;
    double bt = INF;
    for (size_t k : fo) {
        const double tot = dist[L.fin[k]] + L.finw[k];
        if (tot < bt) { bt = tot; bf = L.fin[k]; }
    }
    if (bf < 0 || bt == INF) return fail(WB_ERR_LATTICE, "lattice has no complete start-to-final path");
    std::vector<int32_t> ol, il;
    for (int64_t i = bf; back[i] >= 0;) {
        const Arc &a = L.arcs[back[i]];
        if (a.ol != 0) ol.push_back(a.ol);
        if (a.il != 0) il.push_back(a.il);
        i = a.from;
    }
    std::reverse(ol.begin(), ol.end());
    std::reverse(il.begin(), il.end());
    *cost = bt;
    *n_olabels = (int32_t)ol.size();
    *n_ilabels = (int32_t)il.size();
    if ((int32_t)ol.size() > capacity || (int32_t)il.size() > capacity)
        return fail(WB_ERR_CAPACITY, "label buffer too small");
    if (olabels) std::copy(ol.begin(), ol.end(), olabels);
    if (ilabels) std::copy(il.begin(), il.end(), ilabels);
    return WB_OK;
}

}  // extern "C"
