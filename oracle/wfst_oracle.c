/*
 * wfst_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A plain-C restatement of the reference `lsd_wfst` serial decoder and raw-lattice code
 * (/root/reference/pkg/src/lsd_wfst/decoder.py, lattice.py).  Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference leg may load
 * this library.  The product path (paper_1808_00687_b200) never links or calls it.
 *
 * Every function names the reference lines it follows.  Arithmetic is IEEE float64 in the
 * reference's association order: emitting (tcost + w) + ac (decoder.py:221), epsilon
 * ucost + w (decoder.py:166), final cost + fw (decoder.py:267), lattice forward
 * (fw + g) + a (lattice.py:338), backward (g + a) + bw (lattice.py:352), prune test
 * ((fw + g) + a) + bw <= (best + beam) + 1e-9 (lattice.py:380,386).
 *
 * Two trace modes:
 *   canonical = 0  reproduces the reference exactly, including its FIFO epsilon queue and
 *                  the stale-backpointer behaviour under exact cost ties;
 *   canonical = 1  winner-consistent traces: each state's trace follows its final winner
 *                  (what a frontier-parallel device closure produces).  Identical to mode 0
 *                  on tie-free inputs.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OG_OK 0
#define OG_ERR_LATTICE 3   /* LatticeError */
#define OG_ERR_VALUE 2     /* ValueError */
#define OG_ERR_NOMEM 5

#define ROOT_TRACE (-1)
static const double INF = 1.0 / 0.0;
#define COST_EPS 1e-9      /* lattice.py:26 */
#define PATH_KEY_CAP 500000 /* lattice.py:465 */

typedef struct {
    int32_t num_states, start, num_arcs, _pad;
    const int32_t *row_ptr;   /* [S+1] arc_offsets (wfst.py:185-190) */
    const int32_t *eps_end;   /* [S]   eps_split     (wfst.py:192-198) */
    const int32_t *dst, *ilabel, *olabel;  /* [A] arcs sorted (src,ilabel,dst,olabel,weight) */
    const double *weight;     /* [A] */
    const double *final_w;    /* [S] +inf = not final (wfst.py:183) */
} og_graph;

typedef struct {
    double beam;            /* DecodeConfig.beam (decoder.py:80) */
    int32_t max_active;     /* 0 = None */
    int32_t mode;           /* 0 fsd, 1 lsd */
    double blank_threshold; /* strict '>' (posteriors.py:122) */
    int32_t record_lattice;
    int32_t canonical;
} og_config;

typedef struct {
    double total_cost;
    int64_t tokens_expanded;
    int32_t search_steps, reached_final, died_at_step, n_olabels, n_ilabels, final_state, final_step, status;
    int32_t *olabels, *ilabels; /* malloc'ed; free with og_result_free */
    /* lattice recording (record_lattice): per node step k, survivors(k) sorted by state */
    int32_t n_node_steps;
    int64_t *surv_off;  /* [n_node_steps+1] */
    int32_t *surv;      /* flat */
    /* recorded emitting events (node step, src, arc, ac) and epsilon events (node step, src, arc) */
    int64_t n_emit, n_eps;
    int32_t *emit_step, *emit_src, *emit_arc; double *emit_ac;
    int32_t *eps_step, *eps_src, *eps_arc;
} og_result;

typedef struct {
    int32_t empty;           /* start_id is None */
    int64_t n_nodes, n_arcs, n_finals;
    int32_t *node_state, *node_step;
    int64_t *arc_from, *arc_to, *arc_tie;
    int32_t *arc_il, *arc_ol;
    double *arc_g, *arc_a;
    int64_t *final_node; double *final_w;
} og_lattice;

/* ------------------------------------------------------------------ growable vectors */
#define VEC_PUSH(ptr, n, cap, val, T)                                               \
    do {                                                                            \
        if ((n) >= (cap)) {                                                         \
            int64_t nc_ = (cap) ? (cap) * 2 : 64;                                   \
            T *np_ = (T *)realloc((ptr), (size_t)nc_ * sizeof(T));                  \
            if (!np_) abort();                                                      \
            (ptr) = np_; (cap) = nc_;                                               \
        }                                                                           \
        (ptr)[(n)++] = (val);                                                       \
    } while (0)

/* ------------------------------------------------------------------ decoder state */
typedef struct { int64_t *prev; int32_t *ol, *il; int64_t n, cap; } arena_t;

typedef struct {
    const og_graph *g;
    const og_config *cfg;
    double *c_cost; int32_t *c_src, *c_arc; int64_t *c_trace; uint32_t *c_tag; uint32_t epoch;
    int32_t *touched; int32_t n_touched;
    int32_t *q; int64_t qn, qcap; uint8_t *queued;
    /* canonical-mode extras */
    int64_t *c_tok_trace;   /* emitting winner: the source token's trace */
    int8_t *c_resolved;
    arena_t ar;
    og_result *rec;          /* non-NULL when recording */
    int64_t emit_cap, eps_cap, surv_cap, soff_cap;
} dec_t;

typedef struct { int32_t state; double cost; int64_t trace; } tok_t;

static int64_t arena_add(arena_t *a, int64_t prev, int32_t ol, int32_t il) {
    if (a->n >= a->cap) {
        int64_t nc = a->cap ? a->cap * 2 : 1024;
        a->prev = (int64_t *)realloc(a->prev, nc * sizeof(int64_t));
        a->ol = (int32_t *)realloc(a->ol, nc * sizeof(int32_t));
        a->il = (int32_t *)realloc(a->il, nc * sizeof(int32_t));
        if (!a->prev || !a->ol || !a->il) abort();
        a->cap = nc;
    }
    a->prev[a->n] = prev; a->ol[a->n] = ol; a->il[a->n] = il;
    return a->n++;
}

static void rec_emit(dec_t *d, int32_t k, int32_t src, int32_t ai, double ac) {
    og_result *r = d->rec;
    if (r->n_emit >= d->emit_cap) {
        int64_t nc = d->emit_cap ? d->emit_cap * 2 : 1024;
        r->emit_step = realloc(r->emit_step, nc * sizeof(int32_t));
        r->emit_src = realloc(r->emit_src, nc * sizeof(int32_t));
        r->emit_arc = realloc(r->emit_arc, nc * sizeof(int32_t));
        r->emit_ac = realloc(r->emit_ac, nc * sizeof(double));
        d->emit_cap = nc;
    }
    r->emit_step[r->n_emit] = k; r->emit_src[r->n_emit] = src; r->emit_arc[r->n_emit] = ai;
    r->emit_ac[r->n_emit] = ac; r->n_emit++;
}

static void rec_eps(dec_t *d, int32_t k, int32_t src, int32_t ai) {
    og_result *r = d->rec;
    if (r->n_eps >= d->eps_cap) {
        int64_t nc = d->eps_cap ? d->eps_cap * 2 : 1024;
        r->eps_step = realloc(r->eps_step, nc * sizeof(int32_t));
        r->eps_src = realloc(r->eps_src, nc * sizeof(int32_t));
        r->eps_arc = realloc(r->eps_arc, nc * sizeof(int32_t));
        d->eps_cap = nc;
    }
    r->eps_step[r->n_eps] = k; r->eps_src[r->n_eps] = src; r->eps_arc[r->n_eps] = ai; r->n_eps++;
}

static void rec_survivors(dec_t *d, const int32_t *states, int32_t n) {
    og_result *r = d->rec;
    if (r->n_node_steps + 2 > d->soff_cap) {
        int64_t nc = d->soff_cap ? d->soff_cap * 2 : 256;
        r->surv_off = realloc(r->surv_off, nc * sizeof(int64_t));
        if (d->soff_cap == 0) r->surv_off[0] = 0;
        d->soff_cap = nc;
    }
    int64_t base = r->surv_off[r->n_node_steps];
    while (base + n > d->surv_cap) {
        int64_t nc = d->surv_cap ? d->surv_cap * 2 : 1024;
        r->surv = realloc(r->surv, nc * sizeof(int32_t));
        d->surv_cap = nc;
    }
    memcpy(r->surv + base, states, (size_t)n * sizeof(int32_t));
    r->n_node_steps++;
    r->surv_off[r->n_node_steps] = base + n;
}

/* _relax, decoder.py:121-135: min under (cost, src state, arc index); equal keys rejected. */
static int relax(dec_t *d, int32_t dst, double cost, int32_t src, int32_t arc, int64_t prev_trace,
                 int32_t ol, int32_t il, int64_t tok_trace) {
    if (d->c_tag[dst] == d->epoch) {
        double ec = d->c_cost[dst];
        if (cost > ec) return 0;
        if (cost == ec) {
            if (src > d->c_src[dst] || (src == d->c_src[dst] && arc >= d->c_arc[dst])) return 0;
        }
    } else {
        d->c_tag[dst] = d->epoch;
        d->touched[d->n_touched++] = dst;
    }
    d->c_cost[dst] = cost; d->c_src[dst] = src; d->c_arc[dst] = arc;
    if (d->cfg->canonical) {
        d->c_trace[dst] = -2; /* resolved after the fixpoint */
        d->c_tok_trace[dst] = tok_trace;
    } else {
        d->c_trace[dst] = arena_add(&d->ar, prev_trace, ol, il);
    }
    return 1;
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

static void q_push(dec_t *d, int32_t s) { VEC_PUSH(d->q, d->qn, d->qcap, s, int32_t); }

/* _epsilon_fixpoint, decoder.py:138-171: FIFO seeded with sorted(cand); self-loops skipped. */
static void epsilon_fixpoint(dec_t *d, int32_t node_step, int has_eps) {
    const og_graph *g = d->g;
    if (!has_eps) return;
    int32_t *seed = (int32_t *)malloc(sizeof(int32_t) * (d->n_touched ? d->n_touched : 1));
    memcpy(seed, d->touched, sizeof(int32_t) * d->n_touched);
    qsort(seed, d->n_touched, sizeof(int32_t), cmp_i32);
    d->qn = 0;
    for (int32_t i = 0; i < d->n_touched; i++) { q_push(d, seed[i]); d->queued[seed[i]] = 1; }
    free(seed);
    int64_t head = 0;
    while (head < d->qn) {
        int32_t u = d->q[head++];
        d->queued[u] = 0;
        double ucost = d->c_cost[u];
        int64_t utrace = d->c_trace[u];
        for (int32_t ai = g->row_ptr[u]; ai < g->eps_end[u]; ai++) {
            int32_t dst = g->dst[ai];
            if (dst == u) continue;
            if (d->rec) rec_eps(d, node_step, u, ai);
            double c = ucost + g->weight[ai];
            if (relax(d, dst, c, u, ai, utrace, g->olabel[ai], g->ilabel[ai], -1)) {
                if (!d->queued[dst]) { q_push(d, dst); d->queued[dst] = 1; }
            }
        }
        /* compact the queue now and then so positive eps cycles cannot grow it forever */
        if (head > 1048576 && head * 2 > d->qn) {
            memmove(d->q, d->q + head, (size_t)(d->qn - head) * sizeof(int32_t));
            d->qn -= head; head = 0;
        }
    }
}

/* canonical trace resolution: trace(v) follows v's final winner (memoised, acyclic). */
static int64_t resolve_trace(dec_t *d, int32_t v) {
    const og_graph *g = d->g;
    if (d->c_trace[v] != -2) return d->c_trace[v];
    /* iterative walk up the epsilon-winner chain */
    int32_t stack_local[64]; int32_t *stk = stack_local; int64_t sn = 0, scap = 64;
    int32_t x = v;
    while (d->c_trace[x] == -2 && d->c_arc[x] >= 0 && g->ilabel[d->c_arc[x]] == 0) {
        if (sn >= scap) {
            int32_t *ns = malloc(sizeof(int32_t) * scap * 2);
            memcpy(ns, stk, sizeof(int32_t) * sn);
            if (stk != stack_local) free(stk);
            stk = ns; scap *= 2;
        }
        stk[sn++] = x;
        x = d->c_src[x];
    }
    if (d->c_trace[x] == -2) {
        /* emitting winner or the root start entry */
        int32_t a = d->c_arc[x];
        d->c_trace[x] = arena_add(&d->ar, d->c_tok_trace[x], g->olabel[a], g->ilabel[a]);
    }
    while (sn > 0) {
        int32_t y = stk[--sn];
        int32_t a = d->c_arc[y];
        d->c_trace[y] = arena_add(&d->ar, d->c_trace[d->c_src[y]], g->olabel[a], g->ilabel[a]);
    }
    if (stk != stack_local) free(stk);
    return d->c_trace[v];
}

static int cmp_tok_state(const void *a, const void *b) {
    const tok_t *x = a, *y = b;
    return (x->state > y->state) - (x->state < y->state);
}
static int cmp_tok_cost_state(const void *a, const void *b) {
    const tok_t *x = a, *y = b;
    if (x->cost < y->cost) return -1;
    if (x->cost > y->cost) return 1;
    return (x->state > y->state) - (x->state < y->state);
}

/* _prune_candidates, decoder.py:174-194. Writes survivors (sorted by state) into out. */
static int32_t prune_candidates(dec_t *d, tok_t *out) {
    int32_t n = d->n_touched;
    if (n == 0) return 0;
    if (d->cfg->canonical)
        for (int32_t i = 0; i < n; i++) resolve_trace(d, d->touched[i]);
    double best = INF;
    int first = 1;
    for (int32_t i = 0; i < n; i++) {
        double c = d->c_cost[d->touched[i]];
        if (first || c < best) { best = c; first = 0; }
    }
    double cutoff = best + d->cfg->beam;
    int32_t m = 0;
    for (int32_t i = 0; i < n; i++) {
        int32_t s = d->touched[i];
        double c = d->c_cost[s];
        if (c <= cutoff) { out[m].state = s; out[m].cost = c; out[m].trace = d->c_trace[s]; m++; }
    }
    if (d->cfg->max_active > 0 && m > d->cfg->max_active) {
        qsort(out, m, sizeof(tok_t), cmp_tok_cost_state);
        m = d->cfg->max_active;
    }
    qsort(out, m, sizeof(tok_t), cmp_tok_state);
    return m;
}

static void begin_cand(dec_t *d) {
    d->epoch++;
    if (d->epoch == 0) { memset(d->c_tag, 0, sizeof(uint32_t) * d->g->num_states); d->epoch = 1; }
    d->n_touched = 0;
}

/* viterbi_step, decoder.py:197-233 */
static int32_t viterbi_step(dec_t *d, const tok_t *live, int32_t n_live, const double *costs,
                            int32_t node_step, int has_eps, tok_t *out) {
    const og_graph *g = d->g;
    begin_cand(d);
    for (int32_t t = 0; t < n_live; t++) {
        int32_t s = live[t].state;
        double tcost = live[t].cost;
        int64_t ttrace = live[t].trace;
        for (int32_t ai = g->eps_end[s]; ai < g->row_ptr[s + 1]; ai++) {
            double ac = costs[g->ilabel[ai]];
            if (ac == INF) continue;
            double c = (tcost + g->weight[ai]) + ac;
            if (d->rec) rec_emit(d, node_step, s, ai, ac);
            relax(d, g->dst[ai], c, s, ai, ttrace, g->olabel[ai], g->ilabel[ai], ttrace);
        }
    }
    epsilon_fixpoint(d, node_step, has_eps);
    int32_t m = prune_candidates(d, out);
    if (d->rec) {
        int32_t *st = malloc(sizeof(int32_t) * (m ? m : 1));
        for (int32_t i = 0; i < m; i++) st[i] = out[i].state;
        rec_survivors(d, st, m);
        free(st);
    }
    return m;
}

static int dec_init(dec_t *d, const og_graph *g, const og_config *cfg) {
    memset(d, 0, sizeof(*d));
    d->g = g; d->cfg = cfg;
    size_t S = (size_t)g->num_states;
    d->c_cost = malloc(S * sizeof(double));
    d->c_src = malloc(S * sizeof(int32_t));
    d->c_arc = malloc(S * sizeof(int32_t));
    d->c_trace = malloc(S * sizeof(int64_t));
    d->c_tag = calloc(S, sizeof(uint32_t));
    d->touched = malloc(S * sizeof(int32_t));
    d->queued = calloc(S, 1);
    d->c_tok_trace = malloc(S * sizeof(int64_t));
    if (!d->c_cost || !d->c_src || !d->c_arc || !d->c_trace || !d->c_tag || !d->touched ||
        !d->queued || !d->c_tok_trace) return OG_ERR_NOMEM;
    return OG_OK;
}

static void dec_free(dec_t *d) {
    free(d->c_cost); free(d->c_src); free(d->c_arc); free(d->c_trace); free(d->c_tag);
    free(d->touched); free(d->queued); free(d->q); free(d->c_tok_trace);
    free(d->ar.prev); free(d->ar.ol); free(d->ar.il);
}

void og_result_free(og_result *r) {
    free(r->olabels); free(r->ilabels); free(r->surv_off); free(r->surv);
    free(r->emit_step); free(r->emit_src); free(r->emit_arc); free(r->emit_ac);
    free(r->eps_step); free(r->eps_src); free(r->eps_arc);
    memset(r, 0, sizeof(*r));
}

/* _search + decode_fsd/decode_lsd, decoder.py:302-367.  costs: [T, L1] row-major with
 * column 0 = +inf (frame_costs, posteriors.py:136-144); blank: [T] blank probabilities. */
int og_decode(const og_graph *g, const double *costs, const double *blank, int32_t T, int32_t L1,
              const og_config *cfg, og_result *out) {
    memset(out, 0, sizeof(*out));
    dec_t d;
    int rc = dec_init(&d, g, cfg);
    if (rc) { dec_free(&d); return rc; }
    if (cfg->record_lattice) d.rec = out;
    int has_eps = 0;
    for (int32_t s = 0; s < g->num_states && !has_eps; s++) has_eps = g->eps_end[s] > g->row_ptr[s];

    /* frame selection: select_frames / classify_blank_frames (decoder.py:113-118) */
    int32_t *frames = malloc(sizeof(int32_t) * (T ? T : 1));
    int32_t nf = 0;
    for (int32_t f = 0; f < T; f++)
        if (cfg->mode == 0 || !(blank[f] > cfg->blank_threshold)) frames[nf++] = f;

    tok_t *live = malloc(sizeof(tok_t) * (size_t)g->num_states);
    tok_t *next = malloc(sizeof(tok_t) * (size_t)g->num_states);

    /* _initial_tokens, decoder.py:236-249 */
    begin_cand(&d);
    d.c_tag[g->start] = d.epoch;
    d.touched[d.n_touched++] = g->start;
    d.c_cost[g->start] = 0.0; d.c_src[g->start] = -1; d.c_arc[g->start] = -1;
    d.c_trace[g->start] = ROOT_TRACE;
    epsilon_fixpoint(&d, 0, has_eps);
    int32_t n_live = prune_candidates(&d, live);
    if (d.rec) {
        int32_t *st = malloc(sizeof(int32_t) * (n_live + 1));
        int32_t m = 0, added = 0;
        for (int32_t i = 0; i < n_live; i++) {
            if (!added && live[i].state > g->start) { st[m++] = g->start; added = 1; }
            if (live[i].state == g->start) added = 1;
            st[m++] = live[i].state;
        }
        if (!added) st[m++] = g->start;
        rec_survivors(&d, st, m);
        free(st);
    }

    int64_t expanded = 0;
    int32_t steps_run = 0, died_at = -1;
    for (int32_t s = 0; s < nf; s++) {
        const double *row = costs + (size_t)frames[s] * L1;
        expanded += n_live;
        int32_t m = viterbi_step(&d, live, n_live, row, s + 1, has_eps, next);
        steps_run++;
        if (m == 0) { died_at = s; break; }
        tok_t *tmp = live; live = next; next = tmp; n_live = m;
    }

    tok_t best; int reached = 0; int32_t last_step;
    if (died_at < 0) {
        /* final_transition, decoder.py:252-273 */
        int found = 0;
        for (int32_t i = 0; i < n_live; i++) {
            double fw = g->final_w[live[i].state];
            if (fw == INF) continue;
            double c = live[i].cost + fw;
            if (!found || c < best.cost || (c == best.cost && live[i].state < best.state)) {
                best.state = live[i].state; best.cost = c; best.trace = live[i].trace; found = 1;
            }
        }
        if (found) reached = 1;
        else {
            best = live[0];
            for (int32_t i = 1; i < n_live; i++)
                if (cmp_tok_cost_state(&live[i], &best) < 0) best = live[i];
        }
        last_step = steps_run;
    } else {
        best = live[0];
        for (int32_t i = 1; i < n_live; i++)
            if (cmp_tok_cost_state(&live[i], &best) < 0) best = live[i];
        last_step = died_at;
    }

    /* backtrace, decoder.py:276-291 */
    int32_t n_o = 0, n_i = 0;
    for (int64_t idx = best.trace; idx != ROOT_TRACE; idx = d.ar.prev[idx]) {
        if (d.ar.ol[idx] != 0) n_o++;
        if (d.ar.il[idx] != 0) n_i++;
    }
    out->olabels = malloc(sizeof(int32_t) * (n_o ? n_o : 1));
    out->ilabels = malloc(sizeof(int32_t) * (n_i ? n_i : 1));
    int32_t po = n_o, pi = n_i;
    for (int64_t idx = best.trace; idx != ROOT_TRACE; idx = d.ar.prev[idx]) {
        if (d.ar.ol[idx] != 0) out->olabels[--po] = d.ar.ol[idx];
        if (d.ar.il[idx] != 0) out->ilabels[--pi] = d.ar.il[idx];
    }
    out->n_olabels = n_o; out->n_ilabels = n_i;
    out->total_cost = best.cost;
    out->search_steps = steps_run;
    out->tokens_expanded = expanded;
    out->reached_final = reached;
    out->died_at_step = died_at;
    out->final_state = best.state;
    out->final_step = last_step;
    free(frames); free(live); free(next);
    dec_free(&d);
    return OG_OK;
}

/* ------------------------------------------------------------------ batch (CPU baseline) */
typedef struct {
    const og_graph *g; const og_config *cfg; int32_t n; int32_t L1;
    const double *const *costs; const double *const *blank; const int32_t *T;
    og_result *out; int *rc;
    int32_t next; pthread_mutex_t mu;
} batch_ctx;

static void *batch_worker(void *arg) {
    batch_ctx *b = arg;
    for (;;) {
        pthread_mutex_lock(&b->mu);
        int32_t i = b->next++;
        pthread_mutex_unlock(&b->mu);
        if (i >= b->n) return NULL;
        b->rc[i] = og_decode(b->g, b->costs[i], b->blank[i], b->T[i], b->L1, b->cfg, &b->out[i]);
    }
}

/* Decode n utterances on n_threads host threads (utterances are independent). */
int og_decode_batch(const og_graph *g, int32_t n, const double *const *costs,
                    const double *const *blank, const int32_t *T, int32_t L1, const og_config *cfg,
                    og_result *out, int32_t n_threads) {
    batch_ctx b = {g, cfg, n, L1, costs, blank, T, out, NULL, 0, PTHREAD_MUTEX_INITIALIZER};
    b.rc = calloc(n ? n : 1, sizeof(int));
    if (n_threads < 1) n_threads = 1;
    if (n_threads > n) n_threads = n ? n : 1;
    pthread_t *th = malloc(sizeof(pthread_t) * n_threads);
    for (int32_t t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, batch_worker, &b);
    for (int32_t t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    int rc = 0;
    for (int32_t i = 0; i < n; i++) if (b.rc[i]) rc = b.rc[i];
    free(th); free(b.rc);
    return rc;
}

/* ================================================================== lattice */
/* node identity = (step, state) packed as (step << 32) | state, so key order == (step, state) */
static inline int64_t nkey(int32_t step, int32_t state) { return ((int64_t)step << 32) | (uint32_t)state; }
static inline int32_t key_step(int64_t k) { return (int32_t)(k >> 32); }
static inline int32_t key_state(int64_t k) { return (int32_t)(uint32_t)(k & 0xffffffff); }

typedef struct { int64_t f, t; int32_t il, ol; double g, a; int64_t tie; int64_t ord; } rawarc_t;

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}
static int64_t uniq_i64(int64_t *v, int64_t n) {
    if (n == 0) return 0;
    qsort(v, n, sizeof(int64_t), cmp_i64);
    int64_t m = 1;
    for (int64_t i = 1; i < n; i++) if (v[i] != v[m - 1]) v[m++] = v[i];
    return m;
}
static int64_t find_i64(const int64_t *v, int64_t n, int64_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (v[mid] < x) lo = mid + 1; else hi = mid; }
    return (lo < n && v[lo] == x) ? lo : -1;
}

static int cmp_rawarc_canon(const void *pa, const void *pb) {
    const rawarc_t *a = pa, *b = pb;
    if (a->f != b->f) return a->f < b->f ? -1 : 1;
    if (a->t != b->t) return a->t < b->t ? -1 : 1;
    if (a->il != b->il) return a->il < b->il ? -1 : 1;
    if (a->ol != b->ol) return a->ol < b->ol ? -1 : 1;
    if (a->tie != b->tie) return a->tie < b->tie ? -1 : 1;
    return (a->ord > b->ord) - (a->ord < b->ord);
}

void og_lattice_free(og_lattice *l) {
    free(l->node_state); free(l->node_step); free(l->arc_from); free(l->arc_to); free(l->arc_tie);
    free(l->arc_il); free(l->arc_ol); free(l->arc_g); free(l->arc_a); free(l->final_node);
    free(l->final_w);
    memset(l, 0, sizeof(*l));
}

static void lattice_empty(og_lattice *l) { memset(l, 0, sizeof(*l)); l->empty = 1; }

/* reachability over nodes indexed 0..n-1 with CSR adjacency */
static void reach(int64_t n, const int64_t *off, const int64_t *adj, const int64_t *seeds,
                  int64_t n_seeds, uint8_t *seen) {
    int64_t *stack = malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t sp = 0;
    for (int64_t i = 0; i < n_seeds; i++)
        if (!seen[seeds[i]]) { seen[seeds[i]] = 1; stack[sp++] = seeds[i]; }
    while (sp) {
        int64_t x = stack[--sp];
        for (int64_t j = off[x]; j < off[x + 1]; j++) {
            int64_t y = adj[j];
            if (!seen[y]) { seen[y] = 1; stack[sp++] = y; }
        }
    }
    free(stack);
}

/* _assemble, lattice.py:190-237.  node_keys sorted unique; finals (key, w) in insertion order. */
static void assemble(const int64_t *node_keys, int64_t n_nodeset, rawarc_t *raw, int64_t n_raw,
                     int64_t start, const int64_t *fin_key, const double *fin_w, int64_t n_fin,
                     og_lattice *out) {
    if (find_i64(node_keys, n_nodeset, start) < 0) { lattice_empty(out); return; }
    /* universe U = node_set U endpoints U finals */
    int64_t nu = n_nodeset + 2 * n_raw + n_fin + 1;
    int64_t *U = malloc(sizeof(int64_t) * nu);
    int64_t k = 0;
    memcpy(U, node_keys, sizeof(int64_t) * n_nodeset); k = n_nodeset;
    for (int64_t i = 0; i < n_raw; i++) { U[k++] = raw[i].f; U[k++] = raw[i].t; }
    for (int64_t i = 0; i < n_fin; i++) U[k++] = fin_key[i];
    U[k++] = start;
    nu = uniq_i64(U, k);
    uint8_t *in_set = calloc(nu, 1);
    for (int64_t i = 0; i < n_nodeset; i++) in_set[find_i64(U, nu, node_keys[i])] = 1;
    int64_t *fi = malloc(sizeof(int64_t) * (n_raw ? n_raw : 1)), *ti = malloc(sizeof(int64_t) * (n_raw ? n_raw : 1));
    for (int64_t i = 0; i < n_raw; i++) { fi[i] = find_i64(U, nu, raw[i].f); ti[i] = find_i64(U, nu, raw[i].t); }
    int64_t *foff = calloc(nu + 1, sizeof(int64_t)), *boff = calloc(nu + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n_raw; i++) { foff[fi[i] + 1]++; boff[ti[i] + 1]++; }
    for (int64_t i = 0; i < nu; i++) { foff[i + 1] += foff[i]; boff[i + 1] += boff[i]; }
    int64_t *fadj = malloc(sizeof(int64_t) * (n_raw ? n_raw : 1)), *badj = malloc(sizeof(int64_t) * (n_raw ? n_raw : 1));
    int64_t *fp = malloc(sizeof(int64_t) * (nu + 1)), *bp = malloc(sizeof(int64_t) * (nu + 1));
    memcpy(fp, foff, sizeof(int64_t) * (nu + 1)); memcpy(bp, boff, sizeof(int64_t) * (nu + 1));
    for (int64_t i = 0; i < n_raw; i++) { fadj[fp[fi[i]]++] = ti[i]; badj[bp[ti[i]]++] = fi[i]; }
    uint8_t *fwd = calloc(nu, 1), *bwd = calloc(nu, 1), *livef = calloc(nu, 1), *keep = calloc(nu, 1);
    int64_t si = find_i64(U, nu, start);
    reach(nu, foff, fadj, &si, 1, fwd);
    int64_t *lf_idx = malloc(sizeof(int64_t) * (n_fin ? n_fin : 1));
    double *lf_w = malloc(sizeof(double) * (n_fin ? n_fin : 1));
    int64_t n_lf = 0;
    for (int64_t i = 0; i < n_fin; i++) {
        int64_t x = find_i64(U, nu, fin_key[i]);
        if (fwd[x] && in_set[x]) {
            /* dict semantics: a repeated key keeps its first position, last value */
            int64_t j;
            for (j = 0; j < n_lf; j++) if (lf_idx[j] == x) break;
            if (j < n_lf) lf_w[j] = fin_w[i];
            else { lf_idx[n_lf] = x; lf_w[n_lf] = fin_w[i]; n_lf++; livef[x] = 1; }
        }
    }
    if (n_lf == 0) {
        lattice_empty(out);
    } else {
        reach(nu, boff, badj, lf_idx, n_lf, bwd);
        int64_t nk = 0;
        for (int64_t i = 0; i < nu; i++) {
            keep[i] = ((fwd[i] && bwd[i]) || livef[i]) && (in_set[i] || livef[i]);
            nk += keep[i];
        }
        /* ordered = [start] + sorted(keep - {start}) by (step, state) == key order */
        int64_t *newid = malloc(sizeof(int64_t) * nu);
        out->empty = 0;
        out->n_nodes = nk;
        out->node_state = malloc(sizeof(int32_t) * (nk ? nk : 1));
        out->node_step = malloc(sizeof(int32_t) * (nk ? nk : 1));
        int64_t id = 0;
        out->node_state[0] = key_state(start); out->node_step[0] = key_step(start); newid[si] = 0; id = 1;
        for (int64_t i = 0; i < nu; i++) {
            if (!keep[i] || i == si) continue;
            newid[i] = id; out->node_state[id] = key_state(U[i]); out->node_step[id] = key_step(U[i]); id++;
        }
        rawarc_t *ka = malloc(sizeof(rawarc_t) * (n_raw ? n_raw : 1));
        int64_t na = 0;
        for (int64_t i = 0; i < n_raw; i++) {
            if (keep[fi[i]] && keep[ti[i]] && fwd[fi[i]] && bwd[ti[i]]) { ka[na] = raw[i]; ka[na].ord = i; na++; }
        }
        qsort(ka, na, sizeof(rawarc_t), cmp_rawarc_canon);
        out->n_arcs = na;
        out->arc_from = malloc(sizeof(int64_t) * (na ? na : 1)); out->arc_to = malloc(sizeof(int64_t) * (na ? na : 1));
        out->arc_tie = malloc(sizeof(int64_t) * (na ? na : 1));
        out->arc_il = malloc(sizeof(int32_t) * (na ? na : 1)); out->arc_ol = malloc(sizeof(int32_t) * (na ? na : 1));
        out->arc_g = malloc(sizeof(double) * (na ? na : 1)); out->arc_a = malloc(sizeof(double) * (na ? na : 1));
        for (int64_t i = 0; i < na; i++) {
            out->arc_from[i] = newid[find_i64(U, nu, ka[i].f)];
            out->arc_to[i] = newid[find_i64(U, nu, ka[i].t)];
            out->arc_il[i] = ka[i].il; out->arc_ol[i] = ka[i].ol;
            out->arc_g[i] = ka[i].g; out->arc_a[i] = ka[i].a; out->arc_tie[i] = ka[i].tie;
        }
        out->n_finals = n_lf;
        out->final_node = malloc(sizeof(int64_t) * n_lf); out->final_w = malloc(sizeof(double) * n_lf);
        for (int64_t i = 0; i < n_lf; i++) { out->final_node[i] = newid[lf_idx[i]]; out->final_w[i] = lf_w[i]; }
        free(ka); free(newid);
    }
    free(U); free(in_set); free(fi); free(ti); free(foff); free(boff); free(fadj); free(badj);
    free(fp); free(bp); free(fwd); free(bwd); free(livef); free(keep); free(lf_idx); free(lf_w);
}

typedef struct { int32_t state; int64_t id; } heap_item;
static void heap_push(heap_item *h, int64_t *n, heap_item x) {
    int64_t i = (*n)++;
    h[i] = x;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (h[p].state < h[i].state || (h[p].state == h[i].state && h[p].id <= h[i].id)) break;
        heap_item t = h[p]; h[p] = h[i]; h[i] = t; i = p;
    }
}
static heap_item heap_pop(heap_item *h, int64_t *n) {
    heap_item top = h[0];
    h[0] = h[--(*n)];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && (h[l].state < h[m].state || (h[l].state == h[m].state && h[l].id < h[m].id))) m = l;
        if (r < *n && (h[r].state < h[m].state || (h[r].state == h[m].state && h[r].id < h[m].id))) m = r;
        if (m == i) break;
        heap_item t = h[m]; h[m] = h[i]; h[i] = t; i = m;
    }
    return top;
}

static int cmp_step_id(const void *a, const void *b, void *ctx) {
    const og_lattice *l = ctx;
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    if (l->node_step[x] != l->node_step[y]) return l->node_step[x] < l->node_step[y] ? -1 : 1;
    return (x > y) - (x < y);
}

/* _topo_order, lattice.py:295-326: ascending step, epsilon-topological within a step with a
 * (state, id) min-heap.  Returns OG_ERR_LATTICE on an epsilon cycle among lattice nodes. */
static int topo_order(const og_lattice *l, int64_t *order) {
    int64_t n = l->n_nodes;
    int64_t *by = malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t i = 0; i < n; i++) by[i] = i;
    qsort_r(by, n, sizeof(int64_t), cmp_step_id, (void *)l);
    /* eps successor CSR (same-step arcs), in arc order */
    int64_t *off = calloc(n + 1, sizeof(int64_t));
    for (int64_t a = 0; a < l->n_arcs; a++)
        if (l->node_step[l->arc_from[a]] == l->node_step[l->arc_to[a]]) off[l->arc_from[a] + 1]++;
    for (int64_t i = 0; i < n; i++) off[i + 1] += off[i];
    int64_t *adj = malloc(sizeof(int64_t) * (off[n] ? off[n] : 1));
    int64_t *pos = malloc(sizeof(int64_t) * (n + 1));
    memcpy(pos, off, sizeof(int64_t) * (n + 1));
    for (int64_t a = 0; a < l->n_arcs; a++)
        if (l->node_step[l->arc_from[a]] == l->node_step[l->arc_to[a]]) adj[pos[l->arc_from[a]]++] = l->arc_to[a];
    int64_t *indeg = calloc(n ? n : 1, sizeof(int64_t));
    heap_item *h = malloc(sizeof(heap_item) * (n ? n : 1));
    int64_t on = 0; int rc = OG_OK;
    int64_t i0 = 0;
    while (i0 < n) {
        int64_t i1 = i0;
        while (i1 < n && l->node_step[by[i1]] == l->node_step[by[i0]]) i1++;
        for (int64_t t = i0; t < i1; t++)
            for (int64_t j = off[by[t]]; j < off[by[t] + 1]; j++) indeg[adj[j]]++;
        int64_t hn = 0;
        for (int64_t t = i0; t < i1; t++)
            if (indeg[by[t]] == 0) heap_push(h, &hn, (heap_item){l->node_state[by[t]], by[t]});
        int64_t emitted = 0;
        while (hn) {
            heap_item x = heap_pop(h, &hn);
            order[on++] = x.id; emitted++;
            for (int64_t j = off[x.id]; j < off[x.id + 1]; j++)
                if (--indeg[adj[j]] == 0) heap_push(h, &hn, (heap_item){l->node_state[adj[j]], adj[j]});
        }
        if (emitted != i1 - i0) { rc = OG_ERR_LATTICE; break; }
        i0 = i1;
    }
    free(by); free(off); free(adj); free(pos); free(indeg); free(h);
    return rc;
}

/* out-adjacency in arc order (Lattice.out_adjacency, lattice.py:71-75) */
static void out_csr(const og_lattice *l, int64_t **poff, int64_t **padj) {
    int64_t n = l->n_nodes;
    int64_t *off = calloc(n + 1, sizeof(int64_t));
    for (int64_t a = 0; a < l->n_arcs; a++) off[l->arc_from[a] + 1]++;
    for (int64_t i = 0; i < n; i++) off[i + 1] += off[i];
    int64_t *adj = malloc(sizeof(int64_t) * (l->n_arcs ? l->n_arcs : 1));
    int64_t *pos = malloc(sizeof(int64_t) * (n + 1));
    memcpy(pos, off, sizeof(int64_t) * (n + 1));
    for (int64_t a = 0; a < l->n_arcs; a++) adj[pos[l->arc_from[a]]++] = a;
    free(pos);
    *poff = off; *padj = adj;
}

/* _forward_costs / _backward_costs, lattice.py:329-356 */
static void forward_costs(const og_lattice *l, const int64_t *order, const int64_t *off,
                          const int64_t *adj, double *fw) {
    for (int64_t i = 0; i < l->n_nodes; i++) fw[i] = INF;
    fw[0] = 0.0;
    for (int64_t t = 0; t < l->n_nodes; t++) {
        int64_t i = order[t];
        double base = fw[i];
        if (base == INF) continue;
        for (int64_t j = off[i]; j < off[i + 1]; j++) {
            int64_t a = adj[j];
            double c = (base + l->arc_g[a]) + l->arc_a[a];
            if (c < fw[l->arc_to[a]]) fw[l->arc_to[a]] = c;
        }
    }
}
static void backward_costs(const og_lattice *l, const int64_t *order, const int64_t *off,
                           const int64_t *adj, double *bw) {
    for (int64_t i = 0; i < l->n_nodes; i++) bw[i] = INF;
    for (int64_t f = 0; f < l->n_finals; f++) bw[l->final_node[f]] = l->final_w[f];
    for (int64_t t = l->n_nodes - 1; t >= 0; t--) {
        int64_t i = order[t];
        double best = bw[i];
        for (int64_t j = off[i]; j < off[i + 1]; j++) {
            int64_t a = adj[j];
            double c = (l->arc_g[a] + l->arc_a[a]) + bw[l->arc_to[a]];
            if (c < best) best = c;
        }
        bw[i] = best;
    }
}

/* --- path-exact split (_enforce_path_soundness, lattice.py:400-501) --- */
typedef struct { int64_t node; uint64_t cbits; int32_t shared; } pkey_t;   /* shared: c is None */
typedef struct { pkey_t *keys; int64_t *slot; int64_t cap, n; } pset_t;

static uint64_t dbits(double x) { if (x == 0.0) x = 0.0; uint64_t u; memcpy(&u, &x, 8); return u; }
static double bitsd(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
static uint64_t phash(const pkey_t *k) {
    uint64_t h = (uint64_t)k->node * 0x9E3779B97F4A7C15ull ^ (k->cbits + 0x632BE59BD9B4E019ull);
    h ^= (uint64_t)k->shared * 0xC2B2AE3D27D4EB4Full;
    h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
    return h;
}
static int pkey_eq(const pkey_t *a, const pkey_t *b) {
    return a->node == b->node && a->shared == b->shared && (a->shared || a->cbits == b->cbits);
}
/* returns index (existing or new), *isnew set */
static int64_t pset_insert(pset_t *s, pkey_t k, int *isnew) {
    if (k.shared) k.cbits = 0;
    if ((s->n + 1) * 2 > s->cap) {
        int64_t nc = s->cap ? s->cap * 2 : 1024;
        int64_t *ns = malloc(sizeof(int64_t) * nc);
        for (int64_t i = 0; i < nc; i++) ns[i] = -1;
        for (int64_t i = 0; i < s->cap; i++) {
            if (s->slot[i] < 0) continue;
            uint64_t h = phash(&s->keys[s->slot[i]]) & (nc - 1);
            while (ns[h] >= 0) h = (h + 1) & (nc - 1);
            ns[h] = s->slot[i];
        }
        free(s->slot); s->slot = ns; s->cap = nc;
        s->keys = realloc(s->keys, sizeof(pkey_t) * nc);
    }
    uint64_t h = phash(&k) & (s->cap - 1);
    while (s->slot[h] >= 0) {
        if (pkey_eq(&s->keys[s->slot[h]], &k)) { *isnew = 0; return s->slot[h]; }
        h = (h + 1) & (s->cap - 1);
    }
    s->keys[s->n] = k; s->slot[h] = s->n; *isnew = 1;
    return s->n++;
}

typedef struct { int32_t step, state, flag; double c; int64_t idx; } psort_t;
static int cmp_psort(const void *pa, const void *pb) {
    const psort_t *a = pa, *b = pb;
    if (a->step != b->step) return a->step < b->step ? -1 : 1;
    if (a->state != b->state) return a->state < b->state ? -1 : 1;
    if (a->flag != b->flag) return a->flag < b->flag ? -1 : 1;
    if (a->c != b->c) return a->c < b->c ? -1 : 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}
typedef struct { int32_t fstep, fstate, tstep, tstate, il, ol; int64_t tie, fid, tid; double g, a; } parc_t;
static int cmp_parc(const void *pa, const void *pb) {
    const parc_t *a = pa, *b = pb;
#define C_(x) if (a->x != b->x) return a->x < b->x ? -1 : 1;
    C_(fstep) C_(fstate) C_(tstep) C_(tstate) C_(il) C_(ol) C_(tie) C_(fid) C_(tid)
#undef C_
    return 0;
}

static int enforce_path_soundness(og_lattice *lat, double cutoff, og_lattice *out) {
    int64_t n = lat->n_nodes;
    int64_t *order = malloc(sizeof(int64_t) * (n ? n : 1));
    int rc = topo_order(lat, order);
    if (rc) { free(order); return rc; }
    int64_t *off, *adj;
    out_csr(lat, &off, &adj);
    double NEG = -INF;
    double *fwmax = malloc(sizeof(double) * n), *bwmax = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; i++) { fwmax[i] = NEG; bwmax[i] = NEG; }
    fwmax[0] = 0.0;
    for (int64_t t = 0; t < n; t++) {
        int64_t i = order[t]; double base = fwmax[i];
        if (base == NEG) continue;
        for (int64_t j = off[i]; j < off[i + 1]; j++) {
            int64_t a = adj[j]; double c = (base + lat->arc_g[a]) + lat->arc_a[a];
            if (c > fwmax[lat->arc_to[a]]) fwmax[lat->arc_to[a]] = c;
        }
    }
    for (int64_t f = 0; f < lat->n_finals; f++) bwmax[lat->final_node[f]] = lat->final_w[f];
    for (int64_t t = n - 1; t >= 0; t--) {
        int64_t i = order[t]; double worst = bwmax[i];
        for (int64_t j = off[i]; j < off[i + 1]; j++) {
            int64_t a = adj[j]; double c = (lat->arc_g[a] + lat->arc_a[a]) + bwmax[lat->arc_to[a]];
            if (c > worst) worst = c;
        }
        bwmax[i] = worst;
    }
    uint8_t *safe = malloc(n);
    int all_safe = 1;
    for (int64_t i = 0; i < n; i++) { safe[i] = (fwmax[i] + bwmax[i]) <= cutoff; all_safe &= safe[i]; }
    if (all_safe) {
        *out = *lat; memset(lat, 0, sizeof(*lat));
        free(order); free(off); free(adj); free(fwmax); free(bwmax); free(safe);
        return OG_OK;
    }
    double *bwmin = malloc(sizeof(double) * n);
    backward_costs(lat, order, off, adj, bwmin);
    double *finw = malloc(sizeof(double) * n); uint8_t *isfin = calloc(n, 1);
    for (int64_t f = 0; f < lat->n_finals; f++) { finw[lat->final_node[f]] = lat->final_w[f]; isfin[lat->final_node[f]] = 1; }

    pset_t ps = {0};
    int isnew;
    pkey_t sk = {0, 0, safe[0] ? 1 : 0};
    sk.cbits = dbits(0.0);
    pset_insert(&ps, sk, &isnew);
    int64_t *stack = NULL, sn = 0, scap = 0;
    VEC_PUSH(stack, sn, scap, (int64_t)0, int64_t);
    typedef struct { int64_t from, to, arc; } karc_t;
    karc_t *ka = NULL; int64_t kn = 0, kcap = 0;
    while (sn && rc == OG_OK) {
        int64_t kidx = stack[--sn];
        pkey_t key = ps.keys[kidx];
        int64_t i = key.node;
        for (int64_t j = off[i]; j < off[i + 1]; j++) {
            int64_t a = adj[j]; int64_t to = lat->arc_to[a];
            pkey_t tk;
            if (key.shared) { tk.node = to; tk.shared = 1; tk.cbits = 0; }
            else {
                double c2 = (bitsd(key.cbits) + lat->arc_g[a]) + lat->arc_a[a];
                if (c2 + bwmin[to] > cutoff) continue;
                if (safe[to]) { tk.node = to; tk.shared = 1; tk.cbits = 0; }
                else { tk.node = to; tk.shared = 0; tk.cbits = dbits(c2); }
            }
            int64_t tidx = pset_insert(&ps, tk, &isnew);
            karc_t ke = {kidx, tidx, a};
            VEC_PUSH(ka, kn, kcap, ke, karc_t);
            if (isnew) {
                if (ps.n > PATH_KEY_CAP) { rc = OG_ERR_LATTICE; break; }
                VEC_PUSH(stack, sn, scap, tidx, int64_t);
            }
        }
    }
    if (rc == OG_OK) {
        int64_t nk = ps.n;
        psort_t *srt = malloc(sizeof(psort_t) * nk);
        for (int64_t x = 0; x < nk; x++) {
            pkey_t *k = &ps.keys[x];
            srt[x].step = lat->node_step[k->node]; srt[x].state = lat->node_state[k->node];
            srt[x].flag = k->shared ? 0 : 1; srt[x].c = k->shared ? 0.0 : bitsd(k->cbits); srt[x].idx = x;
        }
        /* start key first, the rest sorted */
        qsort(srt + 1, nk - 1, sizeof(psort_t), cmp_psort);
        int64_t *newid = malloc(sizeof(int64_t) * nk);
        for (int64_t x = 0; x < nk; x++) newid[srt[x].idx] = x;
        out->empty = 0; out->n_nodes = nk;
        out->node_state = malloc(sizeof(int32_t) * nk); out->node_step = malloc(sizeof(int32_t) * nk);
        for (int64_t x = 0; x < nk; x++) {
            int64_t nd = ps.keys[srt[x].idx].node;
            out->node_state[x] = lat->node_state[nd]; out->node_step[x] = lat->node_step[nd];
        }
        parc_t *pa = malloc(sizeof(parc_t) * (kn ? kn : 1));
        for (int64_t e = 0; e < kn; e++) {
            int64_t a = ka[e].arc; int64_t fid = newid[ka[e].from], tid = newid[ka[e].to];
            pa[e] = (parc_t){out->node_step[fid], out->node_state[fid], out->node_step[tid], out->node_state[tid],
                             lat->arc_il[a], lat->arc_ol[a], lat->arc_tie[a], fid, tid, lat->arc_g[a], lat->arc_a[a]};
        }
        qsort(pa, kn, sizeof(parc_t), cmp_parc);
        out->n_arcs = kn;
        out->arc_from = malloc(sizeof(int64_t) * (kn ? kn : 1)); out->arc_to = malloc(sizeof(int64_t) * (kn ? kn : 1));
        out->arc_tie = malloc(sizeof(int64_t) * (kn ? kn : 1));
        out->arc_il = malloc(sizeof(int32_t) * (kn ? kn : 1)); out->arc_ol = malloc(sizeof(int32_t) * (kn ? kn : 1));
        out->arc_g = malloc(sizeof(double) * (kn ? kn : 1)); out->arc_a = malloc(sizeof(double) * (kn ? kn : 1));
        for (int64_t e = 0; e < kn; e++) {
            out->arc_from[e] = pa[e].fid; out->arc_to[e] = pa[e].tid; out->arc_tie[e] = pa[e].tie;
            out->arc_il[e] = pa[e].il; out->arc_ol[e] = pa[e].ol; out->arc_g[e] = pa[e].g; out->arc_a[e] = pa[e].a;
        }
        /* key_finals in key-set iteration order; dict equality is order-free */
        out->final_node = malloc(sizeof(int64_t) * nk); out->final_w = malloc(sizeof(double) * nk);
        int64_t nf = 0;
        for (int64_t x = 0; x < nk; x++) {
            pkey_t *k = &ps.keys[x];
            if (!isfin[k->node]) continue;
            double w = finw[k->node];
            if (k->shared || bitsd(k->cbits) + w <= cutoff) { out->final_node[nf] = newid[x]; out->final_w[nf] = w; nf++; }
        }
        out->n_finals = nf;
        free(srt); free(newid); free(pa);
    }
    free(order); free(off); free(adj); free(fwmax); free(bwmax); free(safe); free(bwmin); free(finw);
    free(isfin); free(ps.keys); free(ps.slot); free(stack); free(ka);
    return rc;
}

/* build_lattice (lattice.py:240-249) from a recorded decode (_Accumulator.add_step/build,
 * lattice.py:148-187).  Returns OG_ERR_LATTICE for a within-step epsilon cycle (lattice.py:186). */
int og_build_lattice(const og_graph *g, const og_result *r, og_lattice *out) {
    memset(out, 0, sizeof(*out));
    if (r->n_node_steps == 0) { lattice_empty(out); return OG_OK; }
    int64_t n_nodes_all = r->surv_off[r->n_node_steps];
    int64_t *nodeset = malloc(sizeof(int64_t) * (n_nodes_all ? n_nodes_all : 1));
    for (int32_t k = 0; k < r->n_node_steps; k++)
        for (int64_t i = r->surv_off[k]; i < r->surv_off[k + 1]; i++) nodeset[i] = nkey(k, r->surv[i]);
    int64_t nns = uniq_i64(nodeset, n_nodes_all);
    rawarc_t *raw = NULL; int64_t nr = 0, rcap = 0;
    /* events are appended in step order; walk them per step */
    int64_t e = 0, q = 0;
    int64_t *epsk = NULL; int64_t en = 0, ecap = 0;
    for (int32_t k = 0; k < r->n_node_steps; k++) {
        const int32_t *surv = r->surv + r->surv_off[k];
        int64_t ns = r->surv_off[k + 1] - r->surv_off[k];
        const int32_t *prev = k > 0 ? r->surv + r->surv_off[k - 1] : NULL;
        int64_t np = k > 0 ? r->surv_off[k] - r->surv_off[k - 1] : 0;
        int64_t e0 = e;
        while (e < r->n_emit && r->emit_step[e] == k) e++;
        if (k > 0) {
            /* (src, ai) dedup of lattice.py:155-160 is a no-op here: a serial decode relaxes
             * each (src, arc) once per step */
            for (int64_t x = e0; x < e; x++) {
                int32_t src = r->emit_src[x], ai = r->emit_arc[x], dst = g->dst[ai];
                int32_t key = src;
                if (bsearch(&key, prev, np, sizeof(int32_t), cmp_i32) && bsearch(&dst, surv, ns, sizeof(int32_t), cmp_i32)) {
                    rawarc_t ra = {nkey(k - 1, src), nkey(k, dst), g->ilabel[ai], g->olabel[ai], g->weight[ai],
                                   r->emit_ac[x], ai, 0};
                    VEC_PUSH(raw, nr, rcap, ra, rawarc_t);
                }
            }
        }
        int64_t q0 = q;
        while (q < r->n_eps && r->eps_step[q] == k) q++;
        en = 0;
        for (int64_t x = q0; x < q; x++) {
            int64_t v = ((int64_t)r->eps_src[x] << 32) | (uint32_t)r->eps_arc[x];
            VEC_PUSH(epsk, en, ecap, v, int64_t);
        }
        en = uniq_i64(epsk, en);   /* sorted(rec.eps) */
        for (int64_t x = 0; x < en; x++) {
            int32_t src = (int32_t)(epsk[x] >> 32), ai = (int32_t)(uint32_t)(epsk[x] & 0xffffffff);
            int32_t dst = g->dst[ai];
            if (dst != src && bsearch(&src, surv, ns, sizeof(int32_t), cmp_i32) &&
                bsearch(&dst, surv, ns, sizeof(int32_t), cmp_i32)) {
                rawarc_t ra = {nkey(k, src), nkey(k, dst), g->ilabel[ai], g->olabel[ai], g->weight[ai], 0.0, ai, 0};
                VEC_PUSH(raw, nr, rcap, ra, rawarc_t);
            }
        }
    }
    /* finals (lattice.py:172-183) */
    int64_t nfmax = 1;
    if (r->reached_final && r->final_step < r->n_node_steps)
        nfmax += r->surv_off[r->final_step + 1] - r->surv_off[r->final_step];
    int64_t *fk = malloc(sizeof(int64_t) * nfmax); double *fwv = malloc(sizeof(double) * nfmax);
    int64_t nfin = 0;
    if (r->reached_final) {
        int32_t fs = r->final_step;
        if (fs < r->n_node_steps) {
            for (int64_t i = r->surv_off[fs]; i < r->surv_off[fs + 1]; i++) {
                double w = g->final_w[r->surv[i]];
                if (w != INF) { fk[nfin] = nkey(fs, r->surv[i]); fwv[nfin] = w; nfin++; }
            }
        }
    } else {
        fk[nfin] = nkey(r->final_step, r->final_state); fwv[nfin] = 0.0; nfin++;
    }
    assemble(nodeset, nns, raw, nr, nkey(0, g->start), fk, fwv, nfin, out);
    int rc = OG_OK;
    if (!out->empty && out->n_finals > 0) {
        int64_t *order = malloc(sizeof(int64_t) * (out->n_nodes ? out->n_nodes : 1));
        rc = topo_order(out, order);
        free(order);
    }
    free(nodeset); free(raw); free(epsk); free(fk); free(fwv);
    return rc;
}

/* prune_lattice, lattice.py:359-397 (stage 1 + the path-exact stage) */
int og_prune_lattice(const og_lattice *lat, double beam, og_lattice *out) {
    memset(out, 0, sizeof(*out));
    if (beam < 0) return OG_ERR_VALUE;
    if (lat->empty || lat->n_finals == 0) { lattice_empty(out); return OG_OK; }
    int64_t n = lat->n_nodes;
    int64_t *order = malloc(sizeof(int64_t) * n);
    int rc = topo_order(lat, order);
    if (rc) { free(order); return rc; }
    int64_t *off, *adj;
    out_csr(lat, &off, &adj);
    double *fw = malloc(sizeof(double) * n), *bw = malloc(sizeof(double) * n);
    forward_costs(lat, order, off, adj, fw);
    backward_costs(lat, order, off, adj, bw);
    double best = bw[0];
    if (best == INF) {
        lattice_empty(out);
        free(order); free(off); free(adj); free(fw); free(bw);
        return OG_OK;
    }
    double cutoff = (best + beam) + COST_EPS;
    rawarc_t *raw = malloc(sizeof(rawarc_t) * (lat->n_arcs ? lat->n_arcs : 1));
    int64_t nr = 0;
    int64_t *nodes = malloc(sizeof(int64_t) * (2 * lat->n_arcs + lat->n_finals + 1));
    int64_t nn = 0;
    for (int64_t a = 0; a < lat->n_arcs; a++) {
        int64_t f = lat->arc_from[a], t = lat->arc_to[a];
        if (((fw[f] + lat->arc_g[a]) + lat->arc_a[a]) + bw[t] <= cutoff) {
            raw[nr++] = (rawarc_t){nkey(lat->node_step[f], lat->node_state[f]), nkey(lat->node_step[t], lat->node_state[t]),
                                   lat->arc_il[a], lat->arc_ol[a], lat->arc_g[a], lat->arc_a[a], lat->arc_tie[a], 0};
            nodes[nn++] = raw[nr - 1].f; nodes[nn++] = raw[nr - 1].t;
        }
    }
    int64_t *fk = malloc(sizeof(int64_t) * (lat->n_finals ? lat->n_finals : 1));
    double *fwv = malloc(sizeof(double) * (lat->n_finals ? lat->n_finals : 1));
    int64_t nf = 0;
    for (int64_t x = 0; x < lat->n_finals; x++) {
        int64_t i = lat->final_node[x];
        if (fw[i] + lat->final_w[x] <= cutoff) {
            fk[nf] = nkey(lat->node_step[i], lat->node_state[i]); fwv[nf] = lat->final_w[x]; nf++;
            nodes[nn++] = fk[nf - 1];
        }
    }
    int64_t sk = nkey(lat->node_step[0], lat->node_state[0]);
    nodes[nn++] = sk;
    nn = uniq_i64(nodes, nn);
    og_lattice kept;
    memset(&kept, 0, sizeof(kept));
    assemble(nodes, nn, raw, nr, sk, fk, fwv, nf, &kept);
    free(order); free(off); free(adj); free(fw); free(bw); free(raw); free(nodes); free(fk); free(fwv);
    if (kept.empty || kept.n_finals == 0) { *out = kept; return OG_OK; }
    rc = enforce_path_soundness(&kept, cutoff, out);
    og_lattice_free(&kept);
    return rc;
}

/* stage one only: exact forward-backward arc pruning + trim (lattice.py:370-394) */
int og_prune_lattice_stage1(const og_lattice *lat, double beam, og_lattice *out, double *cutoff_out) {
    memset(out, 0, sizeof(*out));
    if (beam < 0) return OG_ERR_VALUE;
    if (lat->empty || lat->n_finals == 0) { lattice_empty(out); return OG_OK; }
    int64_t n = lat->n_nodes;
    int64_t *order = malloc(sizeof(int64_t) * n);
    int rc = topo_order(lat, order);
    if (rc) { free(order); return rc; }
    int64_t *off, *adj;
    out_csr(lat, &off, &adj);
    double *fw = malloc(sizeof(double) * n), *bw = malloc(sizeof(double) * n);
    forward_costs(lat, order, off, adj, fw);
    backward_costs(lat, order, off, adj, bw);
    double best = bw[0];
    if (best == INF) {
        lattice_empty(out);
        free(order); free(off); free(adj); free(fw); free(bw);
        return OG_OK;
    }
    double cutoff = (best + beam) + COST_EPS;
    if (cutoff_out) *cutoff_out = cutoff;
    rawarc_t *raw = malloc(sizeof(rawarc_t) * (lat->n_arcs ? lat->n_arcs : 1));
    int64_t nr = 0;
    int64_t *nodes = malloc(sizeof(int64_t) * (2 * lat->n_arcs + lat->n_finals + 1));
    int64_t nn = 0;
    for (int64_t a = 0; a < lat->n_arcs; a++) {
        int64_t f = lat->arc_from[a], t = lat->arc_to[a];
        if (((fw[f] + lat->arc_g[a]) + lat->arc_a[a]) + bw[t] <= cutoff) {
            raw[nr++] = (rawarc_t){nkey(lat->node_step[f], lat->node_state[f]), nkey(lat->node_step[t], lat->node_state[t]),
                                   lat->arc_il[a], lat->arc_ol[a], lat->arc_g[a], lat->arc_a[a], lat->arc_tie[a], 0};
            nodes[nn++] = raw[nr - 1].f; nodes[nn++] = raw[nr - 1].t;
        }
    }
    int64_t *fk = malloc(sizeof(int64_t) * (lat->n_finals ? lat->n_finals : 1));
    double *fwv = malloc(sizeof(double) * (lat->n_finals ? lat->n_finals : 1));
    int64_t nf = 0;
    for (int64_t x = 0; x < lat->n_finals; x++) {
        int64_t i = lat->final_node[x];
        if (fw[i] + lat->final_w[x] <= cutoff) {
            fk[nf] = nkey(lat->node_step[i], lat->node_state[i]); fwv[nf] = lat->final_w[x]; nf++;
            nodes[nn++] = fk[nf - 1];
        }
    }
    int64_t sk = nkey(lat->node_step[0], lat->node_state[0]);
    nodes[nn++] = sk;
    nn = uniq_i64(nodes, nn);
    assemble(nodes, nn, raw, nr, sk, fk, fwv, nf, out);
    free(order); free(off); free(adj); free(fw); free(bw); free(raw); free(nodes); free(fk); free(fwv);
    return OG_OK;
}

/* lattice_best_path, lattice.py:504-559.  Labels are malloc'ed into *olabels / *ilabels. */
int og_lattice_best_path(const og_lattice *lat, double *cost, int32_t **olabels, int32_t *n_o,
                         int32_t **ilabels, int32_t *n_i) {
    if (lat->empty || lat->n_finals == 0) return OG_ERR_LATTICE;
    int64_t n = lat->n_nodes;
    int64_t *order = malloc(sizeof(int64_t) * n);
    int rc = topo_order(lat, order);
    if (rc) { free(order); return rc; }
    /* in-adjacency in arc order */
    int64_t *off = calloc(n + 1, sizeof(int64_t));
    for (int64_t a = 0; a < lat->n_arcs; a++) off[lat->arc_to[a] + 1]++;
    for (int64_t i = 0; i < n; i++) off[i + 1] += off[i];
    int64_t *adj = malloc(sizeof(int64_t) * (lat->n_arcs ? lat->n_arcs : 1));
    int64_t *pos = malloc(sizeof(int64_t) * (n + 1));
    memcpy(pos, off, sizeof(int64_t) * (n + 1));
    for (int64_t a = 0; a < lat->n_arcs; a++) adj[pos[lat->arc_to[a]]++] = a;
    double *dist = malloc(sizeof(double) * n);
    int64_t *back = malloc(sizeof(int64_t) * n);
    for (int64_t i = 0; i < n; i++) { dist[i] = INF; back[i] = -1; }
    dist[0] = 0.0;
    for (int64_t t = 0; t < n; t++) {
        int64_t i = order[t];
        if (i == 0) continue;
        int have = 0; double bc = 0; int32_t bs = 0; int64_t btie = 0, ba = -1;
        for (int64_t j = off[i]; j < off[i + 1]; j++) {
            int64_t a = adj[j];
            double base = dist[lat->arc_from[a]];
            if (base == INF) continue;
            double c = (base + lat->arc_g[a]) + lat->arc_a[a];
            int32_t st = lat->node_state[lat->arc_from[a]];
            int64_t tie = lat->arc_tie[a];
            if (!have || c < bc || (c == bc && (st < bs || (st == bs && tie < btie)))) {
                have = 1; bc = c; bs = st; btie = tie; ba = a;
            }
        }
        if (have) { dist[i] = bc; back[i] = ba; }
    }
    /* finals sorted by node state (stable), strict < */
    int64_t bf = -1; double bt = INF;
    int64_t *fo = malloc(sizeof(int64_t) * lat->n_finals);
    for (int64_t x = 0; x < lat->n_finals; x++) fo[x] = x;
    for (int64_t x = 1; x < lat->n_finals; x++) { /* insertion sort, stable */
        int64_t v = fo[x], y = x - 1;
        while (y >= 0 && lat->node_state[lat->final_node[fo[y]]] > lat->node_state[lat->final_node[v]]) { fo[y + 1] = fo[y]; y--; }
        fo[y + 1] = v;
    }
    for (int64_t x = 0; x < lat->n_finals; x++) {
        int64_t i = lat->final_node[fo[x]];
        double total = dist[i] + lat->final_w[fo[x]];
        if (total < bt) { bt = total; bf = i; }
    }
    if (bf < 0 || bt == INF) rc = OG_ERR_LATTICE;
    else {
        int32_t no = 0, ni = 0;
        for (int64_t i = bf; back[i] >= 0; i = lat->arc_from[back[i]]) {
            if (lat->arc_ol[back[i]] != 0) no++;
            if (lat->arc_il[back[i]] != 0) ni++;
        }
        int32_t *ol = malloc(sizeof(int32_t) * (no ? no : 1)), *il = malloc(sizeof(int32_t) * (ni ? ni : 1));
        int32_t po = no, pi = ni;
        for (int64_t i = bf; back[i] >= 0; i = lat->arc_from[back[i]]) {
            if (lat->arc_ol[back[i]] != 0) ol[--po] = lat->arc_ol[back[i]];
            if (lat->arc_il[back[i]] != 0) il[--pi] = lat->arc_il[back[i]];
        }
        *cost = bt; *olabels = ol; *ilabels = il; *n_o = no; *n_i = ni;
    }
    free(order); free(off); free(adj); free(pos); free(dist); free(back); free(fo);
    return rc;
}

void og_free(void *p) { free(p); }
