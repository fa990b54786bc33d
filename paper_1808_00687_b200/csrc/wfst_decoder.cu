// wfst_decoder.cu -- B200-native batched WFST Viterbi beam search (arXiv 1808.00687).
//
// One persistent kernel decodes a whole batch: each CTA is an "utterance lane" that pulls
// utterances from an atomic queue and runs the complete frame loop for one utterance with
// CTA-level barriers only (no grid syncs, no per-frame launches).  Within a step the CTA's
// warps cooperate:
//
//   expand   warp-level load balancing: a warp takes 32 live tokens, prefix-sums their
//            emitting out-degrees with shuffles and strides its lanes over the flattened
//            token x arc range (the paper's "tokens x arcs assigned by prefix-summed
//            out-degree"); arc records are 16-byte coalescible loads; the frame's cost row
//            is staged in shared memory; recombination is a 128-bit atomic CAS on a dense
//            per-state slot {cost key, arc+1, payload} under the reference's
//            (cost, src state, arc) total order  (decoder.py:205-225, 121-135)
//   closure  frontier rounds over the epsilon arcs of improved states with an epoch-tagged
//            dedup queue (decoder.py:138-171, parallel.py:287-325)
//   prune    exact beam + max-active cut: min/max reduce, 4096-bucket value histogram in
//            shared memory, then an exact (cost, state) rank inside the boundary bucket
//            (radix select fallback) -- no sort (decoder.py:174-194)
//   compact  survivors + the epsilon-chain candidates they trace through get backpointer
//            records in a batch-wide arena; slots are reset O(touched)
//
// Arithmetic is float64 in the reference's association order, so costs, survivor sets,
// tokens_expanded and (on tie-free inputs) labels are bit-identical to decoder.py.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/wfst_b200.h"
#include "device_common.cuh"

namespace wb {

constexpr int NB = 4096;         // prune histogram buckets
constexpr int GCAP = 1024;       // boundary-bucket members ranked in shared memory
constexpr int ROW_SMEM_MAX = 12288;  // cost-row columns staged in shared memory (96 KB)
constexpr u32 F_SURV = 1u, F_MARK = 2u;
constexpr int MAX_EPS_ROUNDS = 1 << 20;
constexpr int UNROLL = 4;

struct GraphDev {
    int S, A, start, has_eps;
    const int4 *info;       // [S] {eps_lo, eps_hi (= emit_lo), emit_hi, 0}
    const int4 *arcs;       // [A] {dst, ilabel, weight_lo, weight_hi}
    const int *olabel;      // [A]
    const double *final_w;  // [S]
};

struct WorkDev {
    Slot *slot;             // [slots][S]
    u32 *cand_of;           // [slots][S]
    u32 *qtag;              // [slots][S]
    u32 *tag_ctr;           // [slots]
    u32 *cand_state;        // [slots][cap]
    u64 *cand_key;
    u32 *cand_arc, *cand_pay, *cand_flags, *cand_arena;
    u32 *front;             // [slots][2][cap]
    int4 *tok_info;         // [slots][2][cap] {state, trace, emit_lo, emit_hi}
    double *tok_cost;       // [slots][2][cap]
    int *frames;            // [slots][T_cap]
    u64 *arena;             // [arena_cap] (arcp1 | prev << 32)
    u64 arena_cap;
    u64 *arena_ctr;
    u32 *utt_ctr;
    long long S;
    int cap, T_cap;
};

struct BatchDev {
    const double *costs;
    const long long *row_off;
    const int *T;
    const double *blank;
    int L1, n;
};

struct CfgDev {
    double beam, thr;
    int max_active, mode, lattice;
};

template <int BLOCK>
struct Smem {
    static constexpr int NW = BLOCK / 32;
    u32 wa[NW + 1], wb[NW + 1];
    u64 r0[NW], r1[NW];
    long long rl[NW];
    int n_cand, n_front, overflow, utt, tag_round, ng, thr_bucket, thr_below;
    u64 thr_key;
    u32 thr_state;
    u64 arena_base;
    union {
        u32 hist[NB];
        struct {
            u64 key[GCAP];
            u32 st[GCAP];
        } g;
    } u;
};

// ------------------------------------------------------------------ block primitives
template <int BLOCK>
__device__ __forceinline__ void block_minmax(u64 &mn, u64 &mx, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    mn = warp_min_u64(mn);
    mx = warp_max_u64(mx);
    if (l == 0) { sh.r0[w] = mn; sh.r1[w] = mx; }
    __syncthreads();
    if (w == 0) {
        u64 a = l < NW ? sh.r0[l] : EMPTY_KEY, b = l < NW ? sh.r1[l] : 0ull;
        a = warp_min_u64(a);
        b = warp_max_u64(b);
        if (l == 0) { sh.r0[0] = a; sh.r1[0] = b; }
    }
    __syncthreads();
    mn = sh.r0[0];
    mx = sh.r1[0];
    __syncthreads();
}

template <int BLOCK>
__device__ __forceinline__ long long block_sum(long long v, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    v = warp_sum_ll(v);
    if (l == 0) sh.rl[w] = v;
    __syncthreads();
    if (w == 0) {
        long long a = l < NW ? sh.rl[l] : 0;
        a = warp_sum_ll(a);
        if (l == 0) sh.rl[0] = a;
    }
    __syncthreads();
    v = sh.rl[0];
    __syncthreads();
    return v;
}

// Two-predicate order-preserving compaction over [0, n): warps own contiguous segments,
// ballots count, one scan over warp totals.  emit(i, ia, ib) gets the running indices of
// predicate a / b (valid only where that predicate holds).  Returns totals via ta / tb.
template <int BLOCK, class PA, class PB, class EMIT>
__device__ __forceinline__ void block_compact2(int n, PA pa, PB pb, EMIT emit, Smem<BLOCK> &sh,
                                               int &ta, int &tb) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int seg = ((n + NW - 1) / NW + 31) & ~31;
    int lo = min(n, w * seg), hi = min(n, lo + seg);
    int ca = 0, cb = 0;
    for (int i0 = lo; i0 < hi; i0 += 32) {
        int i = i0 + l;
        bool a = false, b = false;
        if (i < hi) { a = pa(i); b = pb(i); }
        ca += __popc(__ballot_sync(FULL, a));
        cb += __popc(__ballot_sync(FULL, b));
    }
    if (l == 0) { sh.wa[w] = ca; sh.wb[w] = cb; }
    __syncthreads();
    if (w == 0) {
        int va = l < NW ? sh.wa[l] : 0, vb = l < NW ? sh.wb[l] : 0;
        int ia = warp_incl_scan(va), ib = warp_incl_scan(vb);
        if (l < NW) { sh.wa[l] = ia - va; sh.wb[l] = ib - vb; }
        if (l == 31) { sh.wa[NW] = ia; sh.wb[NW] = ib; }
    }
    __syncthreads();
    int ra = sh.wa[w], rb = sh.wb[w];
    ta = sh.wa[NW];
    tb = sh.wb[NW];
    const u32 lt = lanemask_lt();
    for (int i0 = lo; i0 < hi; i0 += 32) {
        int i = i0 + l;
        bool a = false, b = false;
        if (i < hi) { a = pa(i); b = pb(i); }
        u32 ma = __ballot_sync(FULL, a), mb = __ballot_sync(FULL, b);
        if (a || b) emit(i, ra + __popc(ma & lt), rb + __popc(mb & lt));
        ra += __popc(ma);
        rb += __popc(mb);
    }
    __syncthreads();
}

// ------------------------------------------------------------------ per-utterance state
struct UttCtx {
    Slot *slot;
    u32 *cand_of, *qtag;
    u32 *cand_state, *cand_arc, *cand_pay, *cand_flags, *cand_arena;
    u64 *cand_key;
    u32 *front[2];
    int4 *tok_info[2];
    double *tok_cost[2];
    int *frames;
    const double *row;  // current cost row (shared or global)
    u32 tag;
    // per-thread counters
    long long a_emit, a_fin, e_eps;
};

template <int BLOCK>
__device__ __forceinline__ void append_cand(u32 d, const GraphDev &g, const WorkDev &ws,
                                            UttCtx &c, Smem<BLOCK> &sh, u32 *front_out,
                                            bool push_front) {
    int idx = atomicAdd(&sh.n_cand, 1);
    if (idx < ws.cap) {
        c.cand_state[idx] = d;
        c.cand_of[d] = (u32)idx;
        if (push_front) {
            int4 inf = __ldg(&g.info[d]);
            if (inf.x < inf.y) {
                int f = atomicAdd(&sh.n_front, 1);
                front_out[f] = d;
            }
        }
    } else {
        sh.overflow = 1;
    }
}

// Emitting expansion of all live tokens (viterbi_step's emitting loop, decoder.py:212-225).
template <int BLOCK>
__device__ void expand_emitting(int n_live, int cur, const GraphDev &g, const WorkDev &ws,
                                UttCtx &c, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int4 *tinfo = c.tok_info[cur];
    const double *tcost = c.tok_cost[cur];
    u32 *front0 = c.front[0];
    const bool push = g.has_eps;
    const int nchunks = (n_live + 31) >> 5;
    for (int ch = w; ch < nchunks; ch += NW) {
        int t = (ch << 5) + l;
        int4 ti = make_int4(0, 0, 0, 0);
        double tc = 0.0;
        if (t < n_live) { ti = tinfo[t]; tc = tcost[t]; }
        int deg = t < n_live ? ti.w - ti.z : 0;
        c.a_emit += deg;
        int incl = warp_incl_scan(deg);
        int total = __shfl_sync(FULL, incl, 31);
        int excl = incl - deg;
        for (int j0 = 0; j0 < total; j0 += 32 * UNROLL) {
            int4 rec[UNROLL];
            double cst[UNROLL];
            u32 pay[UNROLL];
            int arc[UNROLL];
            bool ok[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                int j = j0 + u * 32 + l;
                int k = warp_owner(excl, j);
                int lo_k = __shfl_sync(FULL, ti.z, k);
                int ex_k = __shfl_sync(FULL, excl, k);
                cst[u] = __shfl_sync(FULL, tc, k);
                pay[u] = (u32)__shfl_sync(FULL, ti.y, k);
                ok[u] = j < total;
                arc[u] = lo_k + j - ex_k;
                if (ok[u]) rec[u] = __ldg(&g.arcs[arc[u]]);
            }
            Slot cur_s[UNROLL];
            u64 key[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                if (ok[u]) {
                    double ac = c.row[rec[u].y];
                    if (ac == INFINITY) {
                        ok[u] = false;
                    } else {
                        double wgt = __hiloint2double(rec[u].w, rec[u].z);
                        double cc = __dadd_rn(__dadd_rn(cst[u], wgt), ac);
                        key[u] = cost_key(cc);
                        cur_s[u] = ld_slot(&c.slot[rec[u].x]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                if (!ok[u]) continue;
                c.a_fin++;
                Slot *p = &c.slot[rec[u].x];
                Slot want;
                want.key = key[u];
                want.arcp1 = (u32)arc[u] + 1u;
                want.pay = pay[u];
                Slot cs = cur_s[u];
                while (slot_better(want.key, want.arcp1, cs)) {
                    Slot prev = cas_slot(p, cs, want);
                    if (prev.key == cs.key && prev.arcp1 == cs.arcp1 && prev.pay == cs.pay) {
                        if (cs.key == EMPTY_KEY)
                            append_cand<BLOCK>((u32)rec[u].x, g, ws, c, sh, front0, push);
                        break;
                    }
                    cs = prev;
                }
            }
        }
    }
}

// Epsilon closure to a fixpoint by frontier rounds (decoder.py:138-171; Jacobi form
// parallel.py:287-325).  Self-loops are skipped (decoder.py:162-163).  Payload of an epsilon
// winner = candidate index of its source state | EPS_BIT.
template <int BLOCK>
__device__ void epsilon_closure(const GraphDev &g, const WorkDev &ws, UttCtx &c, Smem<BLOCK> &sh,
                                int &status) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int which = 0;
    int rounds = 0;
    for (;;) {
        int n_front = sh.n_front;
        __syncthreads();
        if (n_front == 0) break;
        if (++rounds > MAX_EPS_ROUNDS) { status = WB_ERR_CAPACITY; break; }
        if (threadIdx.x == 0) {
            sh.n_front = 0;
            sh.tag_round = (int)(++c.tag);
        }
        __syncthreads();
        const u32 tag = (u32)sh.tag_round;
        c.tag = tag;
        const u32 *fin = c.front[which];
        u32 *fout = c.front[which ^ 1];
        const int nchunks = (n_front + 31) >> 5;
        for (int ch = w; ch < nchunks; ch += NW) {
            int i = (ch << 5) + l;
            u32 uu = 0;
            int lo = 0, deg = 0;
            double ucost = 0.0;
            u32 ui = 0;
            if (i < n_front) {
                uu = fin[i];
                int4 inf = __ldg(&g.info[uu]);
                lo = inf.x;
                deg = inf.y - inf.x;
                ucost = key_cost(ld_slot(&c.slot[uu]).key);
                ui = c.cand_of[uu];
            }
            int incl = warp_incl_scan(deg);
            int total = __shfl_sync(FULL, incl, 31);
            int excl = incl - deg;
            for (int j0 = 0; j0 < total; j0 += 32) {
                int j = j0 + l;
                int k = warp_owner(excl, j);
                int lo_k = __shfl_sync(FULL, lo, k);
                int ex_k = __shfl_sync(FULL, excl, k);
                double uc_k = __shfl_sync(FULL, ucost, k);
                u32 u_k = __shfl_sync(FULL, uu, k);
                u32 ui_k = __shfl_sync(FULL, ui, k);
                if (j >= total) continue;
                int a = lo_k + j - ex_k;
                int4 rec = __ldg(&g.arcs[a]);
                if ((u32)rec.x == u_k) continue;  // a positive self-loop never improves its state
                c.e_eps++;
                double wgt = __hiloint2double(rec.w, rec.z);
                u64 key = cost_key(__dadd_rn(uc_k, wgt));
                bool first = false, dec = false;
                if (relax_slot(&c.slot[rec.x], key, (u32)a + 1u, ui_k | EPS_BIT, &first, &dec)) {
                    if (first) append_cand<BLOCK>((u32)rec.x, g, ws, c, sh, fout, false);
                    if (first || dec) {
                        int4 dinf = __ldg(&g.info[rec.x]);
                        if (dinf.x < dinf.y && atomicExch(&c.qtag[rec.x], tag) != tag) {
                            int f = atomicAdd(&sh.n_front, 1);
                            if (f < ws.cap) fout[f] = (u32)rec.x;
                            else sh.overflow = 1;
                        }
                    }
                }
            }
        }
        __syncthreads();
        which ^= 1;
    }
}

__device__ __forceinline__ int bucket_of(double cst, double best, double scale) {
    double v = __dmul_rn(__dsub_rn(cst, best), scale);
    if (!(v < (double)(NB - 1))) return NB - 1;
    return (int)v;
}

// Exact max-active cut: find K* = the max_active-th smallest (cost, state) among kept
// candidates (decoder.py:188-191).  Sets sh.thr_bucket / sh.thr_key / sh.thr_state.
template <int BLOCK>
__device__ void select_threshold(int n_cand, int max_active, double best, double cutoff,
                                 double scale, UttCtx &c, Smem<BLOCK> &sh) {
    for (int b = threadIdx.x; b < NB; b += BLOCK) sh.u.hist[b] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
        double cst = key_cost(c.cand_key[i]);
        if (cst <= cutoff) atomicAdd(&sh.u.hist[bucket_of(cst, best, scale)], 1u);
    }
    __syncthreads();
    // smallest b with inclusive prefix >= max_active
    constexpr int PER = NB / BLOCK;
    u32 loc[PER];
    u32 s = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) { loc[q] = sh.u.hist[threadIdx.x * PER + q]; s += loc[q]; }
    // block exclusive scan of s
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int incl = warp_incl_scan((int)s);
    if (l == 31) sh.wa[w] = incl;
    __syncthreads();
    if (w == 0) {
        int v = l < NW ? sh.wa[l] : 0;
        int iv = warp_incl_scan(v);
        if (l < NW) sh.wa[l] = iv - v;
    }
    __syncthreads();
    u32 run = sh.wa[w] + incl - s;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        if (run < (u32)max_active && run + loc[q] >= (u32)max_active) {
            sh.thr_bucket = threadIdx.x * PER + q;
            sh.thr_below = (int)run;
            sh.ng = (int)loc[q];
        }
        run += loc[q];
    }
    __syncthreads();
    const int bstar = sh.thr_bucket;
    int r = max_active - sh.thr_below;  // rank (1-based) inside the boundary bucket
    const int cnt = sh.ng;
    __syncthreads();
    if (cnt <= GCAP) {
        if (threadIdx.x == 0) sh.ng = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
            u64 k = c.cand_key[i];
            double cst = key_cost(k);
            if (cst <= cutoff && bucket_of(cst, best, scale) == bstar) {
                int j = atomicAdd(&sh.ng, 1);
                sh.u.g.key[j] = k;
                sh.u.g.st[j] = c.cand_state[i];
            }
        }
        __syncthreads();
        const int m = sh.ng;
        for (int j = threadIdx.x; j < m; j += BLOCK) {
            u64 kj = sh.u.g.key[j];
            u32 sj = sh.u.g.st[j];
            int rank = 0;
            for (int q = 0; q < m; ++q) {
                u64 kq = sh.u.g.key[q];
                rank += (kq < kj || (kq == kj && sh.u.g.st[q] < sj)) ? 1 : 0;
            }
            if (rank == r - 1) { sh.thr_key = kj; sh.thr_state = sj; }
        }
        __syncthreads();
        return;
    }
    // radix select over the 96-bit (key, state) among boundary-bucket members, MSB first
    u64 kpre = 0, kmask = 0;
    u32 spre = 0, smask = 0;
    for (int dig = 0; dig < 12; ++dig) {
        for (int b = threadIdx.x; b < 256; b += BLOCK) sh.u.hist[b] = 0;
        __syncthreads();
        const bool in_key = dig < 8;
        const int shift = in_key ? (56 - 8 * dig) : (24 - 8 * (dig - 8));
        for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
            u64 k = c.cand_key[i];
            double cst = key_cost(k);
            if (!(cst <= cutoff) || bucket_of(cst, best, scale) != bstar) continue;
            u32 st = c.cand_state[i];
            if ((k & kmask) != kpre || (st & smask) != spre) continue;
            u32 d = in_key ? (u32)((k >> shift) & 0xFF) : ((st >> shift) & 0xFF);
            atomicAdd(&sh.u.hist[d], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            u32 acc = 0;
            int d = 0;
            for (; d < 256; ++d) {
                if (acc + sh.u.hist[d] >= (u32)r) break;
                acc += sh.u.hist[d];
            }
            sh.thr_below = (int)acc;
            sh.ng = d;
        }
        __syncthreads();
        r -= sh.thr_below;
        u32 d = (u32)sh.ng;
        if (in_key) { kpre |= (u64)d << shift; kmask |= 0xFFull << shift; }
        else { spre |= d << shift; smask |= 0xFFu << shift; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { sh.thr_key = kpre; sh.thr_state = spre; }
    __syncthreads();
}

// Finish a step: gather candidates, beam/max-active prune, backpointer records, next tokens.
// Returns the number of survivors (0 = search death).  node step k = step index + 1.
template <int BLOCK>
__device__ int finish_step(int nxt, const GraphDev &g, const WorkDev &ws, const CfgDev &cfg,
                           UttCtx &c, Smem<BLOCK> &sh, int &status, long long &n_rec) {
    const int n_cand = min(sh.n_cand, ws.cap);
    if (sh.overflow) status = WB_ERR_CAPACITY;
    u64 mn = EMPTY_KEY, mx = 0;
    for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
        u32 s = c.cand_state[i];
        Slot v = ld_slot(&c.slot[s]);
        c.cand_key[i] = v.key;
        c.cand_arc[i] = v.arcp1;
        c.cand_pay[i] = v.pay;
        st_slot_empty(&c.slot[s]);
        mn = v.key < mn ? v.key : mn;
        mx = v.key > mx ? v.key : mx;
    }
    block_minmax<BLOCK>(mn, mx, sh);
    if (n_cand == 0) return 0;
    const double best = key_cost(mn);
    const double cutoff = __dadd_rn(best, cfg.beam);  // cutoff = best + beam (decoder.py:186)
    bool need_select = false;
    double scale = 0.0;
    if (cfg.max_active > 0 && n_cand > cfg.max_active) {
        long long kept = 0;
        for (int i = threadIdx.x; i < n_cand; i += BLOCK) kept += key_cost(c.cand_key[i]) <= cutoff;
        kept = block_sum<BLOCK>(kept, sh);
        need_select = kept > cfg.max_active;
        if (need_select) {
            double hi = key_cost(mx);
            double top = cutoff < hi ? cutoff : hi;
            double range = __dsub_rn(top, best);
            if (range > 0.0 && range < INFINITY) scale = __ddiv_rn((double)NB, range);
            select_threshold<BLOCK>(n_cand, cfg.max_active, best, cutoff, scale, c, sh);
        }
    }
    const int bstar = need_select ? sh.thr_bucket : 0;
    const u64 tkey = need_select ? sh.thr_key : 0;
    const u32 tst = need_select ? sh.thr_state : 0;
    for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
        u64 k = c.cand_key[i];
        double cst = key_cost(k);
        bool surv = cst <= cutoff;
        if (surv && need_select) {
            int b = bucket_of(cst, best, scale);
            surv = b < bstar ||
                   (b == bstar && (k < tkey || (k == tkey && c.cand_state[i] <= tst)));
        }
        c.cand_flags[i] = surv ? F_SURV : 0u;
    }
    __syncthreads();
    if (g.has_eps) {
        // survivors reached through epsilon chains keep the chain's candidates alive
        for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
            if (!(__ldcg(&c.cand_flags[i]) & F_SURV)) continue;
            int v = i;
            for (;;) {
                u32 a = c.cand_arc[v], p = c.cand_pay[v];
                if (a == 0u || !(p & EPS_BIT)) break;
                int uix = (int)(p & ~EPS_BIT);
                u32 old = atomicOr(&c.cand_flags[uix], F_MARK);
                if (old & (F_MARK | F_SURV)) break;
                v = uix;
            }
        }
        __syncthreads();
    }
    int n_keep = 0, n_surv = 0;
    u32 *flags = c.cand_flags;
    // flags were updated by L2 atomics (F_MARK): read them L2-coherently from here on
    auto flag = [&](int i) { return __ldcg(&flags[i]); };
    // reserve arena records: count kept first
    long long nk = 0;
    for (int i = threadIdx.x; i < n_cand; i += BLOCK) nk += flag(i) != 0u;
    nk = block_sum<BLOCK>(nk, sh);
    if (threadIdx.x == 0) {
        u64 base = atomicAdd(ws.arena_ctr, (u64)nk);
        if (base + (u64)nk > ws.arena_cap || base + (u64)nk >= (u64)EPS_BIT) sh.overflow = 2;
        sh.arena_base = base;
    }
    __syncthreads();
    if (sh.overflow == 2) { status = WB_ERR_CAPACITY; return 0; }
    const u64 base = sh.arena_base;
    int4 *tinfo = c.tok_info[nxt];
    double *tcost = c.tok_cost[nxt];
    u32 *arena_of = c.cand_arena;
    const u32 *cstate = c.cand_state;
    const u64 *ckey = c.cand_key;
    block_compact2<BLOCK>(
        n_cand, [&](int i) { return flag(i) != 0u; }, [&](int i) { return (flag(i) & F_SURV) != 0u; },
        [&](int i, int ia, int ib) {
            u32 rec = (u32)(base + (u64)ia);
            arena_of[i] = rec;
            if (flag(i) & F_SURV) {
                u32 s = cstate[i];
                int4 inf = __ldg(&g.info[s]);
                tinfo[ib] = make_int4((int)s, (int)rec, inf.y, inf.z);
                tcost[ib] = key_cost(ckey[i]);
            }
        },
        sh, n_keep, n_surv);
    for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
        if (!flag(i)) continue;
        u32 a = c.cand_arc[i], p = c.cand_pay[i];
        u32 prev = a == 0u ? ROOT_PREV : ((p & EPS_BIT) ? arena_of[p & ~EPS_BIT] : p);
        ws.arena[arena_of[i]] = (u64)a | ((u64)prev << 32);
    }
    n_rec += n_keep;
    __syncthreads();
    return n_surv;
}

template <int BLOCK>
__device__ void lsd_prepass(const BatchDev &b, int u, const CfgDev &cfg, UttCtx &c, int T,
                            long long row0, Smem<BLOCK> &sh, int &nf) {
    // classify_blank_frames + nonblank_frames (posteriors.py:116-125,109-110): a frame is
    // blank iff its blank probability strictly exceeds the threshold.
    const double *bl = b.blank + row0;
    const double thr = cfg.thr;
    int *fr = c.frames;
    int ta = 0, tb = 0;
    block_compact2<BLOCK>(
        T, [&](int f) { return !(bl[f] > thr); }, [&](int) { return false; },
        [&](int f, int ia, int) { fr[ia] = f; }, sh, ta, tb);
    nf = ta;
}

// argmin over tokens by (key, state); returns token index (-1 if none) via shared memory
template <int BLOCK>
__device__ int block_argmin_tok(u64 key, u32 st, int idx, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        u64 k2 = __shfl_xor_sync(FULL, key, o);
        u32 s2 = __shfl_xor_sync(FULL, st, o);
        int i2 = __shfl_xor_sync(FULL, idx, o);
        if (k2 < key || (k2 == key && s2 < st)) { key = k2; st = s2; idx = i2; }
    }
    if (l == 0) { sh.r0[w] = key; sh.wa[w] = st; sh.wb[w] = (u32)idx; }
    __syncthreads();
    if (w == 0) {
        key = l < NW ? sh.r0[l] : EMPTY_KEY;
        st = l < NW ? sh.wa[l] : 0xFFFFFFFFu;
        idx = l < NW ? (int)sh.wb[l] : -1;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            u64 k2 = __shfl_xor_sync(FULL, key, o);
            u32 s2 = __shfl_xor_sync(FULL, st, o);
            int i2 = __shfl_xor_sync(FULL, idx, o);
            if (k2 < key || (k2 == key && s2 < st)) { key = k2; st = s2; idx = i2; }
        }
        if (l == 0) { sh.r0[0] = key; sh.wb[0] = (u32)idx; }
    }
    __syncthreads();
    int r = sh.r0[0] == EMPTY_KEY ? -1 : (int)sh.wb[0];
    __syncthreads();
    return r;
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK, 1024 / BLOCK)
decode_kernel(GraphDev g, WorkDev ws, BatchDev b, CfgDev cfg, wb_utt_result *res) {
    extern __shared__ double s_row[];
    __shared__ Smem<BLOCK> sh;
    const int slot_id = blockIdx.x;
    const size_t S = (size_t)ws.S, cap = (size_t)ws.cap;
    UttCtx c;
    c.slot = ws.slot + slot_id * S;
    c.cand_of = ws.cand_of + slot_id * S;
    c.qtag = ws.qtag + slot_id * S;
    c.cand_state = ws.cand_state + slot_id * cap;
    c.cand_key = ws.cand_key + slot_id * cap;
    c.cand_arc = ws.cand_arc + slot_id * cap;
    c.cand_pay = ws.cand_pay + slot_id * cap;
    c.cand_flags = ws.cand_flags + slot_id * cap;
    c.cand_arena = ws.cand_arena + slot_id * cap;
    c.front[0] = ws.front + (size_t)slot_id * 2 * cap;
    c.front[1] = c.front[0] + cap;
    c.tok_info[0] = ws.tok_info + (size_t)slot_id * 2 * cap;
    c.tok_info[1] = c.tok_info[0] + cap;
    c.tok_cost[0] = ws.tok_cost + (size_t)slot_id * 2 * cap;
    c.tok_cost[1] = c.tok_cost[0] + cap;
    c.frames = ws.frames + (size_t)slot_id * ws.T_cap;
    c.tag = ws.tag_ctr[slot_id];
    const bool row_in_smem = b.L1 <= ROW_SMEM_MAX;

    for (;;) {
        if (threadIdx.x == 0) sh.utt = (int)atomicAdd(ws.utt_ctr, 1u);
        __syncthreads();
        const int u = sh.utt;
        if (u >= b.n) break;
        const int T = b.T[u];
        const long long row0 = b.row_off[u];
        int status = WB_OK;
        c.a_emit = c.a_fin = c.e_eps = 0;
        long long n_tok = 0, n_cand_tot = 0, n_surv_tot = 0, n_rec = 0;
        int nf = T;
        if (cfg.mode == 1) lsd_prepass<BLOCK>(b, u, cfg, c, T, row0, sh, nf);

        // ---- initial tokens: start entry + epsilon closure + prune (decoder.py:236-249)
        if (threadIdx.x == 0) {
            Slot st;
            st.key = cost_key(0.0);
            st.arcp1 = 0u;
            st.pay = ROOT_PREV;
            *reinterpret_cast<ulonglong2 *>(&c.slot[g.start]) =
                make_ulonglong2(st.key, (u64)st.arcp1 | ((u64)st.pay << 32));
            c.cand_state[0] = (u32)g.start;
            c.cand_of[g.start] = 0u;
            sh.n_cand = 1;
            sh.overflow = 0;
            int4 inf = g.info[g.start];
            sh.n_front = 0;
            if (g.has_eps && inf.x < inf.y) { c.front[0][0] = (u32)g.start; sh.n_front = 1; }
        }
        __threadfence_block();
        __syncthreads();
        if (g.has_eps) epsilon_closure<BLOCK>(g, ws, c, sh, status);
        n_cand_tot += min(sh.n_cand, ws.cap);
        int cur = 0;
        int n_live = finish_step<BLOCK>(cur, g, ws, cfg, c, sh, status, n_rec);
        n_surv_tot += n_live;
        int steps_run = 0, died_at = -1;
        long long expanded = 0;
        for (int s = 0; s < nf && status == WB_OK; ++s) {
            const int f = cfg.mode == 1 ? c.frames[s] : s;
            const double *grow = b.costs + (size_t)(row0 + f) * b.L1;
            if (row_in_smem) {
                for (int q = threadIdx.x; q < b.L1; q += BLOCK) s_row[q] = __ldg(&grow[q]);
                c.row = s_row;
            } else {
                c.row = grow;
            }
            if (threadIdx.x == 0) { sh.n_cand = 0; sh.n_front = 0; sh.overflow = 0; }
            __syncthreads();
            expanded += n_live;
            n_tok += n_live;
            expand_emitting<BLOCK>(n_live, cur, g, ws, c, sh);
            __syncthreads();
            if (g.has_eps) epsilon_closure<BLOCK>(g, ws, c, sh, status);
            n_cand_tot += min(sh.n_cand, ws.cap);
            int m = finish_step<BLOCK>(cur ^ 1, g, ws, cfg, c, sh, status, n_rec);
            steps_run++;
            if (m == 0) {
                died_at = s;
                break;
            }
            n_surv_tot += m;
            cur ^= 1;
            n_live = m;
        }
        // ---- final transition / death fallback (decoder.py:252-273, 327-333)
        const int4 *tinfo = c.tok_info[cur];
        const double *tcost = c.tok_cost[cur];
        int best_t = -1;
        int reached = 0;
        double best_cost = 0.0;
        if (died_at < 0) {
            u64 k = EMPTY_KEY;
            u32 st = 0xFFFFFFFFu;
            int idx = -1;
            for (int t = threadIdx.x; t < n_live; t += BLOCK) {
                int s = tinfo[t].x;
                double fw = __ldg(&g.final_w[s]);
                if (fw == INFINITY) continue;
                u64 kk = cost_key(__dadd_rn(tcost[t], fw));
                if (kk < k || (kk == k && (u32)s < st)) { k = kk; st = (u32)s; idx = t; }
            }
            best_t = block_argmin_tok<BLOCK>(k, st, idx, sh);
            if (best_t >= 0) {
                reached = 1;
                best_cost = __dadd_rn(tcost[best_t], __ldg(&g.final_w[tinfo[best_t].x]));
            }
        }
        if (best_t < 0) {
            u64 k = EMPTY_KEY;
            u32 st = 0xFFFFFFFFu;
            int idx = -1;
            for (int t = threadIdx.x; t < n_live; t += BLOCK) {
                u64 kk = cost_key(tcost[t]);
                u32 s = (u32)tinfo[t].x;
                if (kk < k || (kk == k && s < st)) { k = kk; st = s; idx = t; }
            }
            best_t = block_argmin_tok<BLOCK>(k, st, idx, sh);
            if (best_t >= 0) best_cost = tcost[best_t];
        }
        long long a_emit = block_sum<BLOCK>(c.a_emit, sh);
        long long a_fin = block_sum<BLOCK>(c.a_fin, sh);
        long long e_eps = block_sum<BLOCK>(c.e_eps, sh);
        if (threadIdx.x == 0) {
            wb_utt_result r;
            memset(&r, 0, sizeof(r));
            r.total_cost = best_cost;
            r.tokens_expanded = expanded;
            r.search_steps = steps_run;
            r.reached_final = reached;
            r.died_at_step = died_at;
            r.final_state = best_t >= 0 ? tinfo[best_t].x : -1;
            r.final_step = died_at < 0 ? steps_run : died_at;
            r.status = status;
            r.best_trace = best_t >= 0 ? (long long)(u32)tinfo[best_t].y : -1;
            r.n_tok = n_tok;
            r.a_emit = a_emit;
            r.a_fin = a_fin;
            r.e_eps = e_eps;
            r.n_cand = n_cand_tot;
            r.n_surv = n_surv_tot;
            r.n_rec = n_rec;
            res[u] = r;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) ws.tag_ctr[slot_id] = c.tag;
}

// Backtrace (decoder.py:276-291): one thread per utterance walks the arena from the winner;
// labels are written back-to-front so they land in path order without a second walk.
__global__ void backtrace_kernel(GraphDev g, const u64 *arena, wb_utt_result *res, int n,
                                 int *olab, int *ilab, int cap) {
    int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    wb_utt_result r = res[u];
    int *ob = olab + (size_t)u * cap, *ib = ilab + (size_t)u * cap;
    int po = cap, pi = cap, no = 0, ni = 0;
    u32 idx = r.best_trace < 0 ? ROOT_PREV : (u32)r.best_trace;
    while (idx != ROOT_PREV) {
        u64 rec = arena[idx];
        u32 a1 = (u32)rec;
        idx = (u32)(rec >> 32);
        if (a1 == 0u) continue;
        int a = (int)a1 - 1;
        int ol = __ldg(&g.olabel[a]);
        int il = __ldg(&g.arcs[a].y);
        if (ol != 0) { ++no; if (po > 0) ob[--po] = ol; }
        if (il != 0) { ++ni; if (pi > 0) ib[--pi] = il; }
    }
    // shift to the front of the row
    for (int i = 0; i < cap - po && no <= cap; ++i) ob[i] = ob[po + i];
    for (int i = 0; i < cap - pi && ni <= cap; ++i) ib[i] = ib[pi + i];
    res[u].n_olabels = no;
    res[u].n_ilabels = ni;
    if ((no > cap || ni > cap) && r.status == WB_OK) res[u].status = WB_ERR_CAPACITY;
}

}  // namespace wb

// ====================================================================== host side
using namespace wb;

static thread_local std::string g_err;

static int set_err(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return set_err(WB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct wb_graph_s {
    int device = 0;
    int S = 0, A = 0, start = 0, has_eps = 0, max_ilabel = 0;
    int4 *info = nullptr, *arcs = nullptr;
    int *olabel = nullptr;
    double *final_w = nullptr;
    size_t bytes = 0;
};

struct wb_decoder_s {
    wb_graph_s *g = nullptr;
    int slots = 0, cap = 0, T_cap = 0, block = 512, num_sms = 0;
    u64 arena_cap = 0;
    Slot *slot = nullptr;
    u32 *cand_of = nullptr, *qtag = nullptr, *tag_ctr = nullptr;
    u32 *cand_state = nullptr, *cand_arc = nullptr, *cand_pay = nullptr, *cand_flags = nullptr,
        *cand_arena = nullptr;
    u64 *cand_key = nullptr;
    u32 *front = nullptr;
    int4 *tok_info = nullptr;
    double *tok_cost = nullptr;
    int *frames = nullptr;
    u64 *arena = nullptr;
    u64 *counters = nullptr;  // [0] arena_ctr, [1] utt_ctr (u32 in low half)
    // host-mode staging
    double *h_costs = nullptr, *h_blank = nullptr;
    size_t h_costs_n = 0, h_blank_n = 0;
    long long *h_off = nullptr;
    int *h_T = nullptr;
    wb_utt_result *h_res = nullptr;
    int *h_lab = nullptr;
    size_t h_n = 0, h_lab_n = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    size_t bytes = 0;
};

template <class T>
static cudaError_t dalloc(T **p, size_t n, size_t &acc) {
    acc += sizeof(T) * std::max<size_t>(n, 1);
    return cudaMalloc(p, sizeof(T) * std::max<size_t>(n, 1));
}

template <int BLOCK>
static cudaError_t launch_decode(int grid, size_t smem, cudaStream_t st, const GraphDev &gd,
                                 const WorkDev &wd, const BatchDev &bd, const CfgDev &cd,
                                 wb_utt_result *res) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<BLOCK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    decode_kernel<BLOCK><<<grid, BLOCK, smem, st>>>(gd, wd, bd, cd, res);
    return cudaGetLastError();
}

extern "C" {

const char *wb_last_error(void) { return g_err.c_str(); }
int wb_version(void) { return 1; }

int wb_device_count(int32_t *n) {
    int c = 0;
    CUDA_TRY(cudaGetDeviceCount(&c));
    *n = c;
    return WB_OK;
}

int wb_graph_create(const wb_graph_desc *d, int32_t device, wb_graph_t *out) {
    if (!d || !out) return set_err(WB_ERR_VALUE, "null argument");
    if (d->num_states <= 0 || d->num_arcs < 0 || d->start < 0 || d->start >= d->num_states)
        return set_err(WB_ERR_VALUE, "bad graph dimensions");
    CUDA_TRY(cudaSetDevice(device));
    const int S = d->num_states, A = d->num_arcs;
    std::vector<int4> info(S), arcs(std::max(A, 1));
    int has_eps = 0, max_il = 0;
    if (d->row_ptr[0] != 0 || d->row_ptr[S] != A) return set_err(WB_ERR_VALUE, "row_ptr mismatch");
    for (int s = 0; s < S; ++s) {
        int lo = d->row_ptr[s], mid = d->eps_end[s], hi = d->row_ptr[s + 1];
        if (lo > mid || mid > hi) return set_err(WB_ERR_VALUE, "eps_end outside the state's arc range");
        info[s] = make_int4(lo, mid, hi, 0);
        if (mid > lo) has_eps = 1;
    }
    for (int a = 0; a < A; ++a) {
        if (d->dst[a] < 0 || d->dst[a] >= S) return set_err(WB_ERR_VALUE, "arc destination out of range");
        if (d->ilabel[a] < 0 || d->olabel[a] < 0) return set_err(WB_ERR_VALUE, "negative label");
        long long wb_;
        std::memcpy(&wb_, &d->weight[a], 8);
        arcs[a] = make_int4(d->dst[a], d->ilabel[a], (int)(wb_ & 0xffffffffll), (int)(wb_ >> 32));
        max_il = std::max(max_il, d->ilabel[a]);
    }
    wb_graph_s *g = new wb_graph_s();
    g->device = device;
    g->S = S;
    g->A = A;
    g->start = d->start;
    g->has_eps = has_eps;
    g->max_ilabel = max_il;
    auto fail = [&](cudaError_t e) {
        cudaFree(g->info); cudaFree(g->arcs); cudaFree(g->olabel); cudaFree(g->final_w);
        delete g;
        return set_err(WB_ERR_CUDA, std::string("graph upload: ") + cudaGetErrorString(e));
    };
    cudaError_t e;
    if ((e = cudaMalloc(&g->info, sizeof(int4) * S)) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&g->arcs, sizeof(int4) * std::max(A, 1))) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&g->olabel, sizeof(int) * std::max(A, 1))) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&g->final_w, sizeof(double) * S)) != cudaSuccess) return fail(e);
    if ((e = cudaMemcpy(g->info, info.data(), sizeof(int4) * S, cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e);
    if (A) {
        if ((e = cudaMemcpy(g->arcs, arcs.data(), sizeof(int4) * A, cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e);
        if ((e = cudaMemcpy(g->olabel, d->olabel, sizeof(int) * A, cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e);
    }
    if ((e = cudaMemcpy(g->final_w, d->final_w, sizeof(double) * S, cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e);
    g->bytes = sizeof(int4) * (size_t)S + (sizeof(int4) + sizeof(int)) * (size_t)A + sizeof(double) * (size_t)S;
    *out = g;
    return WB_OK;
}

int wb_graph_destroy(wb_graph_t g) {
    if (!g) return WB_OK;
    cudaSetDevice(g->device);
    cudaFree(g->info);
    cudaFree(g->arcs);
    cudaFree(g->olabel);
    cudaFree(g->final_w);
    delete g;
    return WB_OK;
}

int wb_graph_device_bytes(wb_graph_t g, int64_t *bytes) {
    *bytes = (int64_t)g->bytes;
    return WB_OK;
}

static void free_decoder(wb_decoder_s *d) {
    void *ptrs[] = {d->slot, d->cand_of, d->qtag, d->tag_ctr, d->cand_state, d->cand_arc, d->cand_pay,
                    d->cand_flags, d->cand_arena, d->cand_key, d->front, d->tok_info, d->tok_cost,
                    d->frames, d->arena, d->counters, d->h_costs, d->h_blank, d->h_off, d->h_T,
                    d->h_res, d->h_lab};
    for (void *p : ptrs) cudaFree(p);
    if (d->ev0) cudaEventDestroy(d->ev0);
    if (d->ev1) cudaEventDestroy(d->ev1);
}

static int alloc_frames(wb_decoder_s *d, int T_cap) {
    cudaFree(d->frames);
    d->frames = nullptr;
    d->T_cap = std::max(T_cap, 1);
    CUDA_TRY(cudaMalloc(&d->frames, sizeof(int) * (size_t)d->slots * d->T_cap));
    return WB_OK;
}

static int alloc_arena(wb_decoder_s *d, u64 cap) {
    cudaFree(d->arena);
    d->arena = nullptr;
    d->arena_cap = std::min<u64>(std::max<u64>(cap, 1024), (u64)EPS_BIT - 1);
    CUDA_TRY(cudaMalloc(&d->arena, sizeof(u64) * d->arena_cap));
    return WB_OK;
}

int wb_decoder_create(wb_graph_t g, const wb_decoder_opts *o, wb_decoder_t *out) {
    if (!g || !out) return set_err(WB_ERR_VALUE, "null argument");
    CUDA_TRY(cudaSetDevice(g->device));
    wb_decoder_opts opts;
    std::memset(&opts, 0, sizeof(opts));
    if (o) opts = *o;
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, g->device));
    wb_decoder_s *d = new wb_decoder_s();
    d->g = g;
    d->num_sms = prop.multiProcessorCount;
    d->block = opts.block_threads ? opts.block_threads : 512;
    if (d->block != 256 && d->block != 512 && d->block != 1024) {
        delete d;
        return set_err(WB_ERR_VALUE, "block_threads must be 256, 512 or 1024");
    }
    int per_sm = d->block >= 1024 ? 1 : 2048 / d->block;
    if (per_sm > 4) per_sm = 4;
    d->slots = opts.max_utts_in_flight > 0 ? opts.max_utts_in_flight : d->num_sms * per_sm;
    d->cap = opts.cand_capacity > 0 ? opts.cand_capacity : std::min(g->S, 1 << 18);
    d->cap = std::max(1, std::min(d->cap, g->S));
    size_t S = (size_t)g->S, slots = (size_t)d->slots, cap = (size_t)d->cap;
    size_t acc = 0;
    cudaError_t e = cudaSuccess;
#define DA(p, n) if (e == cudaSuccess) e = dalloc(&d->p, (n), acc)
    DA(slot, slots * S);
    DA(cand_of, slots * S);
    DA(qtag, slots * S);
    DA(tag_ctr, slots);
    DA(cand_state, slots * cap);
    DA(cand_key, slots * cap);
    DA(cand_arc, slots * cap);
    DA(cand_pay, slots * cap);
    DA(cand_flags, slots * cap);
    DA(cand_arena, slots * cap);
    DA(front, slots * 2 * cap);
    DA(tok_info, slots * 2 * cap);
    DA(tok_cost, slots * 2 * cap);
    DA(counters, 4);
#undef DA
    if (e == cudaSuccess) e = cudaMemset(d->slot, 0xFF, sizeof(Slot) * slots * S);
    if (e == cudaSuccess) e = cudaMemset(d->qtag, 0, sizeof(u32) * slots * S);
    if (e == cudaSuccess) e = cudaMemset(d->tag_ctr, 0, sizeof(u32) * slots);
    if (e == cudaSuccess) e = cudaEventCreate(&d->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&d->ev1);
    if (e != cudaSuccess) {
        free_decoder(d);
        delete d;
        return set_err(e == cudaErrorMemoryAllocation ? WB_ERR_NOMEM : WB_ERR_CUDA,
                       std::string("decoder workspace: ") + cudaGetErrorString(e));
    }
    d->bytes = acc;
    int rc = alloc_frames(d, opts.max_frames > 0 ? opts.max_frames : 2048);
    if (rc == WB_OK) rc = alloc_arena(d, opts.arena_capacity > 0 ? (u64)opts.arena_capacity : (u64)1 << 24);
    if (rc != WB_OK) {
        free_decoder(d);
        delete d;
        return rc;
    }
    *out = d;
    return WB_OK;
}

int wb_decoder_destroy(wb_decoder_t d) {
    if (!d) return WB_OK;
    cudaSetDevice(d->g->device);
    free_decoder(d);
    delete d;
    return WB_OK;
}

int wb_decoder_device_bytes(wb_decoder_t d, int64_t *bytes) {
    *bytes = (int64_t)(d->bytes + sizeof(int) * (size_t)d->slots * d->T_cap + sizeof(u64) * d->arena_cap);
    return WB_OK;
}

int wb_last_kernel_ms(wb_decoder_t d, float *ms) {
    CUDA_TRY(cudaEventElapsedTime(ms, d->ev0, d->ev1));
    return WB_OK;
}

int wb_decode(wb_decoder_t d, int32_t n, const double *costs, const int64_t *row_offset,
              const int32_t *num_frames, int32_t num_cols, const double *blank, const wb_config *cfg,
              wb_utt_result *results, int32_t *olabels, int32_t *ilabels, int32_t label_cap,
              int32_t memory_kind, void *stream) {
    if (!d || !cfg) return set_err(WB_ERR_VALUE, "null argument");
    if (n < 0 || num_cols < 1 || label_cap < 0) return set_err(WB_ERR_VALUE, "bad batch dimensions");
    if (cfg->beam < 0 || std::isnan(cfg->beam)) return set_err(WB_ERR_VALUE, "beam must be >= 0");
    if (cfg->max_active < 0) return set_err(WB_ERR_VALUE, "max_active must be >= 1 or 0 (None)");
    if (cfg->mode != 0 && cfg->mode != 1) return set_err(WB_ERR_VALUE, "mode must be 0 (fsd) or 1 (lsd)");
    wb_graph_s *g = d->g;
    if (g->max_ilabel > num_cols - 1)
        return set_err(WB_ERR_VALUE, "graph uses input label " + std::to_string(g->max_ilabel) +
                                         " but the posterior matrix only covers labels 1.." +
                                         std::to_string(num_cols - 1));
    CUDA_TRY(cudaSetDevice(g->device));
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) return WB_OK;
    const bool host = memory_kind == WB_MEM_HOST;
    int maxT = 0;
    long long rows = 0;
    if (host) {
        for (int i = 0; i < n; ++i) {
            if (num_frames[i] < 0) return set_err(WB_ERR_VALUE, "negative frame count");
            maxT = std::max(maxT, num_frames[i]);
            rows = std::max<long long>(rows, row_offset[i] + num_frames[i]);
        }
    } else {
        // device mode: the caller passes max frames through label_cap's companion contract --
        // read T on the host once (small copy) to size the frame list.
        std::vector<int> hT(n);
        CUDA_TRY(cudaMemcpyAsync(hT.data(), num_frames, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        for (int i = 0; i < n; ++i) maxT = std::max(maxT, hT[i]);
    }
    if (maxT > d->T_cap) {
        int rc = alloc_frames(d, maxT);
        if (rc) return rc;
    }
    const double *dc = costs, *db = blank;
    const long long *doff = (const long long *)row_offset;
    const int *dT = num_frames;
    wb_utt_result *dres = results;
    int *dol = olabels, *dil = ilabels;
    if (host) {
        size_t ncost = (size_t)rows * num_cols;
        if (ncost > d->h_costs_n) {
            cudaFree(d->h_costs);
            d->h_costs = nullptr;
            CUDA_TRY(cudaMalloc(&d->h_costs, sizeof(double) * ncost));
            d->h_costs_n = ncost;
        }
        if ((size_t)rows > d->h_blank_n || !d->h_blank) {
            cudaFree(d->h_blank);
            d->h_blank = nullptr;
            CUDA_TRY(cudaMalloc(&d->h_blank, sizeof(double) * std::max<long long>(rows, 1)));
            d->h_blank_n = std::max<long long>(rows, 1);
        }
        if ((size_t)n > d->h_n) {
            cudaFree(d->h_off); cudaFree(d->h_T); cudaFree(d->h_res);
            d->h_off = nullptr; d->h_T = nullptr; d->h_res = nullptr;
            CUDA_TRY(cudaMalloc(&d->h_off, sizeof(long long) * n));
            CUDA_TRY(cudaMalloc(&d->h_T, sizeof(int) * n));
            CUDA_TRY(cudaMalloc(&d->h_res, sizeof(wb_utt_result) * n));
            d->h_n = n;
        }
        size_t nlab = (size_t)n * std::max(label_cap, 1) * 2;
        if (nlab > d->h_lab_n) {
            cudaFree(d->h_lab);
            d->h_lab = nullptr;
            CUDA_TRY(cudaMalloc(&d->h_lab, sizeof(int) * nlab));
            d->h_lab_n = nlab;
        }
        if (ncost) CUDA_TRY(cudaMemcpyAsync(d->h_costs, costs, sizeof(double) * ncost, cudaMemcpyHostToDevice, st));
        if (rows) CUDA_TRY(cudaMemcpyAsync(d->h_blank, blank, sizeof(double) * rows, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(d->h_off, row_offset, sizeof(long long) * n, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(d->h_T, num_frames, sizeof(int) * n, cudaMemcpyHostToDevice, st));
        dc = d->h_costs; db = d->h_blank; doff = d->h_off; dT = d->h_T; dres = d->h_res;
        dol = d->h_lab; dil = d->h_lab + (size_t)n * std::max(label_cap, 1);
    }
    CUDA_TRY(cudaMemsetAsync(d->counters, 0, sizeof(u64) * 4, st));
    GraphDev gd{g->S, g->A, g->start, g->has_eps, g->info, g->arcs, g->olabel, g->final_w};
    WorkDev wd;
    wd.slot = d->slot; wd.cand_of = d->cand_of; wd.qtag = d->qtag; wd.tag_ctr = d->tag_ctr;
    wd.cand_state = d->cand_state; wd.cand_key = d->cand_key; wd.cand_arc = d->cand_arc;
    wd.cand_pay = d->cand_pay; wd.cand_flags = d->cand_flags; wd.cand_arena = d->cand_arena;
    wd.front = d->front; wd.tok_info = d->tok_info; wd.tok_cost = d->tok_cost; wd.frames = d->frames;
    wd.arena = d->arena; wd.arena_cap = d->arena_cap; wd.arena_ctr = d->counters;
    wd.utt_ctr = reinterpret_cast<u32 *>(d->counters + 1);
    wd.S = g->S; wd.cap = d->cap; wd.T_cap = d->T_cap;
    BatchDev bd{dc, doff, dT, db, num_cols, n};
    CfgDev cd{cfg->beam, cfg->blank_threshold, cfg->max_active, cfg->mode, cfg->lattice};
    int grid = std::min(n, d->slots);
    size_t smem = num_cols <= ROW_SMEM_MAX ? sizeof(double) * (size_t)num_cols : 0;
    CUDA_TRY(cudaEventRecord(d->ev0, st));
    cudaError_t e;
    switch (d->block) {
        case 256: e = launch_decode<256>(grid, smem, st, gd, wd, bd, cd, dres); break;
        case 1024: e = launch_decode<1024>(grid, smem, st, gd, wd, bd, cd, dres); break;
        default: e = launch_decode<512>(grid, smem, st, gd, wd, bd, cd, dres); break;
    }
    if (e != cudaSuccess) return set_err(WB_ERR_CUDA, std::string("decode launch: ") + cudaGetErrorString(e));
    CUDA_TRY(cudaEventRecord(d->ev1, st));
    backtrace_kernel<<<(n + 127) / 128, 128, 0, st>>>(gd, d->arena, dres, n, dol, dil, std::max(label_cap, 1));
    CUDA_TRY(cudaGetLastError());
    if (host) {
        CUDA_TRY(cudaMemcpyAsync(results, dres, sizeof(wb_utt_result) * n, cudaMemcpyDeviceToHost, st));
        if (label_cap > 0) {
            CUDA_TRY(cudaMemcpyAsync(olabels, dol, sizeof(int) * (size_t)n * label_cap, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(ilabels, dil, sizeof(int) * (size_t)n * label_cap, cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    return WB_OK;
}

}  // extern "C"
