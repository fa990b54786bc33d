// decode_kernel.cuh -- the persistent batched WFST Viterbi beam-search kernel (sm_100a).
//
// One CTA = one "utterance lane": it pulls utterances from an atomic queue and runs the whole
// frame loop of one utterance with CTA-level barriers only (no grid syncs, no per-frame
// launches).  Per search step (decoder.py:197-233):
//
//   expand   warp-level load balancing: a warp takes 32 live tokens, prefix-sums their
//            emitting out-degrees with shuffles and strides its lanes over the flattened
//            token x arc range (the paper's "tokens x arcs assigned by prefix-summed
//            out-degree").  Arc records are 32 B: {dst, ilabel, weight | dst's eps/emit
//            ranges, olabel}, so a relaxation needs one 16 B load and a first touch one more
//            from the same sector -- no per-state lookups.  The frame's float64 cost row is
//            staged in shared memory.  Recombination is a 128-bit atomic CAS on a dense
//            per-state slot {cost key, arc+1, payload} under the reference's
//            (cost, src state, arc) total order (decoder.py:121-135).
//   closure  frontier rounds over the epsilon arcs of improved states, epoch-tagged dedup
//            (decoder.py:138-171; Jacobi form parallel.py:287-325).
//   prune    exact beam + max-active cut without a sort: min/max reduce, a 4096-bucket value
//            histogram in shared memory, exact (cost, state) rank inside the boundary bucket
//            (radix-select fallback) (decoder.py:174-194).
//   compact  candidate keys/flags live in shared memory; survivors and the epsilon-chain
//            candidates they trace through get 8-byte backpointer records in a batch-wide
//            arena; slots are reset O(touched).
//
// Arithmetic is float64 in the reference's association order, so costs, survivor sets,
// tokens_expanded and (tie-free) labels are bit-identical to decoder.py.
#pragma once
#include <cuda_runtime.h>

#include "../../include/wfst_b200.h"
#include "device_common.cuh"

namespace wb {

constexpr int NB = 4096;             // prune histogram buckets
constexpr int GCAP = 1024;           // boundary-bucket members ranked in shared memory
constexpr int ROW_SMEM_MAX = 16384;  // cost-row columns staged in shared memory (128 KB)
constexpr u32 F_SURV = 1u, F_MARK = 2u, CA_NONE = 0xFFFFFFFFu;
constexpr int MAX_EPS_ROUNDS = 1 << 20;
constexpr int UNROLL = 4;
constexpr int GATHER = 4;

struct GraphDev {
    int S, A, start, has_eps;
    int4 start_rng;         // {eps_lo, eps_hi (= emit_lo), emit_hi, 0} of the start state
    const int4 *arcs;       // [2*A]: {dst, ilabel, w_lo, w_hi}, {d_eps_lo, d_emit_lo, d_emit_hi, olabel}
    const double *final_w;  // [S] (+inf = not final)
};

struct WorkDev {
    Slot *slot;           // [slots][S]   recombination slots (EMPTY between steps)
    u32 *cand_of;         // [slots][S]   state -> candidate index (epsilon graphs)
    u32 *qtag;            // [slots][S]   epsilon frontier dedup tags
    u32 *tag_ctr;         // [slots]
    u32 *cand_state;      // [slots][cap]
    int4 *cand_rng;       // [slots][cap] {eps_lo, emit_lo, emit_hi, 0}
    u32 *cand_arc, *cand_pay;
    u64 *cand_key;        // [slots][cap] (used when a step overflows shared memory)
    u32 *cand_ca;         // [slots][cap]
    u32 *front;           // [slots][2][cap] frontier states / pending record list
    int4 *tok_info;       // [slots][2][cap] {state, trace, emit_lo, emit_hi}
    double *tok_cost;     // [slots][2][cap]
    int *frames;          // [slots][T_cap]
    u64 *arena;           // [arena_cap] backpointer records (arcp1 | prev << 32)
    u64 arena_cap;
    u64 *arena_ctr;
    u32 *utt_ctr;
    long long S;
    int cap, T_cap, smem_cands, row_in_smem;
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
    int n_cand, n_front, overflow, utt, tag_round, ng, thr_bucket, thr_below, n_pend;
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

// Exclusive scan of one int per warp (lane 0 of each warp supplies v); returns the warp's
// offset, total in *tot.  Two barriers.
template <int BLOCK>
__device__ __forceinline__ int warp_offsets(int v, u32 *buf, int *tot) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) buf[w] = (u32)v;
    __syncthreads();
    if (w == 0) {
        int x = l < NW ? (int)buf[l] : 0;
        int ix = warp_incl_scan(x);
        if (l < NW) buf[l] = (u32)(ix - x);
        if (l == 31) buf[NW] = (u32)ix;
    }
    __syncthreads();
    *tot = (int)buf[NW];
    return (int)buf[w];
}

// ------------------------------------------------------------------ per-utterance lane state
struct Lane {
    Slot *slot;
    u32 *cand_of, *qtag;
    u32 *cand_state, *cand_arc, *cand_pay, *cand_ca;
    int4 *cand_rng;
    u64 *cand_key;
    u32 *front[2];
    int4 *tok_info[2];
    double *tok_cost[2];
    int *frames;
    const double *row;  // current cost row (shared or global)
    u64 *s_key;         // shared-memory candidate keys
    u32 *s_ca;          // shared-memory candidate flags / arena indices
    u32 tag;
    long long a_emit, a_fin, e_eps;  // per-thread counters
};

// First touch of a state in this step: register it as a candidate.  `rng` = the state's
// {eps_lo, emit_lo, emit_hi} taken from the arc record.  Epsilon graphs: remember the
// state -> candidate map and, if asked, queue the state for the epsilon closure.
template <int BLOCK>
__device__ __forceinline__ void append_cand(u32 d, int4 rng, const GraphDev &g, const WorkDev &ws,
                                            Lane &c, Smem<BLOCK> &sh, u32 *front_out,
                                            bool push_front) {
    int idx = atomicAdd(&sh.n_cand, 1);
    if (idx < ws.cap) {
        c.cand_state[idx] = d;
        c.cand_rng[idx] = make_int4(rng.x, rng.y, rng.z, 0);
        if (g.has_eps) {
            c.cand_of[d] = (u32)idx;
            if (push_front && rng.x < rng.y) {
                int f = atomicAdd(&sh.n_front, 1);
                front_out[f] = d;
            }
        }
    } else {
        sh.overflow = 1;
    }
}

// Emitting expansion of all live tokens (viterbi_step's emitting loop, decoder.py:212-225;
// parallel form parallel.py:257-283).
template <int BLOCK>
__device__ void expand_emitting(int n_live, int cur, const GraphDev &g, const WorkDev &ws,
                                Lane &c, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int4 *tinfo = c.tok_info[cur];
    const double *tcost = c.tok_cost[cur];
    u32 *front0 = c.front[0];
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
                if (ok[u]) rec[u] = __ldg(&g.arcs[2 * arc[u]]);
            }
            Slot cur_s[UNROLL];
            u64 key[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                if (ok[u]) {
                    double ac = c.row[rec[u].y];
                    if (ac == INFINITY) {  // decoder.py:219-220: no relaxation, no record
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
                        if (cs.key == EMPTY_KEY) {
                            int4 r1 = __ldg(&g.arcs[2 * arc[u] + 1]);
                            append_cand<BLOCK>((u32)rec[u].x, r1, g, ws, c, sh, front0, true);
                        }
                        break;
                    }
                    cs = prev;
                }
            }
        }
    }
}

// Epsilon closure to a fixpoint by frontier rounds (decoder.py:138-171; parallel.py:287-325).
// Self-loops are skipped (decoder.py:162-163).  An epsilon winner's payload is the candidate
// index of its source | EPS_BIT.  Frontier entries are states; their candidate index is looked
// up one round later, after the barrier has published it.
template <int BLOCK>
__device__ void epsilon_closure(const GraphDev &g, const WorkDev &ws, Lane &c, Smem<BLOCK> &sh,
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
            sh.tag_round = (int)(c.tag + 1u);
        }
        __syncthreads();
        const u32 tag = (u32)sh.tag_round;
        c.tag = tag;
        const u32 *fin = c.front[which];
        u32 *fout = c.front[which ^ 1];
        const int nchunks = (n_front + 31) >> 5;
        for (int ch = w; ch < nchunks; ch += NW) {
            int i = (ch << 5) + l;
            u32 uu = 0, ui = 0;
            int lo = 0, deg = 0;
            double ucost = 0.0;
            if (i < n_front) {
                uu = fin[i];
                ui = c.cand_of[uu];
                Slot us = ld_slot(&c.slot[uu]);
                int4 rg = c.cand_rng[ui];
                lo = rg.x;
                deg = rg.y - rg.x;
                ucost = key_cost(us.key);
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
                int4 rec = __ldg(&g.arcs[2 * a]);
                if ((u32)rec.x == u_k) continue;  // a positive self-loop never improves its state
                c.e_eps++;
                double wgt = __hiloint2double(rec.w, rec.z);
                u64 key = cost_key(__dadd_rn(uc_k, wgt));
                bool first = false, dec = false;
                if (relax_slot(&c.slot[rec.x], key, (u32)a + 1u, ui_k | EPS_BIT, &first, &dec)) {
                    int4 r1 = make_int4(0, 0, 0, 0);
                    if (first) {
                        r1 = __ldg(&g.arcs[2 * a + 1]);
                        append_cand<BLOCK>((u32)rec.x, r1, g, ws, c, sh, fout, false);
                    } else if (dec) {
                        r1 = __ldg(&g.arcs[2 * a + 1]);
                    }
                    if ((first || dec) && r1.x < r1.y &&
                        atomicExch(&c.qtag[rec.x], tag) != tag) {
                        int f = atomicAdd(&sh.n_front, 1);
                        if (f < ws.cap) fout[f] = (u32)rec.x;
                        else sh.overflow = 1;
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

// Exact max-active cut: K* = the max_active-th smallest (cost, state) among kept candidates
// (decoder.py:188-191).  Expects sh.u.hist filled; sets sh.thr_bucket / thr_key / thr_state.
template <int BLOCK>
__device__ void select_threshold(int n_cand, int max_active, double best, double cutoff,
                                 double scale, const u64 *ckey, Lane &c, Smem<BLOCK> &sh) {
    constexpr int PER = NB / BLOCK;
    u32 loc[PER];
    u32 s = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) { loc[q] = sh.u.hist[threadIdx.x * PER + q]; s += loc[q]; }
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
    int r = max_active - sh.thr_below;  // 1-based rank inside the boundary bucket
    const int cnt = sh.ng;
    __syncthreads();
    if (cnt <= GCAP) {
        if (threadIdx.x == 0) sh.ng = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
            u64 k = ckey[i];
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
    // radix select over the 96-bit (key, state) of the boundary-bucket members, MSB first
    u64 kpre = 0, kmask = 0;
    u32 spre = 0, smask = 0;
    for (int dig = 0; dig < 12; ++dig) {
        for (int b = threadIdx.x; b < 256; b += BLOCK) sh.u.hist[b] = 0;
        __syncthreads();
        const bool in_key = dig < 8;
        const int shift = in_key ? (56 - 8 * dig) : (24 - 8 * (dig - 8));
        for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
            u64 k = ckey[i];
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
// Returns the number of survivors (0 = search death).
template <int BLOCK>
__device__ int finish_step(int nxt, const GraphDev &g, const WorkDev &ws, const CfgDev &cfg,
                           Lane &c, Smem<BLOCK> &sh, int &status, long long &n_rec) {
    const int n_cand = min(sh.n_cand, ws.cap);
    if (sh.overflow) status = WB_ERR_CAPACITY;
    const bool in_smem = n_cand <= ws.smem_cands;
    u64 *ckey = in_smem ? c.s_key : c.cand_key;
    u32 *ca = in_smem ? c.s_ca : c.cand_ca;
    volatile u32 *vca = ca;

    // P1: gather slot contents (batched loads), reset slots, min / max
    u64 mn = EMPTY_KEY, mx = 0;
    for (int i0 = threadIdx.x; i0 < n_cand; i0 += BLOCK * GATHER) {
        u32 st[GATHER];
        Slot v[GATHER];
#pragma unroll
        for (int q = 0; q < GATHER; ++q) {
            int i = i0 + q * BLOCK;
            if (i < n_cand) st[q] = c.cand_state[i];
        }
#pragma unroll
        for (int q = 0; q < GATHER; ++q) {
            int i = i0 + q * BLOCK;
            if (i < n_cand) v[q] = ld_slot(&c.slot[st[q]]);
        }
#pragma unroll
        for (int q = 0; q < GATHER; ++q) {
            int i = i0 + q * BLOCK;
            if (i < n_cand) {
                ckey[i] = v[q].key;
                c.cand_arc[i] = v[q].arcp1;
                c.cand_pay[i] = v[q].pay;
                ca[i] = 0u;
                st_slot_empty(&c.slot[st[q]]);
                mn = v[q].key < mn ? v[q].key : mn;
                mx = v[q].key > mx ? v[q].key : mx;
            }
        }
    }
    block_minmax<BLOCK>(mn, mx, sh);
    if (n_cand == 0) return 0;
    const double best = key_cost(mn);
    const double cutoff = __dadd_rn(best, cfg.beam);  // cutoff = best + beam (decoder.py:186)

    // P2: max-active histogram (only when it can bind)
    bool need_select = false;
    double scale = 0.0;
    if (cfg.max_active > 0 && n_cand > cfg.max_active) {
        double hi = key_cost(mx);
        double top = cutoff < hi ? cutoff : hi;
        double range = __dsub_rn(top, best);
        if (range > 0.0 && range < INFINITY) scale = __ddiv_rn((double)NB, range);
        for (int b = threadIdx.x; b < NB; b += BLOCK) sh.u.hist[b] = 0;
        __syncthreads();
        long long kept = 0;
        for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
            double cst = key_cost(ckey[i]);
            if (cst <= cutoff) {
                ++kept;
                atomicAdd(&sh.u.hist[bucket_of(cst, best, scale)], 1u);
            }
        }
        kept = block_sum<BLOCK>(kept, sh);
        need_select = kept > cfg.max_active;
        if (need_select)
            select_threshold<BLOCK>(n_cand, cfg.max_active, best, cutoff, scale, ckey, c, sh);
    }
    const int bstar = need_select ? sh.thr_bucket : 0;
    const u64 tkey = need_select ? sh.thr_key : 0;
    const u32 tst = need_select ? sh.thr_state : 0;

    // P3: survivor flags + epsilon-chain marks (atomicOr: flags of other candidates change)
    for (int i = threadIdx.x; i < n_cand; i += BLOCK) {
        u64 k = ckey[i];
        double cst = key_cost(k);
        bool surv = cst <= cutoff;
        if (surv && need_select) {
            int b = bucket_of(cst, best, scale);
            surv = b < bstar ||
                   (b == bstar && (k < tkey || (k == tkey && c.cand_state[i] <= tst)));
        }
        if (!surv) continue;
        atomicOr(&ca[i], F_SURV);
        if (!g.has_eps) continue;
        int v = i;
        for (;;) {
            u32 a = c.cand_arc[v], p = c.cand_pay[v];
            if (a == 0u || !(p & EPS_BIT)) break;
            int uix = (int)(p & ~EPS_BIT);
            u32 old = atomicOr(&ca[uix], F_MARK);
            if (old & (F_MARK | F_SURV)) break;
            v = uix;
        }
    }
    __syncthreads();

    // P4: order-preserving compaction of kept candidates (arena records) and survivors
    // (next tokens).  Warps own contiguous segments; ballots count; one scan.
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int seg = ((n_cand + NW - 1) / NW + 31) & ~31;
    const int lo = min(n_cand, w * seg), hi = min(n_cand, lo + seg);
    int ck = 0, cs = 0;
    for (int i0 = lo; i0 < hi; i0 += 32) {
        int i = i0 + l;
        u32 f = i < hi ? vca[i] : 0u;
        ck += __popc(__ballot_sync(FULL, f != 0u));
        cs += __popc(__ballot_sync(FULL, (f & F_SURV) != 0u));
    }
    if (l == 0) { sh.wa[w] = ck; sh.wb[w] = cs; }
    __syncthreads();
    if (w == 0) {
        int va = l < NW ? (int)sh.wa[l] : 0, vb = l < NW ? (int)sh.wb[l] : 0;
        int ia = warp_incl_scan(va), ib = warp_incl_scan(vb);
        if (l < NW) { sh.wa[l] = ia - va; sh.wb[l] = ib - vb; }
        if (l == 31) {
            sh.wa[NW] = ia;
            sh.wb[NW] = ib;
            u64 base = atomicAdd(ws.arena_ctr, (u64)ia);
            if (base + (u64)ia > ws.arena_cap || base + (u64)ia >= (u64)EPS_BIT) sh.overflow = 2;
            sh.arena_base = base;
            sh.n_pend = 0;
        }
    }
    __syncthreads();
    const int n_keep = (int)sh.wa[NW], n_surv = (int)sh.wb[NW];
    if (sh.overflow == 2) { status = WB_ERR_CAPACITY; __syncthreads(); return 0; }
    const u64 base = sh.arena_base;
    int4 *tinfo = c.tok_info[nxt];
    double *tcost = c.tok_cost[nxt];
    u32 *pend = c.front[0];
    {
        int ra = (int)sh.wa[w], rb = (int)sh.wb[w];
        const u32 lt = lanemask_lt();
        for (int i0 = lo; i0 < hi; i0 += 32) {
            int i = i0 + l;
            u32 f = i < hi ? vca[i] : 0u;
            bool keep = f != 0u, surv = (f & F_SURV) != 0u;
            u32 mk = __ballot_sync(FULL, keep), ms = __ballot_sync(FULL, surv);
            if (i < hi) {
                u32 rec = keep ? (u32)(base + (u64)(ra + __popc(mk & lt))) : CA_NONE;
                ca[i] = rec;
                if (surv) {
                    int j = rb + __popc(ms & lt);
                    int4 rg = c.cand_rng[i];
                    tinfo[j] = make_int4((int)c.cand_state[i], (int)rec, rg.y, rg.z);
                    tcost[j] = key_cost(ckey[i]);
                }
                if (keep) {
                    u32 a = c.cand_arc[i], p = c.cand_pay[i];
                    if (a != 0u && (p & EPS_BIT)) {
                        int q = atomicAdd(&sh.n_pend, 1);
                        pend[q] = (u32)i;  // epsilon winner: needs its source's record index
                    } else {
                        u32 prev = a == 0u ? ROOT_PREV : p;
                        ws.arena[rec] = (u64)a | ((u64)prev << 32);
                    }
                }
            }
            ra += __popc(mk);
            rb += __popc(ms);
        }
    }
    __syncthreads();
    const int n_pend = sh.n_pend;
    for (int q = threadIdx.x; q < n_pend; q += BLOCK) {
        int i = (int)pend[q];
        u32 a = c.cand_arc[i], p = c.cand_pay[i];
        ws.arena[vca[i]] = (u64)a | ((u64)vca[p & ~EPS_BIT] << 32);
    }
    n_rec += n_keep;
    __syncthreads();
    return n_surv;
}

// LSD pre-pass (classify_blank_frames + nonblank_frames, posteriors.py:116-125,109-110): a
// frame is blank iff its blank probability strictly exceeds the threshold; non-blank frame
// ids are compacted in order.
template <int BLOCK>
__device__ int lsd_prepass(const double *bl, int T, double thr, int *fr, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int seg = ((T + NW - 1) / NW + 31) & ~31;
    const int lo = min(T, w * seg), hi = min(T, lo + seg);
    int cnt = 0;
    for (int i0 = lo; i0 < hi; i0 += 32) {
        int f = i0 + l;
        cnt += __popc(__ballot_sync(FULL, f < hi && !(bl[f] > thr)));
    }
    int tot;
    int r = warp_offsets<BLOCK>(cnt, sh.wa, &tot);
    const u32 lt = lanemask_lt();
    for (int i0 = lo; i0 < hi; i0 += 32) {
        int f = i0 + l;
        bool nb = f < hi && !(bl[f] > thr);
        u32 m = __ballot_sync(FULL, nb);
        if (nb) fr[r + __popc(m & lt)] = f;
        r += __popc(m);
    }
    __syncthreads();
    return tot;
}

// argmin over tokens by (key, state); returns the token index (-1 if none)
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
    extern __shared__ __align__(16) unsigned char s_dyn[];
    __shared__ Smem<BLOCK> sh;
    const int slot_id = blockIdx.x;
    const size_t S = (size_t)ws.S, cap = (size_t)ws.cap;
    Lane c;
    c.slot = ws.slot + slot_id * S;
    c.cand_of = ws.cand_of + slot_id * S;
    c.qtag = ws.qtag + slot_id * S;
    c.cand_state = ws.cand_state + slot_id * cap;
    c.cand_rng = ws.cand_rng + slot_id * cap;
    c.cand_arc = ws.cand_arc + slot_id * cap;
    c.cand_pay = ws.cand_pay + slot_id * cap;
    c.cand_key = ws.cand_key + slot_id * cap;
    c.cand_ca = ws.cand_ca + slot_id * cap;
    c.front[0] = ws.front + (size_t)slot_id * 2 * cap;
    c.front[1] = c.front[0] + cap;
    c.tok_info[0] = ws.tok_info + (size_t)slot_id * 2 * cap;
    c.tok_info[1] = c.tok_info[0] + cap;
    c.tok_cost[0] = ws.tok_cost + (size_t)slot_id * 2 * cap;
    c.tok_cost[1] = c.tok_cost[0] + cap;
    c.frames = ws.frames + (size_t)slot_id * ws.T_cap;
    c.s_key = reinterpret_cast<u64 *>(s_dyn);
    c.s_ca = reinterpret_cast<u32 *>(s_dyn + sizeof(u64) * (size_t)ws.smem_cands);
    c.tag = ws.tag_ctr[slot_id];
    const bool row_in_smem = ws.row_in_smem != 0;
    double *s_row = reinterpret_cast<double *>(s_dyn);

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
        if (cfg.mode == 1) {
            if (T > ws.T_cap) {  // frame list would overflow: report, do not decode
                status = WB_ERR_CAPACITY;
                nf = 0;
            } else {
                nf = lsd_prepass<BLOCK>(b.blank + row0, T, cfg.thr, c.frames, sh);
            }
        }

        // ---- initial tokens: start entry + epsilon closure + prune (decoder.py:236-249)
        if (threadIdx.x == 0) {
            u64 k0 = cost_key(0.0);
            __stcg(reinterpret_cast<ulonglong2 *>(&c.slot[g.start]),
                   make_ulonglong2(k0, (u64)0u | ((u64)ROOT_PREV << 32)));
            c.cand_state[0] = (u32)g.start;
            c.cand_rng[0] = g.start_rng;
            if (g.has_eps) c.cand_of[g.start] = 0u;
            sh.n_cand = 1;
            sh.overflow = 0;
            sh.n_front = 0;
            if (g.has_eps && g.start_rng.x < g.start_rng.y) {
                c.front[0][0] = (u32)g.start;
                sh.n_front = 1;
            }
        }
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
        int il = __ldg(&g.arcs[2 * a].y);
        int ol = __ldg(&g.arcs[2 * a + 1].w);
        if (ol != 0) { ++no; if (po > 0) ob[--po] = ol; }
        if (il != 0) { ++ni; if (pi > 0) ib[--pi] = il; }
    }
    if (no <= cap) for (int i = 0; i < no; ++i) ob[i] = ob[po + i];
    if (ni <= cap) for (int i = 0; i < ni; ++i) ib[i] = ib[pi + i];
    res[u].n_olabels = no;
    res[u].n_ilabels = ni;
    if ((no > cap || ni > cap) && r.status == WB_OK) res[u].status = WB_ERR_CAPACITY;
}

}  // namespace wb
