// wave_kernel.cuh -- grid-wide batched WFST Viterbi beam search (sm_100a).
//
// A "wave" of W utterances advances one search step at a time together.  Every phase of a
// step is spread over ALL SMs (one cooperative persistent launch, phases separated by grid
// barriers), so one utterance's 15-20k relaxations per frame are processed by ~150 SMs
// instead of one.  Work inside a phase is flattened over (utterance lane, chunk of 32 items);
// chunks never straddle lanes, so per-lane counters are updated with warp-aggregated
// atomics.  Per step (decoder.py:197-233):
//
//   E1 expand   tokens x emitting arcs, warp-level load balancing by prefix-summed
//               out-degree; 32-byte arc records {dst, ilabel, weight | dst ranges, olabel};
//               each relaxation is a fire-and-forget 64-bit atomicMin (RED) of its
//               order-preserving cost key into the destination's slot, and is logged
//   E2 ties     logged relaxations whose key equals the slot minimum atomicMin their
//               arc index + 1: the (cost, src state, arc) total order of decoder.py:121-135
//               (arcs are sorted by source state, so arc order == (src, arc) order)
//   E3 winners  the unique relaxation matching (key, arc) stores its payload and registers
//               the state as a candidate -- no 128-bit CAS on the emitting hot path
//   P2 closure  epsilon frontier rounds (128-bit CAS recombination, epoch-tagged dedup)
//               (decoder.py:138-171)
//   P3 gather   slot -> compact candidate arrays, max-active histogram (4096 value
//               buckets) when the cut can bind (decoder.py:174-194)
//   P5 select   per lane: exact (cost, state) threshold = max_active-th smallest, from the
//               histogram + an exact rank inside the boundary bucket (radix-select fallback)
//   P6 survive  survivors get arena backpointer records + next tokens; epsilon-chain
//               candidates they trace through are claimed and recorded too
//   P8 link     epsilon-winner records (need their source's record index), slot reset
//               O(touched), lane bookkeeping
//
// Arithmetic is float64 in the reference's association order; results are bit-identical to
// decoder.py (labels: winner-consistent traces, identical on tie-free inputs).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "../../include/wfst_b200.h"
#include "device_common.cuh"

namespace wb {
namespace wave {

namespace cg = cooperative_groups;

constexpr int NB = 4096;       // max-active histogram buckets per lane
constexpr int GCAP = 2048;     // boundary-bucket members ranked in shared memory
constexpr int MAXW = 1024;     // lanes per wave (shared-memory prefix arrays)
constexpr u32 CA_NONE = 0xFFFFFFFFu, CA_CLAIM = 0xFFFFFFFEu;
constexpr int MAX_EPS_ROUNDS = 1 << 20;
constexpr int U = 4;           // relaxations in flight per lane (expand)
constexpr int GC = 4;          // chunks per warp iteration in the streaming phases

struct GraphDev {
    int S, A, start, has_eps;
    int4 start_rng;         // {eps_lo, eps_hi (= emit_lo), emit_hi, 0} of the start state
    const int4 *arcs;       // [2*A]: {dst, ilabel, w_lo, w_hi}, {d_eps_lo, d_emit_lo, d_emit_hi, olabel}
    const double *final_w;  // [S] (+inf = not final)
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

// Per-step counters of one lane, double-buffered by step parity.
struct LaneCnt {
    int n_cand;        // candidates registered this step
    int nfront[3];     // epsilon frontier sizes, rotating by round
    int n_surv;        // next-step tokens
    int need;          // max-active cut binds
    int n_log;         // logged emitting relaxations
    int _pad;
    unsigned long long kept;  // candidates within the beam (when the cut may bind)
    u64 kmin, khi;     // min / max of installed cost keys (min == min of final slot values)
    unsigned long long n_rec;  // backpointer records this step
};

// Padded to 4 KB: lanes' hot counters (appends, min/max, logs) are hammered by warp-aggregated
// atomics from every SM, and must not share L2 lines / slices with other lanes' counters.
struct __align__(4096) LaneG {
    LaneCnt cnt[2];
    int utt, T, nf, s, cur, n_live, status, died_at, steps_run, done, tbucket;
    u32 tst;
    u64 tkey;
    long long row0;
    unsigned long long n_tok, a_emit, a_fin, e_eps, n_cand_tot, n_surv_tot, n_rec_tot;
};

struct WaveDev {
    Slot *slot;          // [W][S] recombination slots {cost key, arc+1, payload} (EMPTY between steps)
    u32 *cand_of;        // [W][S] candidate index of a state this step (epsilon graphs)
    u32 *qtag;           // [W][S] epsilon frontier dedup tags (epsilon graphs)
    u32 *log_dst, *log_arc, *log_pay;  // [W][logcap] emitting relaxations of the step
    u64 *log_key;        // [W][logcap]
    u32 *cand_state;     // [W][cap]
    u32 *cand_arc, *cand_pay;  // [W][cap] winner arc + 1, payload (after the gather)
    u32 *ca_idx;         // [W][cap] backpointer record of a kept candidate (CA_NONE = dropped)
    u64 *cand_key;       // [W][cap]
    u32 *front;          // [W][2][cap] frontier states
    int4 *tok_info;      // [W][2][cap] {state, trace, emit_lo, emit_hi}
    double *tok_cost;    // [W][2][cap]
    int *frames;         // [W][T_cap]
    u32 *hist;           // [W][NB]
    LaneG *lane;         // [W]
    u32 *gctr;           // global counters: [0..2] eps pushes (rotating), [3..5] lanes needing
                         // a cut, [6..8] active lanes, [9] qtag epoch
    long long *phase;    // [8] phase cycle counters of the launch
    u64 *arena;          // [arena_cap]
    u64 arena_cap;
    u64 *arena_ctr;
    long long S;
    int cap, logcap, T_cap, W, first_utt;
};

__device__ __forceinline__ size_t lso(const WaveDev &ws, int w) { return (size_t)w * (size_t)ws.S; }
__device__ __forceinline__ size_t lco(const WaveDev &ws, int w) { return (size_t)w * (size_t)ws.cap; }
__device__ __forceinline__ size_t llo(const WaveDev &ws, int w) { return (size_t)w * (size_t)ws.logcap; }

__device__ __forceinline__ int bucket_of(double cst, double best, double scale) {
    double v = __dmul_rn(__dsub_rn(cst, best), scale);
    if (!(v < (double)(NB - 1))) return NB - 1;
    return (int)v;
}

// Beam values of a lane for the current step, recomputed identically wherever needed.
struct Beam {
    double best, cutoff, scale;
    bool may_cut;
};
__device__ __forceinline__ Beam lane_beam(const LaneCnt &cn, const CfgDev &cfg, int n_cand) {
    Beam b;
    b.best = key_cost(cn.kmin);
    b.cutoff = __dadd_rn(b.best, cfg.beam);  // cutoff = best + beam (decoder.py:186)
    b.may_cut = cfg.max_active > 0 && n_cand > cfg.max_active;
    double hi = key_cost(cn.khi);
    double top = b.cutoff < hi ? b.cutoff : hi;
    double range = __dsub_rn(top, b.best);
    b.scale = (range > 0.0 && range < INFINITY) ? __ddiv_rn((double)NB, range) : 0.0;
    return b;
}

__device__ __forceinline__ bool finish_relax(Slot *p, const Slot &want, Slot prev, bool *first,
                                             bool *decreased) {
    if (prev.key == EMPTY_KEY && prev.arcp1 == 0xFFFFFFFFu && prev.pay == 0xFFFFFFFFu) {
        *first = true;
        *decreased = true;
        return true;
    }
    *first = false;
    Slot cs = prev;
    while (slot_better(want.key, want.arcp1, cs)) {
        Slot got = cas_slot(p, cs, want);
        if (got.key == cs.key && got.arcp1 == cs.arcp1 && got.pay == cs.pay) {
            *decreased = want.key < cs.key;
            return true;
        }
        cs = got;
    }
    *decreased = false;
    return false;
}

template <int BLOCK>
struct Smem {
    static constexpr int NW = BLOCK / 32;
    u32 pre[MAXW + 1];     // per-lane chunk prefix of the current phase
    u32 wa[NW + 1];
    u64 r0[NW];
    long long t_mark;
    int flag, ng, thr_bucket, thr_below;
    u64 thr_key;
    u32 thr_state;
    union {
        u32 hist[NB];
        struct {
            u64 key[GCAP];
            u32 st[GCAP];
        } g;
    } u;
};

// ------------------------------------------------------------------ flattened iteration
// Build sh.pre = exclusive prefix over lanes of ceil(count(w) / 32); returns total chunks.
template <int BLOCK, class CNT>
__device__ __forceinline__ int lane_chunks(int W, CNT count, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    u32 carry = 0;
    for (int base = 0; base < W; base += BLOCK) {
        int lane = base + threadIdx.x;
        int c = lane < W ? (count(lane) + 31) >> 5 : 0;
        int incl = warp_incl_scan(c);
        if (l == 31) sh.wa[w] = (u32)incl;
        __syncthreads();
        if (w == 0) {
            int v = l < NW ? (int)sh.wa[l] : 0;
            int iv = warp_incl_scan(v);
            if (l < NW) sh.wa[l] = (u32)(iv - v);
            if (l == 31) sh.wa[NW] = (u32)iv;
        }
        __syncthreads();
        if (lane < W) sh.pre[lane] = carry + sh.wa[w] + (u32)(incl - c);
        carry += sh.wa[NW];
        __syncthreads();
    }
    if (threadIdx.x == 0) sh.pre[W] = carry;
    __syncthreads();
    return (int)carry;
}

// lane owning global chunk ch (largest w with pre[w] <= ch)
__device__ __forceinline__ int chunk_lane(const u32 *pre, int W, u32 ch) {
    int lo = 0, hi = W - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= ch) lo = mid; else hi = mid - 1;
    }
    return lo;
}

template <int BLOCK>
__device__ __forceinline__ void phase_tick(const WaveDev &ws, Smem<BLOCK> &sh, int ph) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        long long t = clock64();
        ws.phase[ph] += t - sh.t_mark;
        sh.t_mark = t;
    }
}

// warp-aggregated atomicAdd on one address (all lanes of the warp call it, converged)
__device__ __forceinline__ u32 warp_reserve(u32 *ctr, bool want, u32 *mask_out) {
    const u32 m = __ballot_sync(FULL, want);
    *mask_out = m;
    if (!m) return 0;
    const int leader = __ffs(m) - 1;
    u32 base = 0;
    if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(ctr, (u32)__popc(m));
    base = __shfl_sync(FULL, base, leader);
    return base + __popc(m & lanemask_lt());
}
__device__ __forceinline__ u64 warp_reserve64(u64 *ctr, bool want) {
    const u32 m = __ballot_sync(FULL, want);
    if (!m) return 0;
    const int leader = __ffs(m) - 1;
    u64 base = 0;
    if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(ctr, (u64)__popc(m));
    base = __shfl_sync(FULL, base, leader);
    return base + __popc(m & lanemask_lt());
}

// Register states installed for the first time this step (warp-converged call): candidate
// index from one atomic per warp; `rng` = the state's {eps_lo, emit_lo, emit_hi} from the arc
// record; states with epsilon arcs record their candidate index and, if `push`, join the
// epsilon frontier.
__device__ __forceinline__ void warp_append(bool first, u32 d, int4 rng, bool push, int w,
                                            const GraphDev &g, const WaveDev &ws, LaneG &L,
                                            int par, u32 *front_out, u32 *front_ctr) {
    u32 m;
    u32 idx = warp_reserve((u32 *)&L.cnt[par].n_cand, first, &m);
    if (!m) return;
    bool pf = false;
    if (first) {
        if ((int)idx < ws.cap) {
            ws.cand_state[lco(ws, w) + idx] = d;
            if (g.has_eps && rng.x < rng.y) {
                ws.cand_of[lso(ws, w) + d] = idx;
                pf = push;
            }
        } else {
            L.status = WB_ERR_CAPACITY;
        }
    }
    if (g.has_eps && push) {
        u32 mf;
        u32 f = warp_reserve(front_ctr, pf, &mf);
        if (mf && (threadIdx.x & 31) == (u32)(__ffs(mf) - 1)) atomicAdd(&ws.gctr[0], (u32)__popc(mf));
        if (pf) {
            if ((int)f < ws.cap) front_out[f] = d;
            else L.status = WB_ERR_CAPACITY;
        }
    }
}

// lane min/max of installed keys (warp-converged call)
__device__ __forceinline__ void warp_minmax(LaneCnt &cn, bool ok, u64 key) {
    u64 mn = ok ? key : EMPTY_KEY, mx = ok ? key : 0ull;
    mn = warp_min_u64(mn);
    mx = warp_max_u64(mx);
    if ((threadIdx.x & 31) == 0 && mn != EMPTY_KEY) {
        atomicMin(&cn.kmin, mn);
        atomicMax(&cn.khi, mx);
    }
}

// ------------------------------------------------------------------ E1: emitting expansion
// Fire-and-forget 64-bit atomicMin of every relaxation's cost key into its slot, plus a log
// entry (dst, key, arc + 1, payload) per relaxation.
template <int BLOCK>
__noinline__ __device__ void phase_expand(const GraphDev &g, const WaveDev &ws,
                                          const BatchDev &b, const CfgDev &cfg, int par,
                                          Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int W = ws.W, l = threadIdx.x & 31;
    const int total = lane_chunks<BLOCK>(W, [&](int w) {
        const LaneG &L = ws.lane[w];
        return L.done ? 0 : L.n_live;
    }, sh);
    for (int ch = blockIdx.x * NW + (threadIdx.x >> 5); ch < total; ch += gridDim.x * NW) {
        const int w = chunk_lane(sh.pre, W, (u32)ch);
        LaneG &L = ws.lane[w];
        LaneCnt &cn = L.cnt[par];
        const int n_live = L.n_live, cur = L.cur;
        const int f = cfg.mode == 1 ? ws.frames[(size_t)w * ws.T_cap + L.s] : L.s;
        const double *row = b.costs + (size_t)(L.row0 + f) * b.L1;
        const size_t co2 = 2 * lco(ws, w) + (size_t)cur * ws.cap;
        Slot *slot = ws.slot + lso(ws, w);
        const size_t lo_ = llo(ws, w);
        const int t = (int)(ch - sh.pre[w]) * 32 + l;
        int4 ti = make_int4(0, 0, 0, 0);
        double tc = 0.0;
        if (t < n_live) { ti = ws.tok_info[co2 + t]; tc = ws.tok_cost[co2 + t]; }
        const int deg = t < n_live ? ti.w - ti.z : 0;
        const int incl = warp_incl_scan(deg);
        const int tot = __shfl_sync(FULL, incl, 31);
        const int excl = incl - deg;
        u32 nfin = 0;
        for (int j0 = 0; j0 < tot; j0 += 32 * U) {
            int4 rec[U];
            u32 arcp1[U], pay[U];
            double cst[U];
            bool act[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int j = j0 + u * 32 + l;
                int k = warp_owner(excl, j);
                int lo_k = __shfl_sync(FULL, ti.z, k);
                int ex_k = __shfl_sync(FULL, excl, k);
                cst[u] = __shfl_sync(FULL, tc, k);
                pay[u] = (u32)__shfl_sync(FULL, ti.y, k);
                act[u] = j < tot;
                int arc = lo_k + j - ex_k;
                arcp1[u] = (u32)arc + 1u;
                if (act[u]) rec[u] = __ldg(&g.arcs[2 * arc]);
            }
            u64 key[U];
            u32 nact = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                key[u] = EMPTY_KEY;
                if (!act[u]) continue;
                double ac = __ldg(&row[rec[u].y]);
                if (ac == INFINITY) {  // decoder.py:219-220: no relaxation, no record
                    act[u] = false;
                    continue;
                }
                double wgt = __hiloint2double(rec[u].w, rec[u].z);
                key[u] = cost_key(__dadd_rn(__dadd_rn(cst[u], wgt), ac));
                atomicMin(&slot[rec[u].x].key, key[u]);  // RED.MIN.64: no return, no wait
                ++nact;
            }
            // log the relaxations: one reservation per warp iteration
            const u32 wn = (u32)warp_sum_ll((long long)nact);
            u32 base = 0;
            if (l == 0 && wn) base = atomicAdd((u32 *)&cn.n_log, wn);
            base = __shfl_sync(FULL, base, 0);
            u32 off = (u32)(warp_incl_scan((int)nact) - (int)nact);
            nfin += nact;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!act[u]) continue;
                const u32 e = base + off++;
                if ((int)e < ws.logcap) {
                    ws.log_dst[lo_ + e] = (u32)rec[u].x;
                    ws.log_key[lo_ + e] = key[u];
                    ws.log_arc[lo_ + e] = arcp1[u];
                    ws.log_pay[lo_ + e] = pay[u];
                } else {
                    L.status = WB_ERR_CAPACITY;
                }
            }
        }
        u32 tot_fin = (u32)warp_sum_ll((long long)nfin);
        if (l == 0) {
            atomicAdd(&L.a_emit, (unsigned long long)tot);
            atomicAdd(&L.a_fin, (unsigned long long)tot_fin);
        }
    }
}

// ------------------------------------------------------------------ E2 / E3: exact ties + winners
// E2 (tie): relaxations whose key equals the slot minimum atomicMin their arc + 1 into it.
// E3 (win): the relaxation matching (key, arc + 1) is the unique winner: it stores its
// payload and registers the state as a candidate (round-0 epsilon frontier if it has
// epsilon arcs).  Lane min / max keys are taken over the winners.
template <int BLOCK>
__noinline__ __device__ void phase_emit_resolve(const GraphDev &g, const WaveDev &ws, int par,
                                                bool win, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int W = ws.W, l = threadIdx.x & 31;
    const int total = lane_chunks<BLOCK>(W, [&](int w) {
        const LaneG &L = ws.lane[w];
        return L.done ? 0 : min(L.cnt[par].n_log, ws.logcap);
    }, sh);
    const int gw = blockIdx.x * NW + (threadIdx.x >> 5), nwarps = gridDim.x * NW;
    for (int c0 = gw * GC; c0 < total; c0 += nwarps * GC) {
        int wq[GC];
        u32 dq[GC], aq[GC];
        u64 kq[GC];
        Slot sq[GC];
#pragma unroll
        for (int q = 0; q < GC; ++q) {
            const int ch = c0 + q;
            wq[q] = -1;
            if (ch < total) {
                const int w = chunk_lane(sh.pre, W, (u32)ch);
                const int i = (int)(ch - sh.pre[w]) * 32 + l;
                if (i < min(ws.lane[w].cnt[par].n_log, ws.logcap)) {
                    const size_t e = llo(ws, w) + i;
                    wq[q] = w;
                    dq[q] = ws.log_dst[e];
                    kq[q] = ws.log_key[e];
                    aq[q] = ws.log_arc[e];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < GC; ++q)
            if (wq[q] >= 0) sq[q] = ld_slot(&ws.slot[lso(ws, wq[q]) + dq[q]]);
        if (!win) {
#pragma unroll
            for (int q = 0; q < GC; ++q)
                if (wq[q] >= 0 && sq[q].key == kq[q] && aq[q] < sq[q].arcp1)
                    atomicMin(&ws.slot[lso(ws, wq[q]) + dq[q]].arcp1, aq[q]);
            continue;
        }
#pragma unroll
        for (int q = 0; q < GC; ++q) {
            const int ch = c0 + q;
            if (ch >= total) break;  // warp-uniform
            const int w = chunk_lane(sh.pre, W, (u32)ch);
            LaneG &L = ws.lane[w];
            LaneCnt &cn = L.cnt[par];
            const bool first = wq[q] >= 0 && sq[q].key == kq[q] && sq[q].arcp1 == aq[q];
            int4 r1 = make_int4(0, 0, 0, 0);
            if (first) {
                const size_t e = llo(ws, w) + (size_t)(ch - (int)sh.pre[w]) * 32 + l;
                ws.slot[lso(ws, w) + dq[q]].pay = ws.log_pay[e];
                if (g.has_eps) r1 = __ldg(&g.arcs[2 * (aq[q] - 1u) + 1]);
            }
            warp_minmax(cn, first, kq[q]);
            warp_append(first, dq[q], r1, true, w, g, ws, L, par,
                        ws.front + 2 * lco(ws, w), (u32 *)&cn.nfront[0]);
        }
    }
}

// ------------------------------------------------------------------ P2: epsilon closure round
// Round r reads frontier buffer r&1 (size nfront[r%3]) and pushes into buffer (r+1)&1
// (nfront[(r+1)%3]); nfront[(r+2)%3] and gctr[(r+2)%3] are zeroed for round r+1.  Frontier
// entries are states; an epsilon winner's payload is its source state | EPS_BIT.
template <int BLOCK>
__noinline__ __device__ void phase_eps_round(const GraphDev &g, const WaveDev &ws, int par,
                                             int r, u32 tag, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int W = ws.W, l = threadIdx.x & 31;
    const int rin = r % 3, rout = (r + 1) % 3, rzero = (r + 2) % 3;
    if (blockIdx.x == 0) {
        for (int w = threadIdx.x; w < W; w += BLOCK) ws.lane[w].cnt[par].nfront[rzero] = 0;
        if (threadIdx.x == 0) ws.gctr[rzero] = 0;
    }
    const int total = lane_chunks<BLOCK>(W, [&](int w) {
        const LaneG &L = ws.lane[w];
        return L.done ? 0 : min(L.cnt[par].nfront[rin], ws.cap);
    }, sh);
    const Slot empty = {EMPTY_KEY, 0xFFFFFFFFu, 0xFFFFFFFFu};
    for (int ch = blockIdx.x * NW + (threadIdx.x >> 5); ch < total; ch += gridDim.x * NW) {
        const int w = chunk_lane(sh.pre, W, (u32)ch);
        LaneG &L = ws.lane[w];
        LaneCnt &cn = L.cnt[par];
        const int nfr = min(cn.nfront[rin], ws.cap);
        Slot *slot = ws.slot + lso(ws, w);
        const size_t co = lco(ws, w);
        const u32 *fin = ws.front + 2 * co + (size_t)(r & 1) * ws.cap;
        u32 *fout = ws.front + 2 * co + (size_t)((r + 1) & 1) * ws.cap;
        const int i = (int)(ch - sh.pre[w]) * 32 + l;
        u32 uu = 0;
        int lo = 0, deg = 0;
        double ucost = 0.0;
        if (i < nfr) {
            uu = fin[i];
            Slot us = ld_slot(&slot[uu]);
            int4 rg = us.arcp1 == 0u ? g.start_rng : __ldg(&g.arcs[2 * (us.arcp1 - 1u) + 1]);
            lo = rg.x;
            deg = rg.y - rg.x;
            ucost = key_cost(us.key);
        }
        const int incl = warp_incl_scan(deg);
        const int tot = __shfl_sync(FULL, incl, 31);
        const int excl = incl - deg;
        u32 neps = 0;
        for (int j0 = 0; j0 < tot; j0 += 32) {
            int j = j0 + l;
            int k = warp_owner(excl, j);
            int lo_k = __shfl_sync(FULL, lo, k);
            int ex_k = __shfl_sync(FULL, excl, k);
            double uc_k = __shfl_sync(FULL, ucost, k);
            u32 u_k = __shfl_sync(FULL, uu, k);
            bool act = j < tot;
            int a = lo_k + j - ex_k;
            int4 rec = make_int4(0, 0, 0, 0);
            if (act) {
                rec = __ldg(&g.arcs[2 * a]);
                if ((u32)rec.x == u_k) act = false;  // a positive self-loop never improves its state
            }
            bool first = false, dec = false, ok = false;
            Slot want;
            want.key = EMPTY_KEY;
            if (act) {
                ++neps;
                want.key = cost_key(__dadd_rn(uc_k, __hiloint2double(rec.w, rec.z)));
                want.arcp1 = (u32)a + 1u;
                want.pay = u_k | EPS_BIT;  // epsilon winner: payload = source state
                Slot prev = cas_slot(&slot[rec.x], empty, want);
                ok = finish_relax(&slot[rec.x], want, prev, &first, &dec);
            }
            warp_minmax(cn, ok, want.key);
            int4 r1 = make_int4(0, 0, 0, 0);
            if (ok && dec) r1 = __ldg(&g.arcs[2 * a + 1]);
            warp_append(first, (u32)rec.x, r1, false, w, g, ws, L, par, fout, nullptr);
            // states that are new or got cheaper re-relax their epsilon arcs next round
            bool push = ok && dec && r1.x < r1.y &&
                        atomicExch(&ws.qtag[lso(ws, w) + rec.x], tag) != tag;
            u32 mp;
            u32 fidx = warp_reserve((u32 *)&cn.nfront[rout], push, &mp);
            if (mp && l == __ffs(mp) - 1) atomicAdd(&ws.gctr[rout], (u32)__popc(mp));
            if (push) {
                if ((int)fidx < ws.cap) fout[fidx] = (u32)rec.x;
                else L.status = WB_ERR_CAPACITY;
            }
        }
        u32 te = (u32)warp_sum_ll((long long)neps);
        if (l == 0 && te) atomicAdd(&L.e_eps, (unsigned long long)te);
    }
}

// ------------------------------------------------------------------ P3: gather + histogram
template <int BLOCK>
__noinline__ __device__ void phase_gather(const GraphDev &g, const WaveDev &ws,
                                          const CfgDev &cfg, int par, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int W = ws.W, l = threadIdx.x & 31;
    const int total = lane_chunks<BLOCK>(W, [&](int w) {
        const LaneG &L = ws.lane[w];
        return L.done ? 0 : min(L.cnt[par].n_cand, ws.cap);
    }, sh);
    const int gw = blockIdx.x * NW + (threadIdx.x >> 5), nwarps = gridDim.x * NW;
    for (int c0 = gw * GC; c0 < total; c0 += nwarps * GC) {
        int wq[GC], iq[GC];
        u32 st[GC];
        Slot v[GC];
#pragma unroll
        for (int q = 0; q < GC; ++q) {
            const int ch = c0 + q;
            wq[q] = -1;
            iq[q] = 0;
            if (ch < total) {
                const int w = chunk_lane(sh.pre, W, (u32)ch);
                const int i = (int)(ch - sh.pre[w]) * 32 + l;
                if (i < min(ws.lane[w].cnt[par].n_cand, ws.cap)) {
                    wq[q] = w;
                    iq[q] = i;
                    st[q] = ws.cand_state[lco(ws, w) + i];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < GC; ++q)
            if (wq[q] >= 0) v[q] = ld_slot(&ws.slot[lso(ws, wq[q]) + st[q]]);
#pragma unroll
        for (int q = 0; q < GC; ++q) {
            const int ch = c0 + q;
            if (ch >= total) break;  // warp-uniform
            const int w = chunk_lane(sh.pre, W, (u32)ch);
            LaneCnt &cn = ws.lane[w].cnt[par];
            const Beam bm = lane_beam(cn, cfg, min(cn.n_cand, ws.cap));
            bool in = false;
            if (wq[q] >= 0) {
                const size_t co = lco(ws, w) + iq[q];
                ws.cand_key[co] = v[q].key;
                ws.cand_arc[co] = v[q].arcp1;
                ws.cand_pay[co] = v[q].pay;
                ws.ca_idx[co] = CA_NONE;
                double cst = key_cost(v[q].key);
                in = cst <= bm.cutoff;
                if (bm.may_cut && in)
                    atomicAdd(&ws.hist[(size_t)w * NB + bucket_of(cst, bm.best, bm.scale)], 1u);
            }
            if (bm.may_cut) {
                u32 kept = (u32)__popc(__ballot_sync(FULL, in));
                if (l == 0 && kept) atomicAdd(&cn.kept, (unsigned long long)kept);
                if (ch == (int)sh.pre[w] && l == 0) atomicAdd(&ws.gctr[3 + par], 1u);
            }
        }
    }
}

// ------------------------------------------------------------------ P5: max-active threshold
template <int BLOCK>
__noinline__ __device__ void lane_threshold(const WaveDev &ws, const CfgDev &cfg, int w, int par,
                               Smem<BLOCK> &sh) {
    LaneG &L = ws.lane[w];
    LaneCnt &cn = L.cnt[par];
    const int n = min(cn.n_cand, ws.cap);
    const Beam bm = lane_beam(cn, cfg, n);
    u32 *hist = ws.hist + (size_t)w * NB;
    const int M = cfg.max_active;
    const bool need = !L.done && bm.may_cut && cn.kept > (unsigned long long)M;
    if (!need) {
        if (!L.done && bm.may_cut)
            for (int q = threadIdx.x; q < NB; q += BLOCK) hist[q] = 0u;
        if (threadIdx.x == 0) cn.need = 0;
        __syncthreads();
        return;
    }
    // smallest bucket b with inclusive prefix >= M
    constexpr int PER = NB / BLOCK;
    constexpr int NW = BLOCK / 32;
    const int wp = threadIdx.x >> 5, l = threadIdx.x & 31;
    u32 loc[PER];
    u32 s = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) { loc[q] = hist[threadIdx.x * PER + q]; s += loc[q]; }
    int incl = warp_incl_scan((int)s);
    if (l == 31) sh.wa[wp] = incl;
    __syncthreads();
    if (wp == 0) {
        int v = l < NW ? (int)sh.wa[l] : 0;
        int iv = warp_incl_scan(v);
        if (l < NW) sh.wa[l] = iv - v;
    }
    __syncthreads();
    u32 run = sh.wa[wp] + incl - s;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        if (run < (u32)M && run + loc[q] >= (u32)M) {
            sh.thr_bucket = threadIdx.x * PER + q;
            sh.thr_below = (int)run;
            sh.ng = (int)loc[q];
        }
        run += loc[q];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < NB; q += BLOCK) hist[q] = 0u;
    const int bstar = sh.thr_bucket;
    int r = M - sh.thr_below;  // 1-based rank inside the boundary bucket
    const int cnt = sh.ng;
    __syncthreads();
    const size_t co = lco(ws, w);
    const u64 *ckey = ws.cand_key + co;
    const u32 *cst_ = ws.cand_state + co;
    if (cnt <= GCAP) {
        if (threadIdx.x == 0) sh.ng = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += BLOCK) {
            u64 k = ckey[i];
            double cst = key_cost(k);
            if (cst <= bm.cutoff && bucket_of(cst, bm.best, bm.scale) == bstar) {
                int j = atomicAdd(&sh.ng, 1);
                sh.u.g.key[j] = k;
                sh.u.g.st[j] = cst_[i];
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
    } else {
        // radix select over the 96-bit (key, state) of the boundary-bucket members
        u64 kpre = 0, kmask = 0;
        u32 spre = 0, smask = 0;
        for (int dig = 0; dig < 12; ++dig) {
            for (int q = threadIdx.x; q < 256; q += BLOCK) sh.u.hist[q] = 0;
            __syncthreads();
            const bool in_key = dig < 8;
            const int shift = in_key ? (56 - 8 * dig) : (24 - 8 * (dig - 8));
            for (int i = threadIdx.x; i < n; i += BLOCK) {
                u64 k = ckey[i];
                double cst = key_cost(k);
                if (!(cst <= bm.cutoff) || bucket_of(cst, bm.best, bm.scale) != bstar) continue;
                u32 st = cst_[i];
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
    if (threadIdx.x == 0) {
        L.tbucket = bstar;
        L.tkey = sh.thr_key;
        L.tst = sh.thr_state;
        cn.need = 1;
    }
    __syncthreads();
}

// survival test (decoder.py:185-191): within the beam and, if the cut binds, among the
// max_active smallest by (cost, state)
__device__ __forceinline__ bool survives(u64 k, u32 st, const Beam &bm, const LaneG &L,
                                         int need) {
    double cst = key_cost(k);
    if (!(cst <= bm.cutoff)) return false;
    if (!need) return true;
    int b = bucket_of(cst, bm.best, bm.scale);
    return b < L.tbucket || (b == L.tbucket && (k < L.tkey || (k == L.tkey && st <= L.tst)));
}

// ------------------------------------------------------------------ P6: survivors + records
// Survivors get a backpointer record and a next-step token.  An epsilon winner's record links
// to its source candidate's record (written in P8); sources that are not survivors themselves
// are claimed here (CAS on their record slot) so exactly one thread records each.
template <int BLOCK>
__noinline__ __device__ void phase_survive(const GraphDev &g, const WaveDev &ws,
                                           const CfgDev &cfg, int par, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int W = ws.W, l = threadIdx.x & 31;
    const int total = lane_chunks<BLOCK>(W, [&](int w) {
        const LaneG &L = ws.lane[w];
        return L.done ? 0 : min(L.cnt[par].n_cand, ws.cap);
    }, sh);
    const int gw = blockIdx.x * NW + (threadIdx.x >> 5), nwarps = gridDim.x * NW;
    for (int c0 = gw * GC; c0 < total; c0 += nwarps * GC) {
        u64 kq[GC];
        u32 sq[GC];
        int iq[GC], wq[GC];
#pragma unroll
        for (int q = 0; q < GC; ++q) {
            const int ch = c0 + q;
            wq[q] = -1;
            iq[q] = 0;
            if (ch < total) {
                const int w = chunk_lane(sh.pre, W, (u32)ch);
                const int i = (int)(ch - sh.pre[w]) * 32 + l;
                if (i < min(ws.lane[w].cnt[par].n_cand, ws.cap)) {
                    const size_t co = lco(ws, w) + i;
                    wq[q] = w;
                    iq[q] = i;
                    kq[q] = ws.cand_key[co];
                    sq[q] = ws.cand_state[co];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < GC; ++q) {
            const int ch = c0 + q;
            if (ch >= total) break;  // warp-uniform
            const int w = chunk_lane(sh.pre, W, (u32)ch);
            LaneG &L = ws.lane[w];
            LaneCnt &cn = L.cnt[par];
            const int n = min(cn.n_cand, ws.cap);
            const Beam bm = lane_beam(cn, cfg, n);
            const int need = cn.need;
            const bool surv = wq[q] >= 0 && survives(kq[q], sq[q], bm, L, need);
            const u64 rec = warp_reserve64(ws.arena_ctr, surv);
            u32 mtok;
            const u32 j = warp_reserve((u32 *)&cn.n_surv, surv, &mtok);
            if (mtok && l == __ffs(mtok) - 1) atomicAdd(&cn.n_rec, (unsigned long long)__popc(mtok));
            if (!surv) continue;
            if (rec >= ws.arena_cap || rec >= (u64)EPS_BIT) { L.status = WB_ERR_CAPACITY; continue; }
            const size_t co = lco(ws, w);
            const int i = iq[q];
            ws.ca_idx[co + i] = (u32)rec;
            const u32 a = ws.cand_arc[co + i], p = ws.cand_pay[co + i];
            const int4 r1 = a == 0u ? g.start_rng : __ldg(&g.arcs[2 * (a - 1u) + 1]);
            const size_t nx = 2 * co + (size_t)(L.cur ^ 1) * ws.cap;
            ws.tok_info[nx + j] = make_int4((int)sq[q], (int)rec, r1.y, r1.z);
            ws.tok_cost[nx + j] = key_cost(kq[q]);
            if (a == 0u || !(p & EPS_BIT)) {
                ws.arena[rec] = (u64)a | ((u64)(a == 0u ? ROOT_PREV : p) << 32);
                continue;
            }
            // epsilon winner: claim the non-surviving candidates of its epsilon chain
            u32 src = p & ~EPS_BIT;  // source state
            for (;;) {
                const u32 uc = ws.cand_of[lso(ws, w) + src];
                if (survives(ws.cand_key[co + uc], src, bm, L, need)) break;  // own thread records it
                if (atomicCAS(&ws.ca_idx[co + uc], CA_NONE, CA_CLAIM) != CA_NONE) break;
                const u64 ru = atomicAdd(ws.arena_ctr, 1ull);
                atomicAdd(&cn.n_rec, 1ull);
                if (ru >= ws.arena_cap || ru >= (u64)EPS_BIT) { L.status = WB_ERR_CAPACITY; break; }
                ws.ca_idx[co + uc] = (u32)ru;
                const u32 au = ws.cand_arc[co + uc], pu = ws.cand_pay[co + uc];
                if (au == 0u || !(pu & EPS_BIT)) {
                    ws.arena[ru] = (u64)au | ((u64)(au == 0u ? ROOT_PREV : pu) << 32);
                    break;
                }
                src = pu & ~EPS_BIT;
            }
        }
    }
}

// ------------------------------------------------------------------ P8: epsilon links + lanes
template <int BLOCK>
__noinline__ __device__ void phase_link(const GraphDev &g, const WaveDev &ws, const CfgDev &cfg,
                                        int k, Smem<BLOCK> &sh) {
    constexpr int NW = BLOCK / 32;
    const int par = k & 1;
    const bool search_step = k > 0;
    const int W = ws.W, l = threadIdx.x & 31;
    {
        // epsilon-winner records (their source's record index is final now) and the slot
        // reset O(touched) for the next step
        const int total = lane_chunks<BLOCK>(W, [&](int w) {
            const LaneG &L = ws.lane[w];
            return L.done ? 0 : min(L.cnt[par].n_cand, ws.cap);
        }, sh);
        const int gw = blockIdx.x * NW + (threadIdx.x >> 5), nwarps = gridDim.x * NW;
        for (int c0 = gw * GC; c0 < total; c0 += nwarps * GC) {
            u32 aq[GC], pq[GC], rq[GC], sq[GC];
            int wq[GC];
#pragma unroll
            for (int q = 0; q < GC; ++q) {
                const int ch = c0 + q;
                wq[q] = -1;
                if (ch < total) {
                    const int w = chunk_lane(sh.pre, W, (u32)ch);
                    const int i = (int)(ch - sh.pre[w]) * 32 + l;
                    if (i < min(ws.lane[w].cnt[par].n_cand, ws.cap)) {
                        const size_t co = lco(ws, w) + i;
                        wq[q] = w;
                        sq[q] = ws.cand_state[co];
                        rq[q] = ws.ca_idx[co];
                        aq[q] = ws.cand_arc[co];
                        pq[q] = ws.cand_pay[co];
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < GC; ++q) {
                if (wq[q] < 0) continue;
                const int w = wq[q];
                if (rq[q] < CA_CLAIM && aq[q] != 0u && (pq[q] & EPS_BIT)) {
                    const u32 uc = ws.cand_of[lso(ws, w) + (pq[q] & ~EPS_BIT)];
                    ws.arena[rq[q]] = (u64)aq[q] | ((u64)ws.ca_idx[lco(ws, w) + uc] << 32);
                }
                st_slot_empty(&ws.slot[lso(ws, w) + sq[q]]);
            }
        }
    }
    // lane bookkeeping: one thread per lane; nothing else in this phase reads these fields
    for (int w = blockIdx.x * BLOCK + threadIdx.x; w < W; w += gridDim.x * BLOCK) {
        LaneG &L = ws.lane[w];
        LaneCnt &cn = L.cnt[par];
        LaneCnt &nx = L.cnt[par ^ 1];
        nx.n_cand = 0;
        nx.nfront[0] = nx.nfront[1] = nx.nfront[2] = 0;
        nx.n_surv = 0;
        nx.need = 0;
        nx.n_log = 0;
        nx.kept = 0;
        nx.kmin = EMPTY_KEY;
        nx.khi = 0;
        nx.n_rec = 0;
        if (L.done) continue;
        const int n = min(cn.n_cand, ws.cap);
        if (cn.n_cand > ws.cap || cn.n_log > ws.logcap) L.status = WB_ERR_CAPACITY;
        L.n_cand_tot += n;
        L.n_rec_tot += cn.n_rec;
        if (!search_step) {  // initial tokens (decoder.py:236-249)
            L.n_live = cn.n_surv;
            L.cur ^= 1;
            L.n_surv_tot += cn.n_surv;
        } else {
            L.n_tok += L.n_live;
            L.steps_run += 1;
            if (cn.n_surv == 0) {  // search death (decoder.py:322-324)
                L.died_at = L.s;
                L.done = 1;
            } else {
                L.n_surv_tot += cn.n_surv;
                L.n_live = cn.n_surv;
                L.cur ^= 1;
                L.s += 1;
            }
        }
        if (L.s >= L.nf || L.status != WB_OK) L.done = 1;
        if (!L.done) atomicAdd(&ws.gctr[6 + ((k + 1) % 3)], 1u);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ws.gctr[0] = ws.gctr[1] = ws.gctr[2] = 0;
        ws.gctr[3 + (par ^ 1)] = 0;
        ws.gctr[6 + ((k + 2) % 3)] = 0;
    }
}

// ------------------------------------------------------------------ the persistent kernel
template <int BLOCK, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
wave_kernel(const __grid_constant__ GraphDev g, const __grid_constant__ WaveDev ws,
            const __grid_constant__ BatchDev b, const __grid_constant__ CfgDev cfg,
            wb_utt_result *res) {
    __shared__ Smem<BLOCK> sh;
    cg::grid_group grid = cg::this_grid();
    const int W = ws.W;
    if (blockIdx.x == 0 && threadIdx.x == 0) sh.t_mark = clock64();

    // ---- lane setup + LSD pre-pass (posteriors.py:116-125): one CTA per lane
    for (int w = blockIdx.x; w < W; w += gridDim.x) {
        LaneG &L = ws.lane[w];
        const int u = ws.first_utt + w;
        const bool real = u < b.n;
        const int T = real ? b.T[u] : 0;
        const long long row0 = real ? b.row_off[u] : 0;
        int nf = T, status = WB_OK;
        if (real && cfg.mode == 1) {
            if (T > ws.T_cap) {
                status = WB_ERR_CAPACITY;
                nf = 0;
            } else {
                const double *bl = b.blank + row0;
                int *fr = ws.frames + (size_t)w * ws.T_cap;
                constexpr int NW = BLOCK / 32;
                const int wp = threadIdx.x >> 5, l = threadIdx.x & 31;
                u32 carry = 0;
                for (int base = 0; base < T; base += BLOCK) {
                    int f = base + threadIdx.x;
                    bool nb = f < T && !(bl[f] > cfg.thr);
                    u32 m = __ballot_sync(FULL, nb);
                    if (l == 0) sh.wa[wp] = __popc(m);
                    __syncthreads();
                    if (wp == 0) {
                        int v = l < NW ? (int)sh.wa[l] : 0;
                        int iv = warp_incl_scan(v);
                        if (l < NW) sh.wa[l] = (u32)(iv - v);
                        if (l == 31) sh.wa[NW] = (u32)iv;
                    }
                    __syncthreads();
                    if (nb) fr[carry + sh.wa[wp] + __popc(m & lanemask_lt())] = f;
                    carry += sh.wa[NW];
                    __syncthreads();
                }
                nf = (int)carry;
            }
        }
        if (threadIdx.x == 0) {
            L.utt = real ? u : -1;
            L.T = T;
            L.nf = nf;
            L.s = 0;
            L.cur = 1;  // the initial step writes buffer 0 (cur ^ 1)
            L.n_live = 0;
            L.status = status;
            L.died_at = -1;
            L.steps_run = 0;
            L.done = real ? 0 : 1;
            L.row0 = row0;
            L.n_tok = L.a_emit = L.a_fin = L.e_eps = L.n_cand_tot = L.n_surv_tot = L.n_rec_tot = 0;
            for (int q = 0; q < 2; ++q) {
                LaneCnt &cn = L.cnt[q];
                cn.n_cand = 0;
                cn.nfront[0] = cn.nfront[1] = cn.nfront[2] = 0;
                cn.n_surv = 0;
                cn.need = 0;
                cn.n_log = 0;
                cn.kept = 0;
                cn.kmin = EMPTY_KEY;
                cn.khi = 0;
                cn.n_rec = 0;
            }
            if (real) {
                // start entry (0.0, src -1, arc -1, ROOT) (decoder.py:241); slots are EMPTY
                const size_t so = lso(ws, w), co = lco(ws, w);
                const u64 k0 = cost_key(0.0);
                __stcg(reinterpret_cast<ulonglong2 *>(&ws.slot[so + g.start]),
                       make_ulonglong2(k0, (u64)0u | ((u64)ROOT_PREV << 32)));
                ws.cand_state[co] = (u32)g.start;
                L.cnt[0].n_cand = 1;
                L.cnt[0].kmin = k0;
                L.cnt[0].khi = k0;
                if (g.has_eps && g.start_rng.x < g.start_rng.y) {
                    ws.cand_of[so + g.start] = 0u;
                    ws.front[2 * co] = (u32)g.start;
                    L.cnt[0].nfront[0] = 1;
                    atomicAdd(&ws.gctr[0], 1u);
                }
            }
        }
        __syncthreads();
    }
    grid.sync();
    phase_tick(ws, sh, 7);

    u32 tag = ws.gctr[9];
    for (int k = 0;; ++k) {
        const int par = k & 1;
        if (k > 0) {
            if (ws.gctr[6 + (k % 3)] == 0) break;  // no active lane left
            phase_expand<BLOCK>(g, ws, b, cfg, par, sh);
            grid.sync();
            phase_tick(ws, sh, 0);
            phase_emit_resolve<BLOCK>(g, ws, par, false, sh);
            grid.sync();
            phase_emit_resolve<BLOCK>(g, ws, par, true, sh);
            grid.sync();
            phase_tick(ws, sh, 1);
        }
        if (g.has_eps) {
            for (int r = 0; r < MAX_EPS_ROUNDS; ++r) {
                if (ws.gctr[r % 3] == 0) break;  // nothing was pushed for this round
                ++tag;
                phase_eps_round<BLOCK>(g, ws, par, r, tag, sh);
                grid.sync();
            }
            phase_tick(ws, sh, 2);
        }
        phase_gather<BLOCK>(g, ws, cfg, par, sh);
        grid.sync();
        phase_tick(ws, sh, 3);
        if (ws.gctr[3 + par]) {
            for (int w = blockIdx.x; w < W; w += gridDim.x) lane_threshold<BLOCK>(ws, cfg, w, par, sh);
            grid.sync();
        }
        phase_tick(ws, sh, 4);
        phase_survive<BLOCK>(g, ws, cfg, par, sh);
        grid.sync();
        phase_tick(ws, sh, 5);
        phase_link<BLOCK>(g, ws, cfg, k, sh);
        grid.sync();
        phase_tick(ws, sh, 6);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ws.gctr[9] = tag;

    // ---- final transition / death fallback (decoder.py:252-273, 327-333): CTA per lane
    for (int w = blockIdx.x; w < W; w += gridDim.x) {
        const LaneG &L = ws.lane[w];
        if (L.utt < 0) continue;
        const size_t cb = 2 * lco(ws, w) + (size_t)L.cur * ws.cap;
        const int4 *tinfo = ws.tok_info + cb;
        const double *tcost = ws.tok_cost + cb;
        const int n_live = L.n_live;
        constexpr int NW = BLOCK / 32;
        const int wp = threadIdx.x >> 5, l = threadIdx.x & 31;
        int best_t = -1, reached = 0;
        for (int pass = 0; pass < 2 && best_t < 0; ++pass) {
            if (pass == 0 && L.died_at >= 0) continue;
            u64 kk = EMPTY_KEY;
            u32 st = 0xFFFFFFFFu;
            int idx = -1;
            for (int t = threadIdx.x; t < n_live; t += BLOCK) {
                int s = tinfo[t].x;
                u64 key;
                if (pass == 0) {
                    double fw = __ldg(&g.final_w[s]);
                    if (fw == INFINITY) continue;
                    key = cost_key(__dadd_rn(tcost[t], fw));
                } else {
                    key = cost_key(tcost[t]);
                }
                if (key < kk || (key == kk && (u32)s < st)) { kk = key; st = (u32)s; idx = t; }
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                u64 k2 = __shfl_xor_sync(FULL, kk, o);
                u32 s2 = __shfl_xor_sync(FULL, st, o);
                int i2 = __shfl_xor_sync(FULL, idx, o);
                if (k2 < kk || (k2 == kk && s2 < st)) { kk = k2; st = s2; idx = i2; }
            }
            if (l == 0) { sh.r0[wp] = kk; sh.u.g.st[wp] = st; sh.u.g.st[NW + wp] = (u32)idx; }
            __syncthreads();
            if (threadIdx.x == 0) {
                u64 bk = EMPTY_KEY;
                u32 bs = 0xFFFFFFFFu;
                int bi = -1;
                for (int q = 0; q < NW; ++q) {
                    u64 k2 = sh.r0[q];
                    u32 s2 = sh.u.g.st[q];
                    if (k2 < bk || (k2 == bk && s2 < bs)) { bk = k2; bs = s2; bi = (int)sh.u.g.st[NW + q]; }
                }
                sh.flag = bk == EMPTY_KEY ? -1 : bi;
            }
            __syncthreads();
            best_t = sh.flag;
            __syncthreads();
            if (best_t >= 0 && pass == 0) reached = 1;
        }
        if (threadIdx.x == 0) {
            wb_utt_result r;
            memset(&r, 0, sizeof(r));
            double bc = 0.0;
            if (best_t >= 0) {
                bc = tcost[best_t];
                if (reached) bc = __dadd_rn(bc, __ldg(&g.final_w[tinfo[best_t].x]));
            }
            r.total_cost = bc;
            r.tokens_expanded = (long long)L.n_tok;
            r.search_steps = L.steps_run;
            r.reached_final = reached;
            r.died_at_step = L.died_at;
            r.final_state = best_t >= 0 ? tinfo[best_t].x : -1;
            r.final_step = L.died_at < 0 ? L.steps_run : L.died_at;
            r.status = L.status;
            r.best_trace = best_t >= 0 ? (long long)(u32)tinfo[best_t].y : -1;
            r.n_tok = (long long)L.n_tok;
            r.a_emit = (long long)L.a_emit;
            r.a_fin = (long long)L.a_fin;
            r.e_eps = (long long)L.e_eps;
            r.n_cand = (long long)L.n_cand_tot;
            r.n_surv = (long long)L.n_surv_tot;
            r.n_rec = (long long)L.n_rec_tot;
            for (int q = 0; q < 8; ++q) r.phase_cycles[q] = ws.phase[q];
            res[L.utt] = r;
        }
        __syncthreads();
    }
}

// Backtrace (decoder.py:276-291): one thread per utterance walks the arena from the winner;
// labels are written back-to-front so they land in path order without a second walk.
__global__ void backtrace_kernel(const u64 *arena, const int4 *arcs, wb_utt_result *res, int n,
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
        int il = __ldg(&arcs[2 * a].y);
        int ol = __ldg(&arcs[2 * a + 1].w);
        if (ol != 0) { ++no; if (po > 0) ob[--po] = ol; }
        if (il != 0) { ++ni; if (pi > 0) ib[--pi] = il; }
    }
    if (no <= cap) for (int i = 0; i < no; ++i) ob[i] = ob[po + i];
    if (ni <= cap) for (int i = 0; i < ni; ++i) ib[i] = ib[pi + i];
    res[u].n_olabels = no;
    res[u].n_ilabels = ni;
    if ((no > cap || ni > cap) && r.status == WB_OK) res[u].status = WB_ERR_CAPACITY;
}

}  // namespace wave
}  // namespace wb
