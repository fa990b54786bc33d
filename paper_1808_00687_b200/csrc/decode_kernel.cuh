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
//   prune    exact beam + max-active cut without a sort: min/max reduce, a 2048-bucket value
//            histogram in shared memory, exact (cost, state) rank inside the boundary bucket
//            (radix-select fallback) (decoder.py:174-194).
//   compact  candidate keys/flags live in shared memory; survivors and the epsilon-chain
//            candidates they trace through get 8-byte backpointer records in a batch-wide
//            arena; slots are reset O(touched).
//
// Arithmetic is float64 in the reference's association order, so costs, survivor sets,
// tokens_expanded and (tie-free) labels are bit-identical to decoder.py.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "../../include/wfst_b200.h"
#include "device_common.cuh"

namespace wb {

#ifndef WB_EPS_UNIT_SPLIT
#define WB_EPS_UNIT_SPLIT 8      // closure: frontiers above this many entries per warp use 32-entry units
#endif
#ifndef WB_EPS_UNIT_SHIFT
#define WB_EPS_UNIT_SHIFT 3      // ... else units of 1 << this entries
#endif
#ifndef WB_NB
#define WB_NB 2048
#endif
constexpr int NB = WB_NB;            // prune histogram buckets
constexpr int GCAP = 1024;           // boundary-bucket members ranked in shared memory
constexpr int ROW_SMEM_MAX = 16384;  // cost-row columns staged in shared memory (128 KB)
constexpr u32 F_SURV = 1u, F_MARK = 2u, CA_NONE = 0xFFFFFFFFu;
constexpr int MAX_EPS_ROUNDS = 1 << 20;
constexpr long long STREAM_WAIT_CYCLES = 60ll * 2000000000ll;  // ~60 s at ~2 GHz
// Capacity failures carry their cause above the status byte (reported as capacity_flags)
__host__ __device__ constexpr int wb_cap(int cause) { return WB_ERR_CAPACITY | (cause << 8); }
// relaxations in flight per lane (expand) / gathers per thread (prune): halved for 1024-thread
// CTAs, whose register budget is 64 per thread
#ifndef WB_UNROLL_1024
#define WB_UNROLL_1024 1
#endif
#ifndef WB_GATHER_P1_1024
#define WB_GATHER_P1_1024 2
#endif
#ifndef WB_GATHER_1024
#define WB_GATHER_1024 2
#endif
// CTAs per SM the 512-thread variant is compiled for (2: two lanes per SM at 64 registers)
#ifndef WB_MINB_512
#define WB_MINB_512 1
#endif
#ifndef WB_MINB_256
#define WB_MINB_256 1
#endif
// The step's phase functions are compiled into the kernel body: as separate calls, every
// value live across a call was spilled around it under the 64-register budget and the
// callees read the kernel parameters through generic pointers (config 2: 97.3 ms as calls,
// 87.2 ms inlined).  WB_PHASE_NOINLINE restores the calls (experiments).
#ifdef WB_PHASE_NOINLINE
#define WB_PHASE_FN __noinline__
#else
#define WB_PHASE_FN __forceinline__
#endif
// the lattice recorder's step and trim functions (lattice mode only): inlined as well
// (config 3: 529 -> 518 ms); WB_LATTICE_NOINLINE restores the calls
#ifdef WB_LATTICE_NOINLINE
#define WB_LATTICE_FN __noinline__
#else
#define WB_LATTICE_FN __forceinline__
#endif

template <int BLOCK> struct Tune {
    static constexpr int MINB = BLOCK == 512 ? WB_MINB_512 : BLOCK == 256 ? WB_MINB_256 : 1;
    static constexpr bool R64 = BLOCK * MINB >= 1024;  // 64-register budget
    static constexpr int UNROLL = R64 ? WB_UNROLL_1024 : 4;
    static constexpr int GATHER = R64 ? WB_GATHER_1024 : 4;
    static constexpr int GATHER_P1 = R64 ? WB_GATHER_P1_1024 : 4;  // slot exchange pass
};

struct GraphDev {
    int S, A, start, has_eps;
    int4 start_rng;         // {eps_lo, eps_hi (= emit_lo), emit_hi, 0} of the start state
    const int4 *arcs;       // [2*A]: {dst, ilabel, w_lo, w_hi}, {d_eps_lo, d_emit_lo, d_emit_hi, olabel}
    const double *final_w;  // [S] (+inf = not final)
    int nonneg;             // every arc weight >= 0 (enables the in-expand beam skip)
};

struct WorkDev {
    Slot *slot;           // [slots][S]   recombination slots (EMPTY between steps)
    u64 *cand_of;         // [slots][S]   state -> step stamp << 32 | candidate index (epsilon
                          //              graphs; one store, so a reader sees both or neither)
    u32 *qtag;            // [slots][S]   epsilon frontier dedup tags
    u32 *tag_ctr;         // [slots]
    u32 *cand_state;      // [slots][cap]
    u64 *cand_ap;       // candidate winner (arc + 1) | payload << 32: a slot's high word
    u64 *cand_key;        // [slots][cap] (used when a step overflows shared memory)
    u32 *cand_ca;         // [slots][cap]
    u32 *front;           // [slots][2][cap] frontier states / pending record list
    int4 *frng;           // [slots][2][cap] frontier entry {candidate index | CA_NONE, eps_lo, eps_hi, 0}
    int eps_dedup;        // epsilon frontier: drop repeated pushes of a state within a round
    int ma_early;         // expand: max-active early cutoff (cheaper tokens first, see expand)
    int force_radix;      // prune: radix-select every boundary bucket (test knob, WB_FORCE_RADIX)
    int row_prefetch;     // cost table in device memory: pull the next step's row into L2 early
    // ---- checked build (-DWB_CHECKS, libwfstb200_checked.so): device invariants in place of
    // the reference's ClaimLedger / debug_epoch (parallel.py:41-61, 92-116)
    u32 *chk_claim;       // [CTA slots][cap] expansions of each live token this step (must be 1)
    u32 *chk_seen;        // [slots][S] registrations of each state this step (must be <= 1)
    unsigned long long *chk_err;  // [slots] first violation: code << 32 | source line
    unsigned short *chk_log;      // [slots][chk_log_cap] group (warp) that expanded each token
    long long chk_log_cap;
    int *chk_steps;       // [slots][T_cap + 1] live tokens of each search step (claim ledger)
    int chk_inject;       // test knob: leave one slot un-reset (the stale-slot check must fire)
    int K, kshift;        // CTAs per utterance lane (a thread-block cluster of K = 1 << kshift);
                          // CTA rank r owns candidate / frontier indices [r*cap, (r+1)*cap)
    int lcap;             // K * cap: a lane's candidate / token / frontier capacity
    int4 *tok_info;       // [slots][2][cap] {state, trace, emit_lo, emit_hi}
    double *tok_cost;     // [slots][2][cap]
    int *frames;          // [slots][T_cap]
    u64 *arena;           // [slots][arena_cap] backpointer records (arcp1 | prev << 32), reused
                          // per utterance (the lane backtraces before taking the next one)
    u64 arena_cap;
    u32 *utt_ctr;
    long long S;
    int cap, T_cap, smem_cands, row_in_smem;
    int stage_off;        // dyn-smem byte offset of the per-lane arc prefetch buffers (0 = off)
    int log_rows;         // the cost rows hold log(p): negated as they are read (rows staged)
    int beam_skip;        // expand skips relaxations provably outside the beam
    int exact_min;        // token-filtered exact emitting-minimum pass (needs a non-negative row)
    int xchg_gather;      // gather reads and resets each slot with one 128-bit atomic exchange
                          // (2: with an L2 evict-first policy -- the line is dead until the
                          // state's next touch; 0: load + store)
    // ---- lattice recording (LatticeRecorder / build_lattice, lattice.py:96-249)
    int *tok_eps;         // [slots][2][cap] epsilon-range start of each token's state
    u32 *sbits;           // [slots][ceil(S/32)] survivor bitmap of the current node step (L2-resident)
    u32 *snode;           // [slots][S] node index of a survivor state
    int4 *rlog;           // [slots][rlog_cap] this step's finite emitting relaxations
                          // {token, arc, dst, ilabel} (logged by expand, filtered by record)
    long long rlog_cap;
    u32 *ln_state;        // [slots][lat_cap] raw lattice nodes (state), step-major
    unsigned char *ln_flag;  // [slots][lat_cap] trim flags (forward / backward reach)
    u32 *ln_out;          // [slots][lat_cap] output index of a kept node
    u32 *la_src, *la_dst, *la_arc;  // [slots][lat_cap] raw arcs: src / dst node, wfst arc
    double *la_ac;        // [slots][lat_cap] acoustic cost of a raw arc (0 for epsilon)
    long long lat_cap;
    int4 *lstep;          // [slots][T_cap + 2] {node_base, arc_base, n_nodes, n_emit | n_eps << 0}
    int *lstep_eps;       // [slots][T_cap + 2] epsilon arcs of the step (after its emitting arcs)
    int *lstep_start;     // [slots] step-local index of the start node in step 0
    // trimmed lattice output (global pools, one reservation per utterance)
    int2 *o_node;         // {state, step}
    uint4 *o_arc;         // {from, to, wfst arc, 0} (utterance-local node ids)
    double *o_ac;         // acoustic cost of o_arc
    u32 *o_fin;           // final node (utterance-local)
    double *o_finw;       // its final weight
    long long o_node_cap, o_arc_cap, o_fin_cap;
    unsigned long long *o_ctr;  // [3] node / arc / final reservations
    long long *o_meta;    // [n_utts][6] node_off, n_nodes, arc_off, n_arcs, fin_off, n_fin
};

struct BatchDev {
    const double *costs;
    const long long *row_off;
    const int *T;
    const double *blank;
    int L1, n;
    int *olab, *ilab;  // [n][lab_cap] best-path labels
    int lab_cap;
    const int *ready;  // streaming: frames of utterance u whose cost rows the host has written
                       // (page-locked, mapped); null = all rows present
    const long long *crow_off;  // streaming LSD: rows hold only the searched (non-blank) frames,
                                // utterance u's step s at row crow_off[u] + s; null = by frame
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
    int n_cand, overflow, utt, ng, thr_bucket, thr_below, n_pend;
    int flag, lat_bad;  // lattice sweeps: change flag / output-pool overflow
    int n_log;          // relaxations logged this step (lattice mode)
    u64 run_min;        // smallest emitting relaxation key seen so far this step
    int best_tok;       // a live token of minimal cost (its arcs seed run_min); -1 = unknown
    u64 best_rng;       // its emitting arc range emit_hi << 32 | emit_lo (one 64-bit store)
    u64 best_key;       // its cost key (the step's minimum)
    int next_chunk;     // expand: next unclaimed 32-token chunk (warps claim chunks dynamically)
    int ready_seen;     // streaming: last ready count read for the current utterance
    int pflags;         // WB_PATH_* bits of the current utterance (thread 0 writes)
    // cluster lanes (K > 1): per-CTA values the other CTAs of the lane read through DSMEM
    // after a cluster barrier
    int nfr[2];         // epsilon frontier entries pushed for round parity 0 / 1
    u64 x_mn, x_mx;     // this CTA's candidate key min / max (prune)
    int x_n, x_flags;   // this CTA's candidates this step; bit 0 overflow, bit 1 keys in global
    int x_gn;           // rank 0: boundary-bucket members collected from the lane's CTAs
    int x_stream;       // this CTA timed out waiting for a streamed cost row (cluster lanes)
    long long chk_off;  // checked build: this step's offset in the lane's claim log
    u32 ls_flag[8];     // lane barrier: epoch of the last barrier each peer CTA arrived at
    u32 ls_epoch;       // lane barriers passed by this CTA
    int x_ck, x_cs;     // kept / surviving candidates of this CTA (compaction bases)
    int x_eps_rounds;   // epsilon-closure rounds this CTA ran this step
    u32 stamp;          // this step's stamp in cand_of (the lane's dedup tag at the step start)
    u64 x_run_min;      // this CTA's exact emitting minimum (expand)
    // per-utterance counters kept out of the step loop's registers (with the 64-register
    // budget every value live across the phase calls was spilled around each call)
    unsigned long long cnt[4];  // a_emit, a_fin, a_cas, e_eps: warp-aggregated shared atomics
    long long acc[5];           // thread 0: tokens expanded, candidates, survivors, records, eps rounds
    double tok_lo, tok_hi;  // cost range of the current live tokens (from the last prune)
    float ma_frac;          // max-active early cutoff: split point in [tok_lo, tok_hi]
    u64 ma_thr;             // its bound key for the step
    u64 thr_key;
    u32 thr_state;
    u64 arena_base;
    u64 arena_used;    // records of the lane's current utterance
    long long pc[8];   // phase cycle counters (thread 0)
    long long t_mark;  // last phase boundary (thread 0)
#ifdef WB_PROBE
    long long spin_acc, spin_ph[8];  // probe build: lane-barrier wait cycles of thread 0 per phase
#endif
    union {
        u32 hist[NB];
        struct {
            u64 key[GCAP];
            u32 st[GCAP];
        } g;
    } u;
};

// Dynamic shared memory: [Smem header | cost row (expansion) / candidate keys + flags (prune)]
__device__ __forceinline__ unsigned char *dyn_smem() {
    extern __shared__ __align__(128) unsigned char s_dyn[];
    return s_dyn;
}
template <int BLOCK>
__host__ __device__ constexpr size_t smem_hdr() { return (sizeof(Smem<BLOCK>) + 127) & ~(size_t)127; }
template <int BLOCK>
__device__ __forceinline__ Smem<BLOCK> &SH() { return *reinterpret_cast<Smem<BLOCK> *>(dyn_smem()); }
template <int BLOCK>
__device__ __forceinline__ double *s_row() { return reinterpret_cast<double *>(dyn_smem() + smem_hdr<BLOCK>()); }
template <int BLOCK>
__device__ __forceinline__ u64 *s_key() { return reinterpret_cast<u64 *>(dyn_smem() + smem_hdr<BLOCK>()); }
template <int BLOCK>
__device__ __forceinline__ u32 *s_ca(const WorkDev &ws) {
    return reinterpret_cast<u32 *>(dyn_smem() + smem_hdr<BLOCK>() + sizeof(u64) * (size_t)ws.smem_cands);
}

// Phase timing: thread 0 charges the cycles since the previous mark to phase `ph`.  Called
// right after a barrier, so the time is the CTA's wall time for the phase.
template <int BLOCK>
__device__ __forceinline__ void tick(int ph) {
    Smem<BLOCK> &sh = SH<BLOCK>();
    if (threadIdx.x == 0) {
        long long t = clock64();
        sh.pc[ph] += t - sh.t_mark;
        sh.t_mark = t;
#ifdef WB_PROBE
        sh.spin_ph[ph] += sh.spin_acc;
        sh.spin_acc = 0;
#endif
    }
}

// ------------------------------------------------------------------ cluster lanes (see below)
// With K > 1 an utterance lane is a thread-block cluster: the K CTAs (on K SMs of one GPC)
// split every per-step phase and meet at cluster barriers; per-CTA partial results are read
// by the others straight from their shared memory (DSMEM, mapa).  K == 1 is the plain CTA.
__device__ __forceinline__ int cta_rank() {
    u32 r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return (int)r;
}
// The hardware cluster barrier with acquire semantics (barrier.cluster.wait) invalidates the
// whole L1 (CCTL.IVALL): spilled registers, cached arc records and token data all miss
// afterwards.  Used once, at kernel start; the per-phase barriers are lane_sync below.
__device__ __forceinline__ void cluster_sync_full() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// The same shared-memory object in CTA `rank` of this cluster (generic address into DSMEM).
template <class T>
__device__ __forceinline__ T *peer(T *p, int rank) {
    return cooperative_groups::this_cluster().map_shared_rank(p, (unsigned)rank);
}

// Loads of global data another CTA of the lane wrote in an earlier phase: L2 (the per-phase
// lane barrier does not invalidate this SM's L1).  Plain loads with one CTA per lane.
template <int KC, class T>
__device__ __forceinline__ T ldx(const T *p) {
    if constexpr (KC > 1) return __ldcg(p);
    else return *p;
}

// ------------------------------------------------------------------ checked build
// WB_CHECK(cond, code) records the first violated invariant of a lane; the host turns it into
// an AssertionError (like the reference's ClaimLedger.verify_partitions / debug_epoch).
enum : int {
    CHK_CLAIM = 1,       // a live token was expanded zero or several times in a step
    CHK_DUP = 2,         // a state was registered as a candidate twice in a step
    CHK_STALE = 3,       // a touched slot was not reset at the end of its step
    CHK_STALE_UTT = 4,   // a slot was left non-empty at the end of an utterance
    CHK_BOUNDS = 5,      // an index outside its workspace array
};
#ifdef WB_CHECKS
#define WB_CHECK(ws, cond, code) \
    do { if (!(cond)) check_fail((ws), (code), __LINE__); } while (0)
#else
#define WB_CHECK(ws, cond, code) do { } while (0)
#endif
__device__ __noinline__ void check_fail(const WorkDev &ws, int code, int line) {
    atomicCAS(&ws.chk_err[blockIdx.x >> ws.kshift], 0ull,
              ((unsigned long long)code << 32) | (unsigned)line);
}

// Barrier of every thread of every CTA of a lane.  With K > 1: a flag handshake through
// distributed shared memory between the CTAs' thread 0s, bracketed by CTA barriers, instead of
// barrier.cluster (whose acquire invalidates L1).  `global`: each thread first releases its
// global-memory writes (fence.release, MEMBAR.GPU without an L1 invalidation); the readers of
// such data in other CTAs load it from L2 (ldx).  Shared-memory data needs no fence: it is
// read in place through DSMEM after the handshake.
template <int BLOCK>
__device__ __forceinline__ void lane_sync(int K, bool global = true) {
    if (K == 1) {
        __syncthreads();
        return;
    }
    if (global) asm volatile("fence.release.cluster;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        Smem<BLOCK> &sh = SH<BLOCK>();
        const u32 e = ++sh.ls_epoch;
        const int r = cta_rank();
        for (int q = 0; q < K; ++q)
            if (q != r) *(volatile u32 *)&peer(&sh, q)->ls_flag[r] = e;
#ifdef WB_PROBE
        const long long t0 = clock64();
#endif
        for (int q = 0; q < K; ++q)
            if (q != r)
                while ((int)(*(volatile u32 *)&sh.ls_flag[q] - e) < 0) { }
#ifdef WB_PROBE
        sh.spin_acc += clock64() - t0;
#endif
    }
    __syncthreads();
}

// ------------------------------------------------------------------ block primitives
template <int BLOCK>
__device__ __forceinline__ void block_minmax(u64 &mn, u64 &mx) {
    Smem<BLOCK> &sh = SH<BLOCK>();
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
__device__ __forceinline__ void count_add(int q, u32 v) {
    v = __reduce_add_sync(FULL, v);   // one shared atomic per warp
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&SH<BLOCK>().cnt[q], (unsigned long long)v);
}
template <int BLOCK>
__device__ __forceinline__ void acc_add(int q, long long v) {
    if (threadIdx.x == 0) SH<BLOCK>().acc[q] += v;
}
template <int BLOCK>
__device__ __forceinline__ long long block_sum(long long v) {
    Smem<BLOCK> &sh = SH<BLOCK>();
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
    // Stateless accessor: pointers into this CTA's workspace are recomputed from the kernel
    // parameters on use (constant-bank loads + one IMAD) instead of living in registers or
    // on the stack across the persistent loop.
    const WorkDev &ws;
    // the lane of this CTA: a cluster of K CTAs shares one lane's workspace
    __device__ __forceinline__ size_t lane() const { return (size_t)(blockIdx.x >> ws.kshift); }
    __device__ __forceinline__ size_t so() const { return lane() * (size_t)ws.S; }
    __device__ __forceinline__ size_t co() const { return lane() * (size_t)ws.lcap; }
    __device__ __forceinline__ Slot *slot() const { return ws.slot + so(); }
    __device__ __forceinline__ u64 *cand_of() const { return ws.cand_of + so(); }
    __device__ __forceinline__ u32 *qtag() const { return ws.qtag + so(); }
    __device__ __forceinline__ u32 *cand_state() const { return ws.cand_state + co(); }
    __device__ __forceinline__ u64 *cand_ap() const { return ws.cand_ap + co(); }
    __device__ __forceinline__ u64 *cand_key() const { return ws.cand_key + co(); }
    __device__ __forceinline__ u32 *cand_ca() const { return ws.cand_ca + co(); }
    __device__ __forceinline__ u32 *front(int k) const { return ws.front + 2 * co() + (size_t)k * ws.lcap; }
    __device__ __forceinline__ int4 *frng(int k) const { return ws.frng + 2 * co() + (size_t)k * ws.lcap; }
    __device__ __forceinline__ int4 *tok_info(int k) const {
        return ws.tok_info + 2 * co() + (size_t)k * ws.lcap;
    }
    __device__ __forceinline__ double *tok_cost(int k) const {
        return ws.tok_cost + 2 * co() + (size_t)k * ws.lcap;
    }
    __device__ __forceinline__ int *frames() const { return ws.frames + lane() * ws.T_cap; }
    __device__ __forceinline__ u64 *arena() const { return ws.arena + lane() * ws.arena_cap; }
};



// Warp-cooperative candidate registration (call with the whole warp converged).  Lanes with
// `first` set installed the first entry of state `d` this step; they get consecutive
// candidate indices from one shared-memory atomic per warp.  `rng` = the state's
// {eps_lo, emit_lo, emit_hi} from the arc record.  Epsilon graphs: states with epsilon arcs
// record their candidate index (frontier lookups) and, if `push`, join the frontier.
// Candidate indices of CTA rank r are r*capK + (its local count): appends stay CTA-local.
// Frontier pushes go to this CTA's frontier region (`front_out`, counter `*nfront`).
template <int BLOCK>
__device__ __forceinline__ int warp_append(bool first, u32 d, int4 rng, bool push,
                                           const GraphDev &g, const WorkDev &ws,
                                           u32 *front_out, int4 *frng_out, int *nfront, int cbase) {
    Smem<BLOCK> &sh = SH<BLOCK>();
    const Lane c{ws};
    const u32 m = __ballot_sync(FULL, first);
    if (!m) return -1;
    const int l = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (l == leader) base = atomicAdd(&sh.n_cand, __popc(m));
    base = __shfl_sync(FULL, base, leader);
    const int loc = base + __popc(m & lanemask_lt());
    const int idx = cbase + loc;
    bool pf = false;
    if (first) {
        WB_CHECK(ws, loc >= ws.cap || (idx >= 0 && idx < ws.lcap), CHK_BOUNDS);
        if (loc < ws.cap) {
            c.cand_state()[idx] = d;
            if (g.has_eps && rng.x < rng.y) {
                c.cand_of()[d] = ((u64)sh.stamp << 32) | (u32)idx;
                pf = push;
            }
        } else {
            sh.overflow = 1;
        }
    }
    if (g.has_eps && push) {
        const u32 mf = __ballot_sync(FULL, pf);
        if (mf) {
            const int lf = __ffs(mf) - 1;
            int fb = 0;
            if (l == lf) fb = atomicAdd(nfront, __popc(mf));
            fb = __shfl_sync(FULL, fb, lf);
            if (pf) {
                const int f = fb + __popc(mf & lanemask_lt());
                front_out[f] = d;
                frng_out[f] = make_int4(idx, rng.x, rng.y, 0);
            }
        }
    }
    return (first && loc < ws.cap) ? idx : -1;
}

// Install `want` in *p under the (cost, arc) total order, optimistic first attempt already
// made (prev = value returned by a CAS that expected EMPTY).  Returns true if installed;
// *first = the slot was empty.
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

// Beam-skip pilot (one warp): the cheapest relaxation of live token `bt` against `row` lowers
// the step's running minimum, an upper bound of its best cost.
template <int BLOCK>
__device__ __forceinline__ void pilot_min(int bt, int cur, const double *row, const GraphDev &g,
                                          const WorkDev &ws, bool neg_row = false) {
    const int l = threadIdx.x & 31;
    // the token's arc range and cost as the compaction recorded them with best_tok
    const u64 br = *(volatile u64 *)&SH<BLOCK>().best_rng;
    const double tc = key_cost(SH<BLOCK>().best_key);
    u64 m = EMPTY_KEY;
    for (int a = (int)(u32)br + l; a < (int)(u32)(br >> 32); a += 32) {
        const int4 r = ld_arc(&g.arcs[2 * a]);
        const double ac = neg_row ? -row[r.y] : row[r.y];
        if (ac != INFINITY) {
            const u64 k = cost_key(__dadd_rn(__dadd_rn(tc, __hiloint2double(r.w, r.z)), ac));
            m = k < m ? k : m;
        }
    }
    m = warp_min_u64(m);
    if (l == 0 && m < *(volatile u64 *)&SH<BLOCK>().run_min)
        atomicMin(reinterpret_cast<unsigned long long *>(&SH<BLOCK>().run_min), m);
}

// Emitting expansion of all live tokens (viterbi_step's emitting loop, decoder.py:212-225;
// parallel form parallel.py:257-283).  Per lane, UNROLL relaxations are in flight: their arc
// loads, then their CAS attempts (optimistically expecting an empty slot -- most relaxations
// are first touches), are issued back to back.
struct ExpandCounts {
    u32 a_emit, a_fin, a_cas;
};

__device__ __forceinline__ int bucket_of(double cst, double best, double scale);

// Max-active early cutoff (exact).  Candidate costs only fall and the candidate set only grows
// during a step, so once >= max_active candidates are registered, the largest first-install key
// among the max_active cheapest of them bounds the step's final max-active cutoff from above
// (decoder.py:188-191 keeps the first max_active by (cost, state)): a relaxation costing more
// cannot survive, and with non-negative weights nothing reached from it by epsilon arcs can.
// Called between the two token passes of expand_emitting; returns the bound key (EMPTY_KEY =
// fewer than max_active candidates).  cand_key holds each candidate's first-install key.
template <int BLOCK>
__device__ __noinline__ u64 ma_bound(int max_active, const WorkDev &ws) {
    Smem<BLOCK> &sh = SH<BLOCK>();
    const Lane c{ws};
    const int n = min(sh.n_cand, ws.cap);
    if (n < max_active) return EMPTY_KEY;
    const u64 *ck = c.cand_key();
    u64 mn = EMPTY_KEY, mx = 0;
    for (int i = threadIdx.x; i < n; i += BLOCK) {
        const u64 k = ck[i];
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
    }
    block_minmax<BLOCK>(mn, mx);
    const double lo = key_cost(mn), hi = key_cost(mx);
    const double range = __dsub_rn(hi, lo);
    if (!(range > 0.0 && range < INFINITY)) return EMPTY_KEY;
    const double scale = __ddiv_rn((double)NB, range);
    for (int b = threadIdx.x; b < NB; b += BLOCK) sh.u.hist[b] = 0;
    if (threadIdx.x == 0) { sh.ma_thr = 0; sh.thr_bucket = NB - 1; }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += BLOCK) atomicAdd(&sh.u.hist[bucket_of(key_cost(ck[i]), lo, scale)], 1u);
    __syncthreads();
    constexpr int PER = NB / BLOCK;
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    u32 loc[PER], tot = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) { loc[q] = sh.u.hist[threadIdx.x * PER + q]; tot += loc[q]; }
    const int incl = warp_incl_scan((int)tot);
    if (l == 31) sh.wa[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int v = l < NW ? sh.wa[l] : 0;
        const int iv = warp_incl_scan(v);
        if (l < NW) sh.wa[l] = iv - v;
    }
    __syncthreads();
    u32 run = sh.wa[w] + incl - tot;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        if (run < (u32)max_active && run + loc[q] >= (u32)max_active) sh.thr_bucket = threadIdx.x * PER + q;
        run += loc[q];
    }
    __syncthreads();
    const int bstar = sh.thr_bucket;
    u64 m = 0;
    for (int i = threadIdx.x; i < n; i += BLOCK) {
        const u64 k = ck[i];
        if (bucket_of(key_cost(k), lo, scale) <= bstar && k > m) m = k;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const u64 x = __shfl_xor_sync(FULL, m, o);
        m = x > m ? x : m;
    }
    if (l == 0 && m) atomicMax(reinterpret_cast<unsigned long long *>(&sh.ma_thr), (unsigned long long)m);
    __syncthreads();
    return sh.ma_thr ? sh.ma_thr : EMPTY_KEY;
}

#ifdef WB_CHECKS
// Claim-ledger analogue: count the expansions of live token t and log the expanding group
// (warp) at the step's offset in the lane's claim log.
template <int BLOCK>
__device__ __forceinline__ void claim_token(const WorkDev &ws, int t, int group) {
    const size_t ln = blockIdx.x >> ws.kshift;
    WB_CHECK(ws, t >= 0 && t < ws.lcap, CHK_BOUNDS);
    atomicAdd(&ws.chk_claim[ln * ws.lcap + t], 1u);
    const long long at = SH<BLOCK>().chk_off + t;
    if (at < ws.chk_log_cap) ws.chk_log[ln * ws.chk_log_cap + at] = (unsigned short)group;
}
#endif

template <int BLOCK, int KC>
WB_PHASE_FN __device__ ExpandCounts expand_emitting(int n_live, int cur, const double *row,
                                                     const GraphDev &g, const WorkDev &ws,
                                                     double beam, bool row_nonneg, bool piloted,
                                                     int max_active) {
    const Lane c{ws};
    u32 a_emit = 0, a_fin = 0, a_cas = 0;
    constexpr int NW = BLOCK / 32;
    constexpr int U = Tune<BLOCK>::UNROLL;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int4 *__restrict__ tinfo = c.tok_info(cur);
    const double *__restrict__ tcost = c.tok_cost(cur);
    Slot *slot = c.slot();
    // cluster lanes: this CTA expands the 32-token chunks ch = r + K * j (j = 0, 1, ...) and
    // registers its candidates / frontier pushes in its own index range
    constexpr int KS = KC >= 8 ? 3 : KC >= 4 ? 2 : KC >= 2 ? 1 : 0;
    const int r = KC > 1 ? cta_rank() : 0;
    const int cbase = r * ws.cap;
    u32 *front0 = c.front(0) + cbase;
    int4 *frng0 = c.frng(0) + cbase;
    int *nfr0 = &SH<BLOCK>().nfr[0];
    const int nchunks_all = (n_live + 31) >> 5;
    const int nchunks = (nchunks_all - r + KC - 1) >> KS;   // this CTA's chunks
    auto chunk_of = [&](int j) { return r + (j << KS); };
    const Slot empty = {EMPTY_KEY, 0xFFFFFFFFu, 0xFFFFFFFFu};
    if (ws.stage_off) {
        // Software-pipelined: each lane prefetches its next arc record into shared memory
        // (cp.async, no registers held) while its current relaxation's CAS is in flight, so an
        // iteration costs one memory round trip instead of two.  The two-deep ring is
        // buffer-major ([2][BLOCK] x 16 B): a warp's 16-byte reads are contiguous (4
        // wavefronts, no bank conflicts).  cp.async.cg: the records bypass L1 (config 4
        // 16.9 -> 16.7 ms, config 2 -0.2 %; L1 keeps the spills and the pilot's data).
        int4 *stage = reinterpret_cast<int4 *>(dyn_smem() + ws.stage_off) + threadIdx.x;
        const bool skip_on = g.nonneg && beam < INFINITY && ws.beam_skip;
        auto sh_run_min = [&]() -> u64 { return *(volatile u64 *)&SH<BLOCK>().run_min; };
        bool exact = false;
        if (skip_on) {
            // (1) pilot: evaluate (no CAS) the arcs of a cheapest live token, so the running
            // minimum -- an upper bound of the step's best cost -- is tight from the start
            const int bt = SH<BLOCK>().best_tok;
            if (!piloted) {  // (done by warp 0 during row staging when the row is staged)
                if (w == 0 && bt >= 0 && bt < n_live) pilot_min<BLOCK>(bt, cur, row, g, ws);
                __syncthreads();
            }
            // (2) exact minimum: with non-negative weights and acoustic costs a relaxation of
            // token t costs at least c_t, so only tokens cheaper than the pilot's minimum can
            // lower it -- usually a handful -- and the skip below then uses the step's final
            // cutoff from the first relaxation on
            if (ws.exact_min && row_nonneg && n_live >= 1024) {  // (small steps: pilot only)
                exact = true;
                const u64 rm0 = sh_run_min();
                const double bound = rm0 == EMPTY_KEY ? INFINITY : key_cost(rm0);
                u64 m = EMPTY_KEY;
                for (int ch0 = w; ch0 < nchunks; ch0 += 2 * NW) {
                  // token costs of two chunks in flight; token records only where a token passes
                  double tcs[2];
#pragma unroll
                  for (int q = 0; q < 2; ++q) {
                    const int t = (chunk_of(ch0 + q * NW) << 5) + l;
                    tcs[q] = (ch0 + q * NW < nchunks && t < n_live) ? ldx<KC>(&tcost[t]) : INFINITY;
                  }
#pragma unroll
                  for (int q = 0; q < 2; ++q) {
                    const int t = (chunk_of(ch0 + q * NW) << 5) + l;
                    const double tc = tcs[q];
                    const bool pass = tc < bound && t != bt;
                    if (!__any_sync(FULL, pass)) continue;
                    int4 ti = make_int4(0, 0, 0, 0);
                    if (pass) ti = ldx<KC>(&tinfo[t]);
                    const int deg = pass ? ti.w - ti.z : 0;
                    const int incl = warp_incl_scan(deg);
                    const int total = __shfl_sync(FULL, incl, 31);
                    const int excl = incl - deg;
                    for (int j0 = 0; j0 < total; j0 += 32) {
                        const int j = j0 + l;
                        const int k = warp_owner(excl, j);
                        const int arc = __shfl_sync(FULL, ti.z, k) + j - __shfl_sync(FULL, excl, k);
                        const double cst = __shfl_sync(FULL, tc, k);
                        if (j < total) {
                            const int4 r = ld_arc(&g.arcs[2 * arc]);
                            const double ac = row[r.y];
                            if (ac != INFINITY) {
                                const u64 kk = cost_key(__dadd_rn(__dadd_rn(cst, __hiloint2double(r.w, r.z)), ac));
                                m = kk < m ? kk : m;
                            }
                        }
                    }
                  }
                }
                m = warp_min_u64(m);
                if (l == 0 && m < sh_run_min()) atomicMin(reinterpret_cast<unsigned long long *>(&SH<BLOCK>().run_min), m);
                // a cluster lane's CTAs each saw their own tokens: the lane's exact minimum is
                // the minimum over the CTAs (run_min is not written again this step)
                lane_sync<BLOCK>(KC, false);   // run_min: shared memory only
                if (KC > 1) {
                    u64 lm = sh_run_min();
                    for (int q = 1; q < KC; ++q) {
                        const u64 o = *(volatile u64 *)&peer(&SH<BLOCK>(), (r + q) & (KC - 1))->run_min;
                        lm = o < lm ? o : lm;
                    }
                    if (threadIdx.x == 0) SH<BLOCK>().x_run_min = lm;
                    __syncthreads();
                }
            }
        }
        // the final cutoff key when the exact minimum is known (EMPTY_KEY: running bound)
        u64 exact_thr = EMPTY_KEY;
        if (exact) {
            const u64 rm = KC > 1 ? SH<BLOCK>().x_run_min : sh_run_min();
            if (rm != EMPTY_KEY) exact_thr = cost_key(__dadd_rn(key_cost(rm), beam));
        }
        const u32 s0 = (u32)__cvta_generic_to_shared(stage);
        // max-active early cutoff: pass 0 expands the tokens up to a split cost, ma_bound
        // turns the candidates it registered into a bound, pass 1 expands the rest against it
        const bool ma_on = ws.ma_early > 0 && n_live >= ws.ma_early && max_active > 0 && !ws.rlog &&
                           g.nonneg && ws.beam_skip && KC == 1;
        u64 ma_thr = EMPTY_KEY;
        double split = INFINITY;
        if (ma_on) {
            const Smem<BLOCK> &sh = SH<BLOCK>();
            split = __dadd_rn(sh.tok_lo, (double)sh.ma_frac * __dsub_rn(sh.tok_hi, sh.tok_lo));
        }
        for (int pass = 0; pass < (ma_on ? 2 : 1); ++pass) {
        if (pass == 1) {
            __syncthreads();  // pass 0's registrations and first-install keys are visible
            const u64 mb = ma_bound<BLOCK>(max_active, ws);
            if (threadIdx.x == 0) {
                Smem<BLOCK> &sh = SH<BLOCK>();
                sh.ma_frac = mb != EMPTY_KEY ? fmaxf(0.05f, sh.ma_frac - 0.02f) : fminf(1.0f, sh.ma_frac + 0.1f);
                sh.next_chunk = NW;
            }
            ma_thr = mb;
            __syncthreads();
        }
        // warps claim work units dynamically (first unit = warp id): 32-token chunks, except
        // that the last NW chunks are claimed as 8-token quarters, so the warps run out of work
        // within about a quarter chunk of each other at the closing barrier
        const int nbig = max(0, nchunks - NW);
        const int nunits = nbig + 4 * (nchunks - nbig);
        for (int lc = w; lc < nunits;) {
            int ch_claim = 0;
            if (l == 0) ch_claim = atomicAdd(&SH<BLOCK>().next_chunk, 1);  // used after this unit
            const int qv = lc - nbig;
            const int ch = chunk_of(lc < nbig ? lc : nbig + (qv >> 2));
            const int tlo = lc < nbig ? 0 : (qv & 3) << 3;   // the unit's first token in the chunk
            const int t = (ch << 5) + tlo + l;
            int4 ti = make_int4(0, 0, 0, 0);
            double tc = 0.0;
            if (t < n_live && (lc < nbig || l < 8)) { ti = ldx<KC>(&tinfo[t]); tc = ldx<KC>(&tcost[t]); }
            const bool in_pass = !ma_on || ((tc <= split) == (pass == 0));
            const bool mine = t < n_live && (lc < nbig || l < 8) && in_pass;
            const int deg = mine ? ti.w - ti.z : 0;
#ifdef WB_CHECKS
            if (mine) claim_token<BLOCK>(ws, t, r * NW + w);
#endif
            a_emit += deg;
            const int incl = warp_incl_scan(deg);
            const int total = __shfl_sync(FULL, incl, 31);
            const int excl = incl - deg;
            auto arc_of = [&](int j, int &k) {
                k = warp_owner(excl, j);
                return __shfl_sync(FULL, ti.z, k) + j - __shfl_sync(FULL, excl, k);
            };
            int k_next, arc_next = arc_of(l, k_next);
            if (l < total)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s0), "l"(&g.arcs[2 * arc_next]));
            constexpr u32 RING = 16u * BLOCK;  // byte distance between the two ring buffers
            asm volatile("cp.async.commit_group;");
            for (int j0 = 0, it = 0; j0 < total; j0 += 32, ++it) {
                const int j = j0 + l, k = k_next, arc = arc_next;
                if (j0 + 32 < total) {  // prefetch the next iteration's record
                    arc_next = arc_of(j + 32, k_next);
                    if (j + 32 < total)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s0 + RING * ((it + 1) & 1)),
                                     "l"(&g.arcs[2 * arc_next]));
                }
                asm volatile("cp.async.commit_group;");
                asm volatile("cp.async.wait_group 1;" ::: "memory");
                const double cst = __shfl_sync(FULL, tc, k);
                Slot want;
                want.pay = (u32)__shfl_sync(FULL, ti.y, k);
                want.arcp1 = (u32)arc + 1u;
                bool act = j < total;
                int4 rec = make_int4(0, 0, 0, 0);
                if (act) {
                    rec = stage[(it & 1) * BLOCK];
                    const double ac = row[rec.y];
                    if (ac == INFINITY) {  // decoder.py:219-220: no relaxation, no record
                        act = false;
                    } else {
                        want.key = cost_key(__dadd_rn(__dadd_rn(cst, __hiloint2double(rec.w, rec.z)), ac));
                    }
                }
                if (ws.rlog) {  // lattice mode: log the finite relaxations for record_lattice_step
                    const u32 m = __ballot_sync(FULL, act);
                    if (m) {
                        int base = 0;
                        if (l == __ffs(m) - 1) base = atomicAdd(&SH<BLOCK>().n_log, __popc(m));
                        base = __shfl_sync(FULL, base, __ffs(m) - 1);
                        const long long e = base + __popc(m & lanemask_lt());
                        if (act && e < ws.rlog_cap)
                            ws.rlog[(size_t)blockIdx.x * ws.rlog_cap + e] =
                                make_int4((ch << 5) + tlo + k, arc, rec.x, rec.y);
                    }
                }
                bool first = false, dec = false;
                bool relax = act;
                if (exact_thr != EMPTY_KEY) {
                    // Beam skip (exact) against the step's final cutoff best + beam
                    // (decoder.py:186): such a state cannot survive and, with non-negative
                    // weights, nothing reached from it can either.  The lattice log above
                    // still records it.
                    relax = act && want.key <= exact_thr;
                } else if (skip_on) {
                    // same skip against a running bound: the step's best cost is at most the
                    // smallest key seen so far
                    const u64 wm = warp_min_u64(act ? want.key : EMPTY_KEY);
                    if (l == 0 && wm < sh_run_min()) atomicMin(reinterpret_cast<unsigned long long *>(&SH<BLOCK>().run_min), wm);
                    const u64 rm = sh_run_min();
                    if (relax && rm != EMPTY_KEY && want.key > cost_key(__dadd_rn(key_cost(rm), beam)))
                        relax = false;
                }
                if (want.key > ma_thr) relax = false;  // max-active early cutoff (ma_bound)
                if (act) a_fin++;
                if (relax) {
                    a_cas++;
                    const Slot prev = cas_slot(&slot[rec.x], empty, want);
                    finish_relax(&slot[rec.x], want, prev, &first, &dec);
                }
                int4 r1 = make_int4(0, 0, 0, 0);
                if (first) r1 = __ldg(&g.arcs[2 * arc + 1]);
                const int ci = warp_append<BLOCK>(first, (u32)rec.x, r1, true, g, ws, front0, frng0, nfr0, cbase);
                if (ma_on && pass == 0 && ci >= 0) c.cand_key()[ci] = want.key;
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            lc = __shfl_sync(FULL, ch_claim, 0);
        }
        }
        return ExpandCounts{a_emit, a_fin, a_cas};
    }
    for (int lc = w; lc < nchunks; lc += NW) {
        const int ch = chunk_of(lc);
        int t = (ch << 5) + l;
        int4 ti = make_int4(0, 0, 0, 0);
        double tc = 0.0;
        if (t < n_live) { ti = ldx<KC>(&tinfo[t]); tc = ldx<KC>(&tcost[t]); }
        int deg = t < n_live ? ti.w - ti.z : 0;
#ifdef WB_CHECKS
        if (t < n_live) claim_token<BLOCK>(ws, t, r * NW + w);
#endif
        a_emit += deg;
        int incl = warp_incl_scan(deg);
        int total = __shfl_sync(FULL, incl, 31);
        int excl = incl - deg;
        for (int j0 = 0; j0 < total; j0 += 32 * U) {
            int4 rec[U];
            Slot want[U];
            bool act[U];
            int tk[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int j = j0 + u * 32 + l;
                int k = warp_owner(excl, j);
                tk[u] = (ch << 5) + k;
                int lo_k = __shfl_sync(FULL, ti.z, k);
                int ex_k = __shfl_sync(FULL, excl, k);
                double cst = __shfl_sync(FULL, tc, k);
                want[u].pay = (u32)__shfl_sync(FULL, ti.y, k);
                act[u] = j < total;
                int arc = lo_k + j - ex_k;
                want[u].arcp1 = (u32)arc + 1u;
                if (act[u]) rec[u] = ld_arc(&g.arcs[2 * arc]);
                want[u].key = __double_as_longlong(cst);  // carry the token cost
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!act[u]) continue;
                double ac = row[rec[u].y];
                if (ac == INFINITY) {  // decoder.py:219-220: no relaxation, no record
                    act[u] = false;
                    continue;
                }
                double wgt = __hiloint2double(rec[u].w, rec[u].z);
                double cst = __longlong_as_double((long long)want[u].key);
                want[u].key = cost_key(__dadd_rn(__dadd_rn(cst, wgt), ac));
            }
            if (ws.rlog) {  // lattice mode: log the finite relaxations for record_lattice_step
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const u32 m = __ballot_sync(FULL, act[u]);
                    if (!m) continue;
                    int base = 0;
                    if (l == __ffs(m) - 1) base = atomicAdd(&SH<BLOCK>().n_log, __popc(m));
                    base = __shfl_sync(FULL, base, __ffs(m) - 1);
                    const long long e = base + __popc(m & lanemask_lt());
                    if (act[u] && e < ws.rlog_cap)
                        ws.rlog[(size_t)blockIdx.x * ws.rlog_cap + e] =
                            make_int4(tk[u], (int)want[u].arcp1 - 1, rec[u].x, rec[u].y);
                }
            }
            Slot prev[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (act[u]) prev[u] = cas_slot(&slot[rec[u].x], empty, want[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                bool first = false, dec = false;
                if (act[u]) {
                    a_fin++;
                    a_cas++;
                    finish_relax(&slot[rec[u].x], want[u], prev[u], &first, &dec);
                }
                int4 r1 = make_int4(0, 0, 0, 0);
                if (first) r1 = __ldg(&g.arcs[2 * (want[u].arcp1 - 1u) + 1]);
                warp_append<BLOCK>(first, (u32)rec[u].x, r1, true, g, ws, front0, frng0, nfr0, cbase);
            }
        }
    }
    return ExpandCounts{a_emit, a_fin, a_cas};
}

// Epsilon closure to a fixpoint by frontier rounds (decoder.py:138-171; parallel.py:287-325).
// Self-loops are skipped (decoder.py:162-163).  An epsilon winner's payload is the candidate
// index of its source | EPS_BIT.  Frontier entries are states; their candidate index is looked
// up one round later, after the barrier has published it.
struct EpsOut {
    u32 tag, e_eps;
    int status, rounds;
};

template <int BLOCK, int KC>
WB_PHASE_FN __device__ EpsOut epsilon_closure(const GraphDev &g, const WorkDev &ws, u32 tag_in,
                                               double beam) {
    Smem<BLOCK> &sh = SH<BLOCK>();
    const Lane c{ws};
    // beam skip as in expand: with non-negative weights every candidate of this step costs at
    // least the emitting minimum, and run_min is an upper bound of it (this CTA's minimum), so
    // run_min + beam is at or above the step's final cutoff
    u64 rm = sh.run_min;
    for (int q = 1; q < KC; ++q) {   // the lane's minimum (expand ended with a lane barrier)
        const u64 o = *(volatile u64 *)&peer(&sh, (cta_rank() + q) & (KC - 1))->run_min;
        rm = o < rm ? o : rm;
    }
    const bool skip_on = g.nonneg && ws.beam_skip && beam < INFINITY && rm != EMPTY_KEY;
    const u64 thr = skip_on ? cost_key(__dadd_rn(key_cost(rm), beam)) : EMPTY_KEY;
    u32 tag_cur = tag_in, e_eps = 0;
    int status = WB_OK;
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    constexpr int K = KC;
    const int r = K > 1 ? cta_rank() : 0, cbase = r * ws.cap;
    Slot *slot = c.slot();
    const Slot empty = {EMPTY_KEY, 0xFFFFFFFFu, 0xFFFFFFFFu};
    int n_rounds = 0;
    // a candidate overflow anywhere in the lane leaves frontier states without a candidate
    // index: the step has failed (WB_CAP_CANDIDATES)
    auto lane_overflow = [&]() {
        int ovf = *(volatile int *)&sh.overflow;
        for (int q = 1; q < K; ++q) ovf |= *(volatile int *)peer(&sh.overflow, (r + q) & (K - 1));
        return ovf != 0;
    };
    // Round k consumes the frontier pushed in round k-1 (round 0: by expand) from buffer k & 1
    // and pushes into the other.  Each CTA of a cluster lane drains its own frontier region with
    // CTA barriers (a push always goes to the pusher's region, so no CTA can create work for
    // another); the lane meets once, after the last CTA is done.  Dedup tags are per CTA and
    // round (tag_in + 1 + rounds * K + rank), so one CTA's push never suppresses another's.
    for (int rounds = 0;; ++rounds) {
        const int par = rounds & 1;
        const int n_front = min(sh.nfr[par], ws.cap);  // overflowed pushes were dropped (flagged)
        n_rounds = rounds;
        if (n_front == 0) break;
        // stop before following stale indices
        if (lane_overflow()) { status = wb_cap(WB_CAP_CANDIDATES); break; }
        if (rounds >= MAX_EPS_ROUNDS) { status = wb_cap(WB_CAP_EPS_ROUNDS); break; }
        // the other buffer's count was last read before the barrier that ended the last round
        if (threadIdx.x == 0) sh.nfr[par ^ 1] = 0;
        __syncthreads();
        const u32 tag = tag_in + 1u + (u32)rounds * (u32)K + (u32)r;
        const u32 *fin = c.front(par) + cbase;
        u32 *fout = c.front(par ^ 1) + cbase;
        const int4 *frin = c.frng(par) + cbase;
        int4 *frout = c.frng(par ^ 1) + cbase;
        int *nfout = &sh.nfr[par ^ 1];
        // a small frontier (<= 8 entries per warp) is spread over more warps (units of 8
        // entries): a round's latency is one pass over a unit's epsilon arcs
        const int ush = n_front > WB_EPS_UNIT_SPLIT * NW ? 5 : WB_EPS_UNIT_SHIFT, usz = 1 << ush;
        const int nchunks = (n_front + usz - 1) >> ush;
        for (int ch = w; ch < nchunks; ch += NW) {
            int i = (ch << ush) + l;
            u32 uu = 0, ui = 0;
            int lo = 0, deg = 0;
            double ucost = 0.0;
            if (l < usz && i < n_front) {
                // the entry carries the state's epsilon range (and its candidate index when the
                // pusher knew it), so the arcs load alongside the slot
                uu = fin[i];
                const int4 fe = frin[i];
                Slot us = ld_slot(&slot[uu]);
                if (fe.x >= 0) {
                    ui = (u32)fe.x;
                } else {
                    // the state's candidate index, possibly registered by another CTA that has
                    // not published it yet: valid once it carries this step's stamp
                    for (;;) {
                        const u64 co = ldx<KC>(&c.cand_of()[uu]);
                        ui = min((u32)co, (u32)ws.lcap - 1u);
                        if ((u32)(co >> 32) == sh.stamp || lane_overflow()) break;
                    }
                }
                lo = fe.y;
                deg = fe.z - fe.y;
                ucost = key_cost(us.key);
            }
            int incl = warp_incl_scan(deg);
            int total_d = __shfl_sync(FULL, incl, 31);
            int excl = incl - deg;
            for (int j0 = 0; j0 < total_d; j0 += 32) {
                int j = j0 + l;
                int k = warp_owner(excl, j);
                int lo_k = __shfl_sync(FULL, lo, k);
                int ex_k = __shfl_sync(FULL, excl, k);
                double uc_k = __shfl_sync(FULL, ucost, k);
                u32 u_k = __shfl_sync(FULL, uu, k);
                u32 ui_k = __shfl_sync(FULL, ui, k);
                bool act = j < total_d;
                int a = lo_k + j - ex_k;
                int4 rec = make_int4(0, 0, 0, 0);
                if (act) {
                    rec = ld_arc(&g.arcs[2 * a]);
                    if ((u32)rec.x == u_k) act = false;  // a positive self-loop never improves its state
                }
                bool first = false, dec = false;
                if (act) {
                    e_eps++;
                    Slot want;
                    want.key = cost_key(__dadd_rn(uc_k, __hiloint2double(rec.w, rec.z)));
                    want.arcp1 = (u32)a + 1u;
                    want.pay = ui_k | EPS_BIT;
                    if (want.key <= thr) {
                        Slot prev = cas_slot(&slot[rec.x], empty, want);
                        finish_relax(&slot[rec.x], want, prev, &first, &dec);
                    }
                }
                int4 r1 = make_int4(0, 0, 0, 0);
                if (dec) r1 = __ldg(&g.arcs[2 * a + 1]);
                const int nidx = warp_append<BLOCK>(first, (u32)rec.x, r1, false, g, ws, fout, frout,
                                                    nfout, cbase);
                // states whose cost dropped (or that are new) re-relax their epsilon arcs
                bool push = dec && r1.x < r1.y &&
                            (!ws.eps_dedup || atomicExch(&c.qtag()[rec.x], tag) != tag);
                const u32 mp = __ballot_sync(FULL, push);
                if (mp) {
                    const int lp = __ffs(mp) - 1;
                    int fb = 0;
                    if (l == lp) fb = atomicAdd(nfout, __popc(mp));
                    fb = __shfl_sync(FULL, fb, lp);
                    int f = fb + __popc(mp & lanemask_lt());
                    if (push) {
                        if (f < ws.cap) {
                            fout[f] = (u32)rec.x;
                            frout[f] = make_int4(nidx, r1.x, r1.y, 0);  // nidx -1: look it up
                        } else {
                            sh.overflow = 1;
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    // every CTA's relaxations have landed before the gather; the next step's tags start above
    // every tag any CTA used
    if (threadIdx.x == 0) sh.x_eps_rounds = n_rounds;
    lane_sync<BLOCK>(K);
    int max_rounds = n_rounds;
    for (int q = 1; q < K; ++q)
        max_rounds = max(max_rounds, *(volatile int *)&peer(&sh, (r + q) & (K - 1))->x_eps_rounds);
    tag_cur = tag_in + (u32)(max_rounds + 1) * (u32)K;
    return EpsOut{tag_cur, e_eps, status, n_rounds};
}

__device__ __forceinline__ int bucket_of(double cst, double best, double scale) {
    double v = __dmul_rn(__dsub_rn(cst, best), scale);
    if (!(v < (double)(NB - 1))) return NB - 1;
    return (int)v;
}

// Exact max-active cut: K* = the max_active-th smallest (cost, state) among kept candidates
// (decoder.py:188-191).  Expects sh.u.hist filled with this CTA's candidates; rank 0 of a
// cluster lane merges the CTAs' histograms, finds the boundary bucket, collects its members
// from every CTA and ranks them.  Sets thr_bucket / thr_key / thr_state, returned uniformly.
struct Thr {
    int bucket;
    u64 key;
    u32 state;
};

template <int BLOCK, int KC>
WB_PHASE_FN __device__ Thr select_threshold(int n_loc, int max_active, double best, double cutoff,
                                             double scale, const u64 *ckey, const u32 *cst,
                                             const WorkDev &ws) {
    Smem<BLOCK> &sh = SH<BLOCK>();
    constexpr int PER = NB / BLOCK;
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    constexpr int K = KC;
    const int r = K > 1 ? cta_rank() : 0;
    Smem<BLOCK> &s0 = K > 1 ? *peer(&sh, 0) : sh;   // rank 0's header (itself when K == 1)
    if (K > 1) lane_sync<BLOCK>(K, false);                         // every CTA's histogram is complete
    if (r == 0) {
        if (threadIdx.x == 0) sh.thr_bucket = -1;   // stays -1: max-active does not bind
        u32 loc[PER];
        u32 s = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int b = threadIdx.x * PER + q;
            u32 v = sh.u.hist[b];
            for (int o = 1; o < K; ++o) v += peer(&sh, o)->u.hist[b];
            loc[q] = v;
            s += v;
        }
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
        if (threadIdx.x == 0) sh.x_gn = 0;   // boundary members collected below
    }
    lane_sync<BLOCK>(K, false);
    const int bstar = s0.thr_bucket;
    if (bstar < 0) return Thr{-1, 0, 0};  // at most max_active candidates within the beam
    if (r == 0 && threadIdx.x == 0) sh.pflags |= WB_PATH_SELECT;
    int rk = max_active - s0.thr_below;  // 1-based rank inside the boundary bucket
    const int cnt = s0.ng;
    if (cnt <= GCAP && !ws.force_radix) {
        for (int j = threadIdx.x; j < n_loc; j += BLOCK) {
            const u64 k = ckey[j];
            const double cs = key_cost(k);
            if (cs <= cutoff && bucket_of(cs, best, scale) == bstar) {
                const int q = atomicAdd(&s0.x_gn, 1);
                s0.u.g.key[q] = k;
                s0.u.g.st[q] = cst[j];
            }
        }
        lane_sync<BLOCK>(K, false);
        if (r == 0) {
            const int m = sh.x_gn;
            for (int j = threadIdx.x; j < m; j += BLOCK) {
                const u64 kj = sh.u.g.key[j];
                const u32 sj = sh.u.g.st[j];
                int rank = 0;
                for (int q = 0; q < m; ++q) {
                    const u64 kq = sh.u.g.key[q];
                    rank += (kq < kj || (kq == kj && sh.u.g.st[q] < sj)) ? 1 : 0;
                }
                if (rank == rk - 1) { sh.thr_key = kj; sh.thr_state = sj; }
            }
        }
        lane_sync<BLOCK>(K, false);
        // rank 0 writes thr_key / thr_state again only in the next step's select, many lane
        // barriers after these reads
        return Thr{bstar, s0.thr_key, s0.thr_state};
    }
    // radix select over the 96-bit (key, state) of the boundary-bucket members, MSB first;
    // per digit every CTA counts its members, rank 0 sums the counts and picks the digit
    if (threadIdx.x == 0) sh.pflags |= WB_PATH_RADIX;
    u64 kpre = 0, kmask = 0;
    u32 spre = 0, smask = 0;
    for (int dig = 0; dig < 12; ++dig) {
        for (int b = threadIdx.x; b < 256; b += BLOCK) sh.u.hist[b] = 0;
        __syncthreads();
        const bool in_key = dig < 8;
        const int shift = in_key ? (56 - 8 * dig) : (24 - 8 * (dig - 8));
        for (int j = threadIdx.x; j < n_loc; j += BLOCK) {
            const u64 k = ckey[j];
            const double cs = key_cost(k);
            if (!(cs <= cutoff) || bucket_of(cs, best, scale) != bstar) continue;
            const u32 st = cst[j];
            if ((k & kmask) != kpre || (st & smask) != spre) continue;
            const u32 d = in_key ? (u32)((k >> shift) & 0xFF) : ((st >> shift) & 0xFF);
            atomicAdd(&sh.u.hist[d], 1u);
        }
        lane_sync<BLOCK>(K, false);
        if (r == 0 && threadIdx.x == 0) {
            u32 acc = 0;
            int d = 0;
            for (; d < 256; ++d) {
                u32 h = sh.u.hist[d];
                for (int o = 1; o < K; ++o) h += peer(&sh, o)->u.hist[d];
                if (acc + h >= (u32)rk) break;
                acc += h;
            }
            sh.thr_below = (int)acc;
            sh.ng = d;
        }
        lane_sync<BLOCK>(K, false);
        rk -= s0.thr_below;
        const u32 d = (u32)s0.ng;
        if (in_key) { kpre |= (u64)d << shift; kmask |= 0xFFull << shift; }
        else { spre |= d << shift; smask |= 0xFFu << shift; }
        lane_sync<BLOCK>(K, false);   // rank 0 rewrites thr_below / ng for the next digit
    }
    return Thr{bstar, kpre, spre};
}

// Finish a step: gather candidates, beam/max-active prune, backpointer records, next tokens.
// Returns the number of survivors (0 = search death).  In a cluster lane every CTA handles
// its own candidates; the minimum, the counts, the histogram and the compaction bases are
// combined through DSMEM, and epsilon-chain marks reach other CTAs' flags directly.
struct StepOut {
    int n_surv, n_keep, status, n_cand;
};

template <int BLOCK, int KC>
WB_PHASE_FN __device__ StepOut finish_step(int nxt, const GraphDev &g, const WorkDev &ws,
                                            const CfgDev &cfg) {
    Smem<BLOCK> &sh = SH<BLOCK>();
    const Lane c{ws};
    constexpr int K = KC;
    const int r = K > 1 ? cta_rank() : 0, cbase = r * ws.cap;
    const int n_loc = min(sh.n_cand, ws.cap);
    const bool in_smem = n_loc <= ws.smem_cands;
    if (!in_smem && threadIdx.x == 0) sh.pflags |= WB_PATH_GLOBAL_CANDS;
    // this CTA's candidates, by local index j (lane candidate index cbase + j)
    u64 *ckey = in_smem ? s_key<BLOCK>() : c.cand_key() + cbase;
    u32 *ca = in_smem ? s_ca<BLOCK>(ws) : c.cand_ca() + cbase;
    volatile u32 *vca = ca;
    u32 *cst = c.cand_state() + cbase;
    u64 *cap = c.cand_ap() + cbase;

    // P1: gather slot contents (batched loads), reset slots, min / max
    if (threadIdx.x == 0) sh.best_tok = -1;
    u64 mn = EMPTY_KEY, mx = 0;
    // a cluster CTA holds ~n/K candidates: keep all of a thread's slot exchanges in flight
    constexpr int G1 = KC > 1 ? 4 : Tune<BLOCK>::GATHER_P1;
    for (int i0 = threadIdx.x; i0 < n_loc; i0 += BLOCK * G1) {
        u32 st[G1];
        Slot v[G1];
#pragma unroll
        for (int q = 0; q < G1; ++q) {
            int i = i0 + q * BLOCK;
            if (i < n_loc) st[q] = cst[i];
        }
#pragma unroll
        for (int q = 0; q < G1; ++q) {
            int i = i0 + q * BLOCK;
            if (i < n_loc) {
                if (ws.xchg_gather) v[q] = xchg_slot_empty(&c.slot()[st[q]], ws.xchg_gather > 1);
                else v[q] = ld_slot(&c.slot()[st[q]]);
            }
        }
#pragma unroll
        for (int q = 0; q < G1; ++q) {
            int i = i0 + q * BLOCK;
            if (i < n_loc) {
                ckey[i] = v[q].key;
                cap[i] = (u64)v[q].arcp1 | ((u64)v[q].pay << 32);
                ca[i] = 0u;
                if (!ws.xchg_gather) st_slot_empty(&c.slot()[st[q]]);
#ifdef WB_CHECKS
                {   // one registration per state and step (the first-touch CAS protocol)
                    const u32 old = atomicAdd(&ws.chk_seen[c.so() + st[q]], 1u);
                    WB_CHECK(ws, old == 0u, CHK_DUP);
                    if (ws.chk_inject && r == 0 && i == 0 && sh.chk_off > 0)   // test knob
                        __stcg(reinterpret_cast<ulonglong2 *>(&c.slot()[st[q]]),
                               make_ulonglong2(v[q].key, 0ull));
                }
#endif
                mn = v[q].key < mn ? v[q].key : mn;
                mx = v[q].key > mx ? v[q].key : mx;
            }
        }
    }
    // lane-wide: min / max, candidate count, overflow, where each CTA keeps its flags
    int n_all = n_loc, flags = (sh.overflow ? 1 : 0) | (in_smem ? 0 : 2) | (sh.x_stream ? 4 : 0);
    u32 glob_mask = in_smem ? 0u : 1u << r;   // CTAs whose flags live in global memory
    if (K == 1) {
        block_minmax<BLOCK>(mn, mx);
    } else {
        // warps fold into this CTA's header with shared-memory atomics (reset at the step
        // start), one lane barrier, then every CTA reads every CTA's values through DSMEM
        mn = warp_min_u64(mn);
        mx = warp_max_u64(mx);
        if ((threadIdx.x & 31) == 0) {
            if (mn != EMPTY_KEY) atomicMin(reinterpret_cast<unsigned long long *>(&sh.x_mn), mn);
            if (mx != 0ull) atomicMax(reinterpret_cast<unsigned long long *>(&sh.x_mx), mx);
        }
        if (threadIdx.x == 0) { sh.x_n = n_loc; sh.x_flags = flags; }
        lane_sync<BLOCK>(K);
        mn = *(volatile u64 *)&sh.x_mn;
        mx = *(volatile u64 *)&sh.x_mx;
        for (int q = 1; q < K; ++q) {
            const int o = (r + q) & (K - 1);
            const Smem<BLOCK> *po = peer(&sh, o);
            const u64 a = *(volatile const u64 *)&po->x_mn, b = *(volatile const u64 *)&po->x_mx;
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
            n_all += *(volatile const int *)&po->x_n;
            const int fo = *(volatile const int *)&po->x_flags;
            flags |= fo;
            if (fo & 2) glob_mask |= 1u << o;
        }
    }
    int status = (flags & 4) ? wb_cap(WB_CAP_STREAM) : (flags & 1) ? wb_cap(WB_CAP_CANDIDATES) : WB_OK;
    tick<BLOCK>(3);
    if (n_all == 0) { lane_sync<BLOCK>(K); return StepOut{0, 0, status, 0}; }
    const double best = key_cost(mn);
    const double cutoff = __dadd_rn(best, cfg.beam);  // cutoff = best + beam (decoder.py:186)

    // P2: max-active histogram (only when it can bind)
    bool need_select = false;
    double scale = 0.0;
    Thr thr{0, 0, 0};
    if (cfg.max_active > 0 && n_all > cfg.max_active) {
        double hi = key_cost(mx);
        double top = cutoff < hi ? cutoff : hi;
        double range = __dsub_rn(top, best);
        if (range > 0.0 && range < INFINITY) scale = __ddiv_rn((double)NB, range);
        // histogram of the beam survivors' costs; its total says whether max-active binds
        for (int b = threadIdx.x; b < NB; b += BLOCK) sh.u.hist[b] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n_loc; i += BLOCK) {
            const double cs = key_cost(ckey[i]);
            if (cs <= cutoff) atomicAdd(&sh.u.hist[bucket_of(cs, best, scale)], 1u);
        }
        __syncthreads();
        thr = select_threshold<BLOCK, KC>(n_loc, cfg.max_active, best, cutoff, scale, ckey, cst, ws);
        need_select = thr.bucket >= 0;
    }
    tick<BLOCK>(4);
    if (threadIdx.x == 0) {  // cost range of the next live tokens (the early cutoff's split)
        const double top = key_cost(mx) < cutoff ? key_cost(mx) : cutoff;
        sh.tok_lo = best;
        sh.tok_hi = need_select ? key_cost(thr.key) : top;
    }
    const int bstar = thr.bucket;
    const u64 tkey = thr.key;
    const u32 tst = thr.state;

    // P3: survivor flags + epsilon-chain marks (atomicOr: flags of other candidates change;
    // a chain may continue into another CTA's candidates: its flags via DSMEM or global)
    auto flag_of = [&](u32 uix) -> u32 * {
        if (K == 1) return ca + uix;
        const int o = (int)(uix / (u32)ws.cap);
        const u32 j = uix - (u32)(o * ws.cap);
        if (o == r) return ca + j;
        if (glob_mask & (1u << o)) return c.cand_ca() + uix;
        return peer(s_ca<BLOCK>(ws), o) + j;
    };
    for (int i = threadIdx.x; i < n_loc; i += BLOCK) {
        u64 k = ckey[i];
        double cs = key_cost(k);
        bool surv = cs <= cutoff;
        if (surv && need_select) {
            int b = bucket_of(cs, best, scale);
            surv = b < bstar || (b == bstar && (k < tkey || (k == tkey && cst[i] <= tst)));
        }
        if (!surv) continue;
        atomicOr(&ca[i], F_SURV);
        if (!g.has_eps) continue;
        u32 v = (u32)(cbase + i);
        for (;;) {
            const u64 ap = ldx<KC>(&c.cand_ap()[v]);
            u32 a = (u32)ap, p = (u32)(ap >> 32);
            if (a == 0u || !(p & EPS_BIT)) break;
            u32 uix = p & ~EPS_BIT;
            u32 old = atomicOr(flag_of(uix), F_MARK);
            if (old & (F_MARK | F_SURV)) break;
            v = uix;
        }
    }
    lane_sync<BLOCK>(K);
    tick<BLOCK>(5);

    // P4: order-preserving compaction of kept candidates (arena records) and survivors
    // (next tokens).  Warps own contiguous segments; ballots count; one scan per CTA; the
    // CTAs of a lane take consecutive ranges in rank order.
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int seg = ((n_loc + NW - 1) / NW + 31) & ~31;
    const int lo = min(n_loc, w * seg), hi = min(n_loc, lo + seg);
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
        if (l == 31) { sh.wa[NW] = ia; sh.wb[NW] = ib; sh.x_ck = ia; sh.x_cs = ib; }
    }
    lane_sync<BLOCK>(K, false);
    int keep_before = 0, surv_before = 0, n_keep = (int)sh.wa[NW], n_surv = (int)sh.wb[NW];
    for (int q = 1; q < K; ++q) {
        const int o = (r + q) & (K - 1);
        const Smem<BLOCK> *po = peer(&sh, o);
        const int a = po->x_ck, b = po->x_cs;
        if (o < r) { keep_before += a; surv_before += b; }
        n_keep += a;
        n_surv += b;
    }
    const u64 base = sh.arena_used + (u64)keep_before;
    {
        const u64 used = sh.arena_used + (u64)n_keep;
        if (used > ws.arena_cap || used >= (u64)EPS_BIT) {
            lane_sync<BLOCK>(K);
            return StepOut{0, 0, wb_cap(WB_CAP_ARENA), n_all};
        }
    }
    __syncthreads();   // everyone has read arena_used
    if (threadIdx.x == 0) { sh.arena_used += (u64)n_keep; sh.n_pend = 0; }
    int4 *tinfo = c.tok_info(nxt);
    double *tcost = c.tok_cost(nxt);
    u32 *pend = c.front(0) + cbase;
    {
        // E: one pass over each warp's segment, 32 candidates at a time: ballot ranks give
        // every kept candidate its record index (left in its flag word for epsilon winners
        // that trace through it) and every survivor its next-token slot; the token and the
        // record are written in the same pass.  The candidate arrays are read coalesced, the
        // loads issued before the ballots.
        int ra = (int)sh.wa[w], rb = (int)sh.wb[w] + surv_before;
        const u32 lt = lanemask_lt();
        for (int i0 = lo; i0 < hi; i0 += 32) {
            const int i = i0 + l;
            const bool in = i < hi;
            u32 f = 0u, a = 0u, p = 0u, st = 0u;
            int4 rg = make_int4(0, 0, 0, 0);
            u64 k = 0;
            if (in) {
                f = vca[i];
                const u64 ap = cap[i];
                a = (u32)ap;
                p = (u32)(ap >> 32);
                st = cst[i];
                k = ckey[i];
            }
            const bool keep = f != 0u, surv = (f & F_SURV) != 0u;
            // a survivor's {eps_lo, emit_lo, emit_hi} is the second half of its winning arc's
            // record (the arc ends in this state; its first half was read by expand, so the
            // sector is in cache) -- no per-candidate range array
            if (surv) rg = a == 0u ? g.start_rng : __ldg(&g.arcs[2 * (size_t)(a - 1u) + 1]);
            const u32 mk = __ballot_sync(FULL, keep), ms = __ballot_sync(FULL, surv);
            const u32 rec = (u32)(base + (u64)(ra + __popc(mk & lt)));
            const u32 tj = (u32)(rb + __popc(ms & lt));
            ra += __popc(mk);
            rb += __popc(ms);
            if (!in) continue;
            ca[i] = keep ? rec : CA_NONE;
            if (surv) {
                WB_CHECK(ws, tj < (u32)ws.lcap, CHK_BOUNDS);
                tinfo[tj] = make_int4((int)st, (int)rec, rg.y, rg.z);
                tcost[tj] = key_cost(k);
                if (k == mn) {   // any minimal token will do; every CTA of the lane gets it
                    // with its arc range (one store: concurrent minimal tokens cannot mix
                    // ranges) and its arcs pulled into L2 for the next step's pilot
                    const u64 br = ((u64)(u32)rg.z << 32) | (u32)rg.y;
                    for (int q = 0; q < K; ++q) {
                        Smem<BLOCK> *po = q == 0 ? &sh : peer(&sh, (r + q) & (K - 1));
                        po->best_tok = (int)tj;
                        *(volatile u64 *)&po->best_rng = br;
                        po->best_key = k;
                    }
                    for (int a2 = rg.y; a2 < rg.z; a2 += 4)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(&g.arcs[2 * (size_t)a2]));
                }
                if (ws.tok_eps) ws.tok_eps[2 * c.co() + (size_t)nxt * ws.lcap + tj] = rg.x;
            }
            if (keep) {
                WB_CHECK(ws, (u64)rec < ws.arena_cap, CHK_BOUNDS);
                if (a != 0u && (p & EPS_BIT)) {
                    const int qq = atomicAdd(&sh.n_pend, 1);
                    pend[qq] = (u32)i;  // epsilon winner: needs its source's record index
                } else {
                    const u32 prev = a == 0u ? ROOT_PREV : p;
                    c.arena()[rec] = (u64)a | ((u64)prev << 32);
                }
            }
        }
    }
    // epsilon winners resolve their source's record index, possibly another CTA's
    if (g.has_eps) lane_sync<BLOCK>(K);
#ifdef WB_CHECKS
    // debug_epoch analogue: every slot this step touched is EMPTY again (no relaxation of
    // this step can leak into the next); registration counters are cleared for the next step
    for (int i = threadIdx.x; i < n_loc; i += BLOCK) {
        const u32 st = cst[i];
        WB_CHECK(ws, ld_slot(&c.slot()[st]).key == EMPTY_KEY, CHK_STALE);
        ws.chk_seen[c.so() + st] = 0u;
    }
#endif
    if (!g.has_eps) __syncthreads();
    const int n_pend = sh.n_pend;
    for (int q = threadIdx.x; q < n_pend; q += BLOCK) {
        int i = (int)pend[q];
        const u64 ap = cap[i];
        const u32 a = (u32)ap, p = (u32)(ap >> 32);
        const u32 src = *(volatile u32 *)flag_of(p & ~EPS_BIT);
        c.arena()[vca[i]] = (u64)a | ((u64)src << 32);
    }
    lane_sync<BLOCK>(K);   // next tokens / records complete in every CTA of the lane
    tick<BLOCK>(6);
    return StepOut{n_surv, n_keep, status, n_all};
}

// LSD pre-pass (classify_blank_frames + nonblank_frames, posteriors.py:116-125,109-110): a
// frame is blank iff its blank probability strictly exceeds the threshold; non-blank frame
// ids are compacted in order.
template <int BLOCK>
__device__ int lsd_prepass(const double *bl, int T, double thr, int *fr, bool write) {
    Smem<BLOCK> &sh = SH<BLOCK>();
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
    for (int i0 = lo; write && i0 < hi; i0 += 32) {
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
__device__ int block_argmin_tok(u64 key, u32 st, int idx) {
    Smem<BLOCK> &sh = SH<BLOCK>();
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

// ------------------------------------------------------------------ lattice recording
__device__ __forceinline__ bool surv_bit(const u32 *bits, u32 s) {
    return (__ldcg(&bits[s >> 5]) >> (s & 31)) & 1u;  // L2-coherent: set by this step's atomics
}

// Raw lattice of node step k (lattice.py:148-170): nodes = survivors(k) (plus the start at
// step 0, decoder.py:246-248); emitting arcs = relaxations from live(k-1) with finite
// acoustic cost into survivors(k); epsilon arcs = non-self-loop epsilon arcs between
// survivors(k).  The raw lattice is a pure function of these sets, so no per-relaxation
// recorder is needed.  Node / arc indices are utterance-global positions in this lane's pool.
template <int BLOCK>
WB_LATTICE_FN __device__ int record_lattice_step(int k, int nxt, int n_surv, int prv, int n_prev,
                                                const double *grow, int L1,
                                                const GraphDev &g, const WorkDev &ws) {
    Smem<BLOCK> &sh = SH<BLOCK>();
    const Lane c{ws};
    constexpr int NW = BLOCK / 32;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const size_t so = c.so(), lo = (size_t)blockIdx.x * (size_t)ws.lat_cap;
    const size_t bo = (size_t)blockIdx.x * (size_t)((ws.S + 31) >> 5);
    int4 *lst = ws.lstep + (size_t)blockIdx.x * (ws.T_cap + 2);
    int *lse = ws.lstep_eps + (size_t)blockIdx.x * (ws.T_cap + 2);
    const int node_base = k == 0 ? 0 : lst[k - 1].x + lst[k - 1].z;
    const int arc_base = k == 0 ? 0 : lst[k - 1].y + lst[k - 1].w + lse[k - 1];
    const int prev_base = k == 0 ? 0 : lst[k - 1].x;
    const int4 *tn = c.tok_info(nxt);
    const int *te = ws.tok_eps + 2 * c.co() + (size_t)nxt * ws.lcap;
    int status = WB_OK;
    // step 0 keeps the start node even when the prune dropped it
    if (threadIdx.x == 0) { sh.ng = -1; sh.n_pend = 0; }
    __syncthreads();
    if (k == 0)
        for (int j = threadIdx.x; j < n_surv; j += BLOCK)
            if (tn[j].x == g.start) sh.ng = j;
    __syncthreads();
    const bool extra = k == 0 && sh.ng < 0;
    const int n_nodes = n_surv + (extra ? 1 : 0);
    if ((long long)node_base + n_nodes > ws.lat_cap) return wb_cap(WB_CAP_LATTICE_RAW);
    for (int j = threadIdx.x; j < n_nodes; j += BLOCK) {
        const u32 st = j < n_surv ? (u32)tn[j].x : (u32)g.start;
        atomicOr(&ws.sbits[bo + (st >> 5)], 1u << (st & 31));
        ws.snode[so + st] = (u32)(node_base + j);
        ws.ln_state[lo + node_base + j] = st;
    }
    if (k == 0 && threadIdx.x == 0) ws.lstep_start[blockIdx.x] = node_base + (extra ? n_surv : sh.ng);
    // the step's cost row again in shared memory (the prune reused that space)
    const double *row = grow;
    if (k > 0 && ws.row_in_smem) {
        double *srow = s_row<BLOCK>();
        for (int q = threadIdx.x; q < L1; q += BLOCK) srow[q] = ws.log_rows ? -__ldg(&grow[q]) : __ldg(&grow[q]);
        row = srow;
    }
    __syncthreads();
    const long long room = ws.lat_cap - arc_base;
    // emitting arcs from live(k-1): the finite relaxations expand logged, into survivors
    if (k > 0) {
        const int n_log = sh.n_log;
        if ((long long)n_log > ws.rlog_cap) status = wb_cap(WB_CAP_LATTICE_RAW);
        const int4 *lg = ws.rlog + (size_t)blockIdx.x * ws.rlog_cap;
        const int nl = (int)min((long long)n_log, ws.rlog_cap);
        constexpr int G = 4;  // log entries per thread with their loads in flight
        for (int i0 = 0; i0 < nl; i0 += BLOCK * G) {
            int4 r[G];
            bool rec[G];
            u32 dn[G];
#pragma unroll
            for (int q = 0; q < G; ++q) {
                const int i = i0 + q * BLOCK + (int)threadIdx.x;
                r[q] = i < nl ? lg[i] : make_int4(0, 0, -1, 0);
            }
#pragma unroll
            for (int q = 0; q < G; ++q)
                rec[q] = r[q].z >= 0 && surv_bit(ws.sbits + bo, (u32)r[q].z);
#pragma unroll
            for (int q = 0; q < G; ++q)
                dn[q] = rec[q] ? __ldcg(&ws.snode[so + r[q].z]) : 0u;
#pragma unroll
            for (int q = 0; q < G; ++q) {
                const u32 m = __ballot_sync(FULL, rec[q]);
                if (!m) continue;
                int base = 0;
                if (l == __ffs(m) - 1) base = atomicAdd(&sh.n_pend, __popc(m));
                base = __shfl_sync(FULL, base, __ffs(m) - 1);
                if (rec[q]) {
                    const long long e = base + __popc(m & lanemask_lt());
                    if (e < room) {
                        const size_t ge = lo + arc_base + e;
                        ws.la_src[ge] = (u32)(prev_base + r[q].x);
                        ws.la_dst[ge] = dn[q];
                        ws.la_arc[ge] = (u32)r[q].y;
                        ws.la_ac[ge] = row[r[q].w];
                    }
                }
            }
        }
    }
    __syncthreads();
    const int n_emit = sh.n_pend;
    // epsilon arcs inside step k
    if (g.has_eps) {
        const int nchunks = (n_nodes + 31) >> 5;
        for (int ch = w; ch < nchunks; ch += NW) {
            const int j = (ch << 5) + l;
            int lo_e = 0, deg = 0;
            u32 st = 0;
            if (j < n_surv) {
                st = (u32)tn[j].x;
                lo_e = te[j];
                deg = tn[j].z - lo_e;
            } else if (j < n_nodes) {
                st = (u32)g.start;
                lo_e = g.start_rng.x;
                deg = g.start_rng.y - g.start_rng.x;
            }
            const int incl = warp_incl_scan(deg);
            const int tot = __shfl_sync(FULL, incl, 31);
            const int excl = incl - deg;
            for (int j0 = 0; j0 < tot; j0 += 32) {
                const int q = j0 + l;
                const int kk = warp_owner(excl, q);
                const int lo_k = __shfl_sync(FULL, lo_e, kk);
                const int ex_k = __shfl_sync(FULL, excl, kk);
                const u32 st_k = __shfl_sync(FULL, st, kk);
                const int a = lo_k + q - ex_k;
                bool rec = false;
                int4 r = make_int4(0, 0, 0, 0);
                if (q < tot) {
                    r = __ldg(&g.arcs[2 * a]);
                    rec = (u32)r.x != st_k && surv_bit(ws.sbits + bo, (u32)r.x);
                }
                const u32 m = __ballot_sync(FULL, rec);
                if (!m) continue;
                int base = 0;
                if (l == __ffs(m) - 1) base = atomicAdd(&sh.n_pend, __popc(m));
                base = __shfl_sync(FULL, base, __ffs(m) - 1);
                if (rec) {
                    const long long e = base + __popc(m & lanemask_lt());
                    if (e < room) {
                        const size_t ge = lo + arc_base + e;
                        ws.la_src[ge] = (u32)(node_base + kk + (ch << 5));
                        ws.la_dst[ge] = __ldcg(&ws.snode[so + r.x]);
                        ws.la_arc[ge] = (u32)a;
                        ws.la_ac[ge] = 0.0;
                    }
                }
            }
        }
    }
    __syncthreads();
    const int n_all = sh.n_pend;
    if (n_all > room) status = wb_cap(WB_CAP_LATTICE_RAW);
    for (int j = threadIdx.x; j < n_nodes; j += BLOCK)  // every set bit is one of these nodes
        ws.sbits[bo + (ws.ln_state[lo + node_base + j] >> 5)] = 0u;
    if (threadIdx.x == 0) {
        lst[k] = make_int4(node_base, arc_base, n_nodes, n_emit);
        lse[k] = n_all - n_emit;
    }
    __syncthreads();
    return status;
}

// Trim to nodes on some start-to-final path (_assemble, lattice.py:190-237) by forward and
// backward reachability sweeps over the node steps, then copy the kept nodes / arcs / finals
// to the output pools.  Canonical ordering is left to the host (small lattice).
constexpr unsigned char LF_FWD = 1, LF_BWD = 2;

template <int BLOCK>
WB_LATTICE_FN __device__ void trim_lattice(int u, int K, int reached, int final_state,
                                          const GraphDev &g, const WorkDev &ws) {
    const int final_step = K;  // the last node step with nodes is the winner's step
    Smem<BLOCK> &sh = SH<BLOCK>();
    const size_t lo = (size_t)blockIdx.x * (size_t)ws.lat_cap;
    const int4 *lst = ws.lstep + (size_t)blockIdx.x * (ws.T_cap + 2);
    const int *lse = ws.lstep_eps + (size_t)blockIdx.x * (ws.T_cap + 2);
    unsigned char *fl = ws.ln_flag + lo;
    const u32 *la_src = ws.la_src + lo, *la_dst = ws.la_dst + lo;
    long long *meta = ws.o_meta + 6 * (size_t)u;
    const int n_nodes = lst[K].x + lst[K].z;
    const int n_arcs = lst[K].y + lst[K].w + lse[K];
    if (threadIdx.x == 0) sh.lat_bad = 0;
    for (int i = threadIdx.x; i < n_nodes; i += BLOCK) fl[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) fl[ws.lstep_start[blockIdx.x]] = LF_FWD;
    __syncthreads();
    // forward reach from the start
    for (int k = 0; k <= K; ++k) {
        const int4 st = lst[k];
        for (int e = threadIdx.x; e < st.w; e += BLOCK) {
            const size_t ge = (size_t)st.y + e;
            if (fl[la_src[ge]] & LF_FWD) fl[la_dst[ge]] = LF_FWD;
        }
        __syncthreads();
        const int ne = lse[k];
        while (ne > 0) {
            if (threadIdx.x == 0) sh.flag = 0;
            __syncthreads();
            for (int e = threadIdx.x; e < ne; e += BLOCK) {
                const size_t ge = (size_t)st.y + st.w + e;
                if ((fl[la_src[ge]] & LF_FWD) && !(fl[la_dst[ge]] & LF_FWD)) {
                    fl[la_dst[ge]] = LF_FWD;
                    sh.flag = 1;
                }
            }
            __syncthreads();
            const int changed = sh.flag;
            __syncthreads();
            if (!changed) break;
        }
    }
    // live finals (lattice.py:172-183, 214): reached -> survivors of final_step with a final
    // weight; otherwise the winning state at final_step with weight 0
    if (threadIdx.x == 0) { sh.ng = 0; sh.n_pend = 0; }
    __syncthreads();
    const int4 fs = lst[final_step];
    for (int i = threadIdx.x; i < fs.z; i += BLOCK) {
        const int node = fs.x + i;
        const u32 s = ws.ln_state[lo + node];
        const bool fin = reached ? __ldg(&g.final_w[s]) != INFINITY : (int)s == final_state;
        if (fin && (fl[node] & LF_FWD)) {
            fl[node] = LF_FWD | LF_BWD;
            atomicAdd(&sh.ng, 1);
        }
    }
    __syncthreads();
    const int n_fin = sh.ng;
    __syncthreads();
    if (n_fin == 0) {  // EMPTY_LATTICE
        if (threadIdx.x == 0) for (int q = 0; q < 6; ++q) meta[q] = 0;
        __syncthreads();
        return;
    }
    // backward reach from the live finals
    for (int k = final_step; k >= 0; --k) {
        if (k < K) {
            const int4 nx = lst[k + 1];
            for (int e = threadIdx.x; e < nx.w; e += BLOCK) {
                const size_t ge = (size_t)nx.y + e;
                const u32 sn = la_src[ge];
                if ((fl[la_dst[ge]] & LF_BWD) && (fl[sn] & LF_FWD)) fl[sn] = LF_FWD | LF_BWD;
            }
            __syncthreads();
        }
        const int4 st = lst[k];
        const int ne = lse[k];
        while (ne > 0) {
            if (threadIdx.x == 0) sh.flag = 0;
            __syncthreads();
            for (int e = threadIdx.x; e < ne; e += BLOCK) {
                const size_t ge = (size_t)st.y + st.w + e;
                const u32 sn = la_src[ge];
                if ((fl[la_dst[ge]] & LF_BWD) && (fl[sn] == LF_FWD)) {
                    fl[sn] = LF_FWD | LF_BWD;
                    sh.flag = 1;
                }
            }
            __syncthreads();
            const int changed = sh.flag;
            __syncthreads();
            if (!changed) break;
        }
    }
    // kept = forward & backward reachable; compact nodes (step-major order), arcs, finals
    constexpr int NW = BLOCK / 32;
    const int wp = threadIdx.x >> 5, l = threadIdx.x & 31;
    const u32 lt = lanemask_lt();
    auto kept = [&](int i) { return fl[i] == (LF_FWD | LF_BWD); };
    int cnt = 0;
    const int seg = ((n_nodes + NW - 1) / NW + 31) & ~31;
    const int s0 = min(n_nodes, wp * seg), s1 = min(n_nodes, s0 + seg);
    for (int i0 = s0; i0 < s1; i0 += 32) {
        const int i = i0 + l;
        cnt += __popc(__ballot_sync(FULL, i < s1 && kept(i)));
    }
    int tot;
    int run = warp_offsets<BLOCK>(cnt, sh.wa, &tot);
    if (threadIdx.x == 0) {
        unsigned long long nb = atomicAdd(&ws.o_ctr[0], (unsigned long long)tot);
        sh.arena_base = nb;
        if (nb + tot > (unsigned long long)ws.o_node_cap) sh.lat_bad = 1;
    }
    __syncthreads();
    const unsigned long long nbase = sh.arena_base;
    const bool ok_nodes = sh.lat_bad == 0;
    for (int i0 = s0; i0 < s1; i0 += 32) {
        const int i = i0 + l;
        const bool kp = i < s1 && kept(i);
        const u32 m = __ballot_sync(FULL, kp);
        if (kp) {
            const int oi = run + __popc(m & lt);
            ws.ln_out[lo + i] = (u32)oi;
            if (ok_nodes) {
                int step = 0, a = 0, b = K;
                while (a <= b) {  // node step: last k with lst[k].x <= i
                    const int mid = (a + b) >> 1;
                    if (lst[mid].x <= i) { step = mid; a = mid + 1; } else b = mid - 1;
                }
                ws.o_node[nbase + oi] = make_int2((int)ws.ln_state[lo + i], step);
            }
        }
        run += __popc(m);
    }
    __syncthreads();
    // arcs between kept nodes (kept from-node is forward-reached, kept to-node backward)
    auto karc = [&](int e) { return kept(la_src[e]) && kept(la_dst[e]); };
    cnt = 0;
    const int sega = ((n_arcs + NW - 1) / NW + 31) & ~31;
    const int a0 = min(n_arcs, wp * sega), a1 = min(n_arcs, a0 + sega);
    for (int i0 = a0; i0 < a1; i0 += 32) {
        const int e = i0 + l;
        cnt += __popc(__ballot_sync(FULL, e < a1 && karc(e)));
    }
    int tota;
    run = warp_offsets<BLOCK>(cnt, sh.wa, &tota);
    if (threadIdx.x == 0) {
        unsigned long long ab = atomicAdd(&ws.o_ctr[1], (unsigned long long)tota);
        unsigned long long fb = atomicAdd(&ws.o_ctr[2], (unsigned long long)n_fin);
        sh.arena_base = ab;
        sh.thr_key = fb;
        if (ab + tota > (unsigned long long)ws.o_arc_cap || fb + n_fin > (unsigned long long)ws.o_fin_cap)
            sh.lat_bad = 1;
    }
    __syncthreads();
    const unsigned long long abase = sh.arena_base, fbase = sh.thr_key;
    const bool ok = sh.lat_bad == 0;
    for (int i0 = a0; i0 < a1; i0 += 32) {
        const int e = i0 + l;
        const bool kp = e < a1 && karc(e);
        const u32 m = __ballot_sync(FULL, kp);
        if (kp && ok) {
            const unsigned long long oe = abase + run + __popc(m & lt);
            ws.o_arc[oe] = make_uint4(ws.ln_out[lo + la_src[e]], ws.ln_out[lo + la_dst[e]],
                                      ws.la_arc[lo + e], 0u);
            ws.o_ac[oe] = ws.la_ac[lo + e];
        }
        run += __popc(m);
    }
    if (threadIdx.x == 0) sh.ng = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < fs.z; i += BLOCK) {
        const int node = fs.x + i;
        const u32 s = ws.ln_state[lo + node];
        const bool fin = reached ? __ldg(&g.final_w[s]) != INFINITY : (int)s == final_state;
        if (fin && kept(node) && ok) {
            const int q = atomicAdd(&sh.ng, 1);
            ws.o_fin[fbase + q] = ws.ln_out[lo + node];
            ws.o_finw[fbase + q] = reached ? __ldg(&g.final_w[s]) : 0.0;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        meta[0] = ok ? (long long)nbase : -1;
        meta[1] = tot;
        meta[2] = (long long)abase;
        meta[3] = tota;
        meta[4] = (long long)fbase;
        meta[5] = n_fin;
    }
    __syncthreads();
}

// Backtrace (decoder.py:276-291): the lane's thread 0 walks its arena from the winner before
// the lane takes its next utterance; labels are written back to front so they land in path
// order without a second walk.
__device__ __noinline__ void backtrace(const GraphDev &g, const u64 *arena, long long best,
                                       u64 used, int *ob, int *ib, int cap, int *n_o, int *n_i) {
    int po = cap, pi = cap, no = 0, ni = 0;
    u32 idx = best < 0 ? ROOT_PREV : (u32)best;
    while (idx != ROOT_PREV && (u64)idx < used) {  // records point backwards: bounded walk
        const u64 rec = __ldcg(&arena[idx]);
        const u32 a1 = (u32)rec;
        idx = (u32)(rec >> 32);
        if (a1 == 0u) continue;
        const int a = (int)a1 - 1;
        const int il = __ldg(&g.arcs[2 * a].y);
        const int ol = __ldg(&g.arcs[2 * a + 1].w);
        if (ol != 0) { ++no; if (po > 0) ob[--po] = ol; }
        if (il != 0) { ++ni; if (pi > 0) ib[--pi] = il; }
    }
    if (no <= cap) for (int i = 0; i < no; ++i) ob[i] = ob[po + i];
    if (ni <= cap) for (int i = 0; i < ni; ++i) ib[i] = ib[pi + i];
    *n_o = no;
    *n_i = ni;
}

template <int BLOCK, int KC>
__global__ void __launch_bounds__(BLOCK, Tune<BLOCK>::MINB)
decode_kernel(const __grid_constant__ GraphDev g, const __grid_constant__ WorkDev ws,
              const __grid_constant__ BatchDev b, const __grid_constant__ CfgDev cfg,
              wb_utt_result *res) {
    Smem<BLOCK> &sh = SH<BLOCK>();
    const Lane c{ws};
    constexpr int K = KC;   // a lane = a cluster of K CTAs
    const int rank = K > 1 ? cta_rank() : 0;
    const int slot_id = (int)c.lane();
    u32 tag = ws.tag_ctr[slot_id];
    if (K > 1) {   // lane-barrier flags are zero in every CTA before any peer writes one
        if (threadIdx.x < 8) sh.ls_flag[threadIdx.x] = 0u;
        if (threadIdx.x == 0) sh.ls_epoch = 0u;
        cluster_sync_full();
    }
    const bool row_in_smem = ws.row_in_smem != 0;
    const bool pilot_on = g.nonneg && cfg.beam < INFINITY && ws.beam_skip && ws.stage_off;
    double *srow = s_row<BLOCK>();

    for (;;) {
        if (rank == 0 && threadIdx.x == 0) sh.utt = (int)atomicAdd(ws.utt_ctr, 1u);
        lane_sync<BLOCK>(K);
        const int u = K > 1 ? peer(&sh, 0)->utt : sh.utt;
        if (u >= b.n) break;
        if (threadIdx.x < 8) sh.pc[threadIdx.x] = 0;
#ifdef WB_PROBE
        if (threadIdx.x < 8) sh.spin_ph[threadIdx.x] = 0;
        if (threadIdx.x == 0) sh.spin_acc = 0;
#endif
        if (threadIdx.x < 4) sh.cnt[threadIdx.x] = 0ull;
        if (threadIdx.x < 5) sh.acc[threadIdx.x] = 0ll;
        if (threadIdx.x == 0) {
            sh.t_mark = clock64(); sh.arena_used = 0; sh.ready_seen = 0; sh.run_min = EMPTY_KEY;
            sh.pflags = ws.stage_off ? WB_PATH_PREFETCH : 0;
            sh.best_tok = -1;
            sh.chk_off = 0;
            sh.tok_lo = 0.0; sh.tok_hi = 0.0; sh.ma_frac = 0.5f;
        }
        const int T = b.T[u];
        const long long row0 = b.row_off[u];
        int status = WB_OK;
        int nf = T;
        if (cfg.mode == 1) {
            if (T > ws.T_cap) {  // frame list would overflow: report, do not decode
                status = wb_cap(WB_CAP_FRAMES);
                nf = 0;
            } else {
                nf = lsd_prepass<BLOCK>(b.blank + row0, T, cfg.thr, c.frames(), rank == 0);
            }
        }

        // ---- initial tokens: start entry + epsilon closure + prune (decoder.py:236-249)
        if (threadIdx.x == 0) {   // rank 0 holds the start entry as its candidate 0
            sh.stamp = tag;
            sh.n_cand = 0;
            sh.overflow = 0;
            sh.nfr[0] = sh.nfr[1] = 0;
            sh.x_stream = 0;
            sh.x_mn = EMPTY_KEY; sh.x_mx = 0; sh.x_n = 0; sh.x_flags = 0;
            if (rank == 0) {
                u64 k0 = cost_key(0.0);
                __stcg(reinterpret_cast<ulonglong2 *>(&c.slot()[g.start]),
                       make_ulonglong2(k0, (u64)0u | ((u64)ROOT_PREV << 32)));
                c.cand_state()[0] = (u32)g.start;
                if (g.has_eps) c.cand_of()[g.start] = (u64)sh.stamp << 32;
                sh.n_cand = 1;
                if (g.has_eps && g.start_rng.x < g.start_rng.y) {
                    c.front(0)[0] = (u32)g.start;
                    c.frng(0)[0] = make_int4(0, g.start_rng.x, g.start_rng.y, 0);
                    sh.nfr[0] = 1;
                }
            }
        }
        lane_sync<BLOCK>(K);
        if (g.has_eps) {
            EpsOut eo = epsilon_closure<BLOCK, KC>(g, ws, tag, cfg.beam);
            tag = eo.tag;
            count_add<BLOCK>(3, eo.e_eps);
            if (eo.status) status = eo.status;
            acc_add<BLOCK>(4, eo.rounds);
        }
        int cur = 0;
        StepOut so = finish_step<BLOCK, KC>(cur, g, ws, cfg);
        acc_add<BLOCK>(1, so.n_cand);
        if (so.status) status = so.status;
        acc_add<BLOCK>(3, so.n_keep);
        long long lat_arcs = 0;
        if (cfg.lattice && status == WB_OK) {
            const int rs = record_lattice_step<BLOCK>(0, cur, so.n_surv, 0, 0, nullptr, 0, g, ws);
            if (rs) status = rs;
        }
        int n_live = so.n_surv;
        acc_add<BLOCK>(2, n_live);
        int steps_run = 0, died_at = -1;
        for (int s = 0; s < nf && status == WB_OK; ++s) {
            const int f = cfg.mode == 1 ? ldx<KC>(&c.frames()[s]) : s;
            const int ridx = b.crow_off ? s : f;  // compacted rows are indexed by search step
            const double *grow = b.costs + (size_t)((b.crow_off ? b.crow_off[u] : row0) + ridx) * b.L1;
            const double *row = grow;
            if (b.ready) {  // streaming input: wait until the host has written row ridx
                if (threadIdx.x == 0) {
                    int seen = sh.ready_seen;
                    const long long t0 = clock64();
                    if (seen <= ridx) {
                        // relaxed polls; one acquire fence once a new count is seen, so the
                        // row data it covers is read after the counter
                        for (;;) {
                            asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(seen) : "l"(b.ready + u) : "memory");
                            if (seen > ridx) break;
                            __nanosleep(500);
                            if (clock64() - t0 > STREAM_WAIT_CYCLES) { seen = -1; break; }
                        }
                        asm volatile("fence.acq_rel.sys;" ::: "memory");
                    }
                    sh.ready_seen = seen;
                }
                __syncthreads();
                if (sh.ready_seen < 0) {  // the host never published this row: give up
                    if (K == 1) {
                        status = wb_cap(WB_CAP_STREAM);
                        break;
                    }
                    // a cluster lane finishes the step with the others; the failure is
                    // combined with theirs in the prune (every CTA then stops together)
                    if (threadIdx.x == 0) { sh.x_stream = 1; sh.ready_seen = 0; }
                }
            }
#ifdef WB_PROBE_STAGE
            __syncthreads();
            tick<BLOCK>(7);   // probe build: loop top (frame id, row address) vs staging + pilot
#endif
            int neg = !row_in_smem;  // acoustic costs of this row all >= 0? (checked while staging)
            if (threadIdx.x == 0) {
                sh.n_cand = 0; sh.nfr[0] = sh.nfr[1] = 0; sh.overflow = 0; sh.n_log = 0;
                sh.stamp = tag;   // registrations of this step (expand, closure) carry it
                sh.run_min = EMPTY_KEY;
                sh.next_chunk = BLOCK / 32;
                // this CTA's prune accumulators (peers read them after the prune's barrier)
                sh.x_mn = EMPTY_KEY; sh.x_mx = 0; sh.x_n = 0; sh.x_flags = 0;
            }
            // Pilot of the beam skip (expand_emitting): warp 0 evaluates the arcs of a cheapest
            // live token against the row in global memory while the other warps stage it.
            const bool pilot = row_in_smem && pilot_on && sh.best_tok >= 0 && sh.best_tok < n_live;
            if (pilot && threadIdx.x < 32) {
                __syncwarp();
                pilot_min<BLOCK>(sh.best_tok, cur, grow, g, ws, ws.log_rows != 0);
            }
            if (row_in_smem) {
                const int t0 = pilot ? (int)threadIdx.x - 32 : (int)threadIdx.x;
                const int nt = pilot ? BLOCK - 32 : BLOCK;
                // 8 loads in flight per thread before the stores (one memory round trip for
                // rows up to 8 x BLOCK columns instead of one per column a thread stages)
                for (int q0 = t0; q0 >= 0 && q0 < b.L1; q0 += 8 * nt) {
                    double v[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int q = q0 + i * nt;
                        v[i] = q < b.L1 ? __ldg(&grow[q]) : 0.0;
                        if (ws.log_rows) v[i] = -v[i];   // log(p) rows: the cost is -log(p)
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int q = q0 + i * nt;
                        if (q < b.L1) {
                            neg |= v[i] < 0.0;
                            srow[q] = v[i];
                        }
                    }
                }
                row = srow;
            }
            const bool row_nonneg = !__syncthreads_or(neg);
            if (ws.row_prefetch && s + 1 < nf) {
                // the next step's row into L2 while this step searches (its staging then hits
                // L2 instead of DRAM): one 128-byte line per thread
                const int fn = cfg.mode == 1 ? ldx<KC>(&c.frames()[s + 1]) : s + 1;
                const double *nrow = b.costs + (size_t)(row0 + fn) * b.L1;
                for (int q = threadIdx.x * 16; q < b.L1; q += BLOCK * 16)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(nrow + q));
            }
            tick<BLOCK>(0);
            acc_add<BLOCK>(0, n_live);
            {
                ExpandCounts ec = expand_emitting<BLOCK, KC>(n_live, cur, row, g, ws, cfg.beam, row_nonneg,
                                                             pilot, cfg.max_active);
                count_add<BLOCK>(0, ec.a_emit);
                count_add<BLOCK>(1, ec.a_fin);
                count_add<BLOCK>(2, ec.a_cas);
            }
            lane_sync<BLOCK>(K);   // every CTA's relaxations have landed in the lane's slots
#ifdef WB_CHECKS
            {   // every live token of the step was expanded by exactly one group
                u32 *cl = ws.chk_claim + c.lane() * ws.lcap;
                for (int t = threadIdx.x + rank * BLOCK; t < n_live; t += BLOCK * K) {
                    WB_CHECK(ws, ldx<KC>(&cl[t]) == 1u, CHK_CLAIM);
                    cl[t] = 0u;
                }
                if (rank == 0 && threadIdx.x == 0 && s <= ws.T_cap)
                    ws.chk_steps[c.lane() * (ws.T_cap + 1) + s] = n_live;
                __syncthreads();
                if (threadIdx.x == 0) sh.chk_off += n_live;
            }
#endif
            tick<BLOCK>(1);
            if (g.has_eps) {
                EpsOut eo = epsilon_closure<BLOCK, KC>(g, ws, tag, cfg.beam);
                tag = eo.tag;
                count_add<BLOCK>(3, eo.e_eps);
                if (eo.status) status = eo.status;
                acc_add<BLOCK>(4, eo.rounds);
            }
            tick<BLOCK>(2);
            so = finish_step<BLOCK, KC>(cur ^ 1, g, ws, cfg);
            acc_add<BLOCK>(1, so.n_cand);
            if (so.status) status = so.status;
            acc_add<BLOCK>(3, so.n_keep);
            steps_run++;
            if (so.n_surv == 0) {
                died_at = s;
                break;
            }
            acc_add<BLOCK>(2, so.n_surv);
            if (cfg.lattice && status == WB_OK) {
                const int rs = record_lattice_step<BLOCK>(s + 1, cur ^ 1, so.n_surv, cur, n_live, grow,
                                                          b.L1, g, ws);
                if (rs) status = rs;
            }
            cur ^= 1;
            n_live = so.n_surv;
        }
#ifdef WB_CHECKS
        if (status == WB_OK) {   // the whole slot array is clean between utterances
            lane_sync<BLOCK>(K);
            const Slot *sl = c.slot();
            for (long long q = threadIdx.x + (long long)rank * BLOCK; q < ws.S; q += (long long)BLOCK * K)
                WB_CHECK(ws, ld_slot(&sl[q]).key == EMPTY_KEY, CHK_STALE_UTT);
        }
#endif
        if (status != WB_OK) {
            // a failed step may leave slots beyond the candidate capacity dirty: restore the
            // lane's whole slot array so later utterances on this lane start clean
            lane_sync<BLOCK>(K);
            Slot *sl = c.slot();
            for (long long q = threadIdx.x + (long long)rank * BLOCK; q < ws.S; q += (long long)BLOCK * K)
                st_slot_empty(&sl[q]);
        }
        if (K > 1) lane_sync<BLOCK>(K, false); else __syncthreads();
        long long t_emit = (long long)sh.cnt[0], t_fin = (long long)sh.cnt[1];
        long long t_cas = (long long)sh.cnt[2], t_eps = (long long)sh.cnt[3];
        int pflags = sh.pflags;
        if (K > 1 && rank == 0) {   // rank 0 reports the lane: sum the other CTAs' counters
            for (int q = 1; q < K; ++q) {
                const Smem<BLOCK> *po = peer(&sh, q);
                t_emit += (long long)po->cnt[0]; t_fin += (long long)po->cnt[1];
                t_cas += (long long)po->cnt[2]; t_eps += (long long)po->cnt[3];
                pflags |= po->pflags;
            }
        }
        if (rank != 0) continue;   // the lane's last writes are visible to rank 0 (lane_sync)
        // ---- final transition / death fallback (decoder.py:252-273, 327-333)
        const int4 *tinfo = c.tok_info(cur);
        const double *tcost = c.tok_cost(cur);
        int best_t = -1;
        int reached = 0;
        double best_cost = 0.0;
        if (died_at < 0) {
            u64 k = EMPTY_KEY;
            u32 st = 0xFFFFFFFFu;
            int idx = -1;
            for (int t = threadIdx.x; t < n_live; t += BLOCK) {
                int s = ldx<KC>(&tinfo[t]).x;
                double fw = __ldg(&g.final_w[s]);
                if (fw == INFINITY) continue;
                u64 kk = cost_key(__dadd_rn(ldx<KC>(&tcost[t]), fw));
                if (kk < k || (kk == k && (u32)s < st)) { k = kk; st = (u32)s; idx = t; }
            }
            best_t = block_argmin_tok<BLOCK>(k, st, idx);
            if (best_t >= 0) {
                reached = 1;
                best_cost = __dadd_rn(ldx<KC>(&tcost[best_t]), __ldg(&g.final_w[ldx<KC>(&tinfo[best_t]).x]));
            }
        }
        if (best_t < 0) {
            u64 k = EMPTY_KEY;
            u32 st = 0xFFFFFFFFu;
            int idx = -1;
            for (int t = threadIdx.x; t < n_live; t += BLOCK) {
                u64 kk = cost_key(ldx<KC>(&tcost[t]));
                u32 s = (u32)ldx<KC>(&tinfo[t]).x;
                if (kk < k || (kk == k && s < st)) { k = kk; st = s; idx = t; }
            }
            best_t = block_argmin_tok<BLOCK>(k, st, idx);
            if (best_t >= 0) best_cost = ldx<KC>(&tcost[best_t]);
        }
        if (cfg.lattice) {
            const int fstep = died_at < 0 ? steps_run : died_at;
            if (status == WB_OK) {
                const int4 lk = ws.lstep[(size_t)blockIdx.x * (ws.T_cap + 2) + fstep];
                lat_arcs = lk.y + lk.w + ws.lstep_eps[(size_t)blockIdx.x * (ws.T_cap + 2) + fstep];
                trim_lattice<BLOCK>(u, fstep, reached, best_t >= 0 ? tinfo[best_t].x : -1, g, ws);
                if (ws.o_meta[6 * (size_t)u] < 0) status = wb_cap(WB_CAP_LATTICE_OUT);
            } else if (threadIdx.x == 0) {
                ws.o_meta[6 * (size_t)u] = -1;
            }
        }
        tick<BLOCK>(7);
        if (threadIdx.x == 0) {
            wb_utt_result r;
            memset(&r, 0, sizeof(r));
            for (int q = 0; q < 8; ++q) r.phase_cycles[q] = sh.pc[q];
#ifdef WB_PROBE
            // probe build: phases 0-6 report thread 0's lane-barrier wait, 7 the total
            for (int q = 0; q < 7; ++q) r.phase_cycles[7] += sh.pc[q];
            for (int q = 0; q < 7; ++q) r.phase_cycles[q] = sh.spin_ph[q];
#endif
            r.total_cost = best_cost;
            r.tokens_expanded = sh.acc[0];
            r.search_steps = steps_run;
            r.reached_final = reached;
            r.died_at_step = died_at;
            r.final_state = best_t >= 0 ? ldx<KC>(&tinfo[best_t]).x : -1;
            r.final_step = died_at < 0 ? steps_run : died_at;
            r.best_trace = best_t >= 0 ? (long long)(u32)ldx<KC>(&tinfo[best_t]).y : -1;
            if (status == WB_OK)  // a failed utterance's tokens / arena are not a valid chain
                backtrace(g, c.arena(), r.best_trace, sh.arena_used, b.olab + (size_t)u * b.lab_cap,
                          b.ilab + (size_t)u * b.lab_cap, b.lab_cap, &r.n_olabels, &r.n_ilabels);
            int capf = status >> 8;
            if (r.n_olabels > b.lab_cap || r.n_ilabels > b.lab_cap) {
                capf |= WB_CAP_LABELS;
                if (status == WB_OK) status = WB_ERR_CAPACITY;
            }
            r.status = status & 0xFF;
            r.capacity_flags = capf;
            r.path_flags = pflags;
            r.n_tok = sh.acc[0];
            r.a_emit = t_emit;
            r.a_fin = t_fin;
            r.a_cas = t_cas;
            r.eps_rounds = sh.acc[4];
            r.e_eps = t_eps;
            r.n_cand = sh.acc[1];
            r.n_surv = sh.acc[2];
            r.n_rec = sh.acc[3];
            r.lat_arcs = lat_arcs;
            res[u] = r;
        }
        __syncthreads();
    }
    if (rank == 0 && threadIdx.x == 0) ws.tag_ctr[slot_id] = tag;
    // no CTA of a cluster may exit while another can still read its shared memory
    if (K > 1) lane_sync<BLOCK>(K, false);
}

}  // namespace wb
