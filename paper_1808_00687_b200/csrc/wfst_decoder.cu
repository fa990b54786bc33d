// wfst_decoder.cu -- host side of the C ABI (include/wfst_b200.h): graph upload, decoder
// workspace, batch launch.  The device code lives in decode_kernel.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/wfst_b200.h"
#include "decode_kernel.cuh"
#include "prune_kernel.cuh"

using namespace wb;

static thread_local std::string g_err;

static int set_err(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int wb_internal_set_error(int code, const char *msg) { return set_err(code, msg); }

#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return set_err(e_ == cudaErrorMemoryAllocation ? WB_ERR_NOMEM : WB_ERR_CUDA,      \
                           std::string(#expr) + ": " + cudaGetErrorString(e_));              \
    } while (0)

struct wb_graph_s {
    int device = 0;
    int S = 0, A = 0, start = 0, has_eps = 0, max_ilabel = 0, nonneg = 1;
    int4 start_rng{0, 0, 0, 0};
    int4 *arcs = nullptr;      // [2*A] 32-byte arc records
    double *final_w = nullptr;
    size_t bytes = 0;
};

struct wb_decoder_s {
    wb_graph_s *g = nullptr;
    int slots = 0, cap = 0, T_cap = 0, block = 0, num_sms = 0;
    int cluster = 0, last_cluster = 1;   // CTAs per lane requested (0 = auto) / used last
    int kmax = 1;   // candidate-side workspace holds slots * kmax CTAs (clusters of kmax CTAs)
    // checked build (-DWB_CHECKS): invariant counters, first violation per lane, claim log
    u32 *chk_claim = nullptr, *chk_seen = nullptr;
    unsigned long long *chk_err = nullptr;
    unsigned short *chk_log = nullptr;
    long long chk_log_cap = 0;
    int *chk_steps = nullptr;
    u64 arena_cap = 0;
    Slot *slot = nullptr;
    u64 *cand_of = nullptr;
    u32 *qtag = nullptr, *tag_ctr = nullptr;
    u32 *cand_state = nullptr, *cand_ca = nullptr;
    u64 *cand_ap = nullptr;
    u64 *cand_key = nullptr;
    u32 *front = nullptr;
    int4 *frng = nullptr;
    int4 *tok_info = nullptr;
    double *tok_cost = nullptr;
    int *frames = nullptr;
    u64 *arena = nullptr;
    u64 *counters = nullptr;  // [0] arena_ctr, [1] utt_ctr (u32 in the low half)
    // host-mode staging buffers (grown on demand)
    double *h_costs = nullptr, *h_blank = nullptr;
    size_t h_costs_n = 0, h_blank_n = 0;
    long long *h_off = nullptr, *h_crow = nullptr;
    size_t h_crow_n = 0;
    int *h_T = nullptr;
    wb_utt_result *h_res = nullptr;
    int *h_lab = nullptr;
    size_t h_off_n = 0, h_T_n = 0, h_res_n = 0, h_lab_n = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // H2D pipeline of a page-locked FSD cost table: step-range chunks on a copy stream, each
    // followed by the per-utterance ready counts the kernel polls (see decode_impl)
    cudaStream_t copy_st = nullptr;
    cudaEvent_t cev_a = nullptr, cev_b = nullptr, cev_c = nullptr;
    int *dma_ready = nullptr;          // device [n] ready counters
    size_t dma_ready_n = 0;
    int *dma_counts = nullptr;         // page-locked host [chunks][n] counts to publish
    size_t dma_counts_n = 0;
    size_t bytes = 0;
    long long last_h2d = 0;   // bytes moved host -> device by the last WB_MEM_HOST call
    int last_zero_copy = 0;
    // lattice mode (allocated on the first lattice decode)
    long long lat_cap = 0, lat_cap_want = 0, lat_out_want = 0;
    int lat_T = 0;
    int *tok_eps = nullptr;
    u32 *sbits = nullptr, *snode = nullptr, *ln_state = nullptr, *ln_out = nullptr;
    unsigned char *ln_flag = nullptr;
    u32 *la_src = nullptr, *la_dst = nullptr, *la_arc = nullptr;
    double *la_ac = nullptr;
    int4 *rlog = nullptr;
    long long rlog_cap = 0;
    int4 *lstep = nullptr;
    int *lstep_eps = nullptr, *lstep_start = nullptr;
    int2 *o_node = nullptr;
    uint4 *o_arc = nullptr;
    double *o_ac = nullptr, *o_finw = nullptr;
    u32 *o_fin = nullptr;
    size_t o_node_n = 0, o_arc_n = 0, o_fin_n = 0, o_meta_n = 0;
    unsigned long long *o_ctr = nullptr;
    long long *o_meta = nullptr;
    int lat_n = 0;                 // utterances of the last lattice decode
    // device lattice-beam pruning (pools sized like the o_* pools; scratch per pool node / arc)
    int2 *p_node = nullptr;
    uint4 *p_arc = nullptr;
    double *p_ac = nullptr, *p_finw = nullptr;
    u32 *p_fin = nullptr;
    u64 *p_fw = nullptr, *p_bw = nullptr;
    unsigned char *p_nflag = nullptr, *p_aflag = nullptr;
    int *p_depth = nullptr, *p_steps = nullptr;
    unsigned long long *p_ctr = nullptr;
    long long *p_meta = nullptr;
    size_t p_node_n = 0, p_arc_n = 0, p_fin_n = 0, p_meta_n = 0, p_steps_n = 0;
    size_t p_fw_n = 0, p_bw_n = 0, p_nflag_n = 0, p_depth_n = 0, p_aflag_n = 0, p_ac_n = 0,
           p_finw_n = 0, p_ctr_n = 0;
    int pruned_n = 0;
    // the last host-mode launch, for wb_decode_finish
    int pend_n = 0, pend_label_cap = 0, pend_lcap = 1, pend_cols = 0, pend_lattice = 0;
    bool pend_zc = false;
    cudaStream_t pend_stream = nullptr;
    cudaStream_t lat_stream = nullptr;
    size_t lat_bytes = 0;
};

extern "C" {

const char *wb_last_error(void) { return g_err.c_str(); }
int wb_version(void) { return 2; }

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
    const int S = d->num_states, A = d->num_arcs;
    if (d->row_ptr[0] != 0 || d->row_ptr[S] != A) return set_err(WB_ERR_VALUE, "row_ptr mismatch");
    int has_eps = 0, max_il = 0, nonneg = 1;
    for (int s = 0; s < S; ++s) {
        int lo = d->row_ptr[s], mid = d->eps_end[s], hi = d->row_ptr[s + 1];
        if (lo > mid || mid > hi) return set_err(WB_ERR_VALUE, "eps_end outside the state's arc range");
        if (mid > lo) has_eps = 1;
    }
    // 32-byte arc records: {dst, ilabel, weight} + the destination's {eps_lo, emit_lo, emit_hi}
    // and the olabel, so relaxation and first touch need no per-state lookups.
    std::vector<int4> arcs(2 * (size_t)std::max(A, 1));
    for (int a = 0; a < A; ++a) {
        int dst = d->dst[a];
        if (dst < 0 || dst >= S) return set_err(WB_ERR_VALUE, "arc destination out of range");
        if (d->ilabel[a] < 0 || d->olabel[a] < 0) return set_err(WB_ERR_VALUE, "negative label");
        long long wbits;
        std::memcpy(&wbits, &d->weight[a], 8);
        arcs[2 * (size_t)a] = make_int4(dst, d->ilabel[a], (int)(wbits & 0xffffffffll), (int)(wbits >> 32));
        arcs[2 * (size_t)a + 1] =
            make_int4(d->row_ptr[dst], d->eps_end[dst], d->row_ptr[dst + 1], d->olabel[a]);
        max_il = std::max(max_il, d->ilabel[a]);
        if (!(d->weight[a] >= 0.0)) nonneg = 0;
    }
    for (int s = 0; s < S; ++s)
        if (std::isnan(d->final_w[s])) return set_err(WB_ERR_VALUE, "NaN final weight");
    CUDA_TRY(cudaSetDevice(device));
    wb_graph_s *g = new wb_graph_s();
    g->device = device;
    g->S = S;
    g->A = A;
    g->start = d->start;
    g->has_eps = has_eps;
    g->max_ilabel = max_il;
    g->nonneg = nonneg;
    g->start_rng = make_int4(d->row_ptr[d->start], d->eps_end[d->start], d->row_ptr[d->start + 1], 0);
    cudaError_t e = cudaMalloc(&g->arcs, sizeof(int4) * arcs.size());
    if (e == cudaSuccess) e = cudaMalloc(&g->final_w, sizeof(double) * S);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->arcs, arcs.data(), sizeof(int4) * arcs.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->final_w, d->final_w, sizeof(double) * S, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(g->arcs);
        cudaFree(g->final_w);
        delete g;
        return set_err(e == cudaErrorMemoryAllocation ? WB_ERR_NOMEM : WB_ERR_CUDA,
                       std::string("graph upload: ") + cudaGetErrorString(e));
    }
    g->bytes = sizeof(int4) * arcs.size() + sizeof(double) * (size_t)S;
    *out = g;
    return WB_OK;
}

int wb_graph_destroy(wb_graph_t g) {
    if (!g) return WB_OK;
    cudaSetDevice(g->device);
    cudaFree(g->arcs);
    cudaFree(g->final_w);
    delete g;
    return WB_OK;
}

int wb_graph_device_bytes(wb_graph_t g, int64_t *bytes) {
    *bytes = (int64_t)g->bytes;
    return WB_OK;
}

}  // extern "C"

static void free_decoder(wb_decoder_s *d) {
    if (d->copy_st) cudaStreamSynchronize(d->copy_st);
    cudaFree(d->dma_ready);
    cudaFreeHost(d->dma_counts);
    for (cudaEvent_t ev : {d->cev_a, d->cev_b, d->cev_c}) if (ev) cudaEventDestroy(ev);
    if (d->copy_st) cudaStreamDestroy(d->copy_st);
    void *chk[] = {d->chk_claim, d->chk_seen, d->chk_err, d->chk_log, d->chk_steps};
    for (void *p : chk) cudaFree(p);
    void *ptrs[] = {d->slot, d->cand_of, d->qtag, d->tag_ctr, d->cand_state,
                    d->cand_ap, d->cand_key, d->cand_ca, d->front, d->frng, d->tok_info,
                    d->tok_cost, d->frames, d->arena, d->counters, d->h_costs, d->h_blank,
                    d->h_off, d->h_crow, d->h_T, d->h_res, d->h_lab, d->tok_eps, d->sbits, d->snode,
                    d->ln_state, d->ln_out, d->ln_flag, d->la_src, d->la_dst, d->la_arc,
                    d->la_ac, d->lstep, d->lstep_eps, d->lstep_start, d->o_node, d->o_arc,
                    d->o_ac, d->o_finw, d->o_fin, d->o_ctr, d->o_meta, d->rlog, d->p_node,
                    d->p_arc, d->p_ac, d->p_finw, d->p_fin, d->p_fw, d->p_bw, d->p_nflag,
                    d->p_aflag, d->p_depth, d->p_steps, d->p_ctr, d->p_meta};
    for (void *p : ptrs) cudaFree(p);
    if (d->ev0) cudaEventDestroy(d->ev0);
    if (d->ev1) cudaEventDestroy(d->ev1);
}

template <class T>
static cudaError_t dalloc(T **p, size_t n, size_t &acc) {
    acc += sizeof(T) * std::max<size_t>(n, 1);
    return cudaMalloc(p, sizeof(T) * std::max<size_t>(n, 1));
}

static int alloc_frames(wb_decoder_s *d, int T_cap) {
    cudaFree(d->frames);
    d->frames = nullptr;
    d->T_cap = std::max(T_cap, 1);
    CUDA_TRY(cudaMalloc(&d->frames, sizeof(int) * (size_t)d->slots * d->T_cap));
#ifdef WB_CHECKS
    cudaFree(d->chk_steps);
    d->chk_steps = nullptr;
    CUDA_TRY(cudaMalloc(&d->chk_steps, sizeof(int) * (size_t)d->slots * (d->T_cap + 1)));
#endif
    return WB_OK;
}

static int alloc_arena(wb_decoder_s *d, u64 cap) {
    cudaFree(d->arena);
    d->arena = nullptr;
    d->arena_cap = std::min<u64>(std::max<u64>(cap, 1024), (u64)EPS_BIT - 1);  // per lane
    CUDA_TRY(cudaMalloc(&d->arena, sizeof(u64) * d->arena_cap * (size_t)d->slots));
    return WB_OK;
}

// Lattice workspace: per-lane raw node / arc pools (lat_cap each), per-step metadata and the
// survivor tags; allocated on the first lattice decode so plain decoding pays nothing.
static int alloc_lattice(wb_decoder_s *d) {
    void *ptrs[] = {d->tok_eps, d->sbits, d->snode, d->ln_state, d->ln_out, d->ln_flag,
                    d->la_src, d->la_dst, d->la_arc, d->la_ac, d->lstep, d->lstep_eps,
                    d->lstep_start, d->o_ctr, d->rlog};
    for (void *p : ptrs) cudaFree(p);
    d->tok_eps = nullptr; d->sbits = d->ln_state = d->ln_out = nullptr; d->snode = nullptr; d->rlog = nullptr;
    d->ln_flag = nullptr; d->la_src = d->la_dst = d->la_arc = nullptr; d->la_ac = nullptr;
    d->lstep = nullptr; d->lstep_eps = d->lstep_start = nullptr; d->o_ctr = nullptr;
    d->lat_cap = 0;
    const size_t slots = (size_t)d->slots, S = (size_t)d->g->S, cap = (size_t)d->cap;
    const long long want = d->lat_cap_want > 0 ? d->lat_cap_want
                                               : std::min<long long>((long long)(d->T_cap + 1) * std::min<long long>(d->cap, 4096), 1ll << 22);
    const size_t L = (size_t)std::max<long long>(want, 1024), TS = (size_t)d->T_cap + 2;
    size_t acc = 0;
    cudaError_t e = cudaSuccess;
#define DA(p, n) if (e == cudaSuccess) e = dalloc(&d->p, (n), acc)
    DA(tok_eps, slots * 2 * cap);
    DA(sbits, slots * ((S + 31) / 32));
    DA(snode, slots * S);
    d->rlog_cap = std::min<long long>((long long)L, 16ll * (long long)cap);
    DA(rlog, slots * (size_t)d->rlog_cap);
    DA(ln_state, slots * L);
    DA(ln_out, slots * L);
    DA(ln_flag, slots * L);
    DA(la_src, slots * L);
    DA(la_dst, slots * L);
    DA(la_arc, slots * L);
    DA(la_ac, slots * L);
    DA(lstep, slots * TS);
    DA(lstep_eps, slots * TS);
    DA(lstep_start, slots);
    DA(o_ctr, 4);
#undef DA
    if (e == cudaSuccess) e = cudaMemset(d->sbits, 0, sizeof(u32) * slots * ((S + 31) / 32));
    if (e != cudaSuccess)
        return set_err(e == cudaErrorMemoryAllocation ? WB_ERR_NOMEM : WB_ERR_CUDA,
                       std::string("lattice workspace: ") + cudaGetErrorString(e));
    d->lat_cap = (long long)L;
    d->lat_T = d->T_cap;
    d->lat_bytes = acc;
    return WB_OK;
}

template <int BLOCK, int K>
static cudaError_t launch_decode(int max_grid, int num_sms, int num_cols, cudaStream_t st,
                                 const GraphDev &gd, WorkDev wd, const BatchDev &bd,
                                 const CfgDev &cd, wb_utt_result *res, bool zero_copy) {
    // One lane per SM: dynamic shared memory holds the cost row during expansion, then the
    // step's candidate keys + flags (as many as fit; larger steps spill to global memory).
    // lift the 48 KB default first: the occupancy query honours the current attribute
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(decode_kernel<BLOCK, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    size_t avail = 0;
    e = cudaOccupancyAvailableDynamicSMemPerBlock(&avail, decode_kernel<BLOCK, K>, 1, BLOCK);
    if (e != cudaSuccess) return e;
    const size_t hdr = smem_hdr<BLOCK>();
    // Cap the carve-out at 100 KB: the rest of the SM's 256 KB stays L1 for the graph's arc
    // records and the call stack.  Measured (config 2): 48-160 KB all ~207 ms, the full 227 KB
    // 331 ms (L1 shrinks to 28 KB and stack reloads miss).  WB_SMEM_KB overrides (tuning).
    size_t cap = 100 * 1024;
    if (const char *cap_kb = std::getenv("WB_SMEM_KB")) cap = (size_t)std::atoi(cap_kb) * 1024;
    if (cap > 0 && cap < avail) avail = cap;
    avail = avail > 1024 + hdr ? avail - 1024 - hdr : 0;
    size_t row = num_cols <= ROW_SMEM_MAX ? sizeof(double) * (size_t)num_cols : 0;
    if (row > avail) row = 0;  // the kernel reads the row from global memory instead
    if (zero_copy && row == 0) return cudaErrorNotSupported;  // host rows must be staged
    // K CTAs per lane (a thread-block cluster): CTA r owns candidate indices [r*cap, (r+1)*cap)
    wd.K = K;
    wd.kshift = K >= 8 ? 3 : K >= 4 ? 2 : K >= 2 ? 1 : 0;
    wd.lcap = K * wd.cap;
    wd.smem_cands = (int)std::min<size_t>(avail / (sizeof(u64) + sizeof(u32)), (size_t)wd.cap);
    // WB_SMEM_CANDS caps the candidates kept in shared memory (tests force the global path)
    if (const char *sc = std::getenv("WB_SMEM_CANDS")) wd.smem_cands = std::min(wd.smem_cands, std::max(0, std::atoi(sc)));
    wd.row_in_smem = row > 0;
    if (wd.log_rows && !wd.row_in_smem) return cudaErrorNotSupported;   // log(p) rows are negated as staged
    // per-lane arc prefetch buffers (2 x 16 B) after the staged row, when they fit
    const size_t row_r = (row + 127) & ~(size_t)127, stage = (size_t)BLOCK * 32;
    const char *pf = std::getenv("WB_PREFETCH");
    wd.stage_off = (row > 0 && row_r + stage <= avail && !(pf && pf[0] == '0')) ? (int)(hdr + row_r) : 0;
    const char *bs = std::getenv("WB_BEAM_SKIP");
    wd.beam_skip = (bs && bs[0] == '0') ? 0 : 1;
    const char *em = std::getenv("WB_EXACT_MIN");
    wd.exact_min = (em && em[0] == '0') ? 0 : 1;
    const char *xg = std::getenv("WB_XCHG_GATHER");
    wd.xchg_gather = xg ? std::atoi(xg) : 2;
    const char *ed = std::getenv("WB_EPS_DEDUP");
    wd.eps_dedup = ed ? std::atoi(ed) : 1;
    const char *ma = std::getenv("WB_MA_EARLY");
    wd.ma_early = ma ? std::atoi(ma) : 0;
    const char *fr = std::getenv("WB_FORCE_RADIX");  // tests: rank every boundary bucket by radix select
    wd.force_radix = (fr && fr[0] == '1') ? 1 : 0;
    const char *ci = std::getenv("WB_CHECK_INJECT");
    wd.chk_inject = ci && ci[0] == '1';
    const char *rp = std::getenv("WB_ROW_PREFETCH");
    wd.row_prefetch = !zero_copy && !bd.ready && !bd.crow_off && !(rp && rp[0] == '0');
    size_t smem = hdr + std::max(wd.stage_off ? row_r + stage : row,
                                 (size_t)wd.smem_cands * (sizeof(u64) + sizeof(u32)));
    smem = (smem + 15) & ~(size_t)15;
    e = cudaFuncSetAttribute(decode_kernel<BLOCK, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return e;
    if (K == 1) {
        int occ = 1;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, decode_kernel<BLOCK, K>, BLOCK, smem);
        if (e != cudaSuccess) return e;
        int grid = std::min(max_grid, num_sms * std::max(occ, 1));
        decode_kernel<BLOCK, K><<<grid, BLOCK, smem, st>>>(gd, wd, bd, cd, res);
        return cudaGetLastError();
    }
    // cluster lanes: as many K-CTA clusters as fit at once (each CTA on its own SM of a GPC)
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)K;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.blockDim = dim3(BLOCK);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    lc.attrs = at;
    lc.numAttrs = 1;
    lc.gridDim = dim3((unsigned)(max_grid * K));
    int clusters = 0;
    e = cudaOccupancyMaxActiveClusters(&clusters, decode_kernel<BLOCK, K>, &lc);
    if (e != cudaSuccess) return e;
    if (clusters < 1) return cudaErrorNotSupported;
    lc.gridDim = dim3((unsigned)(std::min(max_grid, clusters) * K));
    e = cudaLaunchKernelEx(&lc, decode_kernel<BLOCK, K>, gd, wd, bd, cd, res);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <class T>
static int grow(T **p, size_t &have, size_t need) {
    need = std::max<size_t>(need, 1);
    if (need <= have && *p) return WB_OK;
    cudaFree(*p);
    *p = nullptr;
    have = 0;
    CUDA_TRY(cudaMalloc(p, sizeof(T) * need));
    have = need;
    return WB_OK;
}

extern "C" {

int wb_decoder_create(wb_graph_t g, const wb_decoder_opts *o, wb_decoder_t *out) {
    if (!g || !out) return set_err(WB_ERR_VALUE, "null argument");
    CUDA_TRY(cudaSetDevice(g->device));
    wb_decoder_opts opts;
    std::memset(&opts, 0, sizeof(opts));
    if (o) opts = *o;
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, g->device));
    if (opts.block_threads && opts.block_threads != 256 && opts.block_threads != 512 &&
        opts.block_threads != 1024)
        return set_err(WB_ERR_VALUE, "block_threads must be 256, 512 or 1024 (or 0 = auto)");
    wb_decoder_s *d = new wb_decoder_s();
    d->g = g;
    d->num_sms = prop.multiProcessorCount;
    d->block = opts.block_threads;
    d->cluster = opts.cluster_ctas;
    d->cap = opts.cand_capacity > 0 ? opts.cand_capacity : std::min(g->S, 1 << 18);
    d->cap = std::max(1, std::min(d->cap, g->S));
    // one persistent lane per SM (the kernel's shared-memory candidate store fills an SM) --
    // unless the dense per-state arrays of that many lanes do not fit in device memory (a
    // large graph: S x 24 B per lane): then fewer lanes, each a cluster of 2 or 4 CTAs, so the
    // SMs still fill
    d->slots = opts.max_utts_in_flight > 0 ? opts.max_utts_in_flight : d->num_sms;
    if (opts.max_utts_in_flight <= 0) {
        size_t free_b = 0, total_b = 0;
        CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
        double budget = 0.75 * (double)free_b;
        if (const char *mb = std::getenv("WB_MEM_BUDGET_GB")) budget = std::atof(mb) * 1e9;
        const double per_lane = (double)g->S * (sizeof(Slot) + (g->has_eps ? sizeof(u64) + sizeof(u32) : 0)) +
                                (double)sizeof(u64) * (4 << 20);   // dense slots (+ eps maps), default arena
        const double per_cta = (double)d->cap * 96.0;               // candidate / token / frontier regions
        auto fits = [&](int lanes, int k) { return lanes * per_lane + lanes * k * per_cta <= budget; };
        int lanes = d->num_sms, k = 1;
        while (k <= 4 && !fits(lanes = std::max(1, d->num_sms / k), k)) k *= 2;   // smallest K that fits
        if (k > 4)
            while (lanes > 1 && !fits(lanes, 4)) --lanes;
        d->slots = lanes;
    }
    // cluster lanes: when the lanes leave SMs idle, a lane may be a cluster of up to 4 CTAs
    // (8 on request), each with its own candidate / token / frontier region
    d->kmax = std::max(1, opts.cluster_ctas);
    while (d->kmax < 4 && d->slots * d->kmax * 2 <= d->num_sms) d->kmax *= 2;
    size_t S = (size_t)g->S, slots = (size_t)d->slots, cap = (size_t)d->cap;
    const size_t cslots = slots * (size_t)d->kmax;   // CTAs with candidate workspace
    size_t acc = 0;
    cudaError_t e = cudaSuccess;
#define DA(p, n) if (e == cudaSuccess) e = dalloc(&d->p, (n), acc)
    DA(slot, slots * S);
    DA(cand_of, g->has_eps ? slots * S : 1);
    DA(qtag, g->has_eps ? slots * S : 1);
    DA(tag_ctr, slots);
    DA(cand_state, cslots * cap);
    DA(cand_ap, cslots * cap);
    DA(cand_key, cslots * cap);
    DA(cand_ca, cslots * cap);
    DA(front, cslots * 2 * cap);
    DA(frng, g->has_eps ? cslots * 2 * cap : 1);
    DA(tok_info, cslots * 2 * cap);
    DA(tok_cost, cslots * 2 * cap);
    DA(counters, 4);
#ifdef WB_CHECKS
    d->chk_log_cap = 1ll << 20;   // claim-log entries (tokens expanded) per lane
    if (const char *lc = std::getenv("WB_CHECK_LOG")) d->chk_log_cap = std::atoll(lc);
    DA(chk_claim, cslots * cap);
    DA(chk_seen, slots * S);
    DA(chk_err, slots);
    DA(chk_log, slots * (size_t)d->chk_log_cap);
#endif
#undef DA
    if (e == cudaSuccess) e = cudaMemset(d->slot, 0xFF, sizeof(Slot) * slots * S);
    if (e == cudaSuccess && g->has_eps) e = cudaMemset(d->qtag, 0, sizeof(u32) * slots * S);
    // stamp 0xFFFFFFFF: no step's (the lane's tags start at 0)
    if (e == cudaSuccess && g->has_eps) e = cudaMemset(d->cand_of, 0xFF, sizeof(u64) * slots * S);
    if (e == cudaSuccess) e = cudaMemset(d->tag_ctr, 0, sizeof(u32) * slots);
#ifdef WB_CHECKS
    if (e == cudaSuccess) e = cudaMemset(d->chk_claim, 0, sizeof(u32) * cslots * cap);
    if (e == cudaSuccess) e = cudaMemset(d->chk_seen, 0, sizeof(u32) * slots * S);
    if (e == cudaSuccess) e = cudaMemset(d->chk_err, 0, sizeof(unsigned long long) * slots);
#endif
    if (e == cudaSuccess) e = cudaEventCreate(&d->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&d->ev1);
    if (e != cudaSuccess) {
        free_decoder(d);
        delete d;
        return set_err(e == cudaErrorMemoryAllocation ? WB_ERR_NOMEM : WB_ERR_CUDA,
                       std::string("decoder workspace: ") + cudaGetErrorString(e));
    }
    d->bytes = acc;
    d->lat_cap_want = opts.lattice_capacity;
    d->lat_out_want = opts.lattice_out_capacity;
    int rc = alloc_frames(d, opts.max_frames > 0 ? opts.max_frames : 2048);
    if (rc == WB_OK)
        rc = alloc_arena(d, opts.arena_capacity > 0 ? (u64)opts.arena_capacity : (u64)1 << 22);
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
    *bytes = (int64_t)(d->bytes + sizeof(int) * (size_t)d->slots * d->T_cap +
                       sizeof(u64) * d->arena_cap * (size_t)d->slots + d->lat_bytes +
                       sizeof(int2) * d->o_node_n + (sizeof(uint4) + sizeof(double)) * d->o_arc_n +
                       (sizeof(u32) + sizeof(double)) * d->o_fin_n);
    return WB_OK;
}

int wb_checks_enabled(void) {
#ifdef WB_CHECKS
    return 1;
#else
    return 0;
#endif
}

int wb_check_report(wb_decoder_t d, int32_t n_lanes, int64_t *first_violation) {
    if (!d || !first_violation || n_lanes < 0) return set_err(WB_ERR_VALUE, "bad argument");
    const int n = std::min(n_lanes, d->slots);
    for (int i = 0; i < n_lanes; ++i) first_violation[i] = 0;
    if (!d->chk_err || n == 0) return WB_OK;
    CUDA_TRY(cudaSetDevice(d->g->device));
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(first_violation, d->chk_err, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemset(d->chk_err, 0, sizeof(unsigned long long) * d->slots));
    return WB_OK;
}

int wb_claim_log(wb_decoder_t d, int32_t lane, int32_t n_steps, int32_t *queue_len,
                 uint16_t *groups, int64_t groups_cap, int64_t *n_logged) {
    if (!d || !queue_len || !groups || !n_logged) return set_err(WB_ERR_VALUE, "null argument");
    *n_logged = 0;
    if (!d->chk_log) return set_err(WB_ERR_VALUE, "claim logs need the checked library");
    if (lane < 0 || lane >= d->slots || n_steps < 0 || n_steps > d->T_cap + 1)
        return set_err(WB_ERR_VALUE, "lane / step count out of range");
    CUDA_TRY(cudaSetDevice(d->g->device));
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(queue_len, d->chk_steps + (size_t)lane * (d->T_cap + 1),
                        sizeof(int) * n_steps, cudaMemcpyDeviceToHost));
    long long tot = 0;
    for (int s = 0; s < n_steps; ++s) tot += queue_len[s];
    const long long n = std::min<long long>(std::min<long long>(tot, d->chk_log_cap), groups_cap);
    if (n > 0)
        CUDA_TRY(cudaMemcpy(groups, d->chk_log + (size_t)lane * d->chk_log_cap,
                            sizeof(uint16_t) * n, cudaMemcpyDeviceToHost));
    *n_logged = n;
    return WB_OK;
}

int wb_decoder_lanes(wb_decoder_t d, int32_t *lanes, int32_t *max_cluster) {
    if (!d || !lanes || !max_cluster) return set_err(WB_ERR_VALUE, "null argument");
    *lanes = d->slots;
    *max_cluster = d->kmax;
    return WB_OK;
}

int wb_last_launch(wb_decoder_t d, int32_t *cluster_ctas) {
    if (!d || !cluster_ctas) return set_err(WB_ERR_VALUE, "null argument");
    *cluster_ctas = d->last_cluster;
    return WB_OK;
}

int wb_last_kernel_ms(wb_decoder_t d, float *ms) {
    CUDA_TRY(cudaEventElapsedTime(ms, d->ev0, d->ev1));
    return WB_OK;
}

}  // extern "C"

static int finish_impl(wb_decoder_t d, wb_utt_result *results, int32_t *olabels, int32_t *ilabels);

// The body of wb_decode / wb_decode_stream.  `ready` (streaming, host mode only): page-locked
// per-utterance counts of frames whose cost rows are written; `defer` leaves the result copy
// and the synchronisation to wb_decode_finish.
static int decode_impl(wb_decoder_t d, int32_t n, const double *costs, const int64_t *row_offset,
                       const int32_t *num_frames, int32_t num_cols, const double *blank,
                       const wb_config *cfg, wb_utt_result *results, int32_t *olabels,
                       int32_t *ilabels, int32_t label_cap, int32_t memory_kind, void *stream,
                       const int32_t *ready, bool defer, const int64_t *crow = nullptr) {
    if (!d || !cfg) return set_err(WB_ERR_VALUE, "null argument");
    if (n < 0 || num_cols < 1 || label_cap < 0) return set_err(WB_ERR_VALUE, "bad batch dimensions");
    if (cfg->beam < 0 || std::isnan(cfg->beam)) return set_err(WB_ERR_VALUE, "beam must be >= 0");
    if (cfg->max_active < 0) return set_err(WB_ERR_VALUE, "max_active must be >= 1 or 0 (None)");
    if (cfg->mode != 0 && cfg->mode != 1)
        return set_err(WB_ERR_VALUE, "mode must be 0 (fsd) or 1 (lsd)");
    wb_graph_s *g = d->g;
    if (g->max_ilabel > num_cols - 1)
        return set_err(WB_ERR_VALUE, "graph uses input label " + std::to_string(g->max_ilabel) +
                                         " but the posterior matrix only covers labels 1.." +
                                         std::to_string(num_cols - 1));
    CUDA_TRY(cudaSetDevice(g->device));
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) return WB_OK;
    const bool host = memory_kind == WB_MEM_HOST;
    bool zc = false;
    const double *zc_ptr = nullptr;
    const int *ready_dev = nullptr;
    const double *dc = costs, *db = blank;
    const long long *doff = (const long long *)row_offset;
    const int *dT = num_frames;
    wb_utt_result *dres = results;
    int *dol = olabels, *dil = ilabels;
    const int lcap = std::max(label_cap, 1);
    bool dma = false;   // H2D pipeline of the cost table (below)
    if (host) {
        int maxT = 0;
        long long rows = 0;
        for (int i = 0; i < n; ++i) {
            if (num_frames[i] < 0 || row_offset[i] < 0)
                return set_err(WB_ERR_VALUE, "negative frame count / offset");
            maxT = std::max(maxT, num_frames[i]);
            rows = std::max<long long>(rows, row_offset[i] + num_frames[i]);
        }
        if (maxT > d->T_cap) {
            int rc = alloc_frames(d, maxT);
            if (rc) return rc;
        }
        size_t ncost = (size_t)rows * num_cols, nn = (size_t)n;
        int rc;
        if ((rc = grow(&d->h_costs, d->h_costs_n, ncost))) return rc;
        if ((rc = grow(&d->h_blank, d->h_blank_n, (size_t)rows))) return rc;
        if ((rc = grow(&d->h_off, d->h_off_n, nn))) return rc;
        if ((rc = grow(&d->h_T, d->h_T_n, nn))) return rc;
        if ((rc = grow(&d->h_res, d->h_res_n, nn))) return rc;
        if ((rc = grow(&d->h_lab, d->h_lab_n, nn * lcap * 2))) return rc;
        // Zero-copy: a page-locked cost table is read by the kernel straight from host memory,
        // one staged row per search step, so the transfer overlaps the search and LSD reads
        // only non-blank rows.  Pageable tables (or rows too wide to stage) are copied first.
        zc = false;
        const char *zc_env = std::getenv("WB_ZERO_COPY");
        if (ncost && !(zc_env && zc_env[0] == '0')) {
            cudaPointerAttributes pa;
            if (cudaPointerGetAttributes(&pa, costs) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                pa.devicePointer)
                zc = true, zc_ptr = (const double *)pa.devicePointer;
            else
                cudaGetLastError();
        }
        if (ready) {
            cudaPointerAttributes pr;
            if (!zc || cudaPointerGetAttributes(&pr, ready) != cudaSuccess ||
                pr.type != cudaMemoryTypeHost || !pr.devicePointer) {
                cudaGetLastError();
                return set_err(WB_ERR_VALUE, "streaming decode needs page-locked cost and ready buffers");
            }
            ready_dev = (const int *)pr.devicePointer;
        }
        // H2D pipeline (FSD, page-locked table, every utterance T rows at a common stride): the
        // copy engine moves step-range chunks of all utterances into device memory while the
        // kernel runs, publishing per-utterance ready counts after each chunk; the kernel reads
        // its rows from HBM instead of staging each one over PCIe.  WB_H2D_PIPELINE=0: off.
        const char *dp = std::getenv("WB_H2D_PIPELINE");
        if (zc && !ready && cfg->mode == 0 && n > 0 && !(dp && dp[0] == '0')) {
            const long long T0 = num_frames[0], stride = n > 1 ? row_offset[1] - row_offset[0] : T0;
            dma = T0 > 0 && stride >= T0;
            for (int i = 0; i < n && dma; ++i)
                dma = num_frames[i] == T0 && row_offset[i] == row_offset[0] + (long long)i * stride;
        }
        if (dma) {
            const int T0 = num_frames[0];
            const long long stride = n > 1 ? row_offset[1] - row_offset[0] : T0;
            // chunk boundaries in steps: 8, 16, then 32-step chunks (the first rows land fast)
            std::vector<int> cut{0};
            for (int c = 8; cut.back() < T0; c = std::min(32, c * 2)) cut.push_back(std::min(T0, cut.back() + c));
            const size_t nch = cut.size() - 1;
            if (!d->copy_st) {
                CUDA_TRY(cudaStreamCreateWithFlags(&d->copy_st, cudaStreamNonBlocking));
                CUDA_TRY(cudaEventCreateWithFlags(&d->cev_a, cudaEventDisableTiming));
                CUDA_TRY(cudaEventCreateWithFlags(&d->cev_b, cudaEventDisableTiming));
                CUDA_TRY(cudaEventCreateWithFlags(&d->cev_c, cudaEventDisableTiming));
            }
            if ((rc = grow(&d->dma_ready, d->dma_ready_n, nn))) return rc;
            CUDA_TRY(cudaStreamSynchronize(d->copy_st));   // the host counts below are reused
            if (d->dma_counts_n < nch * nn) {
                cudaFreeHost(d->dma_counts);
                d->dma_counts = nullptr;
                d->dma_counts_n = 0;
                CUDA_TRY(cudaMallocHost(&d->dma_counts, sizeof(int) * nch * nn));
                d->dma_counts_n = nch * nn;
            }
            for (size_t k = 0; k < nch; ++k)
                for (size_t i = 0; i < nn; ++i) d->dma_counts[k * nn + i] = cut[k + 1];
            // the copies overwrite the device table only after the work queued before this call
            // (a previous decode reading it) is done; the kernel starts after the counts are zero
            CUDA_TRY(cudaEventRecord(d->cev_a, st));
            CUDA_TRY(cudaStreamWaitEvent(d->copy_st, d->cev_a, 0));
            CUDA_TRY(cudaMemsetAsync(d->dma_ready, 0, sizeof(int) * nn, d->copy_st));
            CUDA_TRY(cudaEventRecord(d->cev_b, d->copy_st));
            // in the order the lanes consume them: a wave of `slots` utterances (the lanes take
            // utterances from a queue in index order) at a time, its step chunks in turn
            const size_t rowb = sizeof(double) * (size_t)num_cols, pitch = rowb * (size_t)stride;
            const size_t wave = (size_t)std::max(1, d->slots);
            for (size_t u0 = 0; u0 < nn; u0 += wave) {
                const size_t nu = std::min(wave, nn - u0);
                for (size_t k = 0; k < nch; ++k) {
                    const size_t off = rowb * ((size_t)row_offset[u0] + (size_t)cut[k]);
                    CUDA_TRY(cudaMemcpy2DAsync(reinterpret_cast<char *>(d->h_costs) + off, pitch,
                                               reinterpret_cast<const char *>(costs) + off, pitch,
                                               rowb * (size_t)(cut[k + 1] - cut[k]), nu,
                                               cudaMemcpyHostToDevice, d->copy_st));
                    CUDA_TRY(cudaMemcpyAsync(d->dma_ready + u0, d->dma_counts + k * nn + u0,
                                             sizeof(int) * nu, cudaMemcpyHostToDevice, d->copy_st));
                }
            }
            CUDA_TRY(cudaEventRecord(d->cev_c, d->copy_st));
            CUDA_TRY(cudaStreamWaitEvent(st, d->cev_b, 0));
            zc = false;
            ready_dev = d->dma_ready;
        }
        if (ncost && !zc && !dma)
            CUDA_TRY(cudaMemcpyAsync(d->h_costs, costs, sizeof(double) * ncost, cudaMemcpyHostToDevice, st));
        d->last_h2d = (long long)(sizeof(double) * (zc ? 0 : ncost) + sizeof(double) * rows +
                                  (sizeof(long long) + sizeof(int)) * nn);
        if (rows)
            CUDA_TRY(cudaMemcpyAsync(d->h_blank, blank, sizeof(double) * rows, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(d->h_off, row_offset, sizeof(long long) * n, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(d->h_T, num_frames, sizeof(int) * n, cudaMemcpyHostToDevice, st));
        dc = zc ? zc_ptr : d->h_costs; db = d->h_blank; doff = d->h_off; dT = d->h_T; dres = d->h_res;
        dol = d->h_lab; dil = d->h_lab + nn * lcap;
    }
    // device mode: frame counts stay on the device; an LSD utterance longer than the frame
    // list capacity reports WB_ERR_CAPACITY (callers size it with max_frames)
    CUDA_TRY(cudaMemsetAsync(d->counters, 0, sizeof(u64) * 4, st));
    GraphDev gd{g->S, g->A, g->start, g->has_eps, g->start_rng, g->arcs, g->final_w, g->nonneg};
    WorkDev wd;
    std::memset(&wd, 0, sizeof(wd));
    wd.slot = d->slot; wd.cand_of = d->cand_of; wd.qtag = d->qtag; wd.tag_ctr = d->tag_ctr;
    wd.cand_state = d->cand_state; wd.cand_ap = d->cand_ap; wd.cand_key = d->cand_key; wd.cand_ca = d->cand_ca;
    wd.front = d->front; wd.frng = d->frng; wd.tok_info = d->tok_info; wd.tok_cost = d->tok_cost;
    wd.frames = d->frames;
    wd.arena = d->arena; wd.arena_cap = d->arena_cap;
    wd.chk_claim = d->chk_claim; wd.chk_seen = d->chk_seen; wd.chk_err = d->chk_err;
    wd.chk_log = d->chk_log; wd.chk_log_cap = d->chk_log_cap; wd.chk_steps = d->chk_steps;
    wd.utt_ctr = reinterpret_cast<u32 *>(d->counters + 1);
    wd.S = g->S; wd.cap = d->cap; wd.T_cap = d->T_cap;
    if (cfg->lattice) {
        if (!d->la_src || d->lat_T < d->T_cap) {
            int rc = alloc_lattice(d);
            if (rc) return rc;
        }
        const size_t out = (size_t)(d->lat_out_want > 0 ? d->lat_out_want : (1ll << 22));
        int rc;
        if ((rc = grow(&d->o_node, d->o_node_n, out))) return rc;
        if ((rc = grow(&d->o_arc, d->o_arc_n, out))) return rc;
        size_t have = d->o_arc_n;
        if ((rc = grow(&d->o_ac, have, out))) return rc;
        if ((rc = grow(&d->o_fin, d->o_fin_n, out))) return rc;
        have = d->o_fin_n;
        if ((rc = grow(&d->o_finw, have, out))) return rc;
        if ((rc = grow(&d->o_meta, d->o_meta_n, (size_t)n * 6))) return rc;
        CUDA_TRY(cudaMemsetAsync(d->o_ctr, 0, sizeof(unsigned long long) * 4, st));
        wd.tok_eps = d->tok_eps; wd.sbits = d->sbits; wd.snode = d->snode; wd.rlog = d->rlog; wd.rlog_cap = d->rlog_cap;
        wd.ln_state = d->ln_state; wd.ln_flag = d->ln_flag; wd.ln_out = d->ln_out;
        wd.la_src = d->la_src; wd.la_dst = d->la_dst; wd.la_arc = d->la_arc; wd.la_ac = d->la_ac;
        wd.lat_cap = d->lat_cap; wd.lstep = d->lstep; wd.lstep_eps = d->lstep_eps;
        wd.lstep_start = d->lstep_start;
        wd.o_node = d->o_node; wd.o_arc = d->o_arc; wd.o_ac = d->o_ac; wd.o_fin = d->o_fin;
        wd.o_finw = d->o_finw; wd.o_node_cap = (long long)d->o_node_n;
        wd.o_arc_cap = (long long)d->o_arc_n; wd.o_fin_cap = (long long)d->o_fin_n;
        wd.o_ctr = d->o_ctr; wd.o_meta = d->o_meta;
        d->lat_n = n;
        d->lat_stream = st;
    }
    const long long *crow_dev = nullptr;
    if (crow) {  // compacted-row streaming (LSD): per-utterance row offsets to the device
        int rc;
        if ((rc = grow(&d->h_crow, d->h_crow_n, (size_t)n))) return rc;
        CUDA_TRY(cudaMemcpyAsync(d->h_crow, crow, sizeof(long long) * n, cudaMemcpyHostToDevice, st));
        crow_dev = d->h_crow;
    }
    BatchDev bd{dc, doff, dT, db, num_cols, n, dol, dil, lcap, ready_dev, crow_dev};
    CfgDev cd{cfg->beam, cfg->blank_threshold, cfg->max_active, cfg->mode, cfg->lattice};
    wd.log_rows = cfg->log_rows ? 1 : 0;
    const bool prune = cfg->lattice && cfg->lattice_beam >= 0;
    if (cfg->lattice && !(cfg->lattice_beam < 0) && std::isnan(cfg->lattice_beam))
        return set_err(WB_ERR_VALUE, "lattice_beam must be >= 0");
    d->pruned_n = 0;
    if (prune) {
        // Size the prune pools BEFORE the decode launch: cudaFree synchronises the device, and a
        // streaming decode's kernel may be waiting for cost rows the caller publishes only
        // after this call returns.
        const size_t nn = d->o_node_n, na = d->o_arc_n, nf = d->o_fin_n;
        const size_t T2 = (size_t)d->T_cap + 3;
        int rc;
        if ((rc = grow(&d->p_node, d->p_node_n, nn)) || (rc = grow(&d->p_arc, d->p_arc_n, na)) ||
            (rc = grow(&d->p_ac, d->p_ac_n, na)) || (rc = grow(&d->p_fin, d->p_fin_n, nf)) ||
            (rc = grow(&d->p_finw, d->p_finw_n, nf)) || (rc = grow(&d->p_fw, d->p_fw_n, nn)) ||
            (rc = grow(&d->p_bw, d->p_bw_n, nn)) || (rc = grow(&d->p_nflag, d->p_nflag_n, nn + 4)) ||
            (rc = grow(&d->p_depth, d->p_depth_n, nn)) || (rc = grow(&d->p_aflag, d->p_aflag_n, na)) ||
            (rc = grow(&d->p_steps, d->p_steps_n, (size_t)n * T2 * 3)) ||
            (rc = grow(&d->p_ctr, d->p_ctr_n, 4)) || (rc = grow(&d->p_meta, d->p_meta_n, (size_t)n * 8)))
            return rc;
    }
    // 1024 threads per CTA, one persistent CTA (utterance lane) per SM; with fewer utterances
    // than SMs a lane becomes a cluster of K CTAs so the idle SMs share the search
    int block = d->block ? d->block : 1024;
    int max_grid = std::min(n, d->slots);
    int K = d->cluster;
    if (const char *kc = std::getenv("WB_CLUSTER")) K = std::atoi(kc);
    if (K <= 0) {   // auto: the largest K in {1, 2, 4} with max_grid * K CTAs within the SMs
        K = 1;
        while (K < 4 && max_grid * K * 2 <= d->num_sms) K *= 2;
    }
    if (K != 1 && K != 2 && K != 4 && K != 8)
        return set_err(WB_ERR_VALUE, "cluster_ctas must be 1, 2, 4 or 8 (0 = auto)");
    if (cfg->lattice || block != 1024) K = 1;   // lattice recording / tuning blocks: one CTA per lane
    // a lane of K CTAs uses K CTAs' worth of candidate / token workspace
    max_grid = std::min(max_grid, std::max(1, d->slots * d->kmax / K));
    d->last_cluster = K;
    CUDA_TRY(cudaEventRecord(d->ev0, st));
    cudaError_t e;
    auto launch = [&]() {
        switch (block) {
            case 256: return launch_decode<256, 1>(max_grid, d->num_sms, num_cols, st, gd, wd, bd, cd, dres, zc);
            case 512: return launch_decode<512, 1>(max_grid, d->num_sms, num_cols, st, gd, wd, bd, cd, dres, zc);
            default:
                switch (K) {
                    case 2: return launch_decode<1024, 2>(max_grid, d->num_sms, num_cols, st, gd, wd, bd, cd, dres, zc);
                    case 4: return launch_decode<1024, 4>(max_grid, d->num_sms, num_cols, st, gd, wd, bd, cd, dres, zc);
                    case 8: return launch_decode<1024, 8>(max_grid, d->num_sms, num_cols, st, gd, wd, bd, cd, dres, zc);
                    default: return launch_decode<1024, 1>(max_grid, d->num_sms, num_cols, st, gd, wd, bd, cd, dres, zc);
                }
        }
    };
    e = launch();
    if (e == cudaErrorNotSupported && zc && ready_dev)
        return set_err(WB_ERR_VALUE, "streaming decode: cost rows too wide to stage in shared memory");
    if (e == cudaErrorNotSupported && zc) {  // rows too wide to stage: copy the table instead
        zc = false;
        long long rows = 0;
        for (int i = 0; i < n; ++i) rows = std::max<long long>(rows, row_offset[i] + num_frames[i]);
        const size_t ncost = (size_t)rows * num_cols;
        CUDA_TRY(cudaMemcpyAsync(d->h_costs, costs, sizeof(double) * ncost, cudaMemcpyHostToDevice, st));
        d->last_h2d += (long long)(sizeof(double) * ncost);
        bd.costs = d->h_costs;
        e = launch();
    }
    d->last_zero_copy = zc ? 1 : dma ? 2 : 0;
    // the call's stream completes only after the whole table copy (the next call may reuse it)
    if (dma) CUDA_TRY(cudaStreamWaitEvent(st, d->cev_c, 0));
    if (e == cudaSuccess && prune) {
        const size_t T2 = (size_t)d->T_cap + 3;
        CUDA_TRY(cudaMemsetAsync(d->p_ctr, 0, sizeof(unsigned long long) * 4, st));
        PruneDev P;
        std::memset(&P, 0, sizeof(P));
        P.node = d->o_node; P.arc = d->o_arc; P.ac = d->o_ac; P.fin = d->o_fin; P.finw = d->o_finw;
        P.meta = d->o_meta; P.garcs = g->arcs; P.n = n; P.start = g->start; P.T2 = (int)T2;
        P.lbeam = cfg->lattice_beam;
        P.fw = d->p_fw; P.bw = d->p_bw; P.nflag = d->p_nflag; P.aflag = d->p_aflag;
        P.depth = d->p_depth;
        P.nstart = d->p_steps; P.gstart = d->p_steps + (size_t)n * T2; P.gsplit = d->p_steps + 2 * (size_t)n * T2;
        P.p_node = d->p_node; P.p_arc = d->p_arc; P.p_ac = d->p_ac; P.p_fin = d->p_fin;
        P.p_finw = d->p_finw; P.p_node_cap = (long long)d->p_node_n; P.p_arc_cap = (long long)d->p_arc_n;
        P.p_fin_cap = (long long)d->p_fin_n; P.p_ctr = d->p_ctr; P.p_meta = d->p_meta;
        prune_kernel<128><<<n, 128, 0, st>>>(P);
        CUDA_TRY(cudaGetLastError());
        d->pruned_n = n;
    }
    if (e != cudaSuccess)
        return set_err(WB_ERR_CUDA, std::string("decode launch: ") + cudaGetErrorString(e));
    CUDA_TRY(cudaEventRecord(d->ev1, st));
    d->pend_n = 0;
    if (!host) return WB_OK;
    d->pend_n = n;
    d->pend_label_cap = label_cap;
    d->pend_lcap = lcap;
    d->pend_cols = num_cols;
    d->pend_lattice = cfg->lattice;
    d->pend_zc = zc;
    d->pend_stream = st;
    if (host && !defer) return finish_impl(d, results, olabels, ilabels);
    return WB_OK;
}

// Copy a host-mode decode's results out and synchronise (wb_decode; wb_decode_finish).
static int finish_impl(wb_decoder_t d, wb_utt_result *results, int32_t *olabels, int32_t *ilabels) {
    const int n = d->pend_n;
    cudaStream_t st = d->pend_stream;
    if (n <= 0) return WB_OK;
    CUDA_TRY(cudaMemcpyAsync(results, d->h_res, sizeof(wb_utt_result) * n, cudaMemcpyDeviceToHost, st));
    if (d->pend_label_cap > 0) {
        CUDA_TRY(cudaMemcpyAsync(olabels, d->h_lab, sizeof(int) * (size_t)n * d->pend_label_cap,
                                 cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(ilabels, d->h_lab + (size_t)n * d->pend_lcap,
                                 sizeof(int) * (size_t)n * d->pend_label_cap, cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    if (d->pend_zc) {  // rows the kernel staged from host memory: one per search step (+ lattice)
        long long steps = 0;
        for (int i = 0; i < n; ++i) steps += results[i].search_steps;
        d->last_h2d += steps * (long long)d->pend_cols * (long long)sizeof(double) * (d->pend_lattice ? 2 : 1);
    }
    d->pend_n = 0;
    return WB_OK;
}

extern "C" {

int wb_decode(wb_decoder_t d, int32_t n, const double *costs, const int64_t *row_offset,
              const int32_t *num_frames, int32_t num_cols, const double *blank, const wb_config *cfg,
              wb_utt_result *results, int32_t *olabels, int32_t *ilabels, int32_t label_cap,
              int32_t memory_kind, void *stream) {
    return decode_impl(d, n, costs, row_offset, num_frames, num_cols, blank, cfg, results,
                       olabels, ilabels, label_cap, memory_kind, stream, nullptr, false);
}

int wb_decode_stream(wb_decoder_t d, int32_t n, const double *costs, const int64_t *row_offset,
                     const int32_t *num_frames, int32_t num_cols, const double *blank,
                     const wb_config *cfg, int32_t label_capacity, const int32_t *ready,
                     const int64_t *step_row_offset, void *stream) {
    if (!ready) return set_err(WB_ERR_VALUE, "null ready counters");
    if (step_row_offset && cfg && cfg->mode != 1)
        return set_err(WB_ERR_VALUE, "compacted rows are for label-synchronous decoding");
    return decode_impl(d, n, costs, row_offset, num_frames, num_cols, blank, cfg, nullptr,
                       nullptr, nullptr, label_capacity, WB_MEM_HOST, stream, ready, true,
                       step_row_offset);
}

void wb_gather_rows(const double *src, int64_t src_ld, const int32_t *idx, int64_t n, int32_t col0,
                    int32_t ncols, double *dst, int64_t dst_ld, int32_t dst_col0) {
    for (int64_t i = 0; i < n; ++i)
        std::memcpy(dst + i * dst_ld + dst_col0, src + (int64_t)idx[i] * src_ld + col0,
                    sizeof(double) * (size_t)ncols);
}

int wb_decode_finish(wb_decoder_t d, wb_utt_result *results, int32_t *olabels, int32_t *ilabels) {
    if (!d || !results) return set_err(WB_ERR_VALUE, "null argument");
    return finish_impl(d, results, olabels, ilabels);
}

int wb_lattice_pruned_totals(wb_decoder_t d, int32_t *n_utts, int64_t *n_nodes, int64_t *n_arcs,
                             int64_t *n_finals) {
    if (!d || !n_utts || !n_nodes || !n_arcs || !n_finals) return set_err(WB_ERR_VALUE, "null argument");
    *n_utts = 0; *n_nodes = *n_arcs = *n_finals = 0;
    if (!d->p_ctr || d->pruned_n == 0) return WB_OK;
    CUDA_TRY(cudaSetDevice(d->g->device));
    CUDA_TRY(cudaStreamSynchronize(d->lat_stream));
    unsigned long long c[4];
    CUDA_TRY(cudaMemcpy(c, d->p_ctr, sizeof(c), cudaMemcpyDeviceToHost));
    *n_utts = d->pruned_n;
    *n_nodes = (int64_t)c[0];
    *n_arcs = (int64_t)c[1];
    *n_finals = (int64_t)c[2];
    return WB_OK;
}

int wb_lattice_pruned_fetch(wb_decoder_t d, int64_t *meta, int32_t *nodes, uint32_t *arcs,
                            double *arc_ac, uint32_t *finals, double *final_w) {
    if (!d || !meta) return set_err(WB_ERR_VALUE, "null argument");
    int32_t n;
    int64_t nn, na, nf;
    int rc = wb_lattice_pruned_totals(d, &n, &nn, &na, &nf);
    if (rc) return rc;
    if (n == 0) return WB_OK;
    nn = std::min<int64_t>(nn, (int64_t)d->p_node_n);
    na = std::min<int64_t>(na, (int64_t)d->p_arc_n);
    nf = std::min<int64_t>(nf, (int64_t)d->p_fin_n);
    CUDA_TRY(cudaMemcpy(meta, d->p_meta, sizeof(long long) * 8 * (size_t)n, cudaMemcpyDeviceToHost));
    if (nn && nodes) CUDA_TRY(cudaMemcpy(nodes, d->p_node, sizeof(int2) * nn, cudaMemcpyDeviceToHost));
    if (na && arcs) CUDA_TRY(cudaMemcpy(arcs, d->p_arc, sizeof(uint4) * na, cudaMemcpyDeviceToHost));
    if (na && arc_ac) CUDA_TRY(cudaMemcpy(arc_ac, d->p_ac, sizeof(double) * na, cudaMemcpyDeviceToHost));
    if (nf && finals) CUDA_TRY(cudaMemcpy(finals, d->p_fin, sizeof(u32) * nf, cudaMemcpyDeviceToHost));
    if (nf && final_w) CUDA_TRY(cudaMemcpy(final_w, d->p_finw, sizeof(double) * nf, cudaMemcpyDeviceToHost));
    return WB_OK;
}

int wb_last_transfer(wb_decoder_t d, int64_t *h2d_bytes, int32_t *zero_copy) {
    if (!d || !h2d_bytes || !zero_copy) return set_err(WB_ERR_VALUE, "null argument");
    *h2d_bytes = d->last_h2d;
    *zero_copy = d->last_zero_copy;
    return WB_OK;
}

int wb_lattice_totals(wb_decoder_t d, int32_t *n_utts, int64_t *n_nodes, int64_t *n_arcs,
                      int64_t *n_finals) {
    if (!d || !n_utts || !n_nodes || !n_arcs || !n_finals) return set_err(WB_ERR_VALUE, "null argument");
    if (!d->o_ctr || d->lat_n == 0) {
        *n_utts = 0; *n_nodes = *n_arcs = *n_finals = 0;
        return WB_OK;
    }
    CUDA_TRY(cudaSetDevice(d->g->device));
    CUDA_TRY(cudaStreamSynchronize(d->lat_stream));
    unsigned long long c[4];
    CUDA_TRY(cudaMemcpy(c, d->o_ctr, sizeof(c), cudaMemcpyDeviceToHost));
    *n_utts = d->lat_n;
    // requested sizes: larger than the pools when the call overflowed them
    *n_nodes = (int64_t)c[0];
    *n_arcs = (int64_t)c[1];
    *n_finals = (int64_t)c[2];
    return WB_OK;
}

int wb_lattice_fetch(wb_decoder_t d, int64_t *meta, int32_t *nodes, uint32_t *arcs, double *arc_ac,
                     uint32_t *finals, double *final_w) {
    if (!d || !meta) return set_err(WB_ERR_VALUE, "null argument");
    int32_t n;
    int64_t nn, na, nf;
    int rc = wb_lattice_totals(d, &n, &nn, &na, &nf);
    if (rc) return rc;
    if (n == 0) return WB_OK;
    nn = std::min<int64_t>(nn, (int64_t)d->o_node_n);
    na = std::min<int64_t>(na, (int64_t)d->o_arc_n);
    nf = std::min<int64_t>(nf, (int64_t)d->o_fin_n);
    CUDA_TRY(cudaMemcpy(meta, d->o_meta, sizeof(long long) * 6 * (size_t)n, cudaMemcpyDeviceToHost));
    if (nn && nodes) CUDA_TRY(cudaMemcpy(nodes, d->o_node, sizeof(int2) * nn, cudaMemcpyDeviceToHost));
    if (na && arcs) CUDA_TRY(cudaMemcpy(arcs, d->o_arc, sizeof(uint4) * na, cudaMemcpyDeviceToHost));
    if (na && arc_ac) CUDA_TRY(cudaMemcpy(arc_ac, d->o_ac, sizeof(double) * na, cudaMemcpyDeviceToHost));
    if (nf && finals) CUDA_TRY(cudaMemcpy(finals, d->o_fin, sizeof(u32) * nf, cudaMemcpyDeviceToHost));
    if (nf && final_w) CUDA_TRY(cudaMemcpy(final_w, d->o_finw, sizeof(double) * nf, cudaMemcpyDeviceToHost));
    return WB_OK;
}

}  // extern "C"
