// wfst_decoder.cu -- host side of the C ABI (include/wfst_b200.h): graph upload, decoder
// workspace, batch launch.  The device code lives in decode_kernel.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/wfst_b200.h"
#include "wave_kernel.cuh"

using namespace wb;
using wb::wave::LaneG;

#ifndef WB_WAVE_MINB
#define WB_WAVE_MINB 1  // CTAs per SM the wave kernel is register-budgeted for
#endif

static thread_local std::string g_err;

static int set_err(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return set_err(e_ == cudaErrorMemoryAllocation ? WB_ERR_NOMEM : WB_ERR_CUDA,      \
                           std::string(#expr) + ": " + cudaGetErrorString(e_));              \
    } while (0)

struct wb_graph_s {
    int device = 0;
    int S = 0, A = 0, start = 0, has_eps = 0, max_ilabel = 0, max_emit_deg = 0;
    int4 start_rng{0, 0, 0, 0};
    int4 *arcs = nullptr;      // [2*A] 32-byte arc records
    double *final_w = nullptr;
    size_t bytes = 0;
};

struct wb_decoder_s {
    wb_graph_s *g = nullptr;
    int W = 0, cap = 0, T_cap = 0, block = 512, num_sms = 0, grid = 0;
    u64 arena_cap = 0;
    int logcap = 0;
    Slot *slot = nullptr;
    u32 *cand_of = nullptr, *qtag = nullptr;
    u32 *log_dst = nullptr, *log_arc = nullptr, *log_pay = nullptr;
    u64 *log_key = nullptr;
    u32 *cand_state = nullptr, *cand_arc = nullptr, *cand_pay = nullptr, *ca_idx = nullptr;
    u64 *cand_key = nullptr;
    u32 *front = nullptr;
    int4 *tok_info = nullptr;
    double *tok_cost = nullptr;
    int *frames = nullptr;
    u32 *hist = nullptr;
    LaneG *lane = nullptr;
    u32 *gctr = nullptr;
    long long *phase = nullptr;
    u64 *arena = nullptr;
    u64 *arena_ctr = nullptr;
    // host-mode staging buffers (grown on demand)
    double *h_costs = nullptr, *h_blank = nullptr;
    size_t h_costs_n = 0, h_blank_n = 0;
    long long *h_off = nullptr;
    int *h_T = nullptr;
    wb_utt_result *h_res = nullptr;
    int *h_lab = nullptr;
    size_t h_off_n = 0, h_T_n = 0, h_res_n = 0, h_lab_n = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    size_t bytes = 0;
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
    int has_eps = 0, max_il = 0, max_deg = 0;
    for (int s = 0; s < S; ++s) {
        int lo = d->row_ptr[s], mid = d->eps_end[s], hi = d->row_ptr[s + 1];
        if (lo > mid || mid > hi) return set_err(WB_ERR_VALUE, "eps_end outside the state's arc range");
        if (mid > lo) has_eps = 1;
        max_deg = std::max(max_deg, hi - mid);
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
    g->max_emit_deg = max_deg;
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
    void *ptrs[] = {d->slot, d->cand_of, d->qtag, d->log_dst, d->log_arc, d->log_pay,
                    d->log_key, d->cand_state, d->cand_arc,
                    d->cand_pay, d->ca_idx, d->cand_key, d->front, d->tok_info,
                    d->tok_cost, d->frames, d->hist, d->lane, d->gctr, d->phase, d->arena,
                    d->arena_ctr, d->h_costs, d->h_blank, d->h_off, d->h_T, d->h_res, d->h_lab};
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
    CUDA_TRY(cudaMalloc(&d->frames, sizeof(int) * (size_t)d->W * d->T_cap));
    return WB_OK;
}

static int alloc_arena(wb_decoder_s *d, u64 cap) {
    cudaFree(d->arena);
    d->arena = nullptr;
    d->arena_cap = std::min<u64>(std::max<u64>(cap, 1024), (u64)EPS_BIT - 1);
    CUDA_TRY(cudaMalloc(&d->arena, sizeof(u64) * d->arena_cap));
    return WB_OK;
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
    if (opts.block_threads && opts.block_threads != 512)
        return set_err(WB_ERR_VALUE, "block_threads must be 512 (or 0 = auto)");
    wb_decoder_s *d = new wb_decoder_s();
    d->g = g;
    d->num_sms = prop.multiProcessorCount;
    // utterance lanes per wave: every phase of a step is spread over all SMs
    d->W = opts.max_utts_in_flight > 0 ? opts.max_utts_in_flight : 64;
    d->W = std::min(d->W, wave::MAXW);
    d->cap = opts.cand_capacity > 0 ? opts.cand_capacity : std::min(g->S, 1 << 18);
    d->cap = std::max(1, std::min(d->cap, g->S));
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wave::wave_kernel<512, WB_WAVE_MINB>, 512, 0);
    if (e != cudaSuccess || occ < 1) {
        delete d;
        return set_err(WB_ERR_CUDA, "wave kernel occupancy query failed");
    }
    d->grid = d->num_sms * std::min(occ, 2);
    // relaxation log per lane: every emitting arc of every candidate of one step
    d->logcap = (int)std::min<int64_t>((int64_t)d->cap * std::max(g->max_emit_deg, 1) + 1024,
                                       (int64_t)1 << 30);
    size_t S = (size_t)g->S, W = (size_t)d->W, cap = (size_t)d->cap, lcap = (size_t)d->logcap;
    size_t acc = 0;
    e = cudaSuccess;
#define DA(p, n) if (e == cudaSuccess) e = dalloc(&d->p, (n), acc)
    DA(slot, W * S);
    DA(cand_of, g->has_eps ? W * S : 1);
    DA(qtag, g->has_eps ? W * S : 1);
    DA(log_dst, W * lcap);
    DA(log_arc, W * lcap);
    DA(log_pay, W * lcap);
    DA(log_key, W * lcap);
    DA(cand_state, W * cap);
    DA(cand_arc, W * cap);
    DA(cand_pay, W * cap);
    DA(ca_idx, W * cap);
    DA(cand_key, W * cap);
    DA(front, W * 2 * cap);
    DA(tok_info, W * 2 * cap);
    DA(tok_cost, W * 2 * cap);
    DA(hist, W * wave::NB);
    DA(lane, W);
    DA(gctr, 16);
    DA(phase, 8);
    DA(arena_ctr, 1);
#undef DA
    if (e == cudaSuccess) e = cudaMemset(d->slot, 0xFF, sizeof(Slot) * W * S);
    if (e == cudaSuccess && g->has_eps) e = cudaMemset(d->qtag, 0, sizeof(u32) * W * S);
    if (e == cudaSuccess) e = cudaMemset(d->hist, 0, sizeof(u32) * W * wave::NB);
    if (e == cudaSuccess) e = cudaMemset(d->gctr, 0, sizeof(u32) * 16);
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
    if (rc == WB_OK)
        rc = alloc_arena(d, opts.arena_capacity > 0 ? (u64)opts.arena_capacity : (u64)1 << 24);
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
    *bytes = (int64_t)(d->bytes + sizeof(int) * (size_t)d->W * d->T_cap +
                       sizeof(u64) * d->arena_cap);
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
    const double *dc = costs, *db = blank;
    const long long *doff = (const long long *)row_offset;
    const int *dT = num_frames;
    wb_utt_result *dres = results;
    int *dol = olabels, *dil = ilabels;
    const int lcap = std::max(label_cap, 1);
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
        if (ncost)
            CUDA_TRY(cudaMemcpyAsync(d->h_costs, costs, sizeof(double) * ncost, cudaMemcpyHostToDevice, st));
        if (rows)
            CUDA_TRY(cudaMemcpyAsync(d->h_blank, blank, sizeof(double) * rows, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(d->h_off, row_offset, sizeof(long long) * n, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(d->h_T, num_frames, sizeof(int) * n, cudaMemcpyHostToDevice, st));
        dc = d->h_costs; db = d->h_blank; doff = d->h_off; dT = d->h_T; dres = d->h_res;
        dol = d->h_lab; dil = d->h_lab + nn * lcap;
    }
    // device mode: frame counts stay on the device; an LSD utterance longer than the frame
    // list capacity reports WB_ERR_CAPACITY (callers size it with max_frames)
    wave::GraphDev gd{g->S, g->A, g->start, g->has_eps, g->start_rng, g->arcs, g->final_w};
    wave::BatchDev bd{dc, doff, dT, db, num_cols, n};
    wave::CfgDev cd{cfg->beam, cfg->blank_threshold, cfg->max_active, cfg->mode, cfg->lattice};
    wave::WaveDev wd;
    std::memset(&wd, 0, sizeof(wd));
    wd.slot = d->slot; wd.cand_of = d->cand_of; wd.qtag = d->qtag;
    wd.log_dst = d->log_dst; wd.log_arc = d->log_arc; wd.log_pay = d->log_pay;
    wd.log_key = d->log_key; wd.logcap = d->logcap;
    wd.cand_state = d->cand_state; wd.cand_arc = d->cand_arc;
    wd.cand_pay = d->cand_pay; wd.ca_idx = d->ca_idx;
    wd.cand_key = d->cand_key; wd.front = d->front; wd.tok_info = d->tok_info;
    wd.tok_cost = d->tok_cost; wd.frames = d->frames; wd.hist = d->hist; wd.lane = d->lane;
    wd.gctr = d->gctr; wd.phase = d->phase; wd.arena = d->arena; wd.arena_cap = d->arena_cap;
    wd.arena_ctr = d->arena_ctr; wd.S = g->S; wd.cap = d->cap; wd.T_cap = d->T_cap;
    CUDA_TRY(cudaEventRecord(d->ev0, st));
    for (int first = 0; first < n; first += d->W) {
        // one wave: W utterances advance step by step on all SMs (cooperative launch)
        wd.first_utt = first;
        wd.W = std::min(d->W, n - first);
        CUDA_TRY(cudaMemsetAsync(d->gctr, 0, sizeof(u32) * 9, st));
        CUDA_TRY(cudaMemsetAsync(d->phase, 0, sizeof(long long) * 8, st));
        CUDA_TRY(cudaMemsetAsync(d->arena_ctr, 0, sizeof(u64), st));
        void *args[] = {(void *)&gd, (void *)&wd, (void *)&bd, (void *)&cd, (void *)&dres};
        CUDA_TRY(cudaLaunchCooperativeKernel((void *)wave::wave_kernel<512, WB_WAVE_MINB>, d->grid, 512, args, 0, st));
        // backtrace (decoder.py:276-291) of this wave before its arena is reused
        wave::backtrace_kernel<<<(wd.W + 127) / 128, 128, 0, st>>>(d->arena, g->arcs, dres + first, wd.W,
                                                             dol + (size_t)first * lcap,
                                                             dil + (size_t)first * lcap, lcap);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaEventRecord(d->ev1, st));
    if (host) {
        CUDA_TRY(cudaMemcpyAsync(results, dres, sizeof(wb_utt_result) * n, cudaMemcpyDeviceToHost, st));
        if (label_cap > 0) {
            CUDA_TRY(cudaMemcpyAsync(olabels, dol, sizeof(int) * (size_t)n * label_cap,
                                     cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(ilabels, dil, sizeof(int) * (size_t)n * label_cap,
                                     cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    return WB_OK;
}

}  // extern "C"
