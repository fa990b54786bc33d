/*
 * wfst_b200.h -- C ABI of the B200-native WFST Viterbi decoder (libwfstb200.so).
 *
 * Drop-in boundary for the reference decode path (`lsd_wfst`, a pure-Python package).  The
 * reference has no C ABI of its own; each entry point below replaces the Python call named
 * beside it (paths relative to /root/reference/pkg/src/lsd_wfst):
 *
 *   wb_graph_create      Wfst.__init__ arc layout (wfst.py:163-206) + epsilon_cycle() cache
 *                        (wfst.py:242-247) + _check_compatible's max-ilabel scan (decoder.py:294)
 *   wb_decode            decode / decode_fsd / decode_lsd (decoder.py:349-367) and
 *                        parallel_decode (parallel.py:205-355) -- whole batches of utterances
 *   wb_lattice_*         LatticeRecorder + build_lattice (lattice.py:96-249) and
 *                        prune_lattice (lattice.py:359-501)
 *
 * Plain pointers and sizes only; no torch types.  Status convention: every function returns
 * an int status, WB_OK == 0; the text of the last failure on the calling thread is available
 * from wb_last_error().  The Python shim maps WB_ERR_VALUE -> ValueError, WB_ERR_WFST ->
 * WfstError, WB_ERR_LATTICE -> LatticeError, others -> RuntimeError.
 *
 * Threading: graph handles are immutable after creation and may be shared by threads using
 * the same device.  A decoder handle owns mutable device workspace: one call at a time.
 */
#ifndef WFST_B200_H
#define WFST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WB_OK 0
#define WB_ERR_CUDA 1
#define WB_ERR_VALUE 2
#define WB_ERR_LATTICE 3
#define WB_ERR_WFST 4
#define WB_ERR_CAPACITY 5  /* a device workspace capacity was exceeded; retry with a larger one */

/* wb_utt_result.capacity_flags: which capacity a WB_ERR_CAPACITY utterance exceeded */
#define WB_CAP_CANDIDATES 1    /* per-step candidates / epsilon frontier (cand_capacity) */
#define WB_CAP_ARENA 2         /* backpointer records (arena_capacity) */
#define WB_CAP_FRAMES 4        /* LSD frame list (max_frames) */
#define WB_CAP_LABELS 8        /* label_capacity of the wb_decode call */
#define WB_CAP_LATTICE_RAW 16  /* raw lattice pools (lattice_capacity) */
#define WB_CAP_LATTICE_OUT 32  /* trimmed lattice output pools (lattice_out_capacity) */
#define WB_CAP_EPS_ROUNDS 64   /* epsilon closure did not converge within 2^20 rounds */
#define WB_CAP_STREAM 128      /* wb_decode_stream: a cost row was not published within ~60 s */
#define WB_ERR_NOMEM 6

#define WB_PARSE_ERROR 7    /* wb_wfst_parse_text: malformed line (ParseError) */
#define WB_PARSE_SYMBOL 8   /* wb_wfst_parse_text: unknown symbol / negative label id (SymbolError) */

#define WB_MEM_DEVICE 0    /* all batch pointers are device pointers; the call is asynchronous */
#define WB_MEM_HOST 1      /* all batch pointers are host pointers; the call copies and syncs */

typedef struct wb_graph_s *wb_graph_t;
typedef struct wb_decoder_s *wb_decoder_t;

/* Host-side CSR description (arrays are read during wb_graph_create only). */
typedef struct {
    int32_t num_states;
    int32_t num_arcs;
    int32_t start;
    int32_t _pad;
    const int32_t *row_ptr;  /* [S+1] arc_offsets               (wfst.py:185-190) */
    const int32_t *eps_end;  /* [S]   eps_split                 (wfst.py:192-198) */
    const int32_t *dst;      /* [A]   arcs sorted by (src, ilabel, dst, olabel, weight) */
    const int32_t *ilabel;   /* [A] */
    const int32_t *olabel;   /* [A] */
    const double *weight;    /* [A] */
    const double *final_w;   /* [S]   +inf = not final          (wfst.py:183) */
} wb_graph_desc;

/* Search configuration (DecodeConfig, decoder.py:78-94). */
typedef struct {
    double beam;             /* +inf allowed */
    double blank_threshold;  /* LSD: a frame is blank iff blank_prob > threshold */
    int32_t max_active;      /* 0 = None */
    int32_t mode;            /* 0 = fsd, 1 = lsd */
    int32_t lattice;         /* 1 = record the raw lattice (LatticeRecorder) */
    int32_t log_rows;        /* 1 = the cost rows hold log(p) (acoustic scale 1): the decoder
                                negates each value as it stages the row, which saves the host a
                                pass; needs rows that fit shared memory (<= 16384 columns) */
    double lattice_beam;     /* >= 0 (lattice mode): also beam-prune the lattices on the device
                                (stage one of prune_lattice, see wb_lattice_pruned_fetch); < 0 off */
} wb_config;

/* wb_utt_result.path_flags (evidence for tests: which prune branches ran) */
#define WB_PATH_GLOBAL_CANDS 1  /* a step's candidate keys spilled from shared to global memory */
#define WB_PATH_SELECT 2        /* max-active bound: the histogram select ran */
#define WB_PATH_RADIX 4         /* ... and its boundary bucket was ranked by radix select */
#define WB_PATH_PREFETCH 8      /* expand used the cp.async prefetch pipeline */

/* Per-utterance result (DecodeResult, decoder.py:97-105) plus device counters. */
typedef struct {
    double total_cost;
    int64_t tokens_expanded;
    int32_t search_steps;
    int32_t reached_final;
    int32_t died_at_step;    /* -1 = None */
    int32_t final_state;     /* state of the winning token */
    int32_t final_step;      /* node step of the winning token (lattice finals) */
    int32_t n_olabels;
    int32_t n_ilabels;
    int32_t status;          /* WB_OK or WB_ERR_CAPACITY */
    int32_t capacity_flags;  /* WB_CAP_* bits of a WB_ERR_CAPACITY utterance */
    int32_t path_flags;      /* WB_PATH_* bits: which prune code paths the utterance took */
    int64_t best_trace;      /* lane-arena index of the winning token's record */
    /* counters for the roofline: summed over the utterance's steps */
    int64_t n_tok;           /* live tokens expanded */
    int64_t a_emit;          /* emitting arcs scanned */
    int64_t a_fin;           /* emitting relaxations with finite acoustic cost */
    int64_t e_eps;           /* epsilon relaxations (self-loops excluded) */
    int64_t n_cand;          /* recombined candidates */
    int64_t n_surv;          /* survivors */
    int64_t n_rec;           /* backpointer records written */
    int64_t lat_arcs;        /* raw lattice arcs recorded (lattice mode) */
    int64_t a_cas;           /* emitting relaxations that reached a slot (not beam-skipped) */
    int64_t eps_rounds;      /* epsilon-closure frontier rounds (summed over steps) */
    /* SM clock cycles spent per phase (CTA thread 0, measured after each phase barrier):
     * [0] cost-row staging, [1] emitting expansion, [2] epsilon closure, [3] candidate
     * gather + min/max, [4] max-active histogram/select, [5] survivor flags + chain marks,
     * [6] compaction + records + next tokens, [7] utterance prologue/epilogue */
    int64_t phase_cycles[8];
} wb_utt_result;

/* Decoder workspace options (0 = automatic). */
typedef struct {
    int32_t max_utts_in_flight;  /* concurrent utterances = persistent CTAs */
    int32_t cand_capacity;       /* per-step candidate capacity per utterance */
    int64_t arena_capacity;      /* backpointer records per utterance lane (reused per utterance) */
    int32_t max_frames;          /* longest utterance a call may contain */
    int32_t block_threads;       /* 256, 512 or 1024 */
    int64_t lattice_capacity;    /* raw lattice nodes (and arcs) per utterance lane */
    int32_t cluster_ctas;        /* CTAs per utterance lane (thread-block cluster): 1, 2, 4, 8;
                                    0 = auto (2 or 4 when utterances leave SMs idle) */
    int32_t _pad;
    int64_t lattice_out_capacity;/* trimmed lattice nodes / arcs / finals per wb_decode call */
} wb_decoder_opts;

const char *wb_last_error(void);
int wb_version(void);
int wb_device_count(int32_t *n);

int wb_graph_create(const wb_graph_desc *desc, int32_t device, wb_graph_t *out);
int wb_graph_destroy(wb_graph_t g);
int wb_graph_device_bytes(wb_graph_t g, int64_t *bytes);

int wb_decoder_create(wb_graph_t g, const wb_decoder_opts *opts, wb_decoder_t *out);
int wb_decoder_destroy(wb_decoder_t d);
int wb_decoder_device_bytes(wb_decoder_t d, int64_t *bytes);

/*
 * Decode a batch of independent utterances in one persistent kernel launch.
 *
 *   costs       [R, num_cols] float64 rows; column 0 must be +inf (frame_costs, posteriors.py:136)
 *   row_offset  [n_utts] first row of each utterance in `costs`
 *   num_frames  [n_utts] T of each utterance
 *   blank       [R] blank probability of each row (LSD pre-pass input)
 *   results     [n_utts]
 *   olabels / ilabels [n_utts * label_capacity]; an utterance whose path is longer than
 *               label_capacity reports its true n_*labels and status WB_ERR_CAPACITY.
 *
 * memory_kind WB_MEM_DEVICE: pointers are device pointers, work is enqueued on `stream`
 * (a cudaStream_t, may be NULL) and the call returns without synchronising.
 * memory_kind WB_MEM_HOST: pointers are host pointers; the call copies inputs in (a
 * page-locked cost table is instead read zero-copy by the kernel, see wb_last_transfer),
 * decodes, copies results out and synchronises.
 */
int wb_decode(wb_decoder_t d, int32_t n_utts, const double *costs, const int64_t *row_offset,
              const int32_t *num_frames, int32_t num_cols, const double *blank,
              const wb_config *cfg, wb_utt_result *results, int32_t *olabels, int32_t *ilabels,
              int32_t label_capacity, int32_t memory_kind, void *stream);

/*
 * Trimmed lattices of the last wb_decode call made with cfg.lattice = 1 (build_lattice,
 * lattice.py:148-249): the raw lattice is recorded on the device step by step and trimmed to
 * nodes on a start-to-final path before anything leaves HBM.  Both calls synchronise with the
 * decode's stream and copy to HOST buffers.
 *
 * wb_lattice_totals: number of utterances and the pool sizes the call requested (nodes,
 *                    arcs, finals) -- above the pool capacity when it overflowed (the
 *                    overflowing utterances then report WB_ERR_CAPACITY).
 * wb_lattice_fetch:  meta [n_utts * 6] = {node_off, n_nodes, arc_off, n_arcs, final_off,
 *                    n_finals} per utterance (n_nodes == 0: EMPTY_LATTICE; node_off < 0: the
 *                    utterance failed); nodes [n_nodes * 2] = {state, step}; arcs
 *                    [n_arcs * 4] = {from, to, wfst arc index, 0} with utterance-local node
 *                    ids; arc_ac [n_arcs] acoustic cost (0 for epsilon arcs); finals
 *                    [n_finals] utterance-local node ids with final_w [n_finals].  Node and arc
 *                    order within an utterance is unspecified (canonical order is (step,
 *                    state), lattice.py:215-230).  Any output pointer may be NULL.
 */
int wb_lattice_totals(wb_decoder_t d, int32_t *n_utts, int64_t *n_nodes, int64_t *n_arcs,
                      int64_t *n_finals);
int wb_lattice_fetch(wb_decoder_t d, int64_t *meta, int32_t *nodes, uint32_t *arcs, double *arc_ac,
                     uint32_t *finals, double *final_w);

/*
 * Lattice in flat arrays (the reference's Lattice, lattice.py:52-83): node i = (state, step);
 * node 0 is the start node; arcs carry graph cost g, acoustic cost a and the tie-break
 * index (the WFST arc index for built lattices); finals are node ids with weights.
 * n_nodes == 0 is EMPTY_LATTICE.  Arrays returned by wb_lattice_prune are owned by the
 * caller and released with wb_lattice_arrays_free.
 */
typedef struct {
    int64_t n_nodes, n_arcs, n_finals;
    int32_t *node_state, *node_step;     /* [n_nodes] */
    int64_t *arc_from, *arc_to, *arc_tie; /* [n_arcs] */
    int32_t *arc_il, *arc_ol;            /* [n_arcs] */
    double *arc_g, *arc_a;               /* [n_arcs] */
    int64_t *final_node;                 /* [n_finals] */
    double *final_w;                     /* [n_finals] */
} wb_lattice_arrays;

/* Canonical order of fetched device lattices (_assemble's numbering, lattice.py:215-230):
 * inputs are wb_lattice_fetch's pools + meta and the graph's per-arc ilabel / olabel / weight;
 * outputs are utterance-ordered flat arrays (out_meta rows like meta, offsets into them), node
 * 0 of each lattice its start node, tie = WFST arc index.  n_threads host threads. */
int wb_lattice_canonical(int32_t n_utts, const int64_t *meta, const int32_t *nodes,
                         const uint32_t *arcs, const double *arc_ac, const uint32_t *finals,
                         const double *final_w, int32_t start_state, const int32_t *g_ilabel,
                         const int32_t *g_olabel, const double *g_weight, int32_t n_threads,
                         int64_t *out_meta, int32_t *node_state, int32_t *node_step,
                         int64_t *arc_from, int64_t *arc_to, int32_t *arc_il, int32_t *arc_ol,
                         double *arc_g, double *arc_a, int64_t *arc_tie, int64_t *final_node,
                         double *final_wo);

/* _topo_order's check (lattice.py:295-326): WB_ERR_LATTICE on an epsilon cycle among nodes. */
int wb_lattice_check(const wb_lattice_arrays *lat);
/* prune_lattice (lattice.py:359-501): exact forward-backward pruning to paths within `beam`
 * of the best, then the path-exact split; WB_ERR_LATTICE past 500,000 split nodes. */
int wb_lattice_prune(const wb_lattice_arrays *lat, double beam, wb_lattice_arrays *out);
void wb_lattice_arrays_free(wb_lattice_arrays *a);
/* _enforce_path_soundness (lattice.py:430-501) on a lattice already cut at `cutoff` (stage one,
 * e.g. from wb_lattice_pruned_fetch): splits nodes whose prefix/suffix recombination could
 * exceed the cutoff; WB_ERR_LATTICE past 500,000 keys. */
int wb_lattice_split(const wb_lattice_arrays *lat, double cutoff, wb_lattice_arrays *out);
/* format_lattice_text / parse_lattice_text (lattice.py:562-627), byte-identical to the
 * reference: the text is malloc'd (release with wb_text_free); parsed arrays are released with
 * wb_lattice_arrays_free (tie = arc position).  WB_ERR_LATTICE / WB_ERR_VALUE (a bad int or
 * float literal) with the reference's messages; no nodes = EMPTY_LATTICE. */
int wb_lattice_format_text(const wb_lattice_arrays *lat, char **text, int64_t *len);
int wb_lattice_parse_text(const char *text, int64_t len, wb_lattice_arrays *out);
void wb_text_free(char *text);
/* lattice_best_path (lattice.py:504-559): tie-exact minimum-cost path and its labels. */
int wb_lattice_best_path(const wb_lattice_arrays *lat, double *cost, int32_t *olabels,
                         int32_t *n_olabels, int32_t *ilabels, int32_t *n_ilabels,
                         int32_t capacity);

/*
 * Device lattice-beam pruning (cfg.lattice_beam >= 0): stage one of prune_lattice
 * (lattice.py:359-394) -- exact forward-backward costs, the cut at (best + beam) + 1e-9 and the
 * re-trim -- runs in a second kernel on the trimmed lattices.  Pools as in wb_lattice_fetch;
 * meta rows have 8 fields: {node_off, n_nodes, arc_off, n_arcs, final_off, n_finals,
 * best (float64 bits: the lattice's best path cost), status (WB_OK, WB_ERR_LATTICE for an
 * epsilon cycle among lattice nodes, WB_ERR_CAPACITY)}.  The path-exact second stage is
 * wb_lattice_split with cutoff = (best + beam) + 1e-9.
 */
int wb_lattice_pruned_totals(wb_decoder_t d, int32_t *n_utts, int64_t *n_nodes, int64_t *n_arcs,
                             int64_t *n_finals);
int wb_lattice_pruned_fetch(wb_decoder_t d, int64_t *meta, int32_t *nodes, uint32_t *arcs,
                            double *arc_ac, uint32_t *finals, double *final_w);

/* Host->device bytes of the last WB_MEM_HOST wb_decode call and how its cost table moved:
 * zero_copy 1 = read zero-copy by the kernel (page-locked host memory, one staged row per
 * search step; LSD reads only the non-blank rows); 2 = page-locked FSD table of equal-length
 * utterances at a common stride, copied by the copy engine in step-range chunks while the
 * kernel decodes (the kernel polls per-utterance ready counts); 0 = copied before the decode
 * (pageable memory). */
int wb_last_transfer(wb_decoder_t d, int64_t *h2d_bytes, int32_t *zero_copy);

/*
 * Streaming host decode: launch a batch whose cost table is still being written.  `costs`
 * (page-locked, read zero-copy) and `ready` (page-locked int32[n_utts]) are host buffers; the
 * kernel stages frame f of utterance u only once ready[u] > f, so the caller computes the rows
 * (frame_costs) while the GPU already searches.  The caller raises each ready[u]
 * monotonically after the rows below it are written (x86 stores are seen in order), must
 * eventually set ready[u] = num_frames[u] (for LSD only non-blank rows need real values), and
 * then calls wb_decode_finish, which copies the results out and synchronises.  `blank` is read
 * up front (the LSD pre-pass).  Labels land in decoder-owned buffers until wb_decode_finish.
 */
int wb_decode_stream(wb_decoder_t d, int32_t n_utts, const double *costs, const int64_t *row_offset,
                     const int32_t *num_frames, int32_t num_cols, const double *blank,
                     const wb_config *cfg, int32_t label_capacity, const int32_t *ready,
                     const int64_t *step_row_offset, void *stream);
/* LSD with step_row_offset (host, page-locked not required): `costs` holds only the searched
 * (non-blank) frames, utterance u's search step s at row step_row_offset[u] + s, and ready[u]
 * counts such rows.  wb_gather_rows copies rows idx[i] (columns col0.., ncols) of a row-major
 * matrix into dst rows i (from column dst_col0): the producer's row compaction. */
void wb_gather_rows(const double *src, int64_t src_ld, const int32_t *idx, int64_t n, int32_t col0,
                    int32_t ncols, double *dst, int64_t dst_ld, int32_t dst_col0);
int wb_decode_finish(wb_decoder_t d, wb_utt_result *results, int32_t *olabels, int32_t *ilabels);
/* The CSR arc order of Wfst (wfst.py:182): `order` receives the permutation that sorts the arcs
 * stably by (src, ilabel, dst, olabel, weight).  States and labels must be >= 0. */
int wb_sort_arcs(int64_t n, const int32_t *src, const int32_t *ilabel, const int32_t *dst,
                 const int32_t *olabel, const double *weight, int64_t *order);

/*
 * parse_wfst_text (wfst.py:315-378): AT&T transducer text -> arc arrays in file order, finals
 * in first-mention order (last weight wins), start = first state mentioned.  `isyms` / `osyms`
 * (may be null): "symbol id" lines; a label token resolves through its table first, then as a
 * bare non-negative integer.  Text must use '\n' (optionally "\r\n") line breaks and ASCII
 * whitespace between fields (the Python shim normalises anything else).  Errors:
 * WB_PARSE_ERROR (ParseError) / WB_PARSE_SYMBOL (SymbolError) with out->error_line (1-based,
 * 0 = no line) and the message in wb_last_error().  Arrays are owned by the caller:
 * wb_parsed_wfst_free.
 */
typedef struct {
    int32_t num_states, start;
    int64_t num_arcs, num_finals;
    int32_t *src, *dst, *ilabel, *olabel;
    double *weight;
    int32_t *final_state;
    double *final_weight;
    int32_t error_line, _pad;
} wb_parsed_wfst;
int wb_wfst_parse_text(const char *text, int64_t len, int32_t allow_negative_weights,
                       const char *isyms, int64_t isyms_len, const char *osyms,
                       int64_t osyms_len, wb_parsed_wfst *out);
void wb_parsed_wfst_free(wb_parsed_wfst *p);

/*
 * POST1 posterior files (load_posteriors' binary form, posteriors.py:147-217): header, and the
 * rows read straight into `dst` (row stride dst_ld doubles) -- typically the decoder's
 * page-locked table, so no pageable staging copy.  WB_ERR_VALUE + message on a malformed file.
 */
int wb_post1_info(const char *path, int32_t *num_frames, int32_t *num_cols, int32_t *blank_col);
int wb_post1_read(const char *path, double *dst, int64_t dst_ld);

/*
 * Checked build (libwfstb200_checked.so, compiled with -DWB_CHECKS): the kernel verifies the
 * search's synchronisation invariants -- the reference's ClaimLedger.verify_partitions and
 * debug_epoch (parallel.py:41-61, 92-116) -- on the device: every live token expanded by
 * exactly one warp per step, every state registered at most once per step (the first-touch
 * CAS protocol), every touched slot reset at the end of its step and the whole slot array
 * clean between utterances, workspace indices in bounds.  wb_check_report copies (and
 * clears) the first violation per lane: code << 32 | kernel source line, 0 = none.
 * wb_claim_log returns the live-token count of each search step of the last utterance on a
 * lane and the group (warp) that expanded each token, step after step.
 */
int wb_checks_enabled(void);
int wb_check_report(wb_decoder_t d, int32_t n_lanes, int64_t *first_violation);
int wb_claim_log(wb_decoder_t d, int32_t lane, int32_t n_steps, int32_t *queue_len,
                 uint16_t *groups, int64_t groups_cap, int64_t *n_logged);

/* Utterance lanes of a decoder (persistent lanes decoding concurrently; fewer than the SMs when
 * a large graph's per-lane dense arrays would not fit) and the largest cluster size its
 * candidate workspace allows. */
int wb_decoder_lanes(wb_decoder_t d, int32_t *lanes, int32_t *max_cluster);

/* CTAs per utterance lane (thread-block cluster size) of the last decode launch. */
int wb_last_launch(wb_decoder_t d, int32_t *cluster_ctas);

/* Device time (ms) of the decode kernel of the last wb_decode call (CUDA events on its stream). */
int wb_last_kernel_ms(wb_decoder_t d, float *ms);

#ifdef __cplusplus
}
#endif
#endif /* WFST_B200_H */
