"""Frame-synchronous and label-synchronous Viterbi beam search on the GPU.

Same public surface as the reference ``lsd_wfst.decoder`` (decoder.py:78-105, 349-367):
``DecodeConfig``, ``DecodeResult``, ``decode`` / ``decode_fsd`` / ``decode_lsd``, plus
``parallel_decode`` (parallel.py:205) and batched entry points.  All search work runs in one
persistent sm_100a kernel per batch (``csrc/wfst_decoder.cu``) reached through the C ABI in
``include/wfst_b200.h``; this module only prepares the float64 cost table (numpy, exactly the
reference's ``frame_costs``), moves buffers and maps status codes to the reference's
exceptions.  There is no CPU search path.
"""
from __future__ import annotations

import ctypes as C
import functools
import math
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .posteriors import PosteriorMatrix, cost_table
from .wfst import Wfst, WfstError

INF = math.inf


@dataclass
class DecodeConfig:
    """Search configuration (decoder.py:78-94)."""
    beam: float = INF
    max_active: int | None = None
    blank_threshold: float = 0.98
    acoustic_scale: float = 1.0
    mode: str = "lsd"

    def __post_init__(self):
        if self.beam < 0:
            raise ValueError(f"beam must be >= 0, got {self.beam}")
        if self.max_active is not None and self.max_active < 1:
            raise ValueError(f"max_active must be >= 1, got {self.max_active}")
        if self.acoustic_scale <= 0:
            raise ValueError(f"acoustic_scale must be positive, got {self.acoustic_scale}")
        if self.mode not in ("fsd", "lsd"):
            raise ValueError(f"mode must be 'fsd' or 'lsd', got {self.mode!r}")


@dataclass(frozen=True)
class DecodeResult:
    """Decode outcome (decoder.py:97-105); compared field by field with the reference."""
    total_cost: float
    olabels: tuple[int, ...]
    ilabels: tuple[int, ...]
    search_steps: int
    tokens_expanded: int
    reached_final: bool
    died_at_step: int | None = None


def result_class():
    """The class decode results are returned as: the reference's own
    ``lsd_wfst.decoder.DecodeResult`` when the caller has the reference loaded (a frozen
    dataclass compares equal only to its own class, so ``lsd_wfst.decode(...) ==
    decode(...)`` holds field for field), else this module's identical ``DecodeResult``.
    The reference is never imported here: only an already loaded one is used."""
    import sys
    ref = sys.modules.get("lsd_wfst.decoder")
    cls = getattr(ref, "DecodeResult", None)
    return cls if cls is not None else DecodeResult


class SearchDied(RuntimeError):
    """For callers that treat an emptied beam as fatal (decoder.py:108-110)."""


def _native_config(cfg, mode: str, lattice: bool = False,
                   lattice_beam: float | None = None, log_rows: bool = False) -> N.Config:
    return N.Config(float(cfg.beam), float(cfg.blank_threshold), int(cfg.max_active or 0),
                    0 if mode == "fsd" else 1, int(bool(lattice)), int(bool(log_rows)),
                    -1.0 if lattice_beam is None else float(lattice_beam))


# ---------------------------------------------------------------- graph residency
_CONVERTED: "weakref.WeakValueDictionary[int, Wfst]" = weakref.WeakValueDictionary()
_REF_KEEP: dict[int, object] = {}


def as_wfst(w) -> Wfst:
    """Accept this package's ``Wfst`` or any reference-shaped transducer (``arcs``,
    ``num_states``, ``start``, ``final_weights``); conversions are cached per object."""
    if isinstance(w, Wfst):
        return w
    key = id(w)
    hit = _CONVERTED.get(key)
    if hit is not None and _REF_KEEP.get(key) is w:
        return hit
    conv = Wfst.from_reference(w)
    _CONVERTED[key] = conv
    _REF_KEEP[key] = w
    w_ref = weakref.ref(conv)
    weakref.finalize(conv, lambda k=key, r=w_ref: _REF_KEEP.pop(k, None))
    return conv


def _current_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return int(torch.cuda.current_device())
    except Exception:  # pragma: no cover - torch is plumbing only
        pass
    return 0


class DeviceGraph:
    """A transducer resident in HBM (``wb_graph_create``): packed 16-byte arc records
    {dst, ilabel, weight}, per-state {eps_lo, emit_lo, emit_hi} ranges, olabels, finals."""

    def __init__(self, wfst, device: int | None = None, checked: bool = False):
        self.wfst = as_wfst(wfst)
        self.device = _current_device() if device is None else int(device)
        self.checked = bool(checked)
        self._L = N.load(self.checked)   # the library (product or checked build) of this handle
        w = self.wfst
        self._arrays = [np.ascontiguousarray(a) for a in (w.row_ptr, w.eps_end, w.dst, w.ilabel,
                                                          w.olabel, w.weight, w.final_w)]
        a = self._arrays
        desc = N.GraphDesc(w.num_states, w.num_arcs, w.start, 0, *(x.ctypes.data for x in a))
        h = C.c_void_p()
        N.check(self._L.wb_graph_create(C.byref(desc), self.device, C.byref(h)), "graph upload")
        self._h = h
        self._fin = weakref.finalize(self, N.defer_destroy, "wb_graph_destroy", h, self._L)

    @property
    def handle(self):
        return self._h

    def device_bytes(self) -> int:
        b = C.c_int64()
        N.check(self._L.wb_graph_device_bytes(self._h, C.byref(b)))
        return int(b.value)


@dataclass
class BatchOutput:
    """Raw per-utterance device results of one batch (numpy record array + labels)."""
    results: np.ndarray  # UTT_RESULT_DTYPE
    olabels: np.ndarray  # [n, cap] int32
    ilabels: np.ndarray
    label_capacity: int

    def decode_result(self, i: int) -> DecodeResult:
        r = self.results[i]
        no, ni = int(r["n_olabels"]), int(r["n_ilabels"])
        died = int(r["died_at_step"])
        return result_class()(
            total_cost=float(r["total_cost"]),
            olabels=tuple(int(x) for x in self.olabels[i, :no]),
            ilabels=tuple(int(x) for x in self.ilabels[i, :ni]),
            search_steps=int(r["search_steps"]),
            tokens_expanded=int(r["tokens_expanded"]),
            reached_final=bool(r["reached_final"]),
            died_at_step=None if died < 0 else died)

    def decode_results(self) -> list[DecodeResult]:
        return [self.decode_result(i) for i in range(len(self.results))]


def _locked(fn):
    """Serialise calls on one decoder: its workspace, page-locked cost table and ready
    counters are mutable state shared by every call (the reference's decode() is pure and its
    Wfst safe for concurrent readers, so concurrent callers must not observe each other)."""
    @functools.wraps(fn)
    def wrapper(self, *a, **k):
        with self.lock:
            return fn(self, *a, **k)
    return wrapper


class BatchDecoder:
    """Device workspace + the batched decode call (``wb_decoder_create`` / ``wb_decode``).

    One persistent kernel decodes a whole batch; every CTA is an utterance lane.  The
    workspace (dense per-state recombination slots per lane, candidate and token buffers, the
    backpointer arena) is allocated once and reused; capacities grow automatically when a
    batch overflows them (results are deterministic, so a retried batch is identical).
    """

    def __init__(self, graph, device: int | None = None, *, max_utts_in_flight: int = 0,
                 cand_capacity: int = 0, arena_capacity: int = 0, max_frames: int = 0,
                 block_threads: int = 0, cluster_ctas: int = 0, lattice_capacity: int = 0,
                 lattice_out_capacity: int = 0, checks: bool = False):
        if isinstance(graph, DeviceGraph):
            if graph.checked != bool(checks):
                raise ValueError("the DeviceGraph was uploaded by the other library build")
            self.graph = graph
        else:
            self.graph = DeviceGraph(graph, device, checked=checks)
        self.checks = bool(checks)   # the -DWB_CHECKS build: device invariants verified
        self._L = self.graph._L
        self.device = self.graph.device
        self.opts = dict(max_utts_in_flight=max_utts_in_flight, cand_capacity=cand_capacity,
                         arena_capacity=arena_capacity, max_frames=max_frames,
                         block_threads=block_threads, cluster_ctas=cluster_ctas,
                         lattice_capacity=lattice_capacity,
                         lattice_out_capacity=lattice_out_capacity)
        self._h = None
        self.lock = threading.RLock()
        self._create()

    def _create(self):
        if self._h is not None:
            self._fin()
        N.flush_destroy()
        o = self.opts
        opts = N.DecoderOpts(o["max_utts_in_flight"], o["cand_capacity"], o["arena_capacity"],
                             o["max_frames"], o["block_threads"], o["lattice_capacity"],
                             o["cluster_ctas"], 0, o["lattice_out_capacity"])
        h = C.c_void_p()
        N.check(self._L.wb_decoder_create(self.graph.handle, C.byref(opts), C.byref(h)),
                "decoder workspace")
        self._h = h
        self._fin = weakref.finalize(self, N.defer_destroy, "wb_decoder_destroy", h, self._L)

    def _grow(self, flags: int, lattice_out_need: int = 0, max_frames: int = 0):
        """Recreate the workspace with the capacities named by ``flags`` (WB_CAP_* bits of
        the failed utterances) enlarged; results are deterministic, so the retry is exact."""
        S = self.graph.wfst.num_states
        if flags & N.WB_CAP_EPS_ROUNDS:
            raise N.CapacityError("epsilon closure did not converge (2^20 rounds)")
        if flags & N.WB_CAP_STREAM:
            raise N.NativeError("streaming decode: cost rows were not published in time")
        if flags & N.WB_CAP_LATTICE_RAW:
            self.opts["lattice_capacity"] = min(2**31 - 2, 4 * (self.opts["lattice_capacity"] or (1 << 20)))
        if flags & N.WB_CAP_LATTICE_OUT:
            out = self.opts["lattice_out_capacity"] or (1 << 22)
            self.opts["lattice_out_capacity"] = max(2 * out, lattice_out_need * 5 // 4)
        if flags & (N.WB_CAP_CANDIDATES | N.WB_CAP_LATTICE_RAW):  # the relaxation log follows cap
            cap = self.opts["cand_capacity"] or min(S, 1 << 18)
            self.opts["cand_capacity"] = min(S, cap * 4)
        if flags & N.WB_CAP_ARENA:
            arena = self.opts["arena_capacity"] or (1 << 22)
            self.opts["arena_capacity"] = min(2**31 - 2, arena * 4)
        if flags & N.WB_CAP_FRAMES:
            self.opts["max_frames"] = max(max_frames, 2 * (self.opts["max_frames"] or 2048))
        self._create()

    def device_bytes(self) -> int:
        b = C.c_int64()
        N.check(self._L.wb_decoder_device_bytes(self._h, C.byref(b)))
        return int(b.value)

    def last_transfer(self) -> tuple[int, int]:
        """(host->device bytes, path) of the last host-buffer decode: path 1 = cost rows read
        zero-copy by the kernel, 2 = table copied in step-range chunks during the decode (H2D
        pipeline), 0 = copied before the decode."""
        b, z = C.c_int64(), C.c_int32()
        N.check(self._L.wb_last_transfer(self._h, C.byref(b), C.byref(z)))
        return int(b.value), int(z.value)

    def check_report(self, n_lanes: int | None = None) -> None:
        """Checked build: raise ``DeviceCheckError`` if a device invariant failed during the
        last decode(s) on any lane (and clear the reports)."""
        if not self.checks:
            return
        n = int(n_lanes or self.opts["max_utts_in_flight"] or 148)
        rep = np.zeros(max(n, 1), np.int64)
        N.check(self._L.wb_check_report(self._h, n, rep.ctypes.data), "check report", self._L)
        bad = np.flatnonzero(rep)
        if len(bad):
            lines = [f"lane {int(i)}: {N.CHECK_NAMES.get(int(rep[i]) >> 32, 'check')} "
                     f"(decode_kernel.cuh:{int(rep[i]) & 0xFFFFFFFF})" for i in bad[:8]]
            raise N.DeviceCheckError("device invariant violated: " + "; ".join(lines))

    def claim_log(self, n_steps: int, lane: int = 0):
        """Checked build: per search step of the last utterance on ``lane``, the live-token
        count and the group (warp) that expanded each token."""
        q = np.zeros(max(n_steps, 1), np.int32)
        cap = 1 << 26
        groups = np.zeros(cap, np.uint16)
        got = C.c_int64()
        N.check(self._L.wb_claim_log(self._h, lane, n_steps, q.ctypes.data, groups.ctypes.data,
                                     cap, C.byref(got)), "claim log", self._L)
        q = q[:n_steps]
        if got.value < int(q.sum()):
            raise ValueError("the claim log overflowed (raise WB_CHECK_LOG)")
        return q, groups[:got.value]

    def lanes(self) -> tuple[int, int]:
        """(utterance lanes, largest cluster size the workspace allows)."""
        a, b = C.c_int32(), C.c_int32()
        N.check(self._L.wb_decoder_lanes(self._h, C.byref(a), C.byref(b)), "lanes", self._L)
        return int(a.value), int(b.value)

    def last_cluster_ctas(self) -> int:
        """CTAs per utterance lane (thread-block cluster size) of the last launch."""
        k = C.c_int32()
        N.check(self._L.wb_last_launch(self._h, C.byref(k)))
        return int(k.value)

    def last_kernel_ms(self) -> float:
        ms = C.c_float()
        N.check(self._L.wb_last_kernel_ms(self._h, C.byref(ms)))
        return float(ms.value)

    def reserve(self, n_frames_total: int, max_active: int | None, max_frames: int,
                lattice: bool = False):
        """Size the backpointer arena / frame list (and the raw-lattice pools of one utterance
        lane when recording lattices) for a batch before launching it."""
        # the arena is per utterance lane and reused per utterance: one utterance's records
        S = self.graph.wfst.num_states
        per_step = min(self.opts["cand_capacity"] or (1 << 18), S,
                       2 * max_active if max_active else 8192)
        need = int(min(2**31 - 2, (max_frames + 2) * max(per_step, 64)))
        changed = False
        if need > (self.opts["arena_capacity"] or (1 << 22)):
            self.opts["arena_capacity"] = need
            changed = True
        if max_frames > (self.opts["max_frames"] or 2048):
            self.opts["max_frames"] = max_frames
            changed = True
        if lattice and not self.opts["lattice_capacity"]:
            S = self.graph.wfst.num_states
            width = min(S, max_active or S, 1 << 16)
            self.opts["lattice_capacity"] = int(min(1 << 23, max(1 << 16, 2 * (max_frames + 1) * width)))
            changed = True
        if changed:
            self._create()

    # ------------------------------------------------------------------ host buffers (e2e)
    @_locked
    def decode_host(self, costs: np.ndarray, row_offset: np.ndarray, num_frames: np.ndarray,
                    blank: np.ndarray, cfg, mode: str, label_capacity: int | None = None,
                    lattice: bool = False, lattice_beam: float | None = None) -> BatchOutput:
        """Decode from host arrays: H2D copies, kernel, D2H results inside one C call."""
        costs = np.ascontiguousarray(costs, dtype=np.float64)
        if costs.ndim == 1:
            costs = costs.reshape(-1, 1)
        n = len(num_frames)
        row_offset = np.ascontiguousarray(row_offset, dtype=np.int64)
        num_frames = np.ascontiguousarray(num_frames, dtype=np.int32)
        blank = np.ascontiguousarray(blank, dtype=np.float64)
        L1 = costs.shape[1]
        maxT = int(num_frames.max()) if n else 0
        self.reserve(int(num_frames.sum()) + n, cfg.max_active, maxT, lattice)
        cap = label_capacity or (maxT + 64)
        if lattice_beam is not None and not lattice_beam >= 0:
            raise ValueError(f"lattice_beam must be >= 0, got {lattice_beam}")
        ncfg = _native_config(cfg, mode, lattice, lattice_beam)
        for _attempt in range(16):
            res = np.zeros(n, dtype=N.UTT_RESULT_DTYPE)
            ol = np.zeros((n, cap), dtype=np.int32)
            il = np.zeros((n, cap), dtype=np.int32)
            rc = self._L.wb_decode(self._h, n, costs.ctypes.data, row_offset.ctypes.data,
                                    num_frames.ctypes.data, L1, blank.ctypes.data,
                                    C.byref(ncfg), res.ctypes.data, ol.ctypes.data,
                                    il.ctypes.data, cap, N.WB_MEM_HOST, None)
            N.check(rc, "decode")
            bad = res["status"] != N.WB_OK
            if not bad.any():
                self.check_report(n)
                return BatchOutput(res, ol, il, cap)
            flags = int(np.bitwise_or.reduce(res["capacity_flags"][bad]))
            if flags & N.WB_CAP_LABELS:           # labels did not fit: rerun with exact room
                cap = int(np.maximum(res["n_olabels"], res["n_ilabels"]).max())
            if flags & ~N.WB_CAP_LABELS:
                need = 0
                if flags & N.WB_CAP_LATTICE_OUT:  # exact output-pool need from the counters
                    nu, nn, na, nf = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64()
                    N.check(self._L.wb_lattice_totals(self._h, C.byref(nu), C.byref(nn),
                                                       C.byref(na), C.byref(nf)), "lattice")
                    need = max(nn.value, na.value, nf.value)
                self._grow(flags, lattice_out_need=need, max_frames=maxT)
        raise N.CapacityError("decode workspace kept overflowing")

    # ------------------------------------------------------------------ posteriors in (e2e)
    def _pinned(self, name: str, shape, dtype):
        """Grow-only page-locked host buffers owned by the decoder (torch is plumbing)."""
        import torch
        n = int(np.prod(shape))
        buf = getattr(self, name, None)
        if buf is None or buf.numel() < n:
            tdt = {np.float64: torch.float64, np.int32: torch.int32}[dtype]
            buf = torch.empty(max(n, 1), dtype=tdt, pin_memory=True)
            setattr(self, name, buf)
        return buf.numpy()[:n].reshape(shape)

    @_locked
    def decode_posteriors(self, posts_list, cfg, mode: str | None = None,
                          label_capacity: int | None = None, lattice: bool = False,
                          lattice_beam: float | None = None, block_frames: int = 128,
                          workers: int | None = None, _attempt: int = 0) -> BatchOutput:
        """Decode from posterior matrices (the public path): host threads compute the
        frame_costs rows straight into a page-locked table in frame-block order while the
        kernel already searches, reading each row zero-copy once its block is published
        (``wb_decode_stream``).  LSD computes only the non-blank rows (select_frames,
        posteriors.py:109-110), gathered into a compacted table indexed by search step.
        Bit-identical to ``decode_host`` on ``cost_table``."""
        import os
        import time
        t_start = time.perf_counter()
        import threading
        from concurrent.futures import ThreadPoolExecutor
        from .posteriors import PosteriorBatch, cost_rows
        mode = mode or cfg.mode
        # a PosteriorBatch's page-locked table becomes the cost table itself: rows are
        # converted in place (the blank column is read out first) and read zero-copy
        batch = posts_list if isinstance(posts_list, PosteriorBatch) else None
        posts_list = batch.matrices() if batch is not None else list(posts_list)
        n = len(posts_list)
        if n == 0:
            return BatchOutput(np.zeros(0, dtype=N.UTT_RESULT_DTYPE), np.zeros((0, 1), np.int32),
                               np.zeros((0, 1), np.int32), 1)
        L1 = posts_list[0].rows.shape[1]
        T = np.asarray([p.rows.shape[0] for p in posts_list], np.int32)
        off = np.zeros(n, np.int64)
        np.cumsum(T[:-1], out=off[1:])
        blank = np.zeros(max(int(T.sum()), 1), np.float64)
        for p, o, t in zip(posts_list, off, T):
            blank[o:o + t] = p.rows[:, p.blank_col]
        # LSD: only the frames the device pre-pass will search (blank <= threshold, strict >
        # for blank), compacted per utterance in search-step order when the label columns
        # are contiguous (blank column 0); otherwise rows stay indexed by frame
        compact = mode == "lsd" and batch is None and all(p.blank_col == 0 for p in posts_list)
        need = [np.flatnonzero(~(p.rows[:, p.blank_col] > cfg.blank_threshold)).astype(np.int32)
                if mode == "lsd" else None for p in posts_list]
        if compact:
            nrow = np.asarray([len(x) for x in need], np.int64)
            crow = np.zeros(n, np.int64)
            np.cumsum(nrow[:-1], out=crow[1:])
            R = max(int(nrow.sum()), 1)
            total = nrow.astype(np.int32)
        else:
            R = max(int(T.sum()), 1)
            total = T
        if batch is not None:
            costs = batch.table
            batch.consumed = True
        else:
            costs = self._pinned("_pin_costs", (R, L1), np.float64)
        ready = self._pinned("_pin_ready", (n,), np.int32)
        ready[:] = 0
        maxT = int(T.max())
        self.reserve(int(T.sum()) + n, cfg.max_active, maxT, lattice)
        cap = label_capacity or (maxT + 64)
        if lattice_beam is not None and not lattice_beam >= 0:
            raise ValueError(f"lattice_beam must be >= 0, got {lattice_beam}")
        # scale 1: the rows keep log(p) and the decoder negates them as it stages each row
        # (exact; one pass less for the producers).  WB_LOG_ROWS=0: costs on the host.
        log_rows = float(cfg.acoustic_scale) == 1.0 and os.environ.get("WB_LOG_ROWS", "1") != "0"
        ncfg = _native_config(cfg, mode, lattice, lattice_beam, log_rows)
        self._last_max_active = cfg.max_active
        N.flush_destroy()
        L = self._L
        t_setup = time.perf_counter()
        # producers: row blocks in block-major order; each utterance's ready count advances
        # over its contiguous finished prefix.  They start BEFORE the launch: when launches are
        # serialised (CUDA_LAUNCH_BLOCKING=1, ncu, compute-sanitizer) wb_decode_stream returns
        # only after the kernel has finished, so the rows must not depend on it returning.
        lock = threading.Lock()
        done = [dict() for _ in range(n)]
        nxt = [0] * n
        # block 0 of every utterance is short (the kernel starts as soon as it is published),
        # later blocks are block_frames long: fewer, larger numpy calls keep the producers
        # off the GIL (measured on the 16-core host: 32-frame blocks 174 ms, 128-frame blocks
        # 49 ms for config 2's 64 x 1000 rows; blocks doubling from 16 frames were slower)
        first = max(1, min(32, block_frames))

        def bounds(u, b):
            lo = 0 if b == 0 else first + (b - 1) * block_frames
            return lo, min(int(total[u]), first if b == 0 else lo + block_frames)
        nblk = [0 if int(t) == 0 else 1 + (max(0, int(t) - first) + block_frames - 1) // block_frames
                for t in total]
        neg = -cfg.acoustic_scale

        def work(u, b):
            lo, hi = bounds(u, b)
            p = posts_list[u]
            if compact:   # gather the searched rows (C++, no GIL), then -scale*log in place
                r0 = int(crow[u]) + lo
                idx = need[u][lo:hi]
                src = p.rows if p.rows.flags.c_contiguous else np.ascontiguousarray(p.rows)
                L.wb_gather_rows(src.ctypes.data, L1, idx.ctypes.data, hi - lo, 1, L1 - 1,
                                 costs[r0:].ctypes.data, L1, 1)
                dst = costs[r0:r0 + hi - lo, 1:]
                with np.errstate(divide="ignore"):
                    np.log(dst, out=dst)
                if log_rows:
                    costs[r0:r0 + hi - lo, 0] = -np.inf
                else:
                    np.multiply(dst, neg, out=dst)
                    costs[r0:r0 + hi - lo, 0] = np.inf
            else:
                view = costs[off[u]:off[u] + T[u]]
                if need[u] is None:
                    cost_rows(p, np.arange(lo, hi), view, cfg.acoustic_scale, log_only=log_rows)
                else:
                    sel = need[u][(need[u] >= lo) & (need[u] < hi)]
                    if len(sel):
                        cost_rows(p, sel, view, cfg.acoustic_scale, log_only=log_rows)
            with lock:
                done[u][b] = hi
                while nxt[u] in done[u]:
                    ready[u] = done[u].pop(nxt[u])
                    nxt[u] += 1
        tasks = [(u, b) for b in range(max(nblk) if nblk else 0) for u in range(n) if b < nblk[u]]
        nw = workers or int(os.environ.get("WB_PRODUCERS", 0)) or len(os.sched_getaffinity(0))
        ex = ThreadPoolExecutor(nw)
        futs: list = []

        def submit_all():   # in block order; a helper thread, so the launch is not delayed
            for u, b in tasks:
                futs.append(ex.submit(work, u, b))
        submitter = threading.Thread(target=submit_all, daemon=True)
        try:
            submitter.start()
            N.check(L.wb_decode_stream(self._h, n, costs.ctypes.data, off.ctypes.data,
                                       T.ctypes.data, L1, blank.ctypes.data, C.byref(ncfg), cap,
                                       ready.ctypes.data, crow.ctypes.data if compact else None,
                                       None), "decode")
            t_launch = time.perf_counter()
            submitter.join()
            for f in futs:
                f.result()
        finally:
            submitter.join()
            ex.shutdown(wait=True)
            ready[:] = total  # every row is written (or the kernel must not wait forever)
        t_rows = time.perf_counter()
        res = np.zeros(n, dtype=N.UTT_RESULT_DTYPE)
        ol = np.zeros((n, cap), dtype=np.int32)
        il = np.zeros((n, cap), dtype=np.int32)
        N.check(L.wb_decode_finish(self._h, res.ctypes.data, ol.ctypes.data, il.ctypes.data),
                "decode")
        # host-side timeline of the last streaming decode (ms since the call): setup done,
        # kernel launched, every cost row published, results back
        self.last_stream_ms = {k: round(1e3 * (v - t_start), 2) for k, v in (
            ("setup", t_setup), ("launched", t_launch), ("rows_published", t_rows),
            ("finished", time.perf_counter()))}
        bad = res["status"] != N.WB_OK
        if bad.any():   # a capacity ran out: grow exactly that one and decode again
            if _attempt >= 16:
                raise N.CapacityError("decode workspace kept overflowing")
            flags = int(np.bitwise_or.reduce(res["capacity_flags"][bad]))
            if flags & N.WB_CAP_LABELS:
                cap = int(np.maximum(res["n_olabels"], res["n_ilabels"]).max())
            if flags & ~N.WB_CAP_LABELS:
                need_out = 0
                if flags & N.WB_CAP_LATTICE_OUT:
                    nu, nn, na, nf = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64()
                    N.check(L.wb_lattice_totals(self._h, C.byref(nu), C.byref(nn), C.byref(na),
                                                C.byref(nf)), "lattice")
                    need_out = max(nn.value, na.value, nf.value)
                self._grow(flags, lattice_out_need=need_out, max_frames=maxT)
            if batch is not None:
                # the batch's rows are costs now (converted in place): retry from the table
                if log_rows:   # (log(p) rows: the costs are their negation, exactly)
                    np.negative(costs, out=costs)
                return self.decode_host(costs, off, T, blank, cfg, mode, cap, lattice,
                                        lattice_beam)
            return self.decode_posteriors(posts_list, cfg, mode, cap, lattice, lattice_beam,
                                          block_frames, workers, _attempt + 1)
        self.check_report(n)
        return BatchOutput(res, ol, il, cap)

    @_locked
    def fetch_lattices(self, wfst: Wfst) -> list:
        """Trimmed lattices of the last lattice-mode decode, canonically ordered."""
        from .lattice import canonical_batch
        L = self._L
        n = C.c_int32()
        nn, na, nf = C.c_int64(), C.c_int64(), C.c_int64()
        N.check(L.wb_lattice_totals(self._h, C.byref(n), C.byref(nn), C.byref(na), C.byref(nf)),
                "lattice")
        meta = np.zeros((max(n.value, 1), 6), np.int64)
        nodes = np.zeros((max(nn.value, 1), 2), np.int32)
        arcs = np.zeros((max(na.value, 1), 4), np.uint32)
        ac = np.zeros(max(na.value, 1), np.float64)
        fin = np.zeros(max(nf.value, 1), np.uint32)
        finw = np.zeros(max(nf.value, 1), np.float64)
        N.check(L.wb_lattice_fetch(self._h, meta.ctypes.data, nodes.ctypes.data, arcs.ctypes.data,
                                   ac.ctypes.data, fin.ctypes.data, finw.ctypes.data), "lattice")
        meta = meta[:n.value]
        if (meta[:, 0] < 0).any():
            raise N.CapacityError("lattice output pool overflowed")
        return canonical_batch(wfst, meta, nodes, arcs, ac, fin, finw)

    @_locked
    def fetch_pruned_lattices(self, wfst: Wfst, lattice_beam: float,
                              max_workers: int | None = None, split: bool = True) -> list:
        """Lattices of the last decode made with ``lattice_beam``: stage one of prune_lattice
        ran on the device; the path-exact split runs here on host threads.  Each element is
        a pruned ``Lattice`` or the ``LatticeError`` the reference would raise for it.  With
        ``split=False`` the stage-one items are returned as (Lattice, cutoff) for the caller
        to finish with ``lattice.split_lattice``."""
        import os
        from concurrent.futures import ThreadPoolExecutor
        from .lattice import LatticeError, canonical_batch, split_lattice, EMPTY_LATTICE, COST_EPS
        L = self._L
        n = C.c_int32()
        nn, na, nf = C.c_int64(), C.c_int64(), C.c_int64()
        N.check(L.wb_lattice_pruned_totals(self._h, C.byref(n), C.byref(nn), C.byref(na),
                                           C.byref(nf)), "lattice")
        meta = np.zeros((max(n.value, 1), 8), np.int64)
        nodes = np.zeros((max(nn.value, 1), 2), np.int32)
        arcs = np.zeros((max(na.value, 1), 4), np.uint32)
        ac = np.zeros(max(na.value, 1), np.float64)
        fin = np.zeros(max(nf.value, 1), np.uint32)
        finw = np.zeros(max(nf.value, 1), np.float64)
        N.check(L.wb_lattice_pruned_fetch(self._h, meta.ctypes.data, nodes.ctypes.data,
                                          arcs.ctypes.data, ac.ctypes.data, fin.ctypes.data,
                                          finw.ctypes.data), "lattice")
        meta = meta[:n.value]
        status = meta[:, 7].copy()
        if ((meta[:, 0] < 0) | (status == N.WB_ERR_CAPACITY)).any():
            raise N.CapacityError("lattice output pool overflowed")
        m6 = meta[:, :6].copy()
        m6[status != N.WB_OK] = 0
        stage1 = canonical_batch(wfst, m6, nodes, arcs, ac, fin, finw)
        best = meta[:, 6].view(np.float64)
        out = []
        for u in range(n.value):
            if status[u] == N.WB_ERR_LATTICE:
                out.append(LatticeError("epsilon cycle among lattice nodes"))
            elif stage1[u].start_id is None:
                out.append(EMPTY_LATTICE)
            else:   # cutoff = best + lattice_beam + COST_EPS (lattice.py:380)
                out.append((stage1[u], (float(best[u]) + float(lattice_beam)) + COST_EPS))
        if not split:
            return out

        def one(item):
            if not isinstance(item, tuple):
                return item
            try:
                return split_lattice(*item)
            except LatticeError as exc:
                return exc
        workers = max_workers or len(os.sched_getaffinity(0))
        with ThreadPoolExecutor(workers) as ex:
            return list(ex.map(one, out))

    # ------------------------------------------------------------------ device buffers
    @_locked
    def decode_device(self, costs, row_offset, num_frames, blank, cfg, mode: str, results,
                      olabels, ilabels, label_capacity: int, stream=None, lattice: bool = False,
                      lattice_beam: float | None = None):
        """Enqueue a decode on device-resident torch tensors (no host sync besides the
        frame-count read); ``results`` is a uint8 CUDA tensor of n * itemsize bytes.  With
        ``lattice`` the trimmed lattices stay on the device until ``fetch_lattices``."""
        n = int(num_frames.numel())
        ncfg = _native_config(cfg, mode, lattice, lattice_beam if lattice else None)
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(self.device).cuda_stream
        rc = self._L.wb_decode(self._h, n, costs.data_ptr(), row_offset.data_ptr(),
                                num_frames.data_ptr(), int(costs.shape[-1]), blank.data_ptr(),
                                C.byref(ncfg), results.data_ptr(), olabels.data_ptr(),
                                ilabels.data_ptr(), int(label_capacity), N.WB_MEM_DEVICE,
                                C.c_void_p(stream))
        N.check(rc, "decode")


# ---------------------------------------------------------------- reference-shaped API
def _check_decodable(w: Wfst, posts) -> None:
    cycle = w.epsilon_cycle()
    if cycle is not None:
        raise WfstError(
            f"epsilon cycle with total weight {cycle.total_weight} through "
            f"states {list(cycle.states)}; non-emitting propagation would not terminate")
    L = posts.rows.shape[1] - 1
    if w.max_ilabel > L:
        raise ValueError(f"graph uses input label {w.max_ilabel} but the posterior matrix "
                         f"only covers labels 1..{L}")


_DECODER_LOCK = threading.Lock()
_RECORDER_PROTOCOL = ("begin_step", "emitting", "epsilon", "survivors", "finish")


def _decoder_for(w: Wfst, checked: bool = False) -> BatchDecoder:
    dev = _current_device()
    with _DECODER_LOCK:
        cache = w.__dict__.setdefault("_b200_decoders", {})
        dec = cache.get((dev, checked))
        if dec is None:
            dec = BatchDecoder(w, dev, checks=checked)
            cache[(dev, checked)] = dec
    return dec


def decode_batch(wfst, posts_list, cfg: DecodeConfig, mode: str | None = None,
                 recorder=None) -> list[DecodeResult]:
    """Decode many utterances in one persistent-kernel launch (utterances are independent,
    SURVEY 8e).  Each element equals ``decode(wfst, posts, cfg)`` of the reference.
    ``recorder``: one ``LatticeRecorder`` per utterance (a list) to record lattices."""
    from .posteriors import PosteriorBatch
    w = as_wfst(wfst)
    mode = mode or cfg.mode
    batch = posts_list if isinstance(posts_list, PosteriorBatch) else None
    posts_list = batch.matrices() if batch is not None else list(posts_list)
    for p in posts_list:
        _check_decodable(w, p)
    if not posts_list:
        return []
    L1s = {p.rows.shape[1] for p in posts_list}
    if len(L1s) != 1:
        raise ValueError("all posterior matrices of a batch must share the label alphabet")
    recorders = None
    if recorder is not None:
        recorders = list(recorder) if isinstance(recorder, (list, tuple)) else [recorder]
        if len(recorders) != len(posts_list):
            raise ValueError("pass one LatticeRecorder per utterance")
        from .lattice import LatticeRecorder
        for rec in recorders:
            if not isinstance(rec, LatticeRecorder) and not all(
                    callable(getattr(rec, m, None)) for m in _RECORDER_PROTOCOL):
                raise TypeError(f"recorder {type(rec).__name__} does not implement "
                                f"{'/'.join(_RECORDER_PROTOCOL)} (lattice.py:112-135)")
    dec = _decoder_for(w)
    with dec.lock:   # the decode and its lattice fetch see one workspace state
        # cost rows are computed on host threads while the kernel already decodes (streaming)
        out = dec.decode_posteriors(batch if batch is not None else posts_list, cfg, mode,
                                    lattice=recorders is not None)
        results = out.decode_results()
        lats = dec.fetch_lattices(w) if recorders is not None else None
    if recorders is not None:
        from .lattice import LatticeRecorder, replay
        for rec, lat, r in zip(recorders, lats, out.results):
            args = (int(r["final_step"]), int(r["final_state"]), bool(r["reached_final"]))
            if isinstance(rec, LatticeRecorder):
                rec._set(lat, *args)
            else:   # e.g. the reference's own lsd_wfst.lattice.LatticeRecorder
                replay(lat, rec, *args)
    return results


def decode_fsd(wfst, posts, cfg: DecodeConfig, recorder=None) -> DecodeResult:
    """Frame-synchronous decoding: one search step per frame (decoder.py:349-352)."""
    return decode_batch(wfst, [posts], cfg, mode="fsd", recorder=recorder)[0]


def decode_lsd(wfst, posts, cfg: DecodeConfig, recorder=None) -> DecodeResult:
    """Label-synchronous decoding: blank frames skipped by the device pre-pass
    (decoder.py:355-359)."""
    return decode_batch(wfst, [posts], cfg, mode="lsd", recorder=recorder)[0]


def decode(wfst, posts, cfg: DecodeConfig, recorder=None) -> DecodeResult:
    """Dispatch on cfg.mode (decoder.py:362-367)."""
    return decode_batch(wfst, [posts], cfg, mode=cfg.mode, recorder=recorder)[0]


def parallel_decode(wfst, posts, cfg: DecodeConfig, workers: int = 1, group_size: int = 32,
                    recorder=None, claim_ledger=None, debug_epoch: bool = False) -> DecodeResult:
    """The reference's parallel engine entry point (parallel.py:205-208).  On the GPU the
    parallelism is the CTA's warps, so ``workers``/``group_size`` are validated for
    compatibility and otherwise unused; the result equals ``decode`` field for field."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if group_size < 1:
        raise ValueError(f"group_size must be >= 1, got {group_size}")
    if claim_ledger is None and not debug_epoch:
        return decode(wfst, posts, cfg, recorder=recorder)
    # the reference's race checks (parallel.py:41-61, 92-116) map to the checked build: the
    # device verifies the per-step claim partition, first-touch registration and slot resets
    # (a violation raises DeviceCheckError, an AssertionError); the claim log fills the ledger
    w = as_wfst(wfst)
    _check_decodable(w, posts)
    dec = _decoder_for(w, checked=True)
    with dec.lock:
        out = dec.decode_posteriors([posts], cfg, cfg.mode, lattice=recorder is not None)
        res = out.decode_result(0)
        lat = dec.fetch_lattices(w)[0] if recorder is not None else None
        if claim_ledger is not None:
            queue, groups = dec.claim_log(res.search_steps)
            at = 0
            for qlen in queue.tolist():
                claims = claim_ledger.begin_step(qlen)
                for t, grp in enumerate(groups[at:at + qlen].tolist()):
                    claims.setdefault(grp, []).append(t)
                at += qlen
    if recorder is not None:
        from .lattice import LatticeRecorder, replay
        r = out.results[0]
        args = (int(r["final_step"]), int(r["final_state"]), bool(r["reached_final"]))
        if isinstance(recorder, LatticeRecorder):
            recorder._set(lat, *args)
        else:
            replay(lat, recorder, *args)
    return res


__all__ = ["BatchDecoder", "BatchOutput", "DecodeConfig", "DecodeResult", "DeviceGraph",
           "SearchDied", "as_wfst", "decode", "decode_batch", "decode_fsd", "decode_lsd",
           "parallel_decode"]
