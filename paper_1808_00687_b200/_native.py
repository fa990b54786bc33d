"""ctypes binding of ``libwfstb200.so`` (the C ABI in ``include/wfst_b200.h``).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).  There is
no fallback: if the library is missing, or no CUDA device is visible, every decode call
raises -- the product path never silently runs on the CPU.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WB_LIB") or os.path.join(_HERE, "_lib", "libwfstb200.so")
# the same kernels compiled with -DWB_CHECKS: device-side invariant checks (claim ledger,
# stale slots, bounds) for tests and parallel_decode(claim_ledger=..., debug_epoch=True)
CHECKED_LIB_PATH = os.path.join(_HERE, "_lib", "libwfstb200_checked.so")

WB_OK, WB_ERR_CUDA, WB_ERR_VALUE, WB_ERR_LATTICE, WB_ERR_WFST, WB_ERR_CAPACITY, WB_ERR_NOMEM = range(7)
WB_PARSE_ERROR, WB_PARSE_SYMBOL = 7, 8
WB_MEM_DEVICE, WB_MEM_HOST = 0, 1
(WB_CAP_CANDIDATES, WB_CAP_ARENA, WB_CAP_FRAMES, WB_CAP_LABELS, WB_CAP_LATTICE_RAW,
 WB_CAP_LATTICE_OUT, WB_CAP_EPS_ROUNDS, WB_CAP_STREAM) = (1, 2, 4, 8, 16, 32, 64, 128)
# wb_utt_result.path_flags: prune / expand branches an utterance took (test evidence)
WB_PATH_GLOBAL_CANDS, WB_PATH_SELECT, WB_PATH_RADIX, WB_PATH_PREFETCH = 1, 2, 4, 8


class NativeError(RuntimeError):
    """A CUDA / native failure reported by libwfstb200."""


class CapacityError(NativeError):
    """A device workspace capacity was exceeded (the caller may retry larger)."""


class GraphDesc(C.Structure):
    _fields_ = [("num_states", C.c_int32), ("num_arcs", C.c_int32), ("start", C.c_int32),
                ("_pad", C.c_int32),
                ("row_ptr", C.c_void_p), ("eps_end", C.c_void_p), ("dst", C.c_void_p),
                ("ilabel", C.c_void_p), ("olabel", C.c_void_p), ("weight", C.c_void_p),
                ("final_w", C.c_void_p)]


class Config(C.Structure):
    _fields_ = [("beam", C.c_double), ("blank_threshold", C.c_double),
                ("max_active", C.c_int32), ("mode", C.c_int32), ("lattice", C.c_int32),
                ("log_rows", C.c_int32), ("lattice_beam", C.c_double)]


class DecoderOpts(C.Structure):
    _fields_ = [("max_utts_in_flight", C.c_int32), ("cand_capacity", C.c_int32),
                ("arena_capacity", C.c_int64), ("max_frames", C.c_int32),
                ("block_threads", C.c_int32), ("lattice_capacity", C.c_int64),
                ("cluster_ctas", C.c_int32), ("_pad", C.c_int32),
                ("lattice_out_capacity", C.c_int64)]


class ParsedWfst(C.Structure):
    _fields_ = [("num_states", C.c_int32), ("start", C.c_int32), ("num_arcs", C.c_int64),
                ("num_finals", C.c_int64), ("src", C.c_void_p), ("dst", C.c_void_p),
                ("ilabel", C.c_void_p), ("olabel", C.c_void_p), ("weight", C.c_void_p),
                ("final_state", C.c_void_p), ("final_weight", C.c_void_p),
                ("error_line", C.c_int32), ("_pad", C.c_int32)]


class LatticeArrays(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_arcs", C.c_int64), ("n_finals", C.c_int64),
                ("node_state", C.c_void_p), ("node_step", C.c_void_p), ("arc_from", C.c_void_p),
                ("arc_to", C.c_void_p), ("arc_tie", C.c_void_p), ("arc_il", C.c_void_p),
                ("arc_ol", C.c_void_p), ("arc_g", C.c_void_p), ("arc_a", C.c_void_p),
                ("final_node", C.c_void_p), ("final_w", C.c_void_p)]


UTT_RESULT_DTYPE = np.dtype([
    ("total_cost", np.float64), ("tokens_expanded", np.int64), ("search_steps", np.int32),
    ("reached_final", np.int32), ("died_at_step", np.int32), ("final_state", np.int32),
    ("final_step", np.int32), ("n_olabels", np.int32), ("n_ilabels", np.int32),
    ("status", np.int32), ("capacity_flags", np.int32), ("path_flags", np.int32),
    ("best_trace", np.int64), ("n_tok", np.int64), ("a_emit", np.int64),
    ("a_fin", np.int64), ("e_eps", np.int64), ("n_cand", np.int64), ("n_surv", np.int64),
    ("n_rec", np.int64), ("lat_arcs", np.int64), ("a_cas", np.int64), ("eps_rounds", np.int64),
    ("phase_cycles", np.int64, (8,))])

_lib = None

# Every symbol include/wfst_b200.h declares (checked by tests/test_native_abi.py).
EXPORTED = ("wb_last_error", "wb_version", "wb_device_count", "wb_graph_create",
            "wb_graph_destroy", "wb_graph_device_bytes", "wb_decoder_create",
            "wb_decoder_destroy", "wb_decoder_device_bytes", "wb_decode", "wb_last_kernel_ms",
            "wb_lattice_totals", "wb_lattice_fetch", "wb_lattice_check", "wb_lattice_prune",
            "wb_lattice_arrays_free", "wb_lattice_best_path", "wb_last_transfer",
            "wb_lattice_canonical", "wb_lattice_pruned_totals", "wb_lattice_pruned_fetch",
            "wb_lattice_split", "wb_decode_stream", "wb_decode_finish", "wb_wfst_parse_text",
            "wb_parsed_wfst_free", "wb_gather_rows", "wb_post1_info", "wb_post1_read", "wb_last_launch",
            "wb_checks_enabled", "wb_check_report", "wb_claim_log", "wb_lattice_format_text",
            "wb_lattice_parse_text", "wb_text_free", "wb_decoder_lanes", "wb_sort_arcs")


_checked_lib = None


def load(checked: bool = False):
    """Load and prototype the library (raises if it has not been built); ``checked`` = the
    -DWB_CHECKS build of the same kernels."""
    global _lib, _checked_lib
    if checked:
        if _checked_lib is None:
            _checked_lib = _open(CHECKED_LIB_PATH)
        return _checked_lib
    if _lib is None:
        _lib = _open(LIB_PATH)
    return _lib


def _open(path):
    if not os.path.exists(path):
        raise NativeError(f"{path} is missing: run __graft_entry__.build() first "
                          "(the decoder has no CPU fallback)")
    L = C.CDLL(path)
    L.wb_last_error.restype = C.c_char_p
    L.wb_version.restype = C.c_int
    L.wb_device_count.argtypes = [C.POINTER(C.c_int32)]
    L.wb_graph_create.argtypes = [C.POINTER(GraphDesc), C.c_int32, C.POINTER(C.c_void_p)]
    L.wb_graph_destroy.argtypes = [C.c_void_p]
    L.wb_graph_device_bytes.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    L.wb_decoder_create.argtypes = [C.c_void_p, C.POINTER(DecoderOpts), C.POINTER(C.c_void_p)]
    L.wb_decoder_destroy.argtypes = [C.c_void_p]
    L.wb_decoder_device_bytes.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    L.wb_decode.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                            C.c_void_p, C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_int32, C.c_int32, C.c_void_p]
    L.wb_last_kernel_ms.argtypes = [C.c_void_p, C.POINTER(C.c_float)]
    L.wb_decode_stream.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int32, C.c_void_p, C.POINTER(Config), C.c_int32,
                                   C.c_void_p, C.c_void_p, C.c_void_p]
    L.wb_sort_arcs.argtypes = [C.c_int64] + [C.c_void_p] * 6
    L.wb_gather_rows.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
                                 C.c_int32, C.c_void_p, C.c_int64, C.c_int32]
    L.wb_gather_rows.restype = None
    L.wb_last_launch.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
    L.wb_decoder_lanes.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.wb_lattice_format_text.argtypes = [C.POINTER(LatticeArrays), C.POINTER(C.c_void_p),
                                         C.POINTER(C.c_int64)]
    L.wb_lattice_parse_text.argtypes = [C.c_char_p, C.c_int64, C.POINTER(LatticeArrays)]
    L.wb_text_free.argtypes = [C.c_void_p]
    L.wb_text_free.restype = None
    L.wb_check_report.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
    L.wb_claim_log.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                               C.c_int64, C.POINTER(C.c_int64)]
    L.wb_post1_info.argtypes = [C.c_char_p] + [C.POINTER(C.c_int32)] * 3
    L.wb_post1_read.argtypes = [C.c_char_p, C.c_void_p, C.c_int64]
    L.wb_decode_finish.argtypes = [C.c_void_p] + [C.c_void_p] * 3
    L.wb_wfst_parse_text.argtypes = [C.c_char_p, C.c_int64, C.c_int32, C.c_char_p, C.c_int64,
                                     C.c_char_p, C.c_int64, C.POINTER(ParsedWfst)]
    L.wb_parsed_wfst_free.argtypes = [C.POINTER(ParsedWfst)]
    L.wb_parsed_wfst_free.restype = None
    L.wb_last_transfer.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    L.wb_lattice_totals.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.wb_lattice_fetch.argtypes = [C.c_void_p] + [C.c_void_p] * 6
    L.wb_lattice_pruned_totals.argtypes = L.wb_lattice_totals.argtypes
    L.wb_lattice_pruned_fetch.argtypes = [C.c_void_p] + [C.c_void_p] * 6
    LP = C.POINTER(LatticeArrays)
    L.wb_lattice_check.argtypes = [LP]
    L.wb_lattice_prune.argtypes = [LP, C.c_double, LP]
    L.wb_lattice_arrays_free.argtypes = [LP]
    L.wb_lattice_split.argtypes = [LP, C.c_double, LP]
    L.wb_lattice_arrays_free.restype = None
    L.wb_lattice_canonical.argtypes = [C.c_int32] + [C.c_void_p] * 6 + [C.c_int32] + \
        [C.c_void_p] * 3 + [C.c_int32] + [C.c_void_p] * 12
    L.wb_lattice_best_path.argtypes = [LP, C.POINTER(C.c_double), C.c_void_p,
                                       C.POINTER(C.c_int32), C.c_void_p, C.POINTER(C.c_int32),
                                       C.c_int32]
    return L


def post1_info(path: str) -> tuple[int, int, int]:
    """(frames, columns, blank column) of a POST1 file (native header check)."""
    from .posteriors import PosteriorFormatError
    T, Cn, b = C.c_int32(), C.c_int32(), C.c_int32()
    if load().wb_post1_info(path.encode(), C.byref(T), C.byref(Cn), C.byref(b)) != WB_OK:
        raise PosteriorFormatError(f"{path}: {last_error()}")
    return T.value, Cn.value, b.value


def post1_read(path: str, dst) -> None:
    """Read a POST1 file's rows into the float64 rows ``dst`` (e.g. a page-locked table)."""
    from .posteriors import PosteriorFormatError
    if load().wb_post1_read(path.encode(), dst.ctypes.data, dst.strides[0] // 8) != WB_OK:
        raise PosteriorFormatError(f"{path}: {last_error()}")


def last_error() -> str:
    """Text of the last failure on the calling thread (wb_last_error)."""
    return (load().wb_last_error() or b"").decode(errors="replace")


CHECK_NAMES = {1: "a live token was expanded zero or several times in one step (claim ledger)",
               2: "a state was registered as a candidate twice in one step (first-touch CAS)",
               3: "a slot touched in a step was not reset at its end (stale epoch)",
               4: "a slot was left non-empty between utterances (stale epoch)",
               5: "a workspace index out of bounds"}


class DeviceCheckError(AssertionError):
    """A device invariant check of the checked build failed (the analogue of the reference's
    ClaimLedger.verify_partitions / debug_epoch AssertionError, parallel.py:52-61, 113-116)."""


def check(rc: int, what: str = "", lib=None) -> None:
    if rc == WB_OK:
        return
    libs = [lib] if lib is not None else [x for x in (_lib, _checked_lib) if x is not None]
    msg = next((m for m in ((x.wb_last_error() or b"").decode(errors="replace") for x in libs)
                if m), "")
    text = f"{what}: {msg}" if what else msg
    if rc == WB_ERR_VALUE:
        raise ValueError(text)
    if rc == WB_ERR_WFST:
        from .wfst import WfstError
        raise WfstError(text)
    if rc == WB_ERR_LATTICE:
        from .lattice import LatticeError
        raise LatticeError(text)
    if rc == WB_ERR_CAPACITY:
        raise CapacityError(text)
    raise NativeError(text)


# ---------------------------------------------------------------- deferred destruction
# Freeing device memory synchronises the device.  A finalizer that runs while a streaming
# decode waits for the host to publish cost rows (wb_decode_stream) would deadlock, so handle
# destruction is queued and done at safe points (before a launch, on workspace re-creation,
# at exit).  Decoders go before graphs (a decoder refers to its graph).
_PENDING: list = []
_PENDING_LOCK = threading.Lock()


def defer_destroy(kind: str, handle, lib=None) -> None:
    with _PENDING_LOCK:
        _PENDING.append((kind, handle, lib))


def flush_destroy() -> None:
    with _PENDING_LOCK:
        items = list(_PENDING)
        _PENDING.clear()
    for kind in ("wb_decoder_destroy", "wb_graph_destroy"):
        for k, h, lib in items:
            L = lib or _lib
            if k == kind and L is not None:
                getattr(L, k)(h)


atexit.register(flush_destroy)


def device_count() -> int:
    n = C.c_int32(0)
    rc = load().wb_device_count(C.byref(n))
    if rc != WB_OK:
        return 0
    return int(n.value)
