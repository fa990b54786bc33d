"""ctypes front end of the C oracle (``wfst_oracle.c``) -- TEST INFRASTRUCTURE ONLY.

The oracle restates the reference serial decoder (``lsd_wfst/decoder.py``) and lattice code
(``lsd_wfst/lattice.py``) in C.  It is pinned against the Python reference (run in the build
container) by ``tests/test_oracle.py`` and the committed golden fixtures under ``tests/golden``.

Graph arguments are duck-typed: any object with ``num_states, start, row_ptr, eps_end, dst,
ilabel, olabel, weight, final_w`` numpy arrays (e.g. ``paper_1808_00687_b200.Wfst``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

OG_OK, OG_ERR_VALUE, OG_ERR_LATTICE = 0, 2, 3


class OracleLatticeError(Exception):
    """The oracle's stand-in for the reference LatticeError."""


class _Graph(C.Structure):
    _fields_ = [("num_states", C.c_int32), ("start", C.c_int32), ("num_arcs", C.c_int32),
                ("_pad", C.c_int32),
                ("row_ptr", C.c_void_p), ("eps_end", C.c_void_p), ("dst", C.c_void_p),
                ("ilabel", C.c_void_p), ("olabel", C.c_void_p), ("weight", C.c_void_p),
                ("final_w", C.c_void_p)]


class _Config(C.Structure):
    _fields_ = [("beam", C.c_double), ("max_active", C.c_int32), ("mode", C.c_int32),
                ("blank_threshold", C.c_double), ("record_lattice", C.c_int32),
                ("canonical", C.c_int32)]


class _Result(C.Structure):
    _fields_ = [("total_cost", C.c_double), ("tokens_expanded", C.c_int64),
                ("search_steps", C.c_int32), ("reached_final", C.c_int32),
                ("died_at_step", C.c_int32), ("n_olabels", C.c_int32), ("n_ilabels", C.c_int32),
                ("final_state", C.c_int32), ("final_step", C.c_int32), ("status", C.c_int32),
                ("olabels", C.POINTER(C.c_int32)), ("ilabels", C.POINTER(C.c_int32)),
                ("n_node_steps", C.c_int32),
                ("surv_off", C.POINTER(C.c_int64)), ("surv", C.POINTER(C.c_int32)),
                ("n_emit", C.c_int64), ("n_eps", C.c_int64),
                ("emit_step", C.c_void_p), ("emit_src", C.c_void_p), ("emit_arc", C.c_void_p),
                ("emit_ac", C.c_void_p),
                ("eps_step", C.c_void_p), ("eps_src", C.c_void_p), ("eps_arc", C.c_void_p)]


class _Lattice(C.Structure):
    _fields_ = [("empty", C.c_int32), ("n_nodes", C.c_int64), ("n_arcs", C.c_int64),
                ("n_finals", C.c_int64),
                ("node_state", C.POINTER(C.c_int32)), ("node_step", C.POINTER(C.c_int32)),
                ("arc_from", C.POINTER(C.c_int64)), ("arc_to", C.POINTER(C.c_int64)),
                ("arc_tie", C.POINTER(C.c_int64)),
                ("arc_il", C.POINTER(C.c_int32)), ("arc_ol", C.POINTER(C.c_int32)),
                ("arc_g", C.POINTER(C.c_double)), ("arc_a", C.POINTER(C.c_double)),
                ("final_node", C.POINTER(C.c_int64)), ("final_w", C.POINTER(C.c_double))]


_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with make (gcc); returns the library path."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "wfst_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.og_decode.argtypes = [C.POINTER(_Graph), C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                C.POINTER(_Config), C.POINTER(_Result)]
        L.og_decode_batch.argtypes = [C.POINTER(_Graph), C.c_int32, C.POINTER(C.c_void_p),
                                      C.POINTER(C.c_void_p), C.c_void_p, C.c_int32,
                                      C.POINTER(_Config), C.POINTER(_Result), C.c_int32]
        L.og_result_free.argtypes = [C.POINTER(_Result)]
        L.og_build_lattice.argtypes = [C.POINTER(_Graph), C.POINTER(_Result), C.POINTER(_Lattice)]
        L.og_prune_lattice.argtypes = [C.POINTER(_Lattice), C.c_double, C.POINTER(_Lattice)]
        L.og_prune_lattice_stage1.argtypes = [C.POINTER(_Lattice), C.c_double, C.POINTER(_Lattice),
                                              C.POINTER(C.c_double)]
        L.og_lattice_best_path.argtypes = [C.POINTER(_Lattice), C.POINTER(C.c_double),
                                           C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.c_int32),
                                           C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.c_int32)]
        L.og_lattice_free.argtypes = [C.POINTER(_Lattice)]
        L.og_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class OracleGraph:
    """Holds contiguous copies of a graph's CSR arrays and the C struct pointing at them."""

    def __init__(self, g):
        self.num_states = int(g.num_states)
        self.start = int(g.start)
        self.row_ptr = np.ascontiguousarray(g.row_ptr, dtype=np.int32)
        self.eps_end = np.ascontiguousarray(g.eps_end, dtype=np.int32)
        self.dst = np.ascontiguousarray(g.dst, dtype=np.int32)
        self.ilabel = np.ascontiguousarray(g.ilabel, dtype=np.int32)
        self.olabel = np.ascontiguousarray(g.olabel, dtype=np.int32)
        self.weight = np.ascontiguousarray(g.weight, dtype=np.float64)
        self.final_w = np.ascontiguousarray(g.final_w, dtype=np.float64)
        self.c = _Graph(self.num_states, self.start, len(self.dst), 0,
                        _ptr(self.row_ptr), _ptr(self.eps_end), _ptr(self.dst), _ptr(self.ilabel),
                        _ptr(self.olabel), _ptr(self.weight), _ptr(self.final_w))


def _as_graph(g) -> OracleGraph:
    return g if isinstance(g, OracleGraph) else OracleGraph(g)


def _config(beam, max_active, mode, blank_threshold, record_lattice=False, canonical=False):
    return _Config(float(beam), int(max_active or 0), 0 if mode == "fsd" else 1,
                   float(blank_threshold), int(bool(record_lattice)), int(bool(canonical)))


@dataclass
class OracleResult:
    total_cost: float
    olabels: tuple
    ilabels: tuple
    search_steps: int
    tokens_expanded: int
    reached_final: bool
    died_at_step: int | None
    final_state: int = -1
    final_step: int = -1
    survivors: list | None = None   # per node step, sorted state arrays (record_lattice)

    def astuple(self):
        return (self.total_cost, self.olabels, self.ilabels, self.search_steps,
                self.tokens_expanded, self.reached_final, self.died_at_step)


def _take_result(r: _Result, with_survivors: bool) -> OracleResult:
    ol = tuple(r.olabels[i] for i in range(r.n_olabels))
    il = tuple(r.ilabels[i] for i in range(r.n_ilabels))
    surv = None
    if with_survivors:
        off = np.ctypeslib.as_array(r.surv_off, shape=(r.n_node_steps + 1,)).copy()
        flat = (np.ctypeslib.as_array(r.surv, shape=(int(off[-1]),)).copy()
                if off[-1] > 0 else np.zeros(0, np.int32))
        surv = [flat[off[k]:off[k + 1]] for k in range(r.n_node_steps)]
    return OracleResult(r.total_cost, ol, il, r.search_steps, r.tokens_expanded,
                        bool(r.reached_final), None if r.died_at_step < 0 else r.died_at_step,
                        r.final_state, r.final_step, surv)


def decode(graph, costs: np.ndarray, blank: np.ndarray, *, beam=float("inf"), max_active=None,
           mode="lsd", blank_threshold=0.98, record_lattice=False, canonical=False,
           return_lattice=False):
    """One utterance.  ``costs`` [T, L'+1] float64 with column 0 = +inf; ``blank`` [T]."""
    g = _as_graph(graph)
    costs = np.ascontiguousarray(costs, dtype=np.float64)
    blank = np.ascontiguousarray(blank, dtype=np.float64)
    T = costs.shape[0]
    L1 = costs.shape[1] if costs.ndim == 2 else 1
    cfg = _config(beam, max_active, mode, blank_threshold, record_lattice or return_lattice, canonical)
    res = _Result()
    rc = lib().og_decode(C.byref(g.c), _ptr(costs), _ptr(blank), T, L1, C.byref(cfg), C.byref(res))
    if rc:
        raise RuntimeError(f"oracle decode failed ({rc})")
    try:
        out = _take_result(res, record_lattice or return_lattice)
        lat = None
        if return_lattice:
            lat = _lattice_call(lambda o: lib().og_build_lattice(C.byref(g.c), C.byref(res), o))
        return (out, lat) if return_lattice else out
    finally:
        lib().og_result_free(C.byref(res))


def decode_batch(graph, costs_list, blank_list, *, beam=float("inf"), max_active=None, mode="lsd",
                 blank_threshold=0.98, n_threads=None, canonical=False):
    """Many utterances on host threads (the CPU baseline).  Returns a list of OracleResult."""
    g = _as_graph(graph)
    n = len(costs_list)
    costs_list = [np.ascontiguousarray(c, dtype=np.float64) for c in costs_list]
    blank_list = [np.ascontiguousarray(b, dtype=np.float64) for b in blank_list]
    L1 = costs_list[0].shape[1] if n else 1
    cp = (C.c_void_p * max(n, 1))(*[_ptr(c) for c in costs_list])
    bp = (C.c_void_p * max(n, 1))(*[_ptr(b) for b in blank_list])
    T = np.asarray([c.shape[0] for c in costs_list], dtype=np.int32)
    cfg = _config(beam, max_active, mode, blank_threshold, False, canonical)
    res = (_Result * max(n, 1))()
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    rc = lib().og_decode_batch(C.byref(g.c), n, cp, bp, _ptr(T), L1, C.byref(cfg), res, n_threads)
    try:
        if rc:
            raise RuntimeError(f"oracle batch decode failed ({rc})")
        return [_take_result(res[i], False) for i in range(n)]
    finally:
        for i in range(n):
            lib().og_result_free(C.byref(res[i]))


@dataclass
class OracleLattice:
    """Array form of a reference Lattice (lattice.py:53-57)."""
    empty: bool
    node_state: np.ndarray
    node_step: np.ndarray
    arc_from: np.ndarray
    arc_to: np.ndarray
    arc_il: np.ndarray
    arc_ol: np.ndarray
    arc_g: np.ndarray
    arc_a: np.ndarray
    arc_tie: np.ndarray
    final_node: np.ndarray
    final_w: np.ndarray

    @property
    def is_empty(self):
        return self.empty or len(self.final_node) == 0

    def key(self):
        """Structural identity as the reference's Lattice.__eq__ sees it (tie excluded)."""
        if self.empty:
            return ("EMPTY",)
        nodes = tuple(zip(self.node_state.tolist(), self.node_step.tolist()))
        arcs = tuple(zip(self.arc_from.tolist(), self.arc_to.tolist(), self.arc_il.tolist(),
                         self.arc_ol.tolist(), self.arc_g.tolist(), self.arc_a.tolist()))
        finals = dict(zip(self.final_node.tolist(), self.final_w.tolist()))
        return (nodes, arcs, 0, finals)

    def _to_c(self):
        self._keep = [np.ascontiguousarray(x) for x in (
            self.node_state.astype(np.int32), self.node_step.astype(np.int32),
            self.arc_from.astype(np.int64), self.arc_to.astype(np.int64), self.arc_tie.astype(np.int64),
            self.arc_il.astype(np.int32), self.arc_ol.astype(np.int32),
            self.arc_g.astype(np.float64), self.arc_a.astype(np.float64),
            self.final_node.astype(np.int64), self.final_w.astype(np.float64))]
        k = self._keep
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
        return _Lattice(int(self.empty), len(k[0]), len(k[2]), len(k[9]),
                        P(k[0], C.c_int32), P(k[1], C.c_int32), P(k[2], C.c_int64),
                        P(k[3], C.c_int64), P(k[4], C.c_int64), P(k[5], C.c_int32),
                        P(k[6], C.c_int32), P(k[7], C.c_double), P(k[8], C.c_double),
                        P(k[9], C.c_int64), P(k[10], C.c_double))


def _empty_lattice():
    z = lambda t: np.zeros(0, t)  # noqa: E731
    return OracleLattice(True, z(np.int32), z(np.int32), z(np.int64), z(np.int64), z(np.int32),
                         z(np.int32), z(np.float64), z(np.float64), z(np.int64), z(np.int64),
                         z(np.float64))


def _from_c(lat: _Lattice) -> OracleLattice:
    if lat.empty:
        return _empty_lattice()

    def arr(p, n):
        return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, p._type_)
    nn, na, nf = lat.n_nodes, lat.n_arcs, lat.n_finals
    return OracleLattice(False, arr(lat.node_state, nn), arr(lat.node_step, nn),
                         arr(lat.arc_from, na), arr(lat.arc_to, na), arr(lat.arc_il, na),
                         arr(lat.arc_ol, na), arr(lat.arc_g, na), arr(lat.arc_a, na),
                         arr(lat.arc_tie, na), arr(lat.final_node, nf), arr(lat.final_w, nf))


def _lattice_call(fn) -> OracleLattice:
    out = _Lattice()
    rc = fn(C.byref(out))
    try:
        if rc == OG_ERR_LATTICE:
            raise OracleLatticeError("lattice error")
        if rc == OG_ERR_VALUE:
            raise ValueError("bad lattice argument")
        if rc:
            raise RuntimeError(f"oracle lattice call failed ({rc})")
        return _from_c(out)
    finally:
        lib().og_lattice_free(C.byref(out))


def prune_lattice(lat: OracleLattice, beam: float) -> OracleLattice:
    cl = lat._to_c()
    return _lattice_call(lambda o: lib().og_prune_lattice(C.byref(cl), float(beam), o))


def prune_lattice_stage1(lat: OracleLattice, beam: float) -> OracleLattice:
    cl = lat._to_c()
    cut = C.c_double(0.0)
    return _lattice_call(lambda o: lib().og_prune_lattice_stage1(C.byref(cl), float(beam), o,
                                                                 C.byref(cut)))


def lattice_best_path(lat: OracleLattice):
    cl = lat._to_c()
    cost = C.c_double()
    ol, il = C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)()
    no, ni = C.c_int32(), C.c_int32()
    rc = lib().og_lattice_best_path(C.byref(cl), C.byref(cost), C.byref(ol), C.byref(no),
                                    C.byref(il), C.byref(ni))
    if rc == OG_ERR_LATTICE:
        raise OracleLatticeError("no best path")
    if rc:
        raise RuntimeError(f"oracle best path failed ({rc})")
    try:
        return cost.value, tuple(ol[i] for i in range(no.value)), tuple(il[i] for i in range(ni.value))
    finally:
        lib().og_free(C.cast(ol, C.c_void_p))
        lib().og_free(C.cast(il, C.c_void_p))


def lattice_from_reference(lat) -> OracleLattice:
    """Convert a reference ``lsd_wfst.lattice.Lattice`` (tests only)."""
    if lat.start_id is None:
        return _empty_lattice()
    return OracleLattice(
        False,
        np.asarray([n.state for n in lat.nodes], np.int32),
        np.asarray([n.step for n in lat.nodes], np.int32),
        np.asarray([a.from_id for a in lat.arcs], np.int64),
        np.asarray([a.to_id for a in lat.arcs], np.int64),
        np.asarray([a.ilabel for a in lat.arcs], np.int32),
        np.asarray([a.olabel for a in lat.arcs], np.int32),
        np.asarray([a.graph_cost for a in lat.arcs], np.float64),
        np.asarray([a.acoustic_cost for a in lat.arcs], np.float64),
        np.asarray([a.tie for a in lat.arcs], np.int64),
        np.asarray(list(lat.finals.keys()), np.int64),
        np.asarray(list(lat.finals.values()), np.float64))
