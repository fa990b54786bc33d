"""Word lattices from the device decoder (the reference's ``lsd_wfst.lattice``).

Same surface as /root/reference/pkg/src/lsd_wfst/lattice.py: ``LatticeNode``, ``LatticeArc``,
``Lattice``, ``EMPTY_LATTICE``, ``LatticeRecorder``, ``build_lattice``, ``prune_lattice``,
``lattice_best_path``, ``format_lattice_text`` / ``parse_lattice_text`` / ``save_lattice`` /
``load_lattice``, ``LatticeError``.

Where the reference records every relaxation into Python lists and assembles the lattice
afterwards (lattice.py:96-249), the decode kernel records the raw lattice of each node step
in HBM (survivor nodes, emitting arcs from the previous step's survivors, within-step epsilon
arcs) and trims it to start-to-final paths before anything leaves the device
(``csrc/decode_kernel.cuh``: ``record_lattice_step`` / ``trim_lattice``).  The host receives
only the trimmed lattice as flat arrays and orders it canonically (lattice.py:215-230).
Pruning and the best path run in C++ over those arrays (``csrc/lattice_host.cpp``).

``Lattice`` is array-backed; ``nodes`` / ``arcs`` materialise the reference's tuples of frozen
dataclasses lazily, and equality follows the reference (``tie`` excluded).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

INF = math.inf
COST_EPS = 1e-9  # lattice.py:26


class LatticeError(Exception):
    """Lattice construction / pruning failure (lattice.py:29)."""


@dataclass(frozen=True)
class LatticeNode:
    state: int
    step: int


@dataclass(frozen=True)
class LatticeArc:
    from_id: int
    to_id: int
    ilabel: int
    olabel: int
    graph_cost: float
    acoustic_cost: float
    tie: int = field(compare=False, default=0)


def _i32(x):
    return np.ascontiguousarray(x, dtype=np.int32)


def _i64(x):
    return np.ascontiguousarray(x, dtype=np.int64)


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


class Lattice:
    """Array-backed lattice.  Node i = (node_state[i], node_step[i]); node 0 is the start
    node; arcs are parallel arrays; finals map node id -> final weight."""

    __slots__ = ("node_state", "node_step", "arc_from", "arc_to", "arc_il", "arc_ol", "arc_g",
                 "arc_a", "arc_tie", "final_node", "final_w", "_nodes", "_arcs", "_finals")

    def __init__(self, node_state=(), node_step=(), arc_from=(), arc_to=(), arc_il=(), arc_ol=(),
                 arc_g=(), arc_a=(), arc_tie=(), final_node=(), final_w=()):
        self.node_state = _i32(node_state)
        self.node_step = _i32(node_step)
        self.arc_from = _i64(arc_from)
        self.arc_to = _i64(arc_to)
        self.arc_il = _i32(arc_il)
        self.arc_ol = _i32(arc_ol)
        self.arc_g = _f64(arc_g)
        self.arc_a = _f64(arc_a)
        self.arc_tie = _i64(arc_tie)
        self.final_node = _i64(final_node)
        self.final_w = _f64(final_w)
        self._nodes = self._arcs = self._finals = None

    # ---------------------------------------------------------------- reference surface
    @property
    def start_id(self):
        return 0 if len(self.node_state) else None

    @property
    def nodes(self) -> tuple:
        if self._nodes is None:
            self._nodes = tuple(LatticeNode(s, t) for s, t in
                                zip(self.node_state.tolist(), self.node_step.tolist()))
        return self._nodes

    @property
    def arcs(self) -> tuple:
        if self._arcs is None:
            self._arcs = tuple(LatticeArc(*x) for x in zip(
                self.arc_from.tolist(), self.arc_to.tolist(), self.arc_il.tolist(),
                self.arc_ol.tolist(), self.arc_g.tolist(), self.arc_a.tolist(),
                self.arc_tie.tolist()))
        return self._arcs

    @property
    def finals(self) -> dict:
        if self._finals is None:
            self._finals = dict(zip(self.final_node.tolist(), self.final_w.tolist()))
        return self._finals

    @property
    def is_empty(self) -> bool:
        return self.start_id is None or len(self.final_node) == 0

    @property
    def num_nodes(self) -> int:
        return len(self.node_state)

    @property
    def num_arcs(self) -> int:
        return len(self.arc_from)

    def out_adjacency(self) -> list:
        adj = [[] for _ in range(self.num_nodes)]
        for a in self.arcs:
            adj[a.from_id].append(a)
        return adj

    def in_adjacency(self) -> list:
        adj = [[] for _ in range(self.num_nodes)]
        for a in self.arcs:
            adj[a.to_id].append(a)
        return adj

    def key(self):
        """Structural identity as the reference's ``Lattice.__eq__`` sees it (tie excluded)."""
        if self.start_id is None:
            return ("EMPTY",)
        nodes = tuple(zip(self.node_state.tolist(), self.node_step.tolist()))
        arcs = tuple(zip(self.arc_from.tolist(), self.arc_to.tolist(), self.arc_il.tolist(),
                         self.arc_ol.tolist(), self.arc_g.tolist(), self.arc_a.tolist()))
        return (nodes, arcs, 0, self.finals)

    def __eq__(self, other):
        if isinstance(other, Lattice):
            return self.key() == other.key()
        if hasattr(other, "nodes") and hasattr(other, "arcs") and hasattr(other, "finals"):
            return self.key() == _reference_key(other)
        return NotImplemented

    def __hash__(self):  # pragma: no cover - frozen-dataclass parity, rarely used
        return hash((self.num_nodes, self.num_arcs))

    def __repr__(self):
        return f"Lattice(nodes={self.num_nodes}, arcs={self.num_arcs}, finals={len(self.final_node)})"

    # ---------------------------------------------------------------- conversions
    @classmethod
    def from_reference(cls, lat) -> "Lattice":
        """Array form of a reference ``lsd_wfst.lattice.Lattice``."""
        if lat.start_id is None:
            return EMPTY_LATTICE
        a = lat.arcs
        fin = list(lat.finals.items())
        return cls([n.state for n in lat.nodes], [n.step for n in lat.nodes],
                   [x.from_id for x in a], [x.to_id for x in a], [x.ilabel for x in a],
                   [x.olabel for x in a], [x.graph_cost for x in a], [x.acoustic_cost for x in a],
                   [x.tie for x in a], [k for k, _ in fin], [w for _, w in fin])

    def _view(self):
        """wb_lattice_arrays over this lattice's buffers (kept alive by self)."""
        from . import _native as N
        P = lambda x: x.ctypes.data  # noqa: E731
        return N.LatticeArrays(self.num_nodes, self.num_arcs, len(self.final_node),
                               P(self.node_state), P(self.node_step), P(self.arc_from),
                               P(self.arc_to), P(self.arc_tie), P(self.arc_il), P(self.arc_ol),
                               P(self.arc_g), P(self.arc_a), P(self.final_node), P(self.final_w))

    @classmethod
    def _from_native(cls, v) -> "Lattice":
        if v.n_nodes == 0:
            return EMPTY_LATTICE

        def arr(p, n, t):
            if n == 0:
                return np.zeros(0, t)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(t))),
                                         shape=(n,)).copy()
        nn, na, nf = v.n_nodes, v.n_arcs, v.n_finals
        return cls(arr(v.node_state, nn, np.int32), arr(v.node_step, nn, np.int32),
                   arr(v.arc_from, na, np.int64), arr(v.arc_to, na, np.int64),
                   arr(v.arc_il, na, np.int32), arr(v.arc_ol, na, np.int32),
                   arr(v.arc_g, na, np.float64), arr(v.arc_a, na, np.float64),
                   arr(v.arc_tie, na, np.int64), arr(v.final_node, nf, np.int64),
                   arr(v.final_w, nf, np.float64))


def _reference_key(lat):
    if lat.start_id is None:
        return ("EMPTY",)
    nodes = tuple((n.state, n.step) for n in lat.nodes)
    arcs = tuple((a.from_id, a.to_id, a.ilabel, a.olabel, a.graph_cost, a.acoustic_cost)
                 for a in lat.arcs)
    return (nodes, arcs, lat.start_id, dict(lat.finals))


EMPTY_LATTICE = Lattice()


# ---------------------------------------------------------------- device lattice -> Lattice
def canonical_from_device(wfst, nodes: np.ndarray, arcs: np.ndarray, arc_ac: np.ndarray,
                          finals: np.ndarray, final_w: np.ndarray) -> Lattice:
    """Order one utterance's trimmed device lattice canonically (_assemble, lattice.py:215-236):
    nodes [start] + sorted by (step, state); arcs sorted by (from.step, from.state, to.step,
    to.state, ilabel, olabel, tie) with tie = the WFST arc index."""
    if len(nodes) == 0:
        return EMPTY_LATTICE
    st = nodes[:, 0].astype(np.int32)
    sp = nodes[:, 1].astype(np.int32)
    is_start = (st == wfst.start) & (sp == 0)
    order = np.lexsort((st, sp, ~is_start))
    newid = np.empty(len(order), dtype=np.int64)
    newid[order] = np.arange(len(order))
    ai = arcs[:, 2].astype(np.int64)
    f = newid[arcs[:, 0].astype(np.int64)]
    t = newid[arcs[:, 1].astype(np.int64)]
    il = wfst.ilabel[ai]
    ol = wfst.olabel[ai]
    nst, nsp = st[order], sp[order]
    aord = np.lexsort((ai, ol, il, nst[t], nsp[t], nst[f], nsp[f]))
    fo = newid[finals.astype(np.int64)]
    return Lattice(nst, nsp, f[aord], t[aord], il[aord], ol[aord], wfst.weight[ai][aord],
                   arc_ac[aord], ai[aord], fo, final_w)


def canonical_batch(wfst, meta, nodes, arcs, arc_ac, finals, final_w,
                    n_threads: int | None = None) -> list:
    """``canonical_from_device`` for a whole batch: the C++ pass (``wb_lattice_canonical``)
    orders every utterance's lattice on host threads, then each ``Lattice`` is a view into
    the flat output arrays.  ``meta`` rows: {node_off, n_nodes, arc_off, n_arcs, final_off,
    n_finals} into the fetched pools."""
    import os
    from . import _native as N
    n = len(meta)
    if n == 0:
        return []
    meta = np.ascontiguousarray(meta, np.int64)
    nn, na, nf = (int(meta[:, i].sum()) for i in (1, 3, 5))
    om = np.zeros((n, 6), np.int64)
    out = dict(st=np.zeros(max(nn, 1), np.int32), sp=np.zeros(max(nn, 1), np.int32),
               f=np.zeros(max(na, 1), np.int64), t=np.zeros(max(na, 1), np.int64),
               il=np.zeros(max(na, 1), np.int32), ol=np.zeros(max(na, 1), np.int32),
               g=np.zeros(max(na, 1), np.float64), a=np.zeros(max(na, 1), np.float64),
               tie=np.zeros(max(na, 1), np.int64), fn=np.zeros(max(nf, 1), np.int64),
               fw=np.zeros(max(nf, 1), np.float64))
    ins = [np.ascontiguousarray(nodes, np.int32), np.ascontiguousarray(arcs, np.uint32),
           np.ascontiguousarray(arc_ac, np.float64), np.ascontiguousarray(finals, np.uint32),
           np.ascontiguousarray(final_w, np.float64)]
    gi = [np.ascontiguousarray(wfst.ilabel, np.int32), np.ascontiguousarray(wfst.olabel, np.int32),
          np.ascontiguousarray(wfst.weight, np.float64)]
    threads = n_threads or len(os.sched_getaffinity(0))
    rc = N.load().wb_lattice_canonical(
        n, meta.ctypes.data, *(x.ctypes.data for x in ins), int(wfst.start),
        *(x.ctypes.data for x in gi), threads, om.ctypes.data,
        *(out[k].ctypes.data for k in ("st", "sp", "f", "t", "il", "ol", "g", "a", "tie", "fn", "fw")))
    N.check(rc, "lattice")
    res = []
    for u in range(n):
        n0, c0, a0, c1, f0, c2 = (int(x) for x in om[u])
        if c0 == 0:
            res.append(EMPTY_LATTICE)
            continue
        ns, as_, fs = slice(n0, n0 + c0), slice(a0, a0 + c1), slice(f0, f0 + c2)
        res.append(Lattice(out["st"][ns], out["sp"][ns], out["f"][as_], out["t"][as_],
                           out["il"][as_], out["ol"][as_], out["g"][as_], out["a"][as_],
                           out["tie"][as_], out["fn"][fs], out["fw"][fs]))
    return res


class StepRecord:
    """One node step of the recorder protocol (the reference's ``_StepRecord``,
    lattice.py:86-93): emitting relaxations (src_state, wfst_arc, acoustic) into step k,
    within-step epsilon relaxations (src_state, wfst_arc), and the step's survivor states."""

    __slots__ = ("emit", "eps", "survivors")

    def __init__(self):
        self.emit: list = []
        self.eps: set = set()
        self.survivors: tuple = ()


def replay(lat: Lattice, recorder, final_step: int, final_state: int, reached: bool) -> None:
    """Drive any object with the reference recorder protocol (``begin_step / emitting /
    epsilon / survivors / finish``, lattice.py:112-135) with a decoded lattice.

    The device records and trims the lattice itself, so the replay carries the trimmed
    lattice: each step's survivors are the lattice nodes of that step, its emitting / epsilon
    calls the lattice arcs into / within it.  The reference's ``build_lattice`` (or its
    ``PipelinedLatticeBuilder``) over these calls assembles exactly ``lat``: trimming an
    already trimmed lattice keeps it, and every live final is one of its nodes."""
    empty = lat.start_id is None
    n_steps = final_step + 1 if final_step is not None and final_step >= 0 else 0
    st = lat.node_state.astype(np.int64)
    sp = lat.node_step.astype(np.int64)
    nodes_at = np.split(np.argsort(sp * (int(st.max(initial=0)) + 1) + st, kind="stable"),
                        np.searchsorted(np.sort(sp), np.arange(1, n_steps)))
    if not empty:
        fs, ts = sp[lat.arc_from], sp[lat.arc_to]
        order = np.lexsort((lat.arc_tie, ts == fs, ts))   # per step: emitting, then epsilon
        bounds = np.searchsorted(ts[order], np.arange(n_steps + 1))
    for k in range(n_steps):
        recorder.begin_step(k)
        if not empty:
            for e in order[bounds[k]:bounds[k + 1]].tolist():
                src, arc = int(st[lat.arc_from[e]]), int(lat.arc_tie[e])
                if fs[e] == k:
                    recorder.epsilon(k, src, arc)
                else:
                    recorder.emitting(k, src, arc, float(lat.arc_a[e]))
        recorder.survivors(k, tuple(int(x) for x in st[nodes_at[k]]) if not empty and
                           k < len(nodes_at) else ())
    recorder.finish(final_step, final_state, reached)


class LatticeRecorder:
    """Pass as ``recorder=`` to ``decode`` / ``decode_fsd`` / ``decode_lsd`` /
    ``parallel_decode`` (lattice.py:96-135); ``build_lattice(recorder, wfst)`` returns the
    lattice the device recorded.  It also implements the reference protocol
    (``begin_step / emitting / epsilon / survivors / finish``): with a ``consumer`` (a
    ``PipelinedLatticeBuilder``, ours or the reference's) the decode replays the lattice
    step by step into it (``feed`` per step, ``close`` at the end), and protocol calls from
    any other source are accumulated like the reference recorder does."""

    def __init__(self, consumer=None):
        self._lattice = None
        self.steps: list[StepRecord] = []
        self.final_step = None
        self.final_state = None
        self.reached_final = False
        self._consumer = consumer

    # ---- the device fast path
    def _set(self, lat: Lattice, final_step: int, final_state: int, reached: bool):
        if self._consumer is not None:   # the consumer sees the step protocol
            replay(lat, self, final_step, final_state, reached)
        self._lattice = lat
        self.final_step, self.final_state, self.reached_final = final_step, final_state, reached

    # ---- the reference protocol
    def begin_step(self, node_step: int) -> None:
        if node_step != len(self.steps):
            raise LatticeError(f"steps must be recorded in order; got {node_step}, "
                               f"expected {len(self.steps)}")
        self.steps.append(StepRecord())

    def emitting(self, node_step: int, src_state: int, wfst_arc: int, acoustic: float) -> None:
        self.steps[node_step].emit.append((src_state, wfst_arc, acoustic))

    def epsilon(self, node_step: int, src_state: int, wfst_arc: int) -> None:
        self.steps[node_step].eps.add((src_state, wfst_arc))

    def survivors(self, node_step: int, states) -> None:
        rec = self.steps[node_step]
        rec.survivors = tuple(states)
        if self._consumer is not None:
            self._consumer.feed(node_step, rec)

    def finish(self, final_step: int, final_state: int, reached_final: bool) -> None:
        self.final_step, self.final_state, self.reached_final = final_step, final_state, reached_final
        if self._consumer is not None:
            self._consumer.close()


class _StepAssembler:
    """Raw lattice from protocol steps (lattice.py:148-183): survivors become nodes; an
    emitting record (deduplicated by (src, arc)) becomes an arc when its source survived step
    k-1 and its destination survives step k; an epsilon record when both ends survive step k
    and it is not a self-loop.  ``build`` trims to start-to-final paths and orders the result
    canonically (``_assemble``, lattice.py:190-237) with numpy / scipy graph searches."""

    def __init__(self, wfst):
        self.wfst = wfst
        self.node_st: list = []
        self.node_sp: list = []
        self.arcs: list = []      # (from_state, from_step, to_state, to_step, wfst_arc, ac)
        self._prev = frozenset()
        self._surv = {}

    def add_step(self, k: int, rec) -> None:
        surv = frozenset(rec.survivors)
        self._surv[k] = surv
        self.node_st.extend(surv)
        self.node_sp.extend([k] * len(surv))
        dst = self.wfst.dst
        if k > 0:
            seen = set()
            for src, ai, ac in rec.emit:
                if (src, ai) not in seen and src in self._prev and int(dst[ai]) in surv:
                    self.arcs.append((src, k - 1, int(dst[ai]), k, ai, ac))
                seen.add((src, ai))
        for src, ai in sorted(rec.eps):
            d = int(dst[ai])
            if src in surv and d in surv and d != src:
                self.arcs.append((src, k, d, k, ai, 0.0))
        self._prev = surv

    def build(self, final_step, final_state, reached_final) -> Lattice:
        from scipy.sparse import csr_matrix
        from scipy.sparse.csgraph import breadth_first_order
        w = self.wfst
        if not self.node_st:
            return EMPTY_LATTICE
        span = max(self.node_sp) + 2
        key = np.unique(np.asarray(self.node_st, np.int64) * span + np.asarray(self.node_sp))
        start_key = w.start * span
        if not np.isin(start_key, key):
            return EMPTY_LATTICE
        if reached_final:
            fs = np.asarray(sorted(self._surv.get(final_step, ())), np.int64)
            fs = fs[w.final_w[fs] != INF] if len(fs) else fs
            fin = {int(s) * span + final_step: float(w.final_w[s]) for s in fs}
        else:
            fin = {final_state * span + final_step: 0.0}
        a = np.asarray(self.arcs, dtype=object).reshape(-1, 6)
        af = np.searchsorted(key, a[:, 0].astype(np.int64) * span + a[:, 1].astype(np.int64))
        at = np.searchsorted(key, a[:, 2].astype(np.int64) * span + a[:, 3].astype(np.int64))
        n = len(key)
        g = csr_matrix((np.ones(len(af)), (af, at)), shape=(n, n))
        fwd = np.zeros(n, bool)
        fwd[breadth_first_order(g, int(np.searchsorted(key, start_key)), return_predecessors=False)] = True
        live = {int(np.searchsorted(key, k)): x for k, x in fin.items()
                if np.isin(k, key) and fwd[np.searchsorted(key, k)]}
        if not live:
            return EMPTY_LATTICE
        bwd = np.zeros(n, bool)
        gt = g.T.tocsr()
        for f in live:
            if not bwd[f]:
                bwd[breadth_first_order(gt, f, return_predecessors=False)] = True
        keep = fwd & bwd
        ka = keep[af] & keep[at]
        ai = a[ka, 4].astype(np.int64)
        nodes = np.stack([key[keep] // span, key[keep] % span], 1).astype(np.int32)
        loc = np.cumsum(keep) - 1
        arcs = np.stack([loc[af[ka]], loc[at[ka]], ai, np.zeros(len(ai), np.int64)], 1)
        fin_ids = np.asarray(sorted(live), np.int64)
        lat = canonical_from_device(w, nodes, arcs.astype(np.uint32), a[ka, 5].astype(np.float64),
                                    loc[fin_ids].astype(np.uint32),
                                    np.asarray([live[f] for f in fin_ids], np.float64))
        _check(lat)
        return lat


class PipelinedLatticeBuilder:
    """The reference's ``PipelinedLatticeBuilder`` (lattice.py:252-292), same use::

        builder = PipelinedLatticeBuilder(wfst)
        rec = LatticeRecorder(consumer=builder)
        decode(wfst, posts, cfg, recorder=rec)      # or parallel_decode
        lat = builder.result_from(rec)

    ``feed(k, step)`` queues a protocol step that a builder thread integrates while the
    producer moves on (the paper's second stream); ``close()`` ends the stream.  With this
    package's decoder the steps come from the device lattice (recorded and trimmed in the
    kernel) replayed at the end of the decode; with the reference decoder they arrive live."""

    def __init__(self, wfst=None):
        import queue
        import threading
        from .decoder import as_wfst
        self._acc = _StepAssembler(as_wfst(wfst)) if wfst is not None else None
        self._q: "queue.Queue" = queue.Queue()
        self._err = None
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()

    def _run(self) -> None:
        while True:
            item = self._q.get()
            if item is None:
                return
            try:
                self._acc.add_step(*item)
            except Exception as exc:  # surfaced by result()
                self._err = exc
                return

    def feed(self, k: int, rec) -> None:
        if self._acc is None:
            raise LatticeError("PipelinedLatticeBuilder needs the transducer")
        self._q.put((k, rec))

    def close(self) -> None:
        self._q.put(None)

    def result(self, final_step: int, final_state: int, reached_final: bool) -> Lattice:
        self._thread.join()
        if self._err is not None:
            raise self._err
        if self._acc is None:
            raise LatticeError("no decode has fed this builder")
        return self._acc.build(final_step, final_state, reached_final)

    def result_from(self, recorder) -> Lattice:
        if recorder.final_step is None:
            raise LatticeError("decode trace is incomplete (finish was never recorded)")
        return self.result(recorder.final_step, recorder.final_state, recorder.reached_final)


def _check(lat: Lattice) -> None:
    from . import _native as N
    if lat.is_empty:
        return
    v = lat._view()
    rc = N.load().wb_lattice_check(C.byref(v))
    N.check(rc, "lattice")


def build_lattice(recorder: LatticeRecorder, wfst=None) -> Lattice:
    """The lattice of the decode ``recorder`` was attached to (lattice.py:240-249); raises
    LatticeError on an epsilon cycle among its nodes (lattice.py:186)."""
    if getattr(recorder, "_lattice", None) is None:
        if recorder.final_step is None:
            if not recorder.steps:
                return EMPTY_LATTICE
            raise LatticeError("decode trace is incomplete (finish was never recorded)")
        if wfst is None:
            raise LatticeError("build_lattice needs the transducer for protocol-recorded steps")
        from .decoder import as_wfst
        acc = _StepAssembler(as_wfst(wfst))
        for k, rec in enumerate(recorder.steps):
            acc.add_step(k, rec)
        return acc.build(recorder.final_step, recorder.final_state, recorder.reached_final)
    _check(recorder._lattice)
    return recorder._lattice


def prune_lattice(lat: Lattice, lattice_beam: float) -> Lattice:
    """Keep exactly the paths within ``lattice_beam`` of the best (lattice.py:359-501)."""
    from . import _native as N
    if lattice_beam < 0:
        raise ValueError(f"lattice_beam must be >= 0, got {lattice_beam}")
    if not isinstance(lat, Lattice):
        lat = Lattice.from_reference(lat)
    if lat.is_empty:
        return EMPTY_LATTICE
    v = lat._view()
    out = N.LatticeArrays()
    rc = N.load().wb_lattice_prune(C.byref(v), float(lattice_beam), C.byref(out))
    try:
        N.check(rc, "prune_lattice")
        return Lattice._from_native(out)
    finally:
        N.load().wb_lattice_arrays_free(C.byref(out))


def split_lattice(lat: Lattice, cutoff: float) -> Lattice:
    """The path-exact second stage of prune_lattice (_enforce_path_soundness,
    lattice.py:430-501) on a lattice already cut at ``cutoff`` (device stage one)."""
    from . import _native as N
    if lat.is_empty:
        return lat if lat.start_id is not None else EMPTY_LATTICE
    v = lat._view()
    out = N.LatticeArrays()
    rc = N.load().wb_lattice_split(C.byref(v), float(cutoff), C.byref(out))
    try:
        N.check(rc, "prune_lattice")
        return Lattice._from_native(out)
    finally:
        N.load().wb_lattice_arrays_free(C.byref(out))


def prune_lattices(lats, lattice_beam: float, max_workers: int | None = None) -> list:
    """``prune_lattice`` over many lattices on host threads (the C++ pass runs without the
    GIL).  A lattice whose split exceeds the cap yields its ``LatticeError`` in its slot."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    def one(lat):
        try:
            return prune_lattice(lat, lattice_beam)
        except LatticeError as exc:
            return exc
    lats = list(lats)
    workers = max_workers or min(len(lats), len(os.sched_getaffinity(0))) or 1
    if workers <= 1:
        return [one(x) for x in lats]
    with ThreadPoolExecutor(workers) as ex:
        return list(ex.map(one, lats))


def lattice_best_path(lat: Lattice) -> tuple[float, tuple[int, ...], tuple[int, ...]]:
    """Minimum-cost start-to-final path (cost, olabels, ilabels), ties as the decoder
    resolves them (lattice.py:504-559)."""
    from . import _native as N
    if not isinstance(lat, Lattice):
        lat = Lattice.from_reference(lat)
    if lat.is_empty:
        raise LatticeError("cannot extract a best path from an empty lattice")
    v = lat._view()
    cap = max(lat.num_arcs, 1)
    ol = np.zeros(cap, np.int32)
    il = np.zeros(cap, np.int32)
    cost = C.c_double()
    no, ni = C.c_int32(), C.c_int32()
    rc = N.load().wb_lattice_best_path(C.byref(v), C.byref(cost), ol.ctypes.data, C.byref(no),
                                       il.ctypes.data, C.byref(ni), cap)
    N.check(rc, "lattice_best_path")
    return float(cost.value), tuple(ol[:no.value].tolist()), tuple(il[:ni.value].tolist())


# ---------------------------------------------------------------- text form (lattice.py:562-627)
def format_lattice_text(lat: Lattice) -> str:
    """Serialise (node id 0 is the start node); native writer (csrc/lattice_text.cpp),
    byte-identical to the reference's (repr floats)."""
    from . import _native as N
    if not isinstance(lat, Lattice):
        lat = Lattice.from_reference(lat)
    v = lat._view()
    ptr, n = C.c_void_p(), C.c_int64()
    L = N.load()
    N.check(L.wb_lattice_format_text(C.byref(v), C.byref(ptr), C.byref(n)), "format_lattice_text")
    try:
        return C.string_at(ptr, n.value).decode("ascii")
    finally:
        L.wb_text_free(ptr)


def format_lattices_text(lats, workers: int | None = None) -> list[str]:
    """``format_lattice_text`` of many lattices on host threads (the native writer runs
    without the GIL)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    lats = list(lats)
    n = workers or min(len(lats), len(os.sched_getaffinity(0))) or 1
    if n <= 1:
        return [format_lattice_text(x) for x in lats]
    with ThreadPoolExecutor(n) as ex:
        return list(ex.map(format_lattice_text, lats))


def parse_lattice_text(text: str) -> Lattice:
    """Inverse of ``format_lattice_text`` (native reader); ``LatticeError`` for malformed
    text, ``ValueError`` for a bad number, as the reference raises them."""
    from . import _native as N
    from .wfst import _native_text
    data = _native_text(text)
    out = N.LatticeArrays()
    L = N.load()
    rc = L.wb_lattice_parse_text(data, len(data), C.byref(out))
    try:
        N.check(rc, "parse_lattice_text")
        return Lattice._from_native(out)
    finally:
        L.wb_lattice_arrays_free(C.byref(out))


def save_lattice(lat: Lattice, path: str) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(format_lattice_text(lat))


def load_lattice(path: str) -> Lattice:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_lattice_text(fh.read())


__all__ = ["COST_EPS", "EMPTY_LATTICE", "Lattice", "LatticeArc", "LatticeError", "LatticeNode",
           "LatticeRecorder", "PipelinedLatticeBuilder", "StepRecord", "build_lattice", "replay", "canonical_batch", "canonical_from_device", "format_lattice_text", "format_lattices_text",
           "lattice_best_path", "load_lattice", "parse_lattice_text", "prune_lattice", "prune_lattices",
           "split_lattice",
           "save_lattice"]
