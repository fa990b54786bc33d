"""Tropical-semiring WFST in CSR form, ready for upload to HBM.

Mirrors the reference data model (``lsd_wfst/wfst.py``): arcs grouped by source state and
sorted by ``(src, ilabel, dst, olabel, weight)`` (wfst.py:182), so every state's range splits
into an epsilon prefix and an emitting suffix (wfst.py:192-198); final weights of +inf are
dropped (wfst.py:183).  Unlike the reference, the storage is a set of numpy arrays
(structure-of-arrays), built with a vectorised lexsort, so million-state graphs construct in
seconds instead of minutes:

    row_ptr[S+1]  int32   arc_offsets           (wfst.py:185-190)
    eps_end[S]    int32   eps_split             (wfst.py:192-198)
    dst/ilabel/olabel[A] int32, weight[A] float64
    final_w[S]    float64 (+inf = not final)

The same arrays are what ``DeviceGraph`` uploads to the GPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

EPSILON = 0
ZERO = math.inf  # tropical "no path"
ONE = 0.0


class WfstError(Exception):
    """Base class for transducer construction and parsing failures (wfst.py:34)."""


class ParseError(WfstError):
    def __init__(self, message: str, line_no: int | None = None):
        if line_no is not None:
            message = f"line {line_no}: {message}"
        super().__init__(message)
        self.line_no = line_no


class SymbolError(WfstError):
    """A label token could not be resolved against a symbol table (wfst.py:46-47)."""


class SymbolTable:
    """Label id <-> symbol string map (reference ``SymbolTable``, wfst.py:67-151).

    Id 0 is always ``<eps>``; a ``<blank>`` entry's id is kept as ``blank_id``.  Remapping a
    symbol or an id to a different partner raises ``SymbolError`` (``ParseError`` from
    ``parse``, with the line number).
    """

    EPS_SYMBOL = "<eps>"
    BLANK_SYMBOL = "<blank>"

    def __init__(self, symbols: dict[str, int] | None = None):
        self._by_sym: dict[str, int] = {self.EPS_SYMBOL: 0}
        self._by_id: dict[int, str] = {0: self.EPS_SYMBOL}
        self.blank_id: int | None = None
        for sym, idx in (symbols or {}).items():
            self.add(sym, idx)

    def add(self, symbol: str, idx: int | None = None) -> int:
        if idx is None:
            idx = max(self._by_id) + 1
        if idx == 0 or symbol == self.EPS_SYMBOL:
            if idx == 0 and symbol == self.EPS_SYMBOL:
                return 0
            raise SymbolError(f"id 0 is reserved for {self.EPS_SYMBOL!r}, got {symbol!r} = {idx}")
        have = self._by_sym.get(symbol)
        if have is not None and have != idx:
            raise SymbolError(f"symbol {symbol!r} already mapped to {have}, cannot remap to {idx}")
        other = self._by_id.get(idx)
        if other is not None and other != symbol:
            raise SymbolError(f"id {idx} already mapped to {other!r}, cannot remap to {symbol!r}")
        self._by_sym[symbol] = idx
        self._by_id[idx] = symbol
        if symbol == self.BLANK_SYMBOL:
            self.blank_id = idx
        return idx

    def find_id(self, symbol: str) -> int | None:
        return self._by_sym.get(symbol)

    def find_symbol(self, idx: int) -> str | None:
        return self._by_id.get(idx)

    def __len__(self) -> int:
        return len(self._by_sym)

    def __contains__(self, symbol: str) -> bool:
        return symbol in self._by_sym

    def __iter__(self):
        return iter(sorted(self._by_id.items()))

    @classmethod
    def parse(cls, text: str) -> "SymbolTable":
        """``symbol id`` lines; ``#`` comments and blank lines skipped; id 0 must be <eps>."""
        table = cls()
        for line_no, raw in enumerate(text.splitlines(), start=1):
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            f = line.split()
            if len(f) != 2:
                raise ParseError(f"expected 'symbol id', got {raw!r}", line_no)
            try:
                idx = int(f[1])
            except ValueError:
                raise ParseError(f"bad id {f[1]!r}", line_no) from None
            if idx == 0:
                if f[0] != cls.EPS_SYMBOL:
                    raise ParseError(f"id 0 must be {cls.EPS_SYMBOL!r}, got {f[0]!r}", line_no)
                continue
            try:
                table.add(f[0], idx)
            except SymbolError as exc:
                raise ParseError(str(exc), line_no) from None
        return table

    def format(self) -> str:
        return "".join(f"{sym} {idx}\n" for idx, sym in sorted(self._by_id.items()))


@dataclass(frozen=True)
class Arc:
    src: int
    dst: int
    ilabel: int
    olabel: int
    weight: float


@dataclass(frozen=True)
class EpsilonCycle:
    """One offending epsilon cycle with non-positive total weight (wfst.py:59-64)."""

    states: tuple[int, ...]
    total_weight: float


class Wfst:
    """Immutable transducer in CSR arrays; same constructor as the reference ``Wfst``.

    ``Wfst(num_states, start, arcs, final_weights)`` takes a list of ``Arc`` (any object with
    ``src, dst, ilabel, olabel, weight``); ``Wfst.from_arrays`` takes parallel arrays.
    """

    def __init__(self, num_states: int, start: int, arcs, final_weights: dict[int, float]):
        arcs = list(arcs)
        n = len(arcs)
        src = np.fromiter((a.src for a in arcs), dtype=np.int64, count=n)
        dst = np.fromiter((a.dst for a in arcs), dtype=np.int64, count=n)
        il = np.fromiter((a.ilabel for a in arcs), dtype=np.int64, count=n)
        ol = np.fromiter((a.olabel for a in arcs), dtype=np.int64, count=n)
        w = np.fromiter((float(a.weight) for a in arcs), dtype=np.float64, count=n)
        self._init_arrays(num_states, start, src, dst, il, ol, w, final_weights)

    @classmethod
    def from_arrays(cls, num_states: int, start: int, src, dst, ilabel, olabel, weight,
                    final_weights) -> "Wfst":
        """Vectorised construction.  ``final_weights``: dict, or a length-S float array with
        +inf for non-final states."""
        self = cls.__new__(cls)
        self._init_arrays(num_states, start, np.asarray(src, np.int64), np.asarray(dst, np.int64),
                          np.asarray(ilabel, np.int64), np.asarray(olabel, np.int64),
                          np.asarray(weight, np.float64), final_weights)
        return self

    @classmethod
    def from_reference(cls, ref) -> "Wfst":
        """Adopt an already-sorted reference ``lsd_wfst.Wfst`` (its arc order is kept)."""
        return cls(ref.num_states, ref.start, ref.arcs, ref.final_weights)

    def _init_arrays(self, num_states, start, src, dst, il, ol, w, final_weights):
        if num_states <= 0:
            raise WfstError("a Wfst needs at least one state")
        if not 0 <= start < num_states:
            raise WfstError(f"start state {start} out of range [0, {num_states})")
        S = int(num_states)
        if len(src):
            if src.min() < 0 or src.max() >= S or dst.min() < 0 or dst.max() >= S:
                raise WfstError("an arc references an invalid state")
            if il.min() < 0 or ol.min() < 0:
                raise WfstError("an arc has a negative label id")
        if np.isnan(w).any():
            raise WfstError("an arc weight is NaN")
        if len(src) >= 2**31 - 1 or S >= 2**31 - 1:
            raise WfstError("graph exceeds the int32 CSR index range")
        if isinstance(final_weights, dict):
            fw = np.full(S, np.inf)
            for s, x in final_weights.items():
                if not 0 <= s < S:
                    raise WfstError(f"final state {s} out of range")
                if math.isnan(x):
                    raise WfstError(f"final weight of state {s} is NaN")
                fw[s] = float(x)
        else:
            fw = np.array(final_weights, dtype=np.float64, copy=True)
            if fw.shape != (S,):
                raise WfstError("final weight array must have one entry per state")
            if np.isnan(fw).any():
                raise WfstError("a final weight is NaN")
        # sort key (src, ilabel, dst, olabel, weight) -- wfst.py:182; lexsort is stable
        order = np.lexsort((w, ol, dst, il, src))
        self.num_states = S
        self.start = int(start)
        self.dst = np.ascontiguousarray(dst[order], dtype=np.int32)
        self.ilabel = np.ascontiguousarray(il[order], dtype=np.int32)
        self.olabel = np.ascontiguousarray(ol[order], dtype=np.int32)
        self.weight = np.ascontiguousarray(w[order], dtype=np.float64)
        src_sorted = src[order]
        counts = np.bincount(src_sorted, minlength=S) if len(src_sorted) else np.zeros(S, np.int64)
        row_ptr = np.zeros(S + 1, dtype=np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        self.row_ptr = row_ptr.astype(np.int32)
        eps_counts = (np.bincount(src_sorted[self.ilabel == EPSILON], minlength=S)
                      if len(src_sorted) else np.zeros(S, np.int64))
        self.eps_end = (row_ptr[:-1] + eps_counts).astype(np.int32)
        self.final_w = fw
        self.has_epsilon_arcs = bool((self.ilabel == EPSILON).any())
        self.max_ilabel = int(self.ilabel.max()) if len(self.ilabel) else 0
        self._eps_cycle_checked = False
        self._eps_cycle = None
        self._arcs = None
        self._src = None
        for a in (self.dst, self.ilabel, self.olabel, self.weight, self.row_ptr, self.eps_end,
                  self.final_w):
            a.setflags(write=False)

    # --- reference-compatible views (built lazily; cheap graphs only) -------------------
    @property
    def num_arcs(self) -> int:
        return int(len(self.dst))

    @property
    def src(self) -> np.ndarray:
        if self._src is None:
            self._src = np.repeat(np.arange(self.num_states, dtype=np.int32),
                                  np.diff(self.row_ptr.astype(np.int64)))
        return self._src

    @property
    def arcs(self) -> list[Arc]:
        if self._arcs is None:
            self._arcs = [Arc(int(s), int(d), int(i), int(o), float(x)) for s, d, i, o, x in
                          zip(self.src, self.dst, self.ilabel, self.olabel, self.weight)]
        return self._arcs

    @property
    def arc_offsets(self) -> list[int]:
        return self.row_ptr.tolist()

    @property
    def eps_split(self) -> list[int]:
        return self.eps_end.tolist()

    @property
    def final_weights(self) -> dict[int, float]:
        idx = np.nonzero(self.final_w != np.inf)[0]
        return {int(s): float(self.final_w[s]) for s in idx}

    def out_arcs(self, state: int) -> list[Arc]:
        self._check_state(state)
        return self.arcs[self.row_ptr[state]:self.row_ptr[state + 1]]

    def out_degree(self, state: int) -> int:
        self._check_state(state)
        return int(self.row_ptr[state + 1] - self.row_ptr[state])

    def final_weight(self, state: int) -> float:
        self._check_state(state)
        return float(self.final_w[state])

    def is_final(self, state: int) -> bool:
        return bool(self.final_w[state] != np.inf)

    def _check_state(self, state: int) -> None:
        if not 0 <= state < self.num_states:
            raise IndexError(f"state {state} out of range [0, {self.num_states})")

    def epsilon_cycle(self) -> EpsilonCycle | None:
        """Cached ``validate_epsilon_acyclic`` (wfst.py:242-247)."""
        if not self._eps_cycle_checked:
            self._eps_cycle = validate_epsilon_acyclic(self)
            self._eps_cycle_checked = True
        return self._eps_cycle


def _eps_edges(w: Wfst):
    m = w.ilabel == EPSILON
    return w.src[m].astype(np.int64), w.dst[m].astype(np.int64), w.weight[m]


def _has_structural_cycle(n: int, u: np.ndarray, v: np.ndarray) -> bool:
    """Kahn's algorithm on the epsilon subgraph (vectorised frontier peeling)."""
    if len(u) == 0:
        return False
    if (u == v).any():
        return True
    indeg = np.bincount(v, minlength=n)
    order = np.argsort(u, kind="stable")
    us, vs = u[order], v[order]
    off = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(us, minlength=n), out=off[1:])
    frontier = np.nonzero(indeg == 0)[0]
    removed = len(frontier)
    while len(frontier):
        starts, ends = off[frontier], off[frontier + 1]
        lens = ends - starts
        if lens.sum() == 0:
            break
        idx = np.repeat(starts, lens) + (np.arange(lens.sum()) - np.repeat(np.cumsum(lens) - lens, lens))
        succ = vs[idx]
        np.subtract.at(indeg, succ, 1)
        cand = np.unique(succ)
        frontier = cand[indeg[cand] == 0]
        removed += len(frontier)
    return removed < n


def validate_epsilon_acyclic(w: Wfst) -> EpsilonCycle | None:
    """Detect an epsilon cycle with total weight <= 0 (wfst.py:412-470).

    Fast path: an epsilon subgraph with no structural cycle at all (the usual case, and every
    graph ``make_random_wfst`` emits) is accepted after a vectorised Kahn peel.  Otherwise the
    reference procedure runs: Bellman-Ford from a virtual zero source, then a cycle search on
    zero-reduced-cost (tight) arcs.
    """
    u, v, wt = _eps_edges(w)
    if len(u) == 0:
        return None
    n = w.num_states
    if not _has_structural_cycle(n, u, v):
        return None
    edges = list(zip(u.tolist(), v.tolist(), wt.tolist()))
    dist = [0.0] * n
    pred = [-1] * n
    relaxed_tail = -1
    for _ in range(n):
        relaxed_tail = -1
        for a, b, x in edges:
            c = dist[a] + x
            if c < dist[b] - 1e-15:
                dist[b] = c
                pred[b] = a
                relaxed_tail = b
        if relaxed_tail < 0:
            break
    if relaxed_tail >= 0:
        x = relaxed_tail
        for _ in range(n):
            x = pred[x]
        cycle = [x]
        y = pred[x]
        while y != x:
            cycle.append(y)
            y = pred[y]
        cycle.reverse()
        return EpsilonCycle(tuple(cycle), _cycle_weight(cycle, edges))
    tight: dict[int, list[int]] = {}
    for a, b, x in edges:
        if dist[a] + x <= dist[b] + 1e-12:
            tight.setdefault(a, []).append(b)
    cycle = _find_cycle(tight, n)
    if cycle is not None:
        return EpsilonCycle(tuple(cycle), _cycle_weight(cycle, edges))
    return None


def _cycle_weight(cycle, edges) -> float:
    lookup: dict[tuple[int, int], float] = {}
    for a, b, x in edges:
        if (a, b) not in lookup or x < lookup[(a, b)]:
            lookup[(a, b)] = x
    return sum(lookup[(a, b)] for a, b in zip(cycle, cycle[1:] + cycle[:1]))


def _find_cycle(succ: dict[int, list[int]], num_states: int):
    color = [0] * num_states
    parent: dict[int, int] = {}
    for root in sorted(succ):
        if color[root]:
            continue
        stack = [(root, iter(succ.get(root, ())))]
        color[root] = 1
        while stack:
            node, it = stack[-1]
            for nxt in it:
                if color[nxt] == 0:
                    color[nxt] = 1
                    parent[nxt] = node
                    stack.append((nxt, iter(succ.get(nxt, ()))))
                    break
                if color[nxt] == 1:
                    cycle = [node]
                    x = node
                    while x != nxt:
                        x = parent[x]
                        cycle.append(x)
                    cycle.reverse()
                    return cycle
            else:
                color[node] = 2
                stack.pop()
    return None


def _parse_fast(text: str, allow_negative_weights: bool):
    """The C++ fast path (csrc/wfst_text.cpp); None when the text needs this module's parser
    (symbols, non-ASCII, malformed lines -- which then raise exactly as the reference)."""
    try:
        from . import _native as N
        L = N.load()
    except Exception:   # library not built: the Python parser is exact, only slower
        return None
    data = text.encode("ascii", errors="replace") if text.isascii() else None
    if data is None:
        return None
    out = N.ParsedWfst()
    rc = L.wb_wfst_parse_text(data, len(data), int(bool(allow_negative_weights)), C.byref(out))
    if rc != N.WB_OK:
        return None
    try:
        def arr(ptr, n, t):
            if n == 0:
                return np.zeros(0, t)
            ct = np.ctypeslib.as_ctypes_type(t)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).copy()
        na, nfin = out.num_arcs, out.num_finals
        fw = np.full(out.num_states, np.inf)
        fw[arr(out.final_state, nfin, np.int32)] = arr(out.final_weight, nfin, np.float64)
        return Wfst.from_arrays(out.num_states, out.start, arr(out.src, na, np.int32),
                                arr(out.dst, na, np.int32), arr(out.ilabel, na, np.int32),
                                arr(out.olabel, na, np.int32), arr(out.weight, na, np.float64),
                                fw)
    finally:
        L.wb_parsed_wfst_free(C.byref(out))


def _label(tok: str, table: SymbolTable | None, line_no: int) -> int:
    """Symbol lookup first, then a bare non-negative integer id (wfst.py:300-312)."""
    if table is not None:
        idx = table.find_id(tok)
        if idx is not None:
            return idx
    try:
        idx = int(tok)
    except ValueError:
        raise SymbolError(f"line {line_no}: unknown symbol {tok!r}") from None
    if idx < 0:
        raise SymbolError(f"line {line_no}: negative label id {idx}")
    return idx


def parse_wfst_text(text: str, isyms: SymbolTable | None = None,
                    osyms: SymbolTable | None = None,
                    allow_negative_weights: bool = False) -> Wfst:
    """AT&T-style transducer text (reference ``parse_wfst_text``, wfst.py:315-378).

    Arc lines ``src dst ilabel olabel [weight]``, final lines ``state [weight]`` (missing
    weight = 0.0); the first state mentioned is the start state; ``#`` comment lines and
    blank lines are skipped.  Labels resolve through ``isyms`` / ``osyms`` when given, with
    bare non-negative integers accepted as raw ids.  Without symbol tables the text goes
    through the C++ fast path (csrc/wfst_text.cpp) when it can reproduce this parser exactly.
    """
    if isyms is None and osyms is None:
        fast = _parse_fast(text, allow_negative_weights)
        if fast is not None:
            return fast
    arcs: list[Arc] = []
    finals: dict[int, float] = {}
    start = None
    max_state = -1

    def state(tok, line_no):
        try:
            x = int(tok)
        except ValueError:
            raise ParseError(f"bad state id {tok!r}", line_no) from None
        if x < 0:
            raise ParseError(f"negative state id {x}", line_no)
        return x

    def weight(tok, line_no):
        try:
            x = float(tok)
        except ValueError:
            raise ParseError(f"bad weight {tok!r}", line_no) from None
        if math.isnan(x):
            raise ParseError("weight is NaN", line_no)
        if x < 0 and not allow_negative_weights:
            raise ParseError(f"negative weight {x} (pass allow_negative_weights to accept)",
                             line_no)
        return x

    for line_no, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        f = line.split()
        if len(f) in (1, 2):
            s = state(f[0], line_no)
            finals[s] = weight(f[1], line_no) if len(f) == 2 else 0.0
            start = s if start is None else start
            max_state = max(max_state, s)
        elif len(f) in (4, 5):
            a, b = state(f[0], line_no), state(f[1], line_no)
            i, o = _label(f[2], isyms, line_no), _label(f[3], osyms, line_no)
            x = weight(f[4], line_no) if len(f) == 5 else 0.0
            arcs.append(Arc(a, b, i, o, x))
            start = a if start is None else start
            max_state = max(max_state, a, b)
        else:
            raise ParseError(f"expected 1-2 (final) or 4-5 (arc) fields, got {len(f)}", line_no)
    if start is None:
        raise ParseError("no states found in transducer text")
    return Wfst(max_state + 1, start, arcs, finals)


def format_wfst_text(w: Wfst) -> str:
    """AT&T text that ``parse_wfst_text`` reads back to the same graph: the start state is
    mentioned first, weights are written with ``repr`` so they round-trip exactly.  Raises
    ``WfstError`` for graphs text cannot express (a start state with neither arcs nor a final
    weight while other states have arcs; trailing states no line mentions)."""
    src = w.src
    fin = w.final_weights
    order = np.argsort(src != w.start, kind="stable")  # the start state's arcs first
    lines = [f"{int(src[k])} {int(w.dst[k])} {int(w.ilabel[k])} {int(w.olabel[k])} "
             f"{float(w.weight[k])!r}" for k in order.tolist()]
    finals = [f"{s} {x!r}" for s, x in sorted(fin.items())]
    if w.start in fin and (not lines or int(src[order[0]]) != w.start):
        finals.remove(f"{w.start} {fin[w.start]!r}")
        lines.insert(0, f"{w.start} {fin[w.start]!r}")
    elif lines and int(src[order[0]]) != w.start:
        raise WfstError("the start state has no arcs and no final weight; text cannot name it")
    mentioned = [w.start, *fin] + ([int(src.max()), int(w.dst.max())] if len(src) else [])
    if max(mentioned) != w.num_states - 1:
        raise WfstError("trailing states with no arcs and no final weight cannot be written")
    return "\n".join(lines + finals) + "\n"


# ------------------------------------------------- binary CSR cache
_CSR_MAGIC = "wfst-b200-csr-v1"


def save_wfst_binary(w: Wfst, path) -> None:
    """Write the canonical CSR arrays (plus the cached epsilon-cycle verdict) so later runs
    skip text parsing, sorting and ``validate_epsilon_acyclic``.  ``.npz``, uncompressed."""
    cyc = w.epsilon_cycle()
    np.savez(path, magic=np.array(_CSR_MAGIC), num_states=np.int64(w.num_states),
             start=np.int64(w.start), row_ptr=w.row_ptr, eps_end=w.eps_end, dst=w.dst,
             ilabel=w.ilabel, olabel=w.olabel, weight=w.weight, final_w=w.final_w,
             eps_cycle_states=np.array(cyc.states if cyc else [], np.int64),
             eps_cycle_weight=np.float64(cyc.total_weight if cyc else np.nan),
             has_eps_cycle=np.bool_(cyc is not None))


def load_wfst_binary(path) -> Wfst:
    """Inverse of ``save_wfst_binary``; the arrays are checked for CSR consistency (and
    re-sorted if a foreign writer left them unsorted) but not re-parsed."""
    with np.load(path, allow_pickle=False) as z:
        if "magic" not in z.files or str(z["magic"]) != _CSR_MAGIC:
            raise WfstError(f"{path}: not a {_CSR_MAGIC} file")
        S = int(z["num_states"])
        row_ptr = z["row_ptr"].astype(np.int64)
        if row_ptr.shape != (S + 1,) or row_ptr[0] != 0 or (np.diff(row_ptr) < 0).any():
            raise WfstError(f"{path}: corrupt row_ptr")
        A = int(row_ptr[-1])
        arrs = [z[k] for k in ("dst", "ilabel", "olabel", "weight")]
        if any(a.shape != (A,) for a in arrs):
            raise WfstError(f"{path}: arc arrays disagree with row_ptr")
        src = np.repeat(np.arange(S, dtype=np.int64), np.diff(row_ptr))
        w = Wfst.from_arrays(S, int(z["start"]), src, *arrs, z["final_w"])
        if not np.array_equal(w.eps_end, z["eps_end"]):
            raise WfstError(f"{path}: corrupt eps_end")
        w._eps_cycle_checked = True
        w._eps_cycle = (EpsilonCycle(tuple(int(x) for x in z["eps_cycle_states"]),
                                     float(z["eps_cycle_weight"]))
                        if bool(z["has_eps_cycle"]) else None)
    return w


def graph_nbytes(w: Wfst) -> int:
    """Device footprint of a graph (CSR + packed arc records + finals)."""
    return int(w.num_states * (4 + 4 + 8) + 4 + w.num_arcs * (16 + 4))


__all__ = ["Arc", "EpsilonCycle", "ParseError", "SymbolError", "SymbolTable", "Wfst", "WfstError",
           "format_wfst_text", "load_wfst_binary", "parse_wfst_text", "save_wfst_binary",
           "validate_epsilon_acyclic", "EPSILON", "ZERO", "ONE"]
