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
    """Label id <-> symbol map for symbolic transducer text and transcripts (the reference's
    ``SymbolTable``, wfst.py:67-151).  Id 0 is ``<eps>``; the id of ``<blank>`` is kept as
    ``blank_id``.  A symbol or id may be bound once (rebinding raises ``SymbolError``)."""

    EPS_SYMBOL, BLANK_SYMBOL = "<eps>", "<blank>"

    def __init__(self, symbols: dict[str, int] | None = None):
        self._id_of = {self.EPS_SYMBOL: 0}
        self._sym_of = {0: self.EPS_SYMBOL}
        for name, ident in (symbols or {}).items():
            self.add(name, ident)

    @property
    def blank_id(self) -> int | None:
        return self._id_of.get(self.BLANK_SYMBOL)

    def add(self, symbol: str, idx: int | None = None) -> int:
        idx = max(self._sym_of) + 1 if idx is None else int(idx)
        bound_id, bound_sym = self._id_of.get(symbol, idx), self._sym_of.get(idx, symbol)
        if (idx == 0) != (symbol == self.EPS_SYMBOL):
            raise SymbolError(f"id 0 is reserved for {self.EPS_SYMBOL!r}, got {symbol!r} = {idx}")
        if bound_id != idx:
            raise SymbolError(f"symbol {symbol!r} already mapped to {bound_id}, cannot remap to {idx}")
        if bound_sym != symbol:
            raise SymbolError(f"id {idx} already mapped to {bound_sym!r}, cannot remap to {symbol!r}")
        self._id_of[symbol], self._sym_of[idx] = idx, symbol
        return idx

    def find_id(self, symbol: str) -> int | None:
        return self._id_of.get(symbol)

    def find_symbol(self, idx: int) -> str | None:
        return self._sym_of.get(idx)

    def __len__(self) -> int:
        return len(self._id_of)

    def __contains__(self, symbol: str) -> bool:
        return symbol in self._id_of

    def __iter__(self):
        return iter(sorted(self._sym_of.items()))

    @classmethod
    def parse(cls, text: str) -> "SymbolTable":
        """``symbol id`` per line (``#`` comments and blank lines skipped)."""
        table = cls()
        rows = [(n, ln.split()) for n, ln in enumerate(text.splitlines(), 1)]
        for n, f in ((n, f) for n, f in rows if f and not f[0].startswith("#")):
            if len(f) != 2 or not f[1].lstrip("+-").isdigit():
                raise ParseError(f"expected 'symbol id', got {' '.join(f)!r}"
                                 if len(f) != 2 else f"bad id {f[1]!r}", n)
            try:
                table.add(f[0], int(f[1]))
            except SymbolError as exc:
                raise ParseError(str(exc), n) from None
        return table

    def format(self) -> str:
        return "".join(f"{sym} {i}\n" for i, sym in sorted(self._sym_of.items()))


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
        # sort key (src, ilabel, dst, olabel, weight) -- wfst.py:182, stable
        order = _arc_order(src, il, dst, ol, w)
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
    """An epsilon cycle whose total weight is <= 0, or None (the check of wfst.py:412-470:
    such a cycle would make non-emitting propagation diverge; strictly positive cycles are
    accepted).  Same tolerances as the reference: an arc improves a potential when it beats it
    by more than 1e-15, and counts as tight when within 1e-12.

    1. A vectorised Kahn peel accepts epsilon subgraphs with no structural cycle at all (the
       usual case, every make_random_wfst graph).
    2. Otherwise only strongly connected components (scipy.sparse.csgraph) can hold a cycle.
       Per component a vectorised (Jacobi) Bellman-Ford from all-zero potentials either keeps
       improving for |C| passes -- a negative cycle, read off the predecessor graph -- or
       converges; then every arc has non-negative reduced cost and a zero-weight cycle is a
       cycle of tight arcs, i.e. a non-trivial strongly connected component of them.
    """
    u, v, wt = _eps_edges(w)
    if len(u) == 0 or not _has_structural_cycle(w.num_states, u, v):
        return None
    for comp in _components(w.num_states, u, v):
        cyc = _component_cycle(comp, u, v, wt)
        if cyc is not None:
            return EpsilonCycle(tuple(int(x) for x in cyc), _cycle_weight(cyc, u, v, wt))
    return None


def _scc_labels(n: int, u: np.ndarray, v: np.ndarray) -> np.ndarray:
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    g = csr_matrix((np.ones(len(u), np.int8), (u, v)), shape=(n, n))
    return connected_components(g, directed=True, connection="strong")[1]


def _components(n: int, u: np.ndarray, v: np.ndarray):
    """Node sets that can carry a cycle: non-trivial SCCs and self-loop states, ordered by
    their smallest state."""
    lab = _scc_labels(n, u, v)
    size = np.bincount(lab)
    cyclic = size[lab] > 1
    cyclic[u[u == v]] = True
    nodes = np.flatnonzero(cyclic)
    order = np.argsort(lab[nodes], kind="stable")
    groups = np.split(nodes[order], np.flatnonzero(np.diff(lab[nodes][order])) + 1)
    return sorted((g for g in groups if len(g)), key=lambda g: int(g.min()))


def _component_cycle(comp: np.ndarray, u, v, wt):
    inside = np.zeros(max(int(u.max()), int(v.max())) + 1, bool)
    inside[comp] = True
    m = inside[u] & inside[v]
    loc = np.full(len(inside), -1, np.int64)
    loc[comp] = np.arange(len(comp))
    a, b, x = loc[u[m]], loc[v[m]], wt[m]
    k = len(comp)
    dist = np.zeros(k)
    pred = np.full(k, -1, np.int64)
    improving = False
    for _ in range(k + 1):
        cand = dist[a] + x
        best = np.full(k, np.inf)
        np.minimum.at(best, b, cand)
        better = best < dist - 1e-15
        improving = bool(better.any())
        if not improving:
            break
        hit = better[b] & (cand == best[b])
        pred[b[hit]] = a[hit]
        dist = np.where(better, best, dist)
    if improving:
        cyc = _functional_cycle(pred)
    else:
        t = dist[a] + x <= dist[b] + 1e-12
        cyc = _tight_cycle(k, a[t], b[t])
    return None if cyc is None else comp[cyc]


def _functional_cycle(nxt: np.ndarray):
    """A cycle of the map i -> nxt[i] (-1 = none), listed in arc direction (reversed walk)."""
    seen = np.full(len(nxt), -1, np.int64)
    for s0 in range(len(nxt)):
        x, path = s0, []
        while x >= 0 and seen[x] < 0:
            seen[x] = s0
            path.append(x)
            x = int(nxt[x])
        if x >= 0 and seen[x] == s0:
            cyc = path[path.index(x):]
            return np.asarray(cyc[::-1], np.int64)
    return None


def _tight_cycle(k: int, a: np.ndarray, b: np.ndarray):
    if len(a) == 0:
        return None
    loops = a[a == b]
    if len(loops):
        return np.asarray([loops.min()], np.int64)
    lab = _scc_labels(k, a, b)
    big = np.flatnonzero(np.bincount(lab) > 1)
    if not len(big):
        return None
    keep = (lab[a] == big[0]) & (lab[b] == big[0])
    first = {}
    for x, y in zip(a[keep].tolist(), b[keep].tolist()):
        first.setdefault(x, y)
    succ = np.full(k, -1, np.int64)
    succ[list(first)] = list(first.values())
    walk = _functional_cycle(succ)
    return None if walk is None else walk[::-1]


def _cycle_weight(cyc, u, v, wt) -> float:
    """Sum over the cycle's consecutive state pairs of the lightest epsilon arc between them."""
    total = 0.0
    for x, y in zip(cyc, np.roll(cyc, -1)):
        total += float(wt[(u == x) & (v == y)].min())
    return total


def _arc_order(src, il, dst, ol, w) -> np.ndarray:
    """Permutation sorting the arcs stably by (src, ilabel, dst, olabel, weight): the native
    packed-key sort (a no-op check when the input is already in order), else np.lexsort."""
    n = len(src)
    if n >= 4096:
        try:
            from . import _native as N
            L = N.load()
        except Exception:   # no library (a CPU-only checkout): numpy
            L = None
        if L is not None:
            arrs = [np.ascontiguousarray(a, dtype=t) for a, t in
                    ((src, np.int32), (il, np.int32), (dst, np.int32), (ol, np.int32), (w, np.float64))]
            order = np.empty(n, np.int64)
            N.check(L.wb_sort_arcs(n, *(a.ctypes.data for a in arrs), order.ctypes.data), "sort arcs")
            return order
    return np.lexsort((w, ol, dst, il, src))


# ASCII bytes the native tokenizers do not treat as Python does (vertical tab, form feed, the
# \x1c-\x1f separators, a lone carriage return); any non-ASCII text is normalised too
_ODD_ASCII = (b"\x0b", b"\x0c", b"\x1c", b"\x1d", b"\x1e", b"\x1f")


def _native_text(text: str) -> bytes:
    """``text`` as the native tokenizers read it: '\\n' lines with ASCII-space fields exactly
    where Python's ``splitlines`` / ``split`` would find them."""
    if text.isascii():
        data = text.encode("ascii")
        if not any(c in data for c in _ODD_ASCII) and data.count(b"\r") == data.count(b"\r\n"):
            return data
    return "\n".join(" ".join(line.split()) for line in text.splitlines()).encode("utf-8")



def parse_wfst_text(text: str, isyms: SymbolTable | None = None,
                    osyms: SymbolTable | None = None,
                    allow_negative_weights: bool = False) -> Wfst:
    """AT&T-style transducer text (the reference's ``parse_wfst_text``, wfst.py:315-378),
    parsed natively (csrc/wfst_text.cpp): arc lines ``src dst ilabel olabel [weight]``, final
    lines ``state [weight]`` (missing weight 0.0), the first state mentioned is the start,
    ``#`` comment and blank lines skipped; labels resolve through ``isyms`` / ``osyms`` first,
    then as bare non-negative integers.  Raises ``ParseError`` (with ``line_no``) /
    ``SymbolError`` as the reference does."""
    from . import _native as N
    L = N.load()
    data = _native_text(text)   # Python line breaks / Unicode whitespace normalised
    tabs = [t.format().encode("utf-8") if t is not None else None for t in (isyms, osyms)]
    out = N.ParsedWfst()
    rc = L.wb_wfst_parse_text(data, len(data), int(bool(allow_negative_weights)),
                              tabs[0], len(tabs[0] or b""), tabs[1], len(tabs[1] or b""),
                              C.byref(out))
    if rc == N.WB_PARSE_ERROR:
        raise ParseError(N.last_error(), out.error_line or None)
    if rc == N.WB_PARSE_SYMBOL:
        raise SymbolError(f"line {out.error_line}: {N.last_error()}")
    N.check(rc, "parse_wfst_text")
    try:
        def take(ptr, n, t):
            if n == 0:
                return np.zeros(0, t)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(t))),
                                         shape=(n,)).copy()
        na, nf = out.num_arcs, out.num_finals
        finals = np.full(out.num_states, np.inf)
        finals[take(out.final_state, nf, np.int32)] = take(out.final_weight, nf, np.float64)
        return Wfst.from_arrays(out.num_states, out.start, take(out.src, na, np.int32),
                                take(out.dst, na, np.int32), take(out.ilabel, na, np.int32),
                                take(out.olabel, na, np.int32), take(out.weight, na, np.float64),
                                finals)
    finally:
        L.wb_parsed_wfst_free(C.byref(out))


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
