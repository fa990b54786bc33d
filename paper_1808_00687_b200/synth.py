"""Seeded synthetic graphs and posteriors at benchmark scale (vectorised numpy).

The reference generators (``lsd_wfst/fixtures.py:62-157``) build Python ``Arc`` objects one
by one (24.5 s for a 3M-arc graph); these produce the same *families* directly as arrays:

* ``random_wfst``      -- make_random_wfst semantics (fixtures.py:62-111): a random spanning
  backbone rooted at 0, optional emitting self-loop on every state (olabel 0), extra random
  arcs of which ``eps_fraction`` are forward-only epsilon arcs (so the epsilon subgraph is
  acyclic), weights ``round(U(0, 3), 6)``, finals with probability ``final_fraction``.
* ``random_posteriors`` -- make_random_posteriors semantics (fixtures.py:114-157): an exact
  count of blank frames at ``blank_prob``; other frames put ``peak`` of the non-blank mass on
  a target label that repeats with probability ``repeat_prob``; rows normalised.

Same seed -> same arrays.  The random streams differ from the reference's ``random.Random``
ones, so parity tests against the Python reference use the reference's own generators (in
the build container) and committed golden fixtures; these generators feed the benchmark and
the on-GPU parity checks against the C oracle.
"""
from __future__ import annotations

import numpy as np

from .posteriors import PosteriorMatrix
from .wfst import Wfst


def _weights(rng: np.random.Generator, n: int) -> np.ndarray:
    return np.round(rng.uniform(0.0, 3.0, size=n), 6)


def random_wfst(seed: int, num_states: int, num_arcs: int, num_labels: int,
                eps_fraction: float = 0.0, selfloops: bool = False,
                final_fraction: float = 0.25) -> Wfst:
    rng = np.random.default_rng(seed)
    S, L = int(num_states), int(num_labels)
    parts_src, parts_dst, parts_il, parts_ol, parts_w = [], [], [], [], []
    if S > 1:
        dst = np.arange(1, S, dtype=np.int64)
        src = (rng.random(S - 1) * dst).astype(np.int64)          # uniform in [0, dst)
        parts_src.append(src); parts_dst.append(dst)
        parts_il.append(rng.integers(1, L + 1, S - 1)); parts_ol.append(rng.integers(1, L + 1, S - 1))
        parts_w.append(_weights(rng, S - 1))
    if selfloops:
        s = np.arange(S, dtype=np.int64)
        parts_src.append(s); parts_dst.append(s)
        parts_il.append(rng.integers(1, L + 1, S)); parts_ol.append(np.zeros(S, np.int64))
        parts_w.append(_weights(rng, S))
    have = sum(len(x) for x in parts_src)
    extra = max(0, int(num_arcs) - have)
    if extra:
        n = int(extra * 1.05) + 16
        src = rng.integers(0, S, n)
        dst = rng.integers(0, S, n)
        is_eps = (rng.random(n) < eps_fraction) & (src != dst)
        keep = is_eps | selfloops | (src != dst)
        src, dst, is_eps = src[keep][:extra], dst[keep][:extra], is_eps[keep][:extra]
        m = len(src)
        lo, hi = np.minimum(src, dst), np.maximum(src, dst)
        src = np.where(is_eps, lo, src)
        dst = np.where(is_eps, hi, dst)
        il = np.where(is_eps, 0, rng.integers(1, L + 1, m))
        ol_eps = np.where(rng.random(m) < 0.5, 0, rng.integers(1, L + 1, m))
        ol = np.where(is_eps, ol_eps, rng.integers(1, L + 1, m))
        parts_src.append(src); parts_dst.append(dst); parts_il.append(il); parts_ol.append(ol)
        parts_w.append(_weights(rng, m))
    cat = (lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64))
    finals = np.full(S, np.inf)
    fmask = rng.random(S) < final_fraction
    if not fmask.any():
        fmask[S - 1] = True
    finals[fmask] = _weights(rng, int(fmask.sum()))
    return Wfst.from_arrays(S, 0, cat(parts_src), cat(parts_dst), cat(parts_il), cat(parts_ol),
                            np.concatenate(parts_w) if parts_w else np.zeros(0), finals)


def hclg_like(seed: int = 0, num_states: int = 1_000_000, num_arcs: int = 3_000_000,
              num_labels: int = 3000, eps_fraction: float = 0.015,
              final_fraction: float = 0.01, selfloops: bool = False) -> Wfst:
    """Config-2/3/5 graph: a spanning backbone plus random cross arcs (out-degree
    ~3), ~1.5 % forward-only epsilon arcs, weights round(U(0,3), 6), 1 % finals.  Without
    self-loops this reproduces the survey's measured steady state at beam 13 / max-active
    7000 (~21k candidates -> 7000 survivors per frame); ``selfloops=True`` gives the CTC/TLG
    family of config 4."""
    return random_wfst(seed, num_states, num_arcs, num_labels, eps_fraction=eps_fraction,
                       selfloops=selfloops, final_fraction=final_fraction)


def random_posterior_rows(seed: int, num_frames: int, num_labels: int,
                          blank_fraction: float = 0.0, blank_col: int = 0,
                          blank_prob: float = 0.995, peak: float = 0.9,
                          repeat_prob: float = 0.4,
                          nonblank_blank_range: tuple[float, float] = (0.002, 0.02)) -> np.ndarray:
    rng = np.random.default_rng(seed)
    T, L = int(num_frames), int(num_labels)
    C1 = L + 1
    label_cols = np.array([c for c in range(C1) if c != blank_col], dtype=np.int64)
    n_blank = int(round(blank_fraction * T))
    is_blank = np.zeros(T, dtype=bool)
    if n_blank:
        is_blank[rng.choice(T, n_blank, replace=False)] = True
    # target label process: repeat with prob repeat_prob, else redraw
    redraw = rng.random(T) >= repeat_prob
    draws = rng.integers(0, L, T)
    first = rng.integers(0, L)
    idx = np.where(redraw & ~is_blank, np.arange(T), -1)
    last = np.maximum.accumulate(idx)
    target = np.where(last >= 0, draws[np.maximum(last, 0)], first)
    rows = np.empty((T, C1), dtype=np.float64)
    bprob = rng.uniform(nonblank_blank_range[0], nonblank_blank_range[1], T)
    remaining = 1.0 - bprob
    spread = remaining * (1.0 - peak) / max(1, L - 1) if L > 1 else np.zeros(T)
    rows[:, label_cols] = spread[:, None]
    rows[np.arange(T), label_cols[target]] = remaining * peak
    rows[:, blank_col] = bprob
    if n_blank:
        rows[is_blank] = (1.0 - blank_prob) / L
        rows[is_blank, blank_col] = blank_prob
    rows /= rows.sum(axis=1, keepdims=True)
    return rows


def random_posteriors(seed: int, num_frames: int, num_labels: int, **kw) -> PosteriorMatrix:
    blank_col = kw.get("blank_col", 0)
    return PosteriorMatrix(random_posterior_rows(seed, num_frames, num_labels, **kw), blank_col,
                           validate=False)


__all__ = ["hclg_like", "random_posterior_rows", "random_posteriors", "random_wfst"]
