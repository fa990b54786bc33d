"""Loader for the committed golden fixtures (tests/golden/cases.{npz,json}).

The fixtures were produced by running the Python reference (tests/golden/make_golden.py); they
travel to the GPU box, where the reference does not exist.
"""
from __future__ import annotations

import functools
import json
import math
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class GraphArrays:
    num_states: int
    start: int
    row_ptr: np.ndarray
    eps_end: np.ndarray
    dst: np.ndarray
    ilabel: np.ndarray
    olabel: np.ndarray
    weight: np.ndarray
    final_w: np.ndarray

    @property
    def num_arcs(self):
        return len(self.dst)

    def to_wfst(self):
        from paper_1808_00687_b200.wfst import Wfst
        src = np.repeat(np.arange(self.num_states), np.diff(self.row_ptr.astype(np.int64)))
        return Wfst.from_arrays(self.num_states, self.start, src, self.dst, self.ilabel,
                                self.olabel, self.weight, self.final_w)


@dataclass
class Case:
    idx: int
    kind: str
    seed: int
    graph: GraphArrays
    costs: np.ndarray
    blank: np.ndarray
    cfg: dict
    expected: tuple
    lattice: object = None      # "error" | "empty" | lattice key tuple | None (not recorded)
    pruned: list | None = None  # per prune beam: "error" | "empty" | key tuple
    best_path: tuple | None = None
    lattice_arrays: dict | None = None  # raw npz arrays of the built lattice (incl. tie)

    def lattice_object(self):
        """The built reference lattice as a package ``Lattice`` (ties included)."""
        from paper_1808_00687_b200.lattice import Lattice
        z = self.lattice_arrays
        n, ai, af = z["nodes"], z["arcs_i"], z["arcs_f"]
        return Lattice(n[:, 0], n[:, 1], ai[:, 0], ai[:, 1], ai[:, 2], ai[:, 3], af[:, 0],
                       af[:, 1], ai[:, 4], z["fin_i"], z["fin_w"])


def _f(x):
    return float.fromhex(x) if isinstance(x, str) else x


def _lat_key(z, prefix, tag):
    if tag in ("error", "empty"):
        return tag
    nodes = tuple(map(tuple, z[prefix + "_nodes"].tolist()))
    ai, af = z[prefix + "_arcs_i"], z[prefix + "_arcs_f"]
    arcs = tuple((int(a[0]), int(a[1]), int(a[2]), int(a[3]), float(f[0]), float(f[1]))
                 for a, f in zip(ai, af))
    finals = dict(zip(z[prefix + "_fin_i"].tolist(), z[prefix + "_fin_w"].tolist()))
    return (tuple((int(s), int(t)) for s, t in nodes), arcs, 0, finals)


@functools.lru_cache(maxsize=1)
def load() -> tuple[list[Case], list[float]]:
    with open(os.path.join(HERE, "cases.json")) as fh:
        meta = json.load(fh)
    z = np.load(os.path.join(HERE, "cases.npz"))
    beams = [_f(b) for b in meta["prune_beams"]]
    out = []
    for i, c in enumerate(meta["cases"]):
        g = GraphArrays(c["num_states"], c["start"], *(z[f"{i}_{k}"] for k in (
            "row_ptr", "eps_end", "dst", "ilabel", "olabel", "weight", "final_w")))
        r = c["result"]
        exp = (_f(r["total_cost"]), tuple(r["olabels"]), tuple(r["ilabels"]), r["search_steps"],
               r["tokens_expanded"], r["reached_final"], r["died_at_step"])
        cfg = {k: (_f(v) if k == "beam" else v) for k, v in c["cfg"].items()}
        case = Case(i, c["kind"], c["seed"], g, z[f"{i}_costs"], z[f"{i}_blank"], cfg, exp)
        if "lattice" in c:
            case.lattice = _lat_key(z, f"{i}_lat", c["lattice"])
            if c["lattice"] not in ("error", "empty"):
                case.lattice_arrays = {k: z[f"{i}_lat_{k}"] for k in
                                       ("nodes", "arcs_i", "arcs_f", "fin_i", "fin_w")}
            if "pruned" in c:
                case.pruned = [_lat_key(z, f"{i}_lat_p{bi}", t) for bi, t in enumerate(c["pruned"])]
            if "best_path" in c:
                bp = c["best_path"]
                case.best_path = (_f(bp[0]), tuple(bp[1]), tuple(bp[2]))
        out.append(case)
    return out, beams


def cases(kind: str | None = None) -> list[Case]:
    cs, _ = load()
    return [c for c in cs if kind is None or c.kind == kind]


def prune_beams() -> list[float]:
    return load()[1]


INF = math.inf
