"""Pin the C oracle: against the committed golden fixtures (always) and against the live
Python reference (build container only).  CPU-only."""
import dataclasses
import math

import numpy as np
import pytest

import golden_cases as GC
import refutil
from oracle import oracle as O

INF = math.inf


def _decode(case, **extra):
    cfg = dict(case.cfg)
    return O.decode(case.graph, case.costs, case.blank, beam=cfg.get("beam", INF),
                    max_active=cfg.get("max_active"), mode=cfg.get("mode", "lsd"), **extra)


@pytest.mark.parametrize("kind", ["c1", "c5", "rnd", "lat", "toy"])
def test_oracle_matches_golden_decode(kind):
    for case in GC.cases(kind):
        got = _decode(case)
        assert got.astuple() == case.expected, (case.kind, case.seed, got, case.expected)


@pytest.mark.parametrize("kind", ["c1", "rnd", "lat", "c5"])
def test_oracle_matches_golden_lattice(kind):
    beams = GC.prune_beams()
    n = 0
    for case in GC.cases(kind):
        if case.lattice is None:
            continue
        res, lat = None, None
        try:
            res, lat = _decode(case, return_lattice=True)
            key = lat.key() if not lat.empty else "empty"
        except O.OracleLatticeError:
            key = "error"
        assert key == case.lattice, (case.kind, case.seed)
        if key in ("error",):
            continue
        for bi, beam in enumerate(beams):
            try:
                pk = O.prune_lattice(lat, beam)
                pk = pk.key() if not pk.empty else "empty"
            except O.OracleLatticeError:
                pk = "error"
            assert pk == case.pruned[bi], (case.kind, case.seed, beam)
        if case.best_path is not None:
            assert O.lattice_best_path(lat) == case.best_path
        n += 1
    assert n > 0


def test_oracle_golden_micro_cases():
    """Known answers of the reference unit tests, through a full decode."""
    from paper_1808_00687_b200.wfst import parse_wfst_text

    def dec(text, rows, **kw):
        w = parse_wfst_text(text)
        rows = np.asarray(rows, dtype=np.float64)
        with np.errstate(divide="ignore"):
            costs = np.concatenate([np.full((len(rows), 1), np.inf), -np.log(rows[:, 1:])], 1)
        return O.decode(w, costs, rows[:, 0].copy(), **kw)

    r = dec("0 1 1 1 0.5\n1 0.0\n", [[0.5, 0.5]], mode="fsd")       # test_decoder.py:139-145
    assert r.total_cost == pytest.approx(0.5 + math.log(2)) and r.olabels == (1,)
    r = dec("0 1 1 1 0.5\n1 0.0\n", [[1.0, 0.0]], mode="fsd")       # death, :161-167
    assert r.died_at_step == 0 and not r.reached_final and r.search_steps == 1
    r = dec("0 0.75", np.zeros((0, 2)), mode="fsd")                 # :132-137
    assert r.reached_final and r.total_cost == pytest.approx(0.75)
    # test_cli.py:34-40 golden transcript "a 1.1931": diamond graph, uniform posteriors
    text = "0 1 1 1 1.0\n1 3 2 2 0.1\n0 2 3 3 0.5\n2 3 4 4 0.9\n3 0.0\n"
    r = dec(text, [[0.1, 0.225, 0.225, 0.225, 0.225]] * 2, mode="fsd")
    assert r.olabels == (1, 2)


needs_ref = pytest.mark.skipif(not refutil.HAVE_REF, reason="reference not present")


@needs_ref
def test_oracle_vs_live_reference_tie_heavy():
    """Tie-heavy grids (weight_grid): the oracle reproduces the reference bit-for-bit,
    including the stale-backpointer behaviour (canonical=False)."""
    L = refutil.ref()
    from paper_1808_00687_b200.wfst import Wfst
    for seed in range(150):
        w, p = refutil.random_instance(seed, weight_grid=[0.0, 0.5, 1.0], eps_fraction=0.3,
                                       max_states=16, max_arcs=50, blank_fraction=0.2)
        for cfgk in (dict(mode="fsd"), dict(mode="lsd", beam=2.0, max_active=4)):
            r = L.decoder.decode(w, p, L.decoder.DecodeConfig(**cfgk))
            o = O.decode(Wfst.from_reference(w), refutil.ref_cost_table(p),
                         p.rows[:, p.blank_col].copy(), **cfgk)
            assert dataclasses.astuple(r) == o.astuple(), (seed, cfgk)


@needs_ref
def test_stale_backpointer_repro():
    """reference decode gives (85, 57); canonical traces give the
    lattice best path (11, 13, 35, 57) at the same cost."""
    L = refutil.ref()
    from paper_1808_00687_b200.wfst import Wfst
    text = ("10 0 2 0 0.0\n10 8 2 0 0.0\n0 1 1 11 0.0\n8 5 1 85 1.0\n1 3 0 13 0.5\n"
            "3 5 0 35 0.5\n5 7 0 57 0.0\n7 0.0\n")
    w = L.wfst.parse_wfst_text(text)
    p = L.posteriors.PosteriorMatrix(np.array([[0, 0, 1], [0, 0.5, 0.5]], float), 0)
    cfg = L.decoder.DecodeConfig(mode="fsd")
    rec = L.lattice.LatticeRecorder()
    r = L.decoder.decode(w, p, cfg, recorder=rec)
    g = Wfst.from_reference(w)
    costs, blank = refutil.ref_cost_table(p), p.rows[:, 0].copy()
    o = O.decode(g, costs, blank, mode="fsd")
    assert o.astuple() == dataclasses.astuple(r) and o.olabels == (85, 57)
    oc = O.decode(g, costs, blank, mode="fsd", canonical=True)
    bp = L.lattice.lattice_best_path(L.lattice.build_lattice(rec, w))
    assert oc.olabels == bp[1] == (11, 13, 35, 57) and oc.total_cost == r.total_cost


@needs_ref
def test_oracle_lattice_vs_live_reference_random():
    L = refutil.ref()
    from paper_1808_00687_b200.wfst import Wfst
    for seed in range(80):
        w, p, cfgk = refutil.equivalence_instance(1000 + seed)
        rec = L.lattice.LatticeRecorder()
        L.decoder.decode(w, p, L.decoder.DecodeConfig(**cfgk), recorder=rec)
        try:
            ref_key = O.lattice_from_reference(L.lattice.build_lattice(rec, w))
            ref_key = ref_key.key() if not ref_key.empty else "empty"
        except L.lattice.LatticeError:
            ref_key = "error"
        try:
            _, lat = O.decode(Wfst.from_reference(w), refutil.ref_cost_table(p),
                              p.rows[:, p.blank_col].copy(), return_lattice=True, **cfgk)
            key = lat.key() if not lat.empty else "empty"
        except O.OracleLatticeError:
            key = "error"
        assert key == ref_key, seed
