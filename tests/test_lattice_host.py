"""Lattice post-processing behind the C ABI (csrc/lattice_host.cpp), CPU only: prune_lattice
and lattice_best_path against the reference's own outputs (golden fixtures), text round trip,
and the reference's error behaviour (lattice.py:359-365, 504-512, 579-627)."""
import math

import numpy as np
import pytest

import golden_cases as GC
import refutil
from paper_1808_00687_b200 import lattice as L

INF = math.inf


def _key(lat):
    return "empty" if lat.start_id is None else lat.key()


def _lattice_cases():
    return [c for c in GC.cases() if c.lattice_arrays is not None]


def test_golden_lattices_load():
    cs = _lattice_cases()
    assert len(cs) > 50
    for c in cs:
        assert c.lattice_object().key() == c.lattice


def test_prune_matches_reference_golden():
    beams = GC.prune_beams()
    n = 0
    for c in _lattice_cases():
        lat = c.lattice_object()
        for b, exp in zip(beams, c.pruned or []):
            try:
                got = _key(L.prune_lattice(lat, b))
            except L.LatticeError:
                got = "error"
            assert got == exp, (c.idx, b)
            n += 1
    assert n > 500


def test_best_path_matches_reference_golden():
    n = 0
    for c in _lattice_cases():
        if c.best_path is None:
            continue
        assert L.lattice_best_path(c.lattice_object()) == c.best_path, c.idx
        n += 1
    assert n > 50


def test_prune_is_idempotent_at_infinite_beam():
    for c in _lattice_cases()[:40]:
        lat = c.lattice_object()
        p = L.prune_lattice(lat, INF)
        assert _key(L.prune_lattice(p, INF)) == _key(p)


def test_text_round_trip():
    for c in _lattice_cases()[:40]:
        lat = c.lattice_object()
        back = L.parse_lattice_text(L.format_lattice_text(lat))
        assert back == lat
    assert L.parse_lattice_text("") is L.EMPTY_LATTICE


def test_errors():
    with pytest.raises(ValueError):
        L.prune_lattice(L.EMPTY_LATTICE, -1.0)
    assert L.prune_lattice(L.EMPTY_LATTICE, 1.0) is L.EMPTY_LATTICE
    with pytest.raises(L.LatticeError):
        L.lattice_best_path(L.EMPTY_LATTICE)
    with pytest.raises(L.LatticeError):
        L.parse_lattice_text("LATTICE nodes=1 arcs=0\nN 0 0 0\nQ\n")
    with pytest.raises(L.LatticeError):
        L.parse_lattice_text("LATTICE nodes=2 arcs=0\nN 0 0 0\n")


def test_epsilon_cycle_is_rejected():
    # two nodes in one step joined by epsilon arcs both ways
    lat = L.Lattice([0, 1], [0, 0], [0, 1], [1, 0], [0, 0], [0, 0], [0.5, 0.5], [0.0, 0.0],
                    [0, 1], [1], [0.0])
    with pytest.raises(L.LatticeError):
        L.prune_lattice(lat, 1.0)
    with pytest.raises(L.LatticeError):
        L._check(lat)


def test_reference_shaped_equality():
    c = _lattice_cases()[0]
    lat = c.lattice_object()
    ref_like = type("RefLat", (), {})()
    ref_like.nodes, ref_like.arcs = lat.nodes, lat.arcs
    ref_like.start_id, ref_like.finals = 0, dict(lat.finals)
    assert lat == ref_like
    assert np.array_equal(L.Lattice.from_reference(ref_like).arc_tie, lat.arc_tie)


def test_prune_lattices_threaded_matches_serial():
    beams = GC.prune_beams()
    lats = [c.lattice_object() for c in _lattice_cases()[:60]]
    for b in beams[:3]:
        par = L.prune_lattices(lats, b, max_workers=4)
        for lat, p in zip(lats, par):
            try:
                want = _key(L.prune_lattice(lat, b))
            except L.LatticeError:
                want = "error"
            got = "error" if isinstance(p, L.LatticeError) else _key(p)
            assert got == want


def test_canonical_batch_matches_per_utterance():
    """The batch-vectorised canonical ordering of device pools == per-utterance ordering."""
    from paper_1808_00687_b200 import synth
    g = synth.random_wfst(1, 50, 300, 8, eps_fraction=0.1)
    rng = np.random.default_rng(0)
    parts = []
    for u in range(8):
        nn = int(rng.integers(0, 12))
        if nn:
            steps = np.sort(rng.integers(0, 4, nn))
            steps[0] = 0
            states = rng.choice(50, nn, replace=False).astype(np.int32)
            states[0] = g.start
            nodes = np.stack([states, steps], 1).astype(np.int32)[rng.permutation(nn)]
            na = int(rng.integers(0, 20))
            arcs = np.stack([rng.integers(0, nn, na), rng.integers(0, nn, na),
                             rng.integers(0, g.num_arcs, na), np.zeros(na)], 1).astype(np.uint32)
            ac = rng.random(na)
            nf = int(rng.integers(1, 3))
            fin, fw = rng.integers(0, nn, nf).astype(np.uint32), rng.random(nf)
        else:
            nodes, arcs = np.zeros((0, 2), np.int32), np.zeros((0, 4), np.uint32)
            ac, fin, fw = np.zeros(0), np.zeros(0, np.uint32), np.zeros(0)
        parts.append((nodes, arcs, ac, fin, fw))
    meta = np.zeros((len(parts), 6), np.int64)
    pools = [[], [], [], [], []]
    c = [0, 0, 0]
    for u in rng.permutation(len(parts)):   # pools filled in arbitrary utterance order
        nodes, arcs, ac, fin, fw = parts[u]
        meta[u] = [c[0], len(nodes), c[1], len(arcs), c[2], len(fin)]
        for p, x in zip(pools, parts[u]):
            p.append(x)
        c = [c[0] + len(nodes), c[1] + len(arcs), c[2] + len(fin)]
    got = L.canonical_batch(g, meta, *(np.concatenate(p) for p in pools))
    for u, (nodes, arcs, ac, fin, fw) in enumerate(parts):
        want = L.canonical_from_device(g, nodes, arcs, ac, fin, fw)
        assert got[u].key() == want.key()
        assert np.array_equal(got[u].arc_tie, want.arc_tie)


@pytest.mark.skipif(not refutil.HAVE_REF, reason="reference not available")
def test_native_lattice_text_matches_reference_byte_for_byte():
    """format_lattice_text (C++ writer, repr floats) produces the reference's exact text for
    the reference's own lattices and random costs; parse_lattice_text reads it back to the
    reference's parse, and malformed text raises what the reference raises."""
    import random
    R = refutil.ref()
    rng = random.Random(3)
    n = 0
    for seed in range(40):
        wfst, posts = refutil.random_instance(seed, max_states=10, max_arcs=30, max_frames=6,
                                              eps_fraction=0.2)
        rec = R.lattice.LatticeRecorder()
        R.decoder.decode(wfst, posts, R.decoder.DecodeConfig(beam=5.0), recorder=rec)
        try:
            ref = R.lattice.build_lattice(rec, wfst)
        except R.lattice.LatticeError:
            continue
        want = R.lattice.format_lattice_text(ref)
        assert L.format_lattice_text(ref) == want
        assert L.format_lattice_text(L.Lattice.from_reference(ref)) == want
        assert L.parse_lattice_text(want) == R.lattice.parse_lattice_text(want)
        n += 1
    assert n > 20
    # repr of awkward doubles: tiny, huge, integral, negative zero, inf, 17-digit values
    vals = [0.0, -0.0, 1.0, 1e16, 1e15, 123456789012345678.0, 1e-4, 9.999e-5, 1e-5, 0.1,
            2.5e-300, 1.7976931348623157e308, math.inf, -math.inf, 5e-324, 100.0, 1e22]
    vals += [rng.uniform(-1e6, 1e6) for _ in range(200)] + [rng.random() * 10 ** rng.randint(-30, 30)
                                                            for _ in range(200)]
    nodes = tuple(R.lattice.LatticeNode(i, i) for i in range(len(vals) + 1))
    arcs = tuple(R.lattice.LatticeArc(i, i + 1, 1, 2, v, -v) for i, v in enumerate(vals))
    big = R.lattice.Lattice(nodes=nodes, arcs=arcs, start_id=0, finals={len(vals): vals[5]})
    want = R.lattice.format_lattice_text(big)
    assert L.format_lattice_text(big) == want
    assert L.parse_lattice_text(want) == R.lattice.parse_lattice_text(want)
    for bad in ("LATTICE nodes=x arcs=0\n", "LATTICE nodes=1 arcs=0\nN 0 0 0\nQ 1\n",
                "LATTICE nodes=2 arcs=0\nN 0 0 0\n", "LATTICE nodes=1 arcs=0\nN 1 0 0\n",
                "LATTICE nodes=1 arcs=0\nN 0 a 0\n", "LATTICE nodes=2 arcs=1\nN 0 0 0\nN 1 0 3\nA 0 1 1 1 0.5 0.5\n",
                "LATTICE nodes=1 arcs=1\nN 0 0 0\nA 0 5 1 1 0.5 0.5\n",
                "LATTICE nodes=1 arcs=1\nN 0 0 0\nA 0 0 1 1 x 0.5\n", "LATTICE nodes=1 arcs=0\nN 0 0 0 final\n"):
        try:
            R.lattice.parse_lattice_text(bad)
            kind = None
        except Exception as exc:   # noqa: BLE001 - the exception type is the contract
            kind = type(exc).__name__
        with pytest.raises(Exception) as ei:
            L.parse_lattice_text(bad)
        assert type(ei.value).__name__ == kind, bad
