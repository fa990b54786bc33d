"""Host-side logic (CPU-only): graph layout, cost table, epsilon-cycle validation, config
validation, synthetic generators, API error behaviour before any device call."""
import dataclasses
import math
import random

import numpy as np
import pytest

import refutil
from paper_1808_00687_b200 import synth
from paper_1808_00687_b200.decoder import DecodeConfig
from paper_1808_00687_b200.posteriors import PosteriorMatrix, cost_table, frame_costs
from paper_1808_00687_b200.wfst import SymbolTable, Arc, Wfst, WfstError, parse_wfst_text, validate_epsilon_acyclic

needs_ref = pytest.mark.skipif(not refutil.HAVE_REF, reason="reference not present")


@needs_ref
def test_wfst_layout_matches_reference():
    """Arc order, arc_offsets, eps_split, final weights (wfst.py:182-198)."""
    L = refutil.ref()
    for seed in range(60):
        rng = random.Random(seed)
        w = L.fixtures.make_random_wfst(rng, rng.randrange(2, 40), rng.randrange(1, 120),
                                        rng.randrange(1, 6), eps_fraction=0.3,
                                        selfloops=seed % 2 == 0,
                                        weight_grid=[0.0, 0.5] if seed % 5 == 0 else None)
        arcs = [Arc(a.src, a.dst, a.ilabel, a.olabel, a.weight) for a in w.arcs]
        random.Random(seed + 1).shuffle(arcs)
        g = Wfst(w.num_states, w.start, arcs, w.final_weights)
        assert [(a.src, a.dst, a.ilabel, a.olabel, a.weight) for a in g.arcs] == \
               [(a.src, a.dst, a.ilabel, a.olabel, a.weight) for a in w.arcs]
        assert g.arc_offsets == w.arc_offsets
        assert g.eps_split == w.eps_split
        assert g.final_weights == w.final_weights
        assert g.has_epsilon_arcs == w.has_epsilon_arcs


@needs_ref
def test_cost_table_bit_exact_vs_frame_costs():
    """The vectorised (and thread-blocked) table equals frame_costs row by row, bit for bit."""
    L = refutil.ref()
    for seed in range(20):
        rng = random.Random(seed)
        labels = rng.randrange(1, 80)
        p = L.fixtures.make_random_posteriors(rng, rng.randrange(0, 40), labels,
                                              blank_fraction=0.3, blank_col=seed % (labels + 1))
        mine = PosteriorMatrix(p.rows, p.blank_col)
        for scale in (1.0, 0.7):
            t = cost_table(mine, scale)
            for f in range(p.num_frames):
                ref = L.posteriors.frame_costs(p, f, scale)
                assert t[f].tobytes() == np.asarray(ref).tobytes()


def test_cost_table_large_threaded_equals_rowwise():
    rows = synth.random_posterior_rows(3, 700, 3000, blank_fraction=0.2)
    p = PosteriorMatrix(rows, 0, validate=False)
    t = cost_table(p)
    for f in (0, 1, 350, 699):
        assert t[f].tobytes() == np.asarray(frame_costs(p, f)).tobytes()


def test_zero_probability_is_infinite_cost():
    p = PosteriorMatrix(np.array([[0.5, 0.5, 0.0], [1.0, 0.0, 0.0]]), 0)
    t = cost_table(p)
    assert math.isinf(t[0, 2]) and math.isinf(t[1, 1]) and math.isinf(t[0, 0])
    assert t[1, 1] > 0


@needs_ref
def test_epsilon_cycle_detection_matches_reference():
    L = refutil.ref()
    texts = ["0 1 0 0 0.0\n1 0 0 0 0.0\n0 2 1 1 0.5\n2 0.0",      # zero-weight cycle
             "0 1 0 0 0.5\n1 0 0 0 0.5\n0 2 1 1 0.5\n2 0.0",      # positive cycle: accepted
             "0 0 0 0 0.0\n0 1 1 1 1\n1",                          # zero self-loop
             "0 0 0 0 0.3\n0 1 1 1 1\n1",                          # positive self-loop
             "0 1 1 1 0.5\n1 0.0"]
    for t in texts:
        ref = L.wfst.parse_wfst_text(t).epsilon_cycle()
        mine = parse_wfst_text(t).epsilon_cycle()
        assert (ref is None) == (mine is None), t
        if ref is not None:
            assert mine.total_weight == ref.total_weight
    for t in ["0 1 0 0 -1.0\n1 0 0 0 0.5\n0 2 1 1 0.5\n2 0.0"]:
        ref = L.wfst.parse_wfst_text(t, allow_negative_weights=True).epsilon_cycle()
        mine = parse_wfst_text(t, allow_negative_weights=True).epsilon_cycle()
        assert (ref is None) == (mine is None)


def test_epsilon_validation_fast_path_on_large_graph():
    g = synth.random_wfst(1, 200_000, 600_000, 100, eps_fraction=0.05)
    assert validate_epsilon_acyclic(g) is None


def test_decode_config_validation():
    with pytest.raises(ValueError):
        DecodeConfig(beam=-1.0)
    with pytest.raises(ValueError):
        DecodeConfig(max_active=0)
    with pytest.raises(ValueError):
        DecodeConfig(acoustic_scale=0.0)
    with pytest.raises(ValueError):
        DecodeConfig(mode="nonsense")


def test_api_errors_raise_before_device_work():
    """WfstError for a non-positive epsilon cycle, ValueError for an alphabet mismatch
    (decoder.py:304-308, 294-299) -- raised on the host, like the reference."""
    import paper_1808_00687_b200 as P
    w = parse_wfst_text("0 1 0 0 0.0\n1 0 0 0 0.0\n0 2 1 1 0.5\n2 0.0")
    p = PosteriorMatrix(np.array([[0.1, 0.9]]), 0)
    with pytest.raises(WfstError):
        P.decode_fsd(w, p, DecodeConfig(mode="fsd"))
    w2 = parse_wfst_text("0 1 7 7 0.5\n1 0.0")
    with pytest.raises(ValueError):
        P.decode_fsd(w2, PosteriorMatrix(np.array([[0.1, 0.45, 0.45]]), 0), DecodeConfig(mode="fsd"))
    with pytest.raises(ValueError):
        P.parallel_decode(w2, p, DecodeConfig(), workers=0)


def test_synth_generators_deterministic_and_well_formed():
    a = synth.random_wfst(5, 1000, 4000, 20, eps_fraction=0.1, selfloops=True)
    b = synth.random_wfst(5, 1000, 4000, 20, eps_fraction=0.1, selfloops=True)
    for f in ("row_ptr", "eps_end", "dst", "ilabel", "olabel", "weight", "final_w"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    assert a.num_arcs == 4000 and validate_epsilon_acyclic(a) is None
    eps = a.ilabel == 0
    assert (a.src[eps] < a.dst[eps]).all()           # forward-only epsilon arcs
    rows = synth.random_posterior_rows(1, 500, 30, blank_fraction=0.4)
    assert np.allclose(rows.sum(1), 1.0) and (rows > 0).all()
    assert int((rows[:, 0] > 0.98).sum()) == 200


@needs_ref
def test_reference_graph_conversion_roundtrip():
    L = refutil.ref()
    from paper_1808_00687_b200.decoder import as_wfst
    w, _ = refutil.random_instance(3)
    g = as_wfst(w)
    assert as_wfst(w) is g
    assert g.arc_offsets == w.arc_offsets and g.eps_split == w.eps_split


def test_cost_rows_is_bit_identical_to_cost_table():
    """The streaming producer's in-place row runs == cost_table == frame_costs arithmetic."""
    import numpy as np
    from paper_1808_00687_b200 import synth
    from paper_1808_00687_b200.posteriors import PosteriorMatrix, cost_rows, cost_table
    for bc in (0, 3):
        rows = synth.random_posterior_rows(5, 200, 40, blank_fraction=0.5, blank_col=bc)
        p = PosteriorMatrix(rows, bc, validate=False)
        ref = cost_table(p, 0.7)
        out = np.full_like(ref, 123.0)
        idx = np.sort(np.random.default_rng(1).choice(200, 90, replace=False))
        cost_rows(p, idx, out, 0.7)
        assert np.array_equal(out[idx], ref[idx])
        assert (np.signbit(out[idx]) == np.signbit(ref[idx])).all()
        assert (out[np.setdiff1d(np.arange(200), idx)] == 123.0).all()


def _wfst_key(w):
    import numpy as np
    return (w.num_states, w.start, w.row_ptr.tolist(), w.eps_end.tolist(), w.dst.tolist(),
            w.ilabel.tolist(), w.olabel.tolist(), w.weight.tolist(),
            np.where(np.isinf(w.final_w), -1.0, w.final_w).tolist())


def _texts():
    import numpy as np
    rng = np.random.default_rng(3)
    out = []
    for k in range(30):
        S = int(rng.integers(1, 40))
        lines = []
        for _ in range(int(rng.integers(0, 120))):
            a, b = rng.integers(0, S, 2)
            i, o = rng.integers(0, 6, 2)
            w = float(np.round(rng.uniform(0, 3), int(rng.integers(0, 8))))
            form = rng.integers(0, 4)
            lines.append(f"{a} {b} {i} {o}" if form == 0 else
                         f"{a}\t{b}  {i} {o} {w!r}" if form == 1 else
                         f"  {a} {b} {i} {o} {w:.3e}  " if form == 2 else f"{a} {b} {i} {o} {w}")
            if rng.random() < 0.1:
                lines.append("# comment")
            if rng.random() < 0.1:
                lines.append("")
        for s in rng.integers(0, S, int(rng.integers(1, 4))):
            lines.append(f"{s} {float(rng.uniform(0, 2))!r}" if rng.random() < 0.7 else f"{s}")
        if rng.random() < 0.3:
            lines.insert(0, f"{int(rng.integers(0, S))} inf")
        sep = "\r\n" if k % 5 == 0 else "\n"
        out.append(sep.join(lines) + (sep if k % 2 else ""))
    return out


def test_wfst_parser_errors_and_number_grammar():
    """The native parser raises ParseError / SymbolError for malformed text and follows
    Python's int()/float() grammar (underscores, inf, no hex) like the reference's parser."""
    from paper_1808_00687_b200.wfst import ParseError, SymbolError
    for bad, exc in (("0 1 2\n", ParseError), ("0 1 a b\n", SymbolError),
                     ("0 1 2 3 nan\n", ParseError), ("0 1 2 3 -1\n", ParseError),
                     ("", ParseError), ("# only\n", ParseError), ("0 1 2 3 0x1p3\n", ParseError),
                     ("-1 2 3 4\n", ParseError), ("0 1 2 3 1__0\n", ParseError),
                     ("0 1 -2 3\n", SymbolError), ("x 1 2 3\n", ParseError)):
        with pytest.raises(exc):
            parse_wfst_text(bad)
    assert parse_wfst_text("0 1 2 3 1_0\n").weight.tolist() == [10.0]
    assert parse_wfst_text("0 1 2 3 -1.5\n1\n", allow_negative_weights=True).weight.tolist() == [-1.5]
    assert parse_wfst_text("0 1 2 3 .5e+1_0\n1 INF\n").num_states == 2
    # Python line breaks / Unicode whitespace are normalised before the native tokenizer
    w = parse_wfst_text("0 1 2 3 0.5\x0b1\u00a02 3 4 1e-3\u20282 0.25\r3 1 1 1")
    assert w.num_arcs == 3 and w.final_w[2] == 0.25


@needs_ref
def test_wfst_parser_fuzz_matches_reference():
    """Random (and randomly corrupted) transducer texts, with and without symbol tables: the
    same graph or the same exception type and message as the reference parser."""
    import numpy as np
    L = refutil.ref()
    rng = np.random.default_rng(11)
    syms = "<eps> 0\na 1\nb 2\n<blank> 3\nc 7\n"
    junk = ["x", "-3", "1__2", "nan", "inf", "-0.0", "1e400", "_1", "1_", "0x10", "+4", "1.5.2",
            "\u00e9", "# c", "3 4 5 6 7 8"]
    for k in range(400):
        base = _texts()[k % 30]
        lines = base.splitlines()
        for _ in range(int(rng.integers(0, 3))):
            if lines:
                i = int(rng.integers(0, len(lines)))
                f = lines[i].split()
                if f:
                    f[int(rng.integers(0, len(f)))] = junk[int(rng.integers(0, len(junk)))]
                    lines[i] = " ".join(f)
        text = "\n".join(lines)
        use_syms = k % 3 == 0
        tabs = ((L.wfst.SymbolTable.parse(syms), L.wfst.SymbolTable.parse(syms)) if use_syms
                else (None, None))
        mine_tabs = ((SymbolTable.parse(syms), SymbolTable.parse(syms)) if use_syms
                     else (None, None))
        try:
            r = L.wfst.parse_wfst_text(text, *tabs, allow_negative_weights=k % 2 == 1)
            want = _wfst_key(Wfst.from_reference(r))
        except Exception as e:
            want = (type(e).__name__, str(e))
        try:
            got = _wfst_key(parse_wfst_text(text, *mine_tabs, allow_negative_weights=k % 2 == 1))
        except Exception as e:
            got = (type(e).__name__, str(e))
        assert got == want, (k, text[:200])


@needs_ref
def test_native_wfst_parser_matches_reference():
    L = refutil.ref()
    for t in _texts()[:10]:
        mine = parse_wfst_text(t)
        ref = L.wfst.parse_wfst_text(t)
        assert _wfst_key(mine) == _wfst_key(Wfst.from_reference(ref))


def test_posterior_files_roundtrip_and_match_reference(tmp_path):
    """load_posteriors / save_posteriors (posteriors.py:147-238): text and POST1 binary round
    trips, and (build container) the reference reads our files and we read its files."""
    import numpy as np
    from paper_1808_00687_b200 import synth
    from paper_1808_00687_b200.posteriors import (PosteriorMatrix, format_posteriors_binary,
                                                   format_posteriors_text, load_posteriors,
                                                   save_posteriors)
    p = synth.random_posteriors(9, 17, 6, blank_col=2)
    for binary in (False, True):
        path = str(tmp_path / f"p{int(binary)}")
        save_posteriors(p, path, binary=binary)
        q = load_posteriors(path)
        assert q.blank_col == 2 and q.rows.tobytes() == p.rows.tobytes()
    assert load_posteriors(format_posteriors_binary(p)).rows.tobytes() == p.rows.tobytes()
    if refutil.HAVE_REF:
        L = refutil.ref()
        ref = L.posteriors.load_posteriors(format_posteriors_text(p).encode())
        assert ref.rows.tobytes() == p.rows.tobytes()
        mine = load_posteriors(L.posteriors.format_posteriors_text(ref).encode())
        assert mine.rows.tobytes() == p.rows.tobytes()


@needs_ref
def test_epsilon_cycle_fuzz_matches_reference():
    """Random epsilon subgraphs with cycles of negative, zero and positive weight (and self-
    loops): the SCC + Bellman-Ford check accepts / rejects exactly the graphs the reference
    rejects."""
    L = refutil.ref()
    rng = random.Random(5)
    for k in range(300):
        S = rng.randrange(2, 14)
        lines = []
        for _ in range(rng.randrange(1, 3 * S)):
            a, b = rng.randrange(S), rng.randrange(S)
            w = rng.choice([0.0, 0.5, 1.0, -0.5, 0.25, 2.0, -1.0])
            lines.append(f"{a} {b} {0 if rng.random() < 0.7 else 1} 0 {w}")
        lines.append(f"{S - 1} 0.0")
        text = "\n".join(lines)
        ref = L.wfst.parse_wfst_text(text, allow_negative_weights=True).epsilon_cycle()
        mine = parse_wfst_text(text, allow_negative_weights=True).epsilon_cycle()
        assert (ref is None) == (mine is None), (k, text)
        if mine is not None:   # the reported cycle is a real epsilon cycle of weight <= 0
            assert mine.total_weight <= 1e-12
            st = list(mine.states)
            w = parse_wfst_text(text, allow_negative_weights=True)
            eps = w.ilabel == 0
            arcs = set(zip(w.src[eps].tolist(), w.dst[eps].tolist()))
            assert all((x, y) in arcs for x, y in zip(st, st[1:] + st[:1])), (k, st)


@needs_ref
def test_post1_native_reader_matches_reference(tmp_path):
    """POST1 files read by the native reader (wb_post1_read, into the PosteriorBatch table)
    equal the reference's load_posteriors; malformed files raise PosteriorFormatError."""
    from paper_1808_00687_b200.posteriors import (PosteriorBatch, PosteriorFormatError,
                                                   format_posteriors_binary, save_posteriors)
    L = refutil.ref()
    mats = [synth.random_posteriors(40 + k, 5 + 7 * k, 9, blank_col=k % 3) for k in range(4)]
    paths = []
    for k, m in enumerate(mats):
        path = tmp_path / f"u{k}.post"
        save_posteriors(m, str(path), binary=k != 1)     # one text file in the batch
        paths.append(str(path))
    batch = PosteriorBatch(paths)
    for path, view in zip(paths, batch.matrices()):
        ref = L.posteriors.load_posteriors(path)
        assert view.rows.tobytes() == ref.rows.tobytes() and view.blank_col == ref.blank_col
    good = format_posteriors_binary(mats[0])
    for bad in (good[:-8], good[:12], good + b"\0" * 8):
        p = tmp_path / "bad.post"
        p.write_bytes(bad)
        with pytest.raises(PosteriorFormatError):
            PosteriorBatch([str(p)])
        with pytest.raises(L.posteriors.PosteriorFormatError):
            L.posteriors.load_posteriors(str(p))
