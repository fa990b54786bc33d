"""Command-line front end (reference pkg/tests/test_cli.py), symbol tables and the CSR cache.

CPU tests: argument / input errors (exit 2 before any GPU work), the ``lattice`` subcommand
(host lattice code), symbol tables and symbol-aware parsing against the reference's own
cases, the binary CSR cache and the text writer.  GPU tests: the reference's decode-command
known answers ("a 1.1931", exit 3 on search death, FSD == LSD at a degenerate threshold,
lattice round trip) plus the batched multi-file form and the bench report.
"""
import json
import math

import numpy as np
import pytest

from refutil import HAVE_REF

from paper_1808_00687_b200 import cli, synth
from paper_1808_00687_b200.lattice import load_lattice
from paper_1808_00687_b200.wfst import (ParseError, SymbolError, SymbolTable, WfstError,
                                        format_wfst_text, load_wfst_binary, parse_wfst_text,
                                        save_wfst_binary)

ONE_ARC_GRAPH = "0 1 1 1 0.5\n1 0.0\n"
ONE_ARC_POSTS = "1 2 blank=0\n0.5 0.5\n"
SYMS = "<eps> 0\na 1\n"
# the one-arc decode's lattice: start (0, 0) -> (1, 1), g = 0.5, a = -ln 0.5
ONE_ARC_LATTICE = ("LATTICE nodes=2 arcs=1\nN 0 0 0\nN 1 1 1 final 0.0\n"
                   f"A 0 1 1 1 0.5 {math.log(2.0)!r}\n")


@pytest.fixture
def files(tmp_path):
    out = {}
    for name, text in (("graph", ONE_ARC_GRAPH), ("posts", ONE_ARC_POSTS), ("syms", SYMS),
                       ("lat", ONE_ARC_LATTICE)):
        p = tmp_path / f"{name}.txt"
        p.write_text(text)
        out[name] = str(p)
    return out


# ----------------------------------------------------------------------------- CPU
def test_missing_graph_exits_2(files, capsys):
    assert cli.main(["decode", "--graph", "/nonexistent/graph.txt", "--posts", files["posts"]]) == 2
    assert "error" in capsys.readouterr().err


def test_malformed_graph_exits_2(tmp_path, files, capsys):
    bad = tmp_path / "bad.txt"
    bad.write_text("0 1 1\n")
    assert cli.main(["decode", "--graph", str(bad), "--posts", files["posts"]]) == 2


def test_bad_workers_exits_2(files, capsys):
    assert cli.main(["decode", "--graph", files["graph"], "--posts", files["posts"],
                     "--workers", "0"]) == 2
    assert "workers" in capsys.readouterr().err


def test_lattice_command_best_path(files, capsys):
    assert cli.main(["lattice", "--lattice-in", files["lat"], "--osyms", files["syms"]]) == 0
    assert capsys.readouterr().out.strip() == "a 1.1931"
    assert cli.main(["lattice", "--lattice-in", files["lat"]]) == 0
    assert capsys.readouterr().out.strip() == "1 1.1931"


def test_lattice_command_prunes_and_writes(tmp_path, files, capsys):
    out = tmp_path / "pruned.lat"
    assert cli.main(["lattice", "--lattice-in", files["lat"], "--lattice-beam", "1.0",
                     "--lattice-out", str(out)]) == 0
    lat = load_lattice(str(out))
    assert (lat.num_nodes, lat.num_arcs) == (2, 1)


def test_bad_lattice_exits_2(tmp_path, capsys):
    bad = tmp_path / "bad.lat"
    bad.write_text("LATTICE nodes=1 arcs=0\nQ\n")
    assert cli.main(["lattice", "--lattice-in", str(bad)]) == 2


def test_symbol_table_reference_cases():
    # pkg/tests/test_wfst.py:182-204
    t = SymbolTable.parse("<eps> 0\na 1\nb 2\n")
    assert (t.find_id("a"), t.find_symbol(2), t.find_id("<eps>")) == (1, "b", 0)
    with pytest.raises(ParseError):
        SymbolTable.parse("a 0\n")
    assert SymbolTable.parse("<eps> 0\n<blank> 3\n").blank_id == 3
    with pytest.raises(ParseError):
        SymbolTable.parse("a 1\na 2\n")
    t = SymbolTable({"a": 1, "b": 2})
    assert list(SymbolTable.parse(t.format())) == list(t)
    with pytest.raises(SymbolError):
        SymbolTable({"a": 1}).add("b", 1)
    assert SymbolTable({"a": 1}).add("c") == 2


def test_symbolic_parse_reference_cases():
    # pkg/tests/test_wfst.py:66-78
    isyms, osyms = SymbolTable({"a": 1, "b": 2}), SymbolTable({"x": 1})
    w = parse_wfst_text("0 1 a x 0.5\n1", isyms, osyms)
    a = w.out_arcs(0)[0]
    assert (a.ilabel, a.olabel) == (1, 1)
    with pytest.raises(SymbolError):
        parse_wfst_text("0 1 zzz a 0.5\n1", SymbolTable({"a": 1}), SymbolTable({"a": 1}))
    with pytest.raises(SymbolError):
        parse_wfst_text("0 1 -3 1 0.5\n1")
    # a table entry wins over the bare-integer reading of the same token
    w = parse_wfst_text("0 1 7 7 0.5\n1", SymbolTable({"7": 2}), None)
    assert (w.ilabel.tolist(), w.olabel.tolist()) == ([2], [7])


@pytest.mark.skipif(not HAVE_REF, reason="reference tree only in the build container")
def test_symbolic_parse_matches_reference():
    from refutil import ref
    L = ref()
    rng = np.random.default_rng(5)
    names = [f"w{i}" for i in range(1, 9)]
    isyms_txt = "<eps> 0\n" + "".join(f"{n} {i + 1}\n" for i, n in enumerate(names))
    mine_t, ref_t = SymbolTable.parse(isyms_txt), L.wfst.SymbolTable.parse(isyms_txt)
    lines = []
    for _ in range(60):
        s, d = rng.integers(0, 12, 2)
        il = names[rng.integers(0, 8)] if rng.random() < 0.7 else str(rng.integers(0, 9))
        ol = names[rng.integers(0, 8)] if rng.random() < 0.5 else str(rng.integers(0, 9))
        lines.append(f"{s} {d} {il} {ol} {rng.uniform(0, 3):.6f}")
    lines += ["3 0.25", "7"]
    text = "\n".join(lines) + "\n"
    mine = parse_wfst_text(text, mine_t, mine_t)
    theirs = L.wfst.parse_wfst_text(text, ref_t, ref_t)
    key = (lambda a: (a.src, a.dst, a.ilabel, a.olabel, a.weight))
    assert [key(a) for a in mine.arcs] == [key(a) for a in theirs.arcs]
    assert mine.final_weights == theirs.final_weights and mine.start == theirs.start


def test_csr_cache_round_trip(tmp_path):
    w = synth.random_wfst(7, 200, 900, 11, eps_fraction=0.05)
    p = str(tmp_path / "g.npz")
    save_wfst_binary(w, p)
    w2 = load_wfst_binary(p)
    for k in ("row_ptr", "eps_end", "dst", "ilabel", "olabel", "weight", "final_w"):
        assert np.array_equal(getattr(w, k), getattr(w2, k)), k
    assert (w2.start, w2.num_states, w2.max_ilabel) == (w.start, w.num_states, w.max_ilabel)
    assert w2._eps_cycle_checked and w2.epsilon_cycle() == w.epsilon_cycle()
    # an epsilon cycle verdict is cached too
    cyc = parse_wfst_text("0 1 0 0 0.0\n1 0 0 0 0.0\n1 0.0")
    save_wfst_binary(cyc, p)
    assert load_wfst_binary(p).epsilon_cycle() == cyc.epsilon_cycle() is not None
    bad = tmp_path / "bad.npz"
    np.savez(bad, x=np.zeros(3))
    with pytest.raises(WfstError):
        load_wfst_binary(str(bad))


def test_text_writer_round_trip():
    for seed in range(4):
        w = synth.random_wfst(seed, 60, 250, 9, eps_fraction=0.1, selfloops=seed % 2 == 1)
        w2 = parse_wfst_text(format_wfst_text(w))
        for k in ("row_ptr", "eps_end", "dst", "ilabel", "olabel", "weight", "final_w"):
            assert np.array_equal(getattr(w, k), getattr(w2, k)), (seed, k)
        assert w2.start == w.start
    assert parse_wfst_text(format_wfst_text(parse_wfst_text("0 0.5\n"))).final_weights == {0: 0.5}


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_decode_one_arc_transcript(cuda, files, capsys):
    # pkg/tests/test_cli.py:34-40
    assert cli.main(["decode", "--graph", files["graph"], "--posts", files["posts"],
                     "--osyms", files["syms"], "--mode", "fsd"]) == 0
    assert capsys.readouterr().out.strip() == "a 1.1931"


@pytest.mark.gpu
def test_lsd_equals_fsd_at_degenerate_threshold(cuda, files, capsys):
    cli.main(["decode", "--graph", files["graph"], "--posts", files["posts"], "--mode", "fsd"])
    fsd = capsys.readouterr().out
    cli.main(["decode", "--graph", files["graph"], "--posts", files["posts"], "--mode", "lsd",
              "--blank-threshold", "1.1"])
    assert capsys.readouterr().out == fsd


@pytest.mark.gpu
def test_search_death_exits_3(cuda, tmp_path, files, capsys):
    dead = tmp_path / "dead.txt"
    dead.write_text("1 2 blank=0\n1.0 0.0\n")
    assert cli.main(["decode", "--graph", files["graph"], "--posts", str(dead),
                     "--mode", "fsd"]) == 3
    cap = capsys.readouterr()
    assert cap.out.strip() == "0.0000"
    assert "died" in cap.err


@pytest.mark.gpu
def test_lattice_out_round_trips(cuda, tmp_path, files, capsys):
    lat_path = tmp_path / "out.lat"
    assert cli.main(["decode", "--graph", files["graph"], "--posts", files["posts"],
                     "--mode", "fsd", "--lattice-out", str(lat_path)]) == 0
    assert not load_lattice(str(lat_path)).is_empty
    capsys.readouterr()
    assert cli.main(["lattice", "--lattice-in", str(lat_path), "--osyms", files["syms"]]) == 0
    assert capsys.readouterr().out.strip() == "a 1.1931"


@pytest.mark.gpu
def test_workers_flag_same_output(cuda, files, capsys):
    cli.main(["decode", "--graph", files["graph"], "--posts", files["posts"], "--mode", "fsd"])
    serial = capsys.readouterr().out
    cli.main(["decode", "--graph", files["graph"], "--posts", files["posts"], "--mode", "fsd",
              "--workers", "4", "--group-size", "2"])
    assert capsys.readouterr().out == serial


def _batch_files(tmp_path, n=5):
    from paper_1808_00687_b200.posteriors import save_posteriors
    w = synth.random_wfst(11, 300, 1500, 20, eps_fraction=0.03, selfloops=True)
    g = tmp_path / "g.txt"
    g.write_text(format_wfst_text(w))
    posts = []
    for i in range(n):
        p = str(tmp_path / f"p{i}.bin")
        save_posteriors(synth.random_posteriors(100 + i, 40 + 7 * i, 20, blank_fraction=0.5), p,
                        binary=i % 2 == 0)
        posts.append(p)
    return w, str(g), posts


@pytest.mark.gpu
def test_decode_batch_of_files_matches_single(cuda, tmp_path, capsys):
    w, g, posts = _batch_files(tmp_path)
    args = ["--beam", "9", "--max-active", "60", "--mode", "lsd"]
    assert cli.main(["decode", "--graph", g, "--posts", *posts, *args]) == 0
    batch = capsys.readouterr().out.splitlines()
    single = []
    for p in posts:
        assert cli.main(["decode", "--graph", g, "--posts", p, *args]) == 0
        single.append(capsys.readouterr().out.strip())
    assert batch == single and len(batch) == len(posts)
    # the CSR cache path gives the same transcripts
    npz = str(tmp_path / "g.npz")
    assert cli.main(["decode", "--graph", g, "--posts", posts[0], "--save-csr", npz, *args]) == 0
    capsys.readouterr()
    assert cli.main(["decode", "--graph", npz, "--posts", posts[0], *args]) == 0
    assert capsys.readouterr().out.strip() == single[0]


@pytest.mark.gpu
def test_bench_report_json(cuda, tmp_path, capsys):
    w, g, posts = _batch_files(tmp_path, 3)
    assert cli.main(["bench", "--graph", g, "--posts", *posts, "--beam", "9", "--repeats", "2",
                     "--report", "json"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["schema"] == "v1" and set(rep["modes"]) == {"fsd-gpu", "lsd-gpu"}
    from paper_1808_00687_b200.posteriors import load_posteriors
    T = sum(load_posteriors(p).num_frames for p in posts)
    assert rep["frames"] == T
    assert rep["modes"]["fsd-gpu"]["search_steps"] == T
    assert rep["modes"]["lsd-gpu"]["search_steps"] == T - rep["blank_frames"]
    assert "fsd-gpu/lsd-gpu" in rep["speedups"]
    assert cli.main(["bench", "--graph", g, "--posts", posts[0], "--repeats", "1",
                     "--modes", "lsd-gpu"]) == 0
    assert "lsd-gpu" in capsys.readouterr().out


def test_pipelined_builder_without_decode_raises():
    # lattice.py:289-292: result_from before the decode finished
    from paper_1808_00687_b200 import LatticeError, LatticeRecorder, PipelinedLatticeBuilder
    b = PipelinedLatticeBuilder(None)
    with pytest.raises(LatticeError):
        b.result_from(LatticeRecorder(consumer=b))
    with pytest.raises(LatticeError):   # no transducer to assemble steps against
        b.feed(0, None)
    b.close()
