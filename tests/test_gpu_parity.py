"""GPU decode vs the CPU oracle on seeded instances (bit-exact DecodeResult)."""
import math

import numpy as np
import pytest

import paper_1808_00687_b200 as P
from paper_1808_00687_b200 import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu
INF = math.inf


def _fields(r):
    return (r.total_cost, r.olabels, r.ilabels, r.search_steps, r.tokens_expanded,
            r.reached_final, r.died_at_step)


def _check_batch(g, posts, cfg, canonical=False):
    got = P.decode_batch(g, posts, cfg)
    for i, (p, r) in enumerate(zip(posts, got)):
        o = O.decode(g, P.cost_table(p, cfg.acoustic_scale), p.rows[:, p.blank_col],
                     beam=cfg.beam, max_active=cfg.max_active, mode=cfg.mode,
                     blank_threshold=cfg.blank_threshold, canonical=canonical)
        assert _fields(r) == o.astuple(), (i, r, o)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("mode", ["fsd", "lsd"])
def test_random_small(cuda, seed, mode):
    rng = np.random.default_rng(seed)
    S = int(rng.integers(2, 60))
    g = synth.random_wfst(seed, S, int(S * rng.uniform(1, 4)), int(rng.integers(1, 6)),
                          eps_fraction=[0.0, 0.15, 0.3][seed % 3], selfloops=seed % 2 == 0,
                          final_fraction=0.3)
    L = int(g.max_ilabel) or 1
    posts = [synth.random_posteriors(seed * 100 + k, int(rng.integers(0, 12)), L,
                                     blank_fraction=0.3) for k in range(5)]
    for beam, ma in ((INF, None), (4.0, None), (INF, 3), (6.0, 5)):
        _check_batch(g, posts, P.DecodeConfig(beam=beam, max_active=ma, mode=mode))


@pytest.mark.parametrize("seed", range(4))
def test_medium_graph(cuda, seed):
    g = synth.random_wfst(seed, 5000, 16000, 50, eps_fraction=0.05, selfloops=True,
                          final_fraction=0.05)
    posts = [synth.random_posteriors(seed * 7 + k, 120, 50, blank_fraction=0.2) for k in range(8)]
    _check_batch(g, posts, P.DecodeConfig(beam=10.0, max_active=300, mode="fsd"))
    _check_batch(g, posts, P.DecodeConfig(beam=7.0, mode="lsd"))


@pytest.mark.parametrize("mode", ["fsd", "lsd"])
def test_zero_copy_pinned_matches_copy_and_oracle(cuda, mode):
    """A page-locked cost table: FSD (equal-length utterances at a common stride) goes through
    the H2D pipeline (step-range chunks copied while the kernel decodes, ready counts polled),
    LSD is read zero-copy (only searched rows cross PCIe); the results equal the copy path's
    and the oracle's."""
    import torch
    from paper_1808_00687_b200.decoder import BatchDecoder
    g = synth.random_wfst(5, 3000, 9000, 40, eps_fraction=0.03, selfloops=mode == "lsd",
                          final_fraction=0.05)
    posts = [synth.random_posteriors(40 + k, 150, 40, blank_fraction=0.6 if mode == "lsd" else 0.0)
             for k in range(7)]
    T = np.asarray([p.num_frames for p in posts], np.int32)
    off = np.zeros(len(T), np.int64)
    np.cumsum(T[:-1], out=off[1:])
    pinned = torch.empty((int(T.sum()), 41), dtype=torch.float64, pin_memory=True)
    blank = np.concatenate([p.rows[:, 0] for p in posts])
    for p, o in zip(posts, off):
        P.cost_table(p, out=pinned.numpy()[o:o + p.num_frames])
    cfg = P.DecodeConfig(beam=9.0, max_active=200, mode=mode)
    dec = BatchDecoder(g, 0)
    zc = dec.decode_host(pinned.numpy(), off, T, blank, cfg, mode)
    h2d, path = dec.last_transfer()
    if mode == "fsd":   # equal-length utterances at a common stride: the H2D pipeline
        assert path == 2
        assert h2d == pinned.numpy().nbytes + blank.nbytes + off.nbytes + T.nbytes
    else:               # LSD: zero-copy, only the searched (non-blank) rows cross PCIe
        assert path == 1
        steps = int(zc.results["search_steps"].sum())
        assert h2d == steps * 41 * 8 + blank.nbytes + off.nbytes + T.nbytes
    cp = dec.decode_host(pinned.numpy().copy(), off, T, blank, cfg, mode)   # pageable -> copy
    assert not dec.last_transfer()[1]
    assert zc.decode_results() == cp.decode_results()
    for p, r in zip(posts, zc.decode_results()):
        o = O.decode(g, P.cost_table(p), p.rows[:, 0], beam=9.0, max_active=200, mode=mode)
        assert _fields(r) == o.astuple()


def test_capacity_flags_and_targeted_retry(cuda):
    """Undersized workspaces report which capacity overflowed (WB_CAP_*) and decode_host
    grows exactly that one; the retried batch equals a decode with ample room."""
    from paper_1808_00687_b200 import _native as N
    from paper_1808_00687_b200.decoder import BatchDecoder, _native_config
    import ctypes as C
    g = synth.random_wfst(8, 2000, 7000, 30, eps_fraction=0.05, final_fraction=0.1)
    posts = [synth.random_posteriors(70 + k, 60, 30) for k in range(5)]
    T = np.asarray([p.num_frames for p in posts], np.int32)
    off = np.zeros(len(T), np.int64)
    np.cumsum(T[:-1], out=off[1:])
    costs = np.concatenate([P.cost_table(p) for p in posts])
    blank = np.concatenate([p.rows[:, 0] for p in posts])
    cfg = P.DecodeConfig(beam=9.0, max_active=150, mode="fsd")
    want = BatchDecoder(g, 0).decode_host(costs, off, T, blank, cfg, "fsd").decode_results()
    # raw call on a tiny workspace: every utterance fails with a named cause
    tiny = BatchDecoder(g, 0, cand_capacity=16, arena_capacity=1024)
    res = np.zeros(len(T), dtype=N.UTT_RESULT_DTYPE)
    lab = np.zeros((len(T), 2), np.int32)
    ncfg = _native_config(cfg, "fsd")
    N.check(N.load().wb_decode(tiny._h, len(T), costs.ctypes.data, off.ctypes.data,
                               T.ctypes.data, costs.shape[1], blank.ctypes.data, C.byref(ncfg),
                               res.ctypes.data, lab.ctypes.data, lab.ctypes.data, 1,
                               N.WB_MEM_HOST, None))
    assert (res["status"] == N.WB_ERR_CAPACITY).all()
    assert (res["capacity_flags"] & (N.WB_CAP_CANDIDATES | N.WB_CAP_ARENA)).all()
    # the Python entry point retries until it fits, with identical results
    got = tiny.decode_host(costs, off, T, blank, cfg, "fsd", label_capacity=1).decode_results()
    assert got == want


def test_ctc_lsd_blank_skip_at_scale(cuda):
    """Config-4 shape at test size: CTC-style graph (self-loops on every state), blank-peaked
    posteriors (80 % blank frames above the 0.98 threshold), LSD blank skipping."""
    g = synth.random_wfst(44, 4000, 16000, 200, eps_fraction=0.01, selfloops=True,
                          final_fraction=0.02)
    posts = [synth.random_posteriors(900 + k, 400, 200, blank_fraction=0.8) for k in range(10)]
    cfg = P.DecodeConfig(beam=13.0, max_active=500, mode="lsd")
    _check_batch(g, posts, cfg)
    got = P.decode_batch(g, posts, cfg)
    # blank skipping really happened: steps == non-blank frames (+0 / the dying step)
    for p, r in zip(posts, got):
        nonblank = int((p.rows[:, 0] <= cfg.blank_threshold).sum())
        assert r.search_steps <= nonblank < p.num_frames


@pytest.mark.parametrize("blank_col", [0, 5])
@pytest.mark.parametrize("mode", ["fsd", "lsd"])
def test_streaming_posteriors_equal_cost_table_path(cuda, mode, blank_col):
    """decode_posteriors (rows computed by host threads while the kernel already runs,
    ready counters in page-locked memory) == decode_host on the finished cost table."""
    from paper_1808_00687_b200.decoder import BatchDecoder
    g = synth.random_wfst(13, 3000, 9000, 60, eps_fraction=0.03, selfloops=mode == "lsd",
                          final_fraction=0.05)
    posts = [synth.random_posteriors(300 + k, 100 + 37 * k, 60, blank_col=blank_col,
                                     blank_fraction=0.7 if mode == "lsd" else 0.0)
             for k in range(9)] + [synth.random_posteriors(999, 0, 60, blank_col=blank_col)]
    cfg = P.DecodeConfig(beam=10.0, max_active=300, mode=mode, acoustic_scale=0.8)
    dec = BatchDecoder(g, 0)
    got = dec.decode_posteriors(posts, cfg, mode, block_frames=8, workers=3).decode_results()
    T = np.asarray([p.num_frames for p in posts], np.int32)
    off = np.zeros(len(T), np.int64)
    np.cumsum(T[:-1], out=off[1:])
    costs = np.concatenate([P.cost_table(p, 0.8) for p in posts if p.num_frames])
    blank = np.concatenate([p.rows[:, p.blank_col] for p in posts])
    want = BatchDecoder(g, 0).decode_host(costs, off, T, blank, cfg, mode).decode_results()
    assert got == want
    h2d, zc = dec.last_transfer()
    assert zc


def test_multi_device_threads_equal_single_batch(cuda):
    """decode_multi_device (one host thread + decoder per device entry; here both entries
    are cuda:0, so two decoders run concurrently on one GPU) == one decode_batch."""
    from paper_1808_00687_b200.shard import decode_multi_device
    g = synth.random_wfst(17, 2000, 7000, 30, eps_fraction=0.05, final_fraction=0.1)
    posts = [synth.random_posteriors(800 + k, 40 + 9 * k, 30) for k in range(11)]
    cfg = P.DecodeConfig(beam=9.0, max_active=100, mode="fsd")
    want = P.decode_batch(g, posts, cfg)
    got = decode_multi_device(g, posts, cfg, devices=[0, 0])
    assert got == want


def test_edge_cases_vs_oracle(cuda):
    """Empty and degenerate inputs: zero frames, all-blank LSD utterances (no search step),
    one frame, beam 0, max-active 1, a graph whose start state has no arcs."""
    g = synth.random_wfst(23, 300, 1200, 12, eps_fraction=0.1, final_fraction=0.2)
    allblank = synth.random_posteriors(5, 20, 12, blank_fraction=1.0)
    posts = [synth.random_posteriors(1, 0, 12), allblank, synth.random_posteriors(2, 1, 12),
             synth.random_posteriors(3, 50, 12, blank_fraction=0.5)]
    for mode in ("fsd", "lsd"):
        for beam, ma in ((0.0, None), (INF, 1), (5.0, 2), (INF, None)):
            _check_batch(g, posts, P.DecodeConfig(beam=beam, max_active=ma, mode=mode))
    r = P.decode(g, allblank, P.DecodeConfig(beam=9.0, mode="lsd"))
    assert r.search_steps == 0 and r.tokens_expanded == 0
    # a start state without arcs: the search dies at the first step
    from paper_1808_00687_b200.wfst import Wfst
    w = Wfst.from_arrays(3, 2, [0, 1], [1, 0], [1, 2], [1, 2], [0.5, 0.5],
                         np.array([np.inf, 0.0, np.inf]))
    p = synth.random_posteriors(4, 5, 2)
    _check_batch(w, [p], P.DecodeConfig(beam=INF, mode="fsd"))


@pytest.mark.parametrize("seed", range(4))
def test_negative_weights_disable_the_skip_exactly(cuda, seed):
    """Graphs with negative arc weights (parse_wfst_text(allow_negative_weights=True)): the
    exact beam skip needs weights >= 0 and is off for them (GraphDev.nonneg); results still
    equal the oracle's.  Epsilon arcs stay forward-only, so no epsilon cycle exists."""
    from paper_1808_00687_b200.wfst import Wfst
    g0 = synth.random_wfst(40 + seed, 400, 1800, 14, eps_fraction=0.05, selfloops=seed % 2 == 1,
                           final_fraction=0.2)
    rng = np.random.default_rng(seed)
    w = g0.weight.copy()
    flip = rng.random(len(w)) < 0.3
    w[flip] = -np.round(rng.uniform(0.0, 0.5, int(flip.sum())), 6)
    g = Wfst.from_arrays(g0.num_states, g0.start, g0.src, g0.dst, g0.ilabel, g0.olabel, w,
                         g0.final_w)
    assert g.epsilon_cycle() is None and (g.weight < 0).any()
    posts = [synth.random_posteriors(300 * seed + k, 30 + 7 * k, 14, blank_fraction=0.3)
             for k in range(6)]
    for mode in ("fsd", "lsd"):
        for beam, ma in ((6.0, 30), (INF, None), (3.0, None)):
            _check_batch(g, posts, P.DecodeConfig(beam=beam, max_active=ma, mode=mode))


def test_acoustic_scale_and_wide_beam_vs_oracle(cuda):
    """Non-unit acoustic scales (costs = -scale * log p) with beams wide enough that the skip
    rarely fires, and narrow ones where it fires on most relaxations."""
    g = synth.random_wfst(77, 1500, 6000, 25, eps_fraction=0.03, final_fraction=0.1)
    posts = [synth.random_posteriors(900 + k, 60, 25, blank_fraction=0.2) for k in range(5)]
    for scale in (0.3, 1.7):
        for beam in (1.5, 40.0):
            _check_batch(g, posts, P.DecodeConfig(beam=beam, max_active=200, mode="fsd",
                                                  acoustic_scale=scale))


@pytest.mark.parametrize("seed", range(3))
def test_max_active_early_cutoff_is_exact(cuda, seed, monkeypatch):
    """WB_MA_EARLY (expand's max-active early cutoff, off by default) on every step: same
    results as the oracle, with max-active binding hard and with beam = inf."""
    monkeypatch.setenv("WB_MA_EARLY", "1")
    g = synth.random_wfst(100 + seed, 5000, 16000, 50, eps_fraction=0.05, selfloops=True,
                          final_fraction=0.05)
    posts = [synth.random_posteriors(seed * 11 + k, 100, 50, blank_fraction=0.2) for k in range(6)]
    for beam, ma in ((10.0, 40), (10.0, 300), (INF, 100)):
        _check_batch(g, posts, P.DecodeConfig(beam=beam, max_active=ma, mode="fsd"))


@pytest.mark.parametrize("mode", ["fsd", "lsd"])
def test_posterior_batch_from_post1_files(cuda, tmp_path, mode):
    """POST1 files read natively into one page-locked table (PosteriorBatch), converted to
    costs in place while the kernel streams them: same results as decoding the matrices."""
    from paper_1808_00687_b200.posteriors import PosteriorBatch, save_posteriors
    g = synth.random_wfst(61, 2500, 8000, 30, eps_fraction=0.03, selfloops=mode == "lsd",
                          final_fraction=0.05)
    mats = [synth.random_posteriors(500 + k, 60 + 17 * k, 30, blank_col=(k % 2) * 4,
                                    blank_fraction=0.6 if mode == "lsd" else 0.0)
            for k in range(6)]
    paths = []
    for k, m in enumerate(mats):
        paths.append(str(tmp_path / f"{k}.post"))
        save_posteriors(m, paths[-1], binary=True)
    cfg = P.DecodeConfig(beam=10.0, max_active=300, mode=mode)
    batch = PosteriorBatch(paths)
    got = P.decode_batch(g, batch, cfg)
    assert batch.consumed
    assert got == P.decode_batch(g, mats, cfg)
    for m, r in zip(mats, got):
        o = O.decode(g, P.cost_table(m), m.rows[:, m.blank_col], beam=10.0, max_active=300,
                     mode=mode)
        assert _fields(r) == o.astuple()


def test_posterior_batch_capacity_retry(cuda, tmp_path):
    """A PosteriorBatch's rows are converted in place; when a capacity overflows, the retry
    decodes the converted table (not the rows a second time) and the results are exact."""
    from paper_1808_00687_b200.decoder import BatchDecoder
    from paper_1808_00687_b200.posteriors import PosteriorBatch
    g = synth.random_wfst(62, 2000, 7000, 20, eps_fraction=0.05, final_fraction=0.1)
    mats = [synth.random_posteriors(600 + k, 50, 20) for k in range(4)]
    cfg = P.DecodeConfig(beam=9.0, max_active=150, mode="fsd")
    tiny = BatchDecoder(g, 0, cand_capacity=16, arena_capacity=1024)
    got = tiny.decode_posteriors(PosteriorBatch(mats), cfg).decode_results()
    assert got == P.decode_batch(g, mats, cfg)


def test_h2d_pipeline_fallbacks(cuda, monkeypatch):
    """The H2D pipeline needs equal-length FSD utterances at a common stride: ragged batches
    and WB_H2D_PIPELINE=0 read the page-locked table zero-copy; all three paths agree."""
    import torch
    from paper_1808_00687_b200.decoder import BatchDecoder
    g = synth.random_wfst(8, 2000, 6000, 30, eps_fraction=0.03, final_fraction=0.05)
    cfg = P.DecodeConfig(beam=9.0, max_active=150, mode="fsd")
    for name, lens in (("equal", [90] * 6), ("ragged", [90, 40, 90, 75, 90, 1])):
        posts = [synth.random_posteriors(70 + k, t, 30) for k, t in enumerate(lens)]
        T = np.asarray(lens, np.int32)
        off = np.zeros(len(T), np.int64)
        np.cumsum(T[:-1], out=off[1:])
        pinned = torch.empty((int(T.sum()), 31), dtype=torch.float64, pin_memory=True)
        for p, o in zip(posts, off):
            P.cost_table(p, out=pinned.numpy()[o:o + p.num_frames])
        blank = np.concatenate([p.rows[:, 0] for p in posts])
        dec = BatchDecoder(g, 0)
        r = dec.decode_host(pinned.numpy(), off, T, blank, cfg, "fsd").decode_results()
        assert dec.last_transfer()[1] == (2 if name == "equal" else 1)
        for p, got in zip(posts, r):
            o = O.decode(g, P.cost_table(p), p.rows[:, 0], beam=9.0, max_active=150, mode="fsd")
            assert _fields(got) == o.astuple()
        if name == "equal":
            monkeypatch.setenv("WB_H2D_PIPELINE", "0")
            assert dec.decode_host(pinned.numpy(), off, T, blank, cfg, "fsd").decode_results() == r
            assert dec.last_transfer()[1] == 1
            monkeypatch.delenv("WB_H2D_PIPELINE")


def test_h2d_pipeline_waves(cuda):
    """More utterances than lanes: the H2D pipeline copies one wave of lanes' utterances at a
    time (in the order the lanes take them); every utterance equals the oracle."""
    import torch
    from paper_1808_00687_b200.decoder import BatchDecoder
    g = synth.random_wfst(11, 2500, 8000, 25, eps_fraction=0.05, final_fraction=0.05)
    cfg = P.DecodeConfig(beam=9.0, max_active=120, mode="fsd")
    posts = [synth.random_posteriors(200 + k, 60, 25) for k in range(9)]
    T = np.full(len(posts), 60, np.int32)
    off = np.arange(len(posts), dtype=np.int64) * 60
    pinned = torch.empty((int(T.sum()), 26), dtype=torch.float64, pin_memory=True)
    for p, o in zip(posts, off):
        P.cost_table(p, out=pinned.numpy()[o:o + 60])
    blank = np.concatenate([p.rows[:, 0] for p in posts])
    dec = BatchDecoder(g, 0, max_utts_in_flight=2)   # 2 lanes: 5 waves
    got = dec.decode_host(pinned.numpy(), off, T, blank, cfg, "fsd").decode_results()
    assert dec.last_transfer()[1] == 2
    for p, r in zip(posts, got):
        o = O.decode(g, P.cost_table(p), p.rows[:, 0], beam=9.0, max_active=120, mode="fsd")
        assert _fields(r) == o.astuple()
