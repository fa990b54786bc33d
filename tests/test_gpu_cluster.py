"""Cluster lanes: one utterance searched by a thread-block cluster of K CTAs (K SMs), the
per-step phases split across the CTAs and combined through distributed shared memory.
Every K gives exactly the oracle's results (and the single-CTA results)."""
import math

import numpy as np
import pytest

import paper_1808_00687_b200 as P
from paper_1808_00687_b200 import _native as N
from paper_1808_00687_b200 import synth
from paper_1808_00687_b200.decoder import BatchDecoder
from oracle import oracle as O

pytestmark = pytest.mark.gpu
INF = math.inf


def _fields(r):
    return (r.total_cost, r.olabels, r.ilabels, r.search_steps, r.tokens_expanded,
            r.reached_final, r.died_at_step)


def _table(posts, scale=1.0):
    T = np.asarray([p.num_frames for p in posts], np.int32)
    off = np.zeros(len(T), np.int64)
    np.cumsum(T[:-1], out=off[1:])
    costs = np.concatenate([P.cost_table(p, scale) for p in posts])
    blank = np.concatenate([p.rows[:, p.blank_col] for p in posts])
    return costs, off, T, blank


def _oracle(g, posts, cfg):
    return [O.decode(g, P.cost_table(p, cfg.acoustic_scale), p.rows[:, p.blank_col],
                     beam=cfg.beam, max_active=cfg.max_active, mode=cfg.mode,
                     blank_threshold=cfg.blank_threshold).astuple() for p in posts]


@pytest.mark.parametrize("K", [2, 4, 8])
@pytest.mark.parametrize("seed", range(6))
def test_cluster_small_graphs_vs_oracle(cuda, K, seed):
    rng = np.random.default_rng(seed)
    S = int(rng.integers(20, 400))
    g = synth.random_wfst(seed, S, int(S * rng.uniform(1.5, 4)), int(rng.integers(2, 12)),
                          eps_fraction=[0.0, 0.1, 0.25][seed % 3], selfloops=seed % 2 == 0,
                          final_fraction=0.2)
    L = int(g.max_ilabel) or 1
    posts = [synth.random_posteriors(seed * 50 + k, int(rng.integers(0, 40)), L,
                                     blank_fraction=0.3) for k in range(5)]
    dec = BatchDecoder(g, 0, cluster_ctas=K)
    for mode in ("fsd", "lsd"):
        for beam, ma in ((INF, None), (5.0, None), (INF, 7), (8.0, 40)):
            cfg = P.DecodeConfig(beam=beam, max_active=ma, mode=mode)
            out = dec.decode_host(*_table(posts), cfg, mode)
            assert dec.last_cluster_ctas() == K
            assert [_fields(r) for r in out.decode_results()] == _oracle(g, posts, cfg), (mode, beam, ma)


@pytest.fixture(scope="module")
def c2():
    g = synth.hclg_like(0)
    return g, O.OracleGraph(g)


@pytest.mark.parametrize("K,env", [(2, {}), (4, {}), (8, {}), (2, {"WB_SMEM_CANDS": "0"}),
                                   (2, {"WB_FORCE_RADIX": "1"}), (4, {"WB_PREFETCH": "0"}),
                                   (4, {"WB_SMEM_CANDS": "1500"})])
def test_cluster_config2_scale(cuda, c2, monkeypatch, K, env):
    g, og = c2
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    posts = [synth.random_posteriors(100 + i, 250, 3000) for i in range(4)]
    cfg = P.DecodeConfig(beam=13.0, max_active=7000, mode="fsd")
    dec = BatchDecoder(g, 0, max_utts_in_flight=4, cluster_ctas=K)
    out = dec.decode_host(*_table(posts), cfg, "fsd")
    assert dec.last_cluster_ctas() == K
    want = O.decode_batch(og, [P.cost_table(p) for p in posts], [p.rows[:, 0] for p in posts],
                          beam=13.0, max_active=7000, mode="fsd")
    assert [_fields(r) for r in out.decode_results()] == [o.astuple() for o in want]
    flags = out.results["path_flags"]
    assert (flags & N.WB_PATH_SELECT).all()


def test_cluster_auto_fills_idle_sms_and_streams(cuda):
    """Fewer utterances than SMs: the automatic choice uses clusters; the public streaming
    path (decode_batch, cost rows published while the kernel runs) agrees with the oracle."""
    g = synth.random_wfst(3, 5000, 16000, 40, eps_fraction=0.05, selfloops=True,
                          final_fraction=0.05)
    posts = [synth.random_posteriors(900 + k, 150, 40, blank_fraction=0.5) for k in range(3)]
    for mode in ("fsd", "lsd"):
        cfg = P.DecodeConfig(beam=10.0, max_active=400, mode=mode)
        got = P.decode_batch(g, posts, cfg)
        assert [_fields(r) for r in got] == _oracle(g, posts, cfg)
    dec = BatchDecoder(g, 0)
    dec.decode_host(*_table(posts), P.DecodeConfig(beam=10.0, mode="fsd"), "fsd")
    assert dec.last_cluster_ctas() == 4


def test_cluster_tie_heavy_radix(cuda):
    from paper_1808_00687_b200.wfst import Wfst
    g0 = synth.random_wfst(5, 50_000, 200_000, 20, eps_fraction=0.0, final_fraction=0.05)
    g = Wfst.from_arrays(g0.num_states, g0.start, g0.src, g0.dst, g0.ilabel, g0.olabel,
                         np.floor(g0.weight), np.floor(g0.final_w))
    posts = [P.PosteriorMatrix(np.full((40 + 10 * i, 21), 1.0 / 21), 0, validate=False)
             for i in range(3)]
    cfg = P.DecodeConfig(beam=INF, max_active=1500, mode="fsd")
    dec = BatchDecoder(g, 0, cluster_ctas=2)
    out = dec.decode_host(*_table(posts), cfg, "fsd")
    assert [_fields(r) for r in out.decode_results()] == _oracle(g, posts, cfg)
    assert (out.results["path_flags"] & N.WB_PATH_RADIX).any()


def test_memory_budget_trades_lanes_for_clusters(cuda, monkeypatch):
    """When the dense per-state arrays of one lane per SM would not fit (a large graph), the
    decoder takes fewer lanes and fills the SMs with clusters; results are unchanged."""
    g = synth.random_wfst(12, 200_000, 600_000, 30, eps_fraction=0.03, final_fraction=0.05)
    posts = [synth.random_posteriors(60 + k, 40, 30) for k in range(90)]
    cfg = P.DecodeConfig(beam=10.0, max_active=500, mode="fsd")
    want = BatchDecoder(g, 0).decode_host(*_table(posts), cfg, "fsd").decode_results()
    # one lane: 200k states x 24 B + a 32 MB arena ~ 37 MB; 148 lanes would need 5.5 GB
    monkeypatch.setenv("WB_MEM_BUDGET_GB", "3.5")
    dec = BatchDecoder(g, 0)
    lanes, kmax = dec.lanes()
    assert lanes <= 74 and kmax >= 2 and lanes * kmax <= 148
    out = dec.decode_host(*_table(posts), cfg, "fsd")
    assert dec.last_cluster_ctas() >= 2
    assert out.decode_results() == want
