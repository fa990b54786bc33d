"""The checked build (libwfstb200_checked.so, -DWB_CHECKS): the device verifies the search's
synchronisation invariants -- the reference's ClaimLedger.verify_partitions and debug_epoch
(parallel.py:41-61, 92-116) -- in place of compute-sanitizer's racecheck (closed on this
pool): each live token expanded by exactly one warp per step, each state registered once per
step (the first-touch CAS protocol), every touched slot reset at the end of its step and the
slot array clean between utterances, workspace indices in bounds."""
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


class Ledger:
    """Same protocol as the reference's ClaimLedger (begin_step / verify_partitions)."""

    def __init__(self):
        self.steps = []

    def begin_step(self, queue_len):
        claims = {}
        self.steps.append((queue_len, claims))
        return claims

    def verify_partitions(self):
        for step, (n, claims) in enumerate(self.steps):
            merged = sorted(i for idx in claims.values() for i in idx)
            if merged != list(range(n)):
                raise AssertionError(f"step {step}: claims do not partition {n}")


def _fields(r):
    return (r.total_cost, r.olabels, r.ilabels, r.search_steps, r.tokens_expanded,
            r.reached_final, r.died_at_step)


def _table(posts):
    T = np.asarray([p.num_frames for p in posts], np.int32)
    off = np.zeros(len(T), np.int64)
    np.cumsum(T[:-1], out=off[1:])
    return (np.concatenate([P.cost_table(p) for p in posts]), off, T,
            np.concatenate([p.rows[:, p.blank_col] for p in posts]))


@pytest.mark.parametrize("K", [1, 2, 4])
@pytest.mark.parametrize("seed", range(5))
def test_checked_build_random_graphs(cuda, K, seed):
    rng = np.random.default_rng(seed)
    S = int(rng.integers(30, 3000))
    g = synth.random_wfst(seed, S, int(S * rng.uniform(1.5, 4)), 20,
                          eps_fraction=[0.0, 0.08, 0.2][seed % 3], selfloops=seed % 2 == 0,
                          final_fraction=0.1)
    posts = [synth.random_posteriors(seed * 40 + k, int(rng.integers(1, 60)), 20,
                                     blank_fraction=0.4) for k in range(6)]
    dec = BatchDecoder(g, 0, cluster_ctas=K, checks=True)
    assert dec.checks
    for mode in ("fsd", "lsd"):
        for beam, ma in ((INF, None), (6.0, 30), (9.0, None), (INF, 4)):
            cfg = P.DecodeConfig(beam=beam, max_active=ma, mode=mode)
            out = dec.decode_host(*_table(posts), cfg, mode)   # raises on a violation
            want = [O.decode(g, P.cost_table(p), p.rows[:, 0], beam=beam, max_active=ma,
                             mode=mode).astuple() for p in posts]
            assert [_fields(r) for r in out.decode_results()] == want


@pytest.mark.parametrize("K", [1, 2])
def test_checked_build_config2_scale(cuda, K):
    g = synth.hclg_like(0)
    posts = [synth.random_posteriors(40 + i, 80, 3000) for i in range(3)]
    cfg = P.DecodeConfig(beam=13.0, max_active=7000, mode="fsd")
    dec = BatchDecoder(g, 0, max_utts_in_flight=3, cluster_ctas=K, checks=True)
    out = dec.decode_host(*_table(posts), cfg, "fsd")
    want = O.decode_batch(g, [P.cost_table(p) for p in posts], [p.rows[:, 0] for p in posts],
                          beam=13.0, max_active=7000, mode="fsd")
    assert [_fields(r) for r in out.decode_results()] == [o.astuple() for o in want]


def test_parallel_decode_fills_the_claim_ledger(cuda):
    """parallel_decode(claim_ledger=..., debug_epoch=True) runs the checked kernels and fills
    the ledger with the device's per-step claims (group = warp); they partition every queue
    (test_parallel.py:235-241), and the result equals decode()."""
    g = synth.random_wfst(2, 2000, 7000, 20, eps_fraction=0.05, final_fraction=0.1)
    p = synth.random_posteriors(9, 50, 20, blank_fraction=0.3)
    for mode in ("fsd", "lsd"):
        cfg = P.DecodeConfig(beam=9.0, max_active=200, mode=mode)
        ledger = Ledger()
        r = P.parallel_decode(g, p, cfg, workers=4, group_size=8, claim_ledger=ledger,
                              debug_epoch=True)
        assert r == P.decode(g, p, cfg)
        assert len(ledger.steps) == r.search_steps
        assert sum(n for n, _ in ledger.steps) == r.tokens_expanded
        assert any(len(c) > 1 for _, c in ledger.steps)   # several warps shared the work
        ledger.verify_partitions()


def test_injected_stale_slot_is_caught(cuda, monkeypatch):
    """A slot deliberately left un-reset (WB_CHECK_INJECT) raises the stale-epoch check, like
    the reference's debug_epoch assertion (test_parallel.py:126-135)."""
    monkeypatch.setenv("WB_CHECK_INJECT", "1")
    g = synth.random_wfst(4, 500, 2000, 10, final_fraction=0.2)
    posts = [synth.random_posteriors(3, 20, 10)]
    dec = BatchDecoder(g, 0, checks=True)
    with pytest.raises(N.DeviceCheckError, match="not reset|non-empty"):
        dec.decode_host(*_table(posts), P.DecodeConfig(beam=INF, mode="fsd"), "fsd")
