"""The public posterior path under serialised launches, growing streaming batches with device
lattice pruning, and concurrent callers (decoder.py:364, wfst_decoder.cu:616,
decoder.py:541)."""
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

import paper_1808_00687_b200 as P
from paper_1808_00687_b200 import lattice as Lt
from paper_1808_00687_b200 import synth
from paper_1808_00687_b200.decoder import BatchDecoder
from paper_1808_00687_b200.pipeline import LatticePipeline
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import sys
sys.path.insert(0, %r)
import paper_1808_00687_b200 as P
from paper_1808_00687_b200 import synth
from oracle import oracle as O
g = synth.random_wfst(3, 2000, 7000, 30, eps_fraction=0.05, selfloops=True, final_fraction=0.1)
posts = [synth.random_posteriors(60 + i, 80 + 11 * i, 30, blank_fraction=0.4) for i in range(5)]
for mode in ("fsd", "lsd"):
    cfg = P.DecodeConfig(beam=9.0, max_active=150, mode=mode)
    got = P.decode_batch(g, posts, cfg)
    for p, r in zip(posts, got):
        o = O.decode(g, P.cost_table(p), p.rows[:, 0], beam=9.0, max_active=150, mode=mode)
        assert (r.total_cost, r.olabels, r.ilabels, r.search_steps, r.tokens_expanded,
                r.reached_final, r.died_at_step) == o.astuple(), (mode, r, o)
    rec = P.LatticeRecorder()
    P.decode(g, posts[0], cfg, recorder=rec)
# the H2D pipeline of a page-locked FSD table (copies enqueued before the launch)
import numpy as np
import torch
from paper_1808_00687_b200.decoder import BatchDecoder
eq = [synth.random_posteriors(90 + i, 70, 30) for i in range(4)]
T = np.full(4, 70, np.int32)
off = np.arange(4, dtype=np.int64) * 70
pin = torch.empty((280, 31), dtype=torch.float64, pin_memory=True)
for p, o in zip(eq, off):
    P.cost_table(p, out=pin.numpy()[o:o + 70])
blank = np.concatenate([p.rows[:, 0] for p in eq])
dec = BatchDecoder(g, 0)
cfg = P.DecodeConfig(beam=9.0, max_active=150, mode="fsd")
res = dec.decode_host(pin.numpy(), off, T, blank, cfg, "fsd").decode_results()
assert dec.last_transfer()[1] == 2, dec.last_transfer()
for p, r in zip(eq, res):
    o = O.decode(g, P.cost_table(p), p.rows[:, 0], beam=9.0, max_active=150, mode="fsd")
    assert (r.total_cost, r.olabels, r.ilabels, r.search_steps, r.tokens_expanded,
            r.reached_final, r.died_at_step) == o.astuple(), (r, o)
print("OK")
""" % ROOT


def test_streaming_decode_with_blocking_launches(cuda):
    """CUDA_LAUNCH_BLOCKING=1 makes every launch return only after its kernel finished (as
    under ncu or compute-sanitizer).  The cost-row producers start before the launch, so the
    streaming kernel still gets its rows and decode() completes with the oracle's results; the
    FSD H2D pipeline's copies are all enqueued before its launch."""
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
    r = subprocess.run([sys.executable, "-c", _CHILD], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_streaming_device_prune_with_growing_batches(cuda):
    """submit_posteriors with a lattice beam and a batch larger than any before it: the prune
    pools grow before the streaming launch (a cudaFree after it would wait on a kernel that
    waits on the host).  Results equal the cost-table path."""
    g = synth.random_wfst(31, 400, 1600, 16, eps_fraction=0.05, final_fraction=0.1)
    cfg = P.DecodeConfig(beam=7.0, max_active=40, mode="fsd")
    batches = [[synth.random_posteriors(10 * b + i, 15 + 9 * b + i, 16) for i in range(2 + 3 * b)]
               for b in range(3)]
    dec = BatchDecoder(g, 0, max_utts_in_flight=4)
    with LatticePipeline(dec, lattice_beam=2.5) as pipe:
        futs = [pipe.submit_posteriors(posts, cfg) for posts in batches]
        got = [f.result(timeout=300) for f in futs]
    ref = BatchDecoder(g, 0)
    for posts, (out, lats) in zip(batches, got):
        T = np.asarray([p.num_frames for p in posts], np.int32)
        off = np.zeros(len(T), np.int64)
        np.cumsum(T[:-1], out=off[1:])
        costs = np.concatenate([P.cost_table(p) for p in posts])
        blank = np.concatenate([p.rows[:, 0] for p in posts])
        rout = ref.decode_host(costs, off, T, blank, cfg, "fsd", lattice=True)
        assert rout.decode_results() == out.decode_results()
        for a, b in zip(ref.fetch_lattices(g), lats):
            try:
                want = a.key() if a.start_id is None else Lt.prune_lattice(a, 2.5).key()
            except Lt.LatticeError:
                want = "error"
            assert ("error" if isinstance(b, Lt.LatticeError) else b.key()) == want


def test_concurrent_decode_calls_on_one_graph(cuda):
    """Threads calling decode() on the same Wfst share one cached decoder: each call holds the
    decoder for its launch + fetch, so every thread gets its own utterance's result."""
    g = synth.random_wfst(41, 3000, 9000, 25, eps_fraction=0.03, final_fraction=0.1)
    posts = [synth.random_posteriors(700 + i, 40 + 13 * i, 25) for i in range(12)]
    cfg = P.DecodeConfig(beam=9.0, max_active=200, mode="fsd")
    want = [O.decode(g, P.cost_table(p), p.rows[:, 0], beam=9.0, max_active=200,
                     mode="fsd").astuple() for p in posts]
    got = [None] * len(posts)
    errs = []

    def run(i):
        try:
            for _ in range(3):
                r = P.decode(g, posts[i], cfg)
                got[i] = (r.total_cost, r.olabels, r.ilabels, r.search_steps, r.tokens_expanded,
                          r.reached_final, r.died_at_step)
        except BaseException as exc:  # pragma: no cover - reported below
            errs.append(exc)
    th = [threading.Thread(target=run, args=(i,)) for i in range(len(posts))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert got == want
