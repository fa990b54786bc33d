"""Device lattice recording + trimming (decode_kernel.cuh record_lattice_step / trim_lattice)
against the reference's built lattices (golden fixtures) and the oracle's build_lattice.

Bit-exact bar: same nodes, arcs (graph + acoustic costs as f64), finals and canonical order
as the reference's build_lattice (lattice.py:148-249); tie = WFST arc index, so the lattice
best path equals the reference's too.
"""
import math

import numpy as np
import pytest

import golden_cases as GC
from oracle import oracle as O
from paper_1808_00687_b200 import lattice as L
from paper_1808_00687_b200 import synth
from paper_1808_00687_b200.decoder import BatchDecoder, DecodeConfig

pytestmark = pytest.mark.gpu
INF = math.inf


def _key(lat):
    return "empty" if lat.start_id is None else lat.key()


def _decode_lattices(g, costs_list, blank_list, cfg, dec=None):
    dec = dec or BatchDecoder(g, 0, max_utts_in_flight=8)
    T = np.asarray([len(c) for c in costs_list], np.int32)
    off = np.zeros(len(T), np.int64)
    np.cumsum(T[:-1], out=off[1:])
    L1 = costs_list[0].shape[1]
    costs = np.concatenate([c.reshape(-1, L1) for c in costs_list]) if T.sum() else np.zeros((1, L1))
    blank = np.concatenate(blank_list) if T.sum() else np.zeros(1)
    out = dec.decode_host(costs, off, T, blank, cfg, cfg.mode, lattice=True)
    lats = dec.fetch_lattices(dec.graph.wfst)
    return out, lats


def test_gpu_lattice_matches_reference_golden(cuda):
    n = 0
    beams = GC.prune_beams()
    for case in GC.cases():
        if case.lattice is None:
            continue
        g = case.graph.to_wfst()
        cfg = DecodeConfig(beam=case.cfg.get("beam", INF), max_active=case.cfg.get("max_active"),
                           mode=case.cfg.get("mode", "lsd"))
        out, lats = _decode_lattices(g, [case.costs], [case.blank], cfg)
        lat = lats[0]
        if case.lattice == "error":
            with pytest.raises(L.LatticeError):
                L._check(lat)
            continue
        assert _key(lat) == case.lattice, (case.kind, case.seed)
        if case.best_path is not None:
            assert L.lattice_best_path(lat) == case.best_path
        for b, exp in zip(beams, case.pruned or []):
            try:
                got = _key(L.prune_lattice(lat, b))
            except L.LatticeError:
                got = "error"
            assert got == exp, (case.kind, case.seed, b)
        n += 1
    assert n > 50


@pytest.mark.parametrize("mode", ["fsd", "lsd"])
def test_gpu_lattice_batch_matches_oracle(cuda, mode):
    """Many utterances per launch, random graphs with epsilon arcs, beam + max-active."""
    for seed in range(4):
        g = synth.random_wfst(seed, 300, 1200, 16, eps_fraction=0.06, selfloops=True,
                              final_fraction=0.1)
        posts = [synth.random_posteriors(1000 * seed + i, 12 + 5 * i, 16, blank_fraction=0.3)
                 for i in range(10)]
        from paper_1808_00687_b200.posteriors import cost_table
        costs = [cost_table(p) for p in posts]
        blanks = [np.ascontiguousarray(p.rows[:, 0]) for p in posts]
        cfg = DecodeConfig(beam=7.0, max_active=40, mode=mode)
        out, lats = _decode_lattices(g, costs, blanks, cfg)
        for i, (c, b) in enumerate(zip(costs, blanks)):
            try:
                res, olat = O.decode(g, c, b, beam=7.0, max_active=40, mode=mode,
                                     return_lattice=True)
                exp = olat.key() if not olat.empty else ("EMPTY",)
            except O.OracleLatticeError:
                with pytest.raises(L.LatticeError):
                    L._check(lats[i])
                continue
            assert lats[i].key() == exp, (seed, i)
            r = out.results[i]
            assert int(r["final_step"]) == res.final_step


def test_gpu_lattice_recorder_api(cuda):
    """decode(..., recorder=LatticeRecorder()) + build_lattice, as the reference is called."""
    import paper_1808_00687_b200 as P
    g = synth.random_wfst(3, 200, 800, 12, eps_fraction=0.05, final_fraction=0.2)
    p = synth.random_posteriors(5, 25, 12)
    rec = L.LatticeRecorder()
    r = P.decode(g, p, P.DecodeConfig(beam=8.0, mode="fsd"), recorder=rec)
    lat = L.build_lattice(rec, g)
    if not lat.is_empty:
        cost, ol, il = L.lattice_best_path(lat)
        assert cost == r.total_cost and ol == r.olabels and il == r.ilabels


def test_gpu_pipelined_builder_api(cuda):
    """The reference's PipelinedLatticeBuilder use (cli.py:104-121): recorder(consumer=builder),
    then builder.result_from(recorder) == build_lattice(recorder)."""
    import paper_1808_00687_b200 as P
    g = synth.random_wfst(4, 200, 800, 12, eps_fraction=0.05, final_fraction=0.2)
    p = synth.random_posteriors(6, 30, 12)
    builder = P.PipelinedLatticeBuilder(g)
    rec = L.LatticeRecorder(consumer=builder)
    P.parallel_decode(g, p, P.DecodeConfig(beam=8.0, mode="lsd"), workers=4, recorder=rec)
    lat = builder.result_from(rec)
    assert _key(lat) == _key(L.build_lattice(rec, g))
    with pytest.raises(L.LatticeError):
        P.PipelinedLatticeBuilder(g).result_from(L.LatticeRecorder())


def test_gpu_lattice_capacity_retry(cuda):
    """Tiny raw-lattice / output pools overflow and are grown transparently."""
    g = synth.random_wfst(11, 300, 1200, 16, eps_fraction=0.05, final_fraction=0.1)
    posts = [synth.random_posteriors(50 + i, 40, 16) for i in range(6)]
    from paper_1808_00687_b200.posteriors import cost_table
    costs = [cost_table(p) for p in posts]
    blanks = [np.ascontiguousarray(p.rows[:, 0]) for p in posts]
    cfg = DecodeConfig(beam=9.0, mode="fsd")
    small = BatchDecoder(g, 0, max_utts_in_flight=3, lattice_capacity=1024,
                         lattice_out_capacity=64)
    _, lats = _decode_lattices(g, costs, blanks, cfg, dec=small)
    _, ref = _decode_lattices(g, costs, blanks, cfg)
    assert [x.key() for x in lats] == [x.key() for x in ref]


def test_gpu_lattice_pipeline_matches_direct(cuda):
    """LatticePipeline (decode of batch i+1 overlapping host pruning of batch i) returns what
    the direct decode + fetch + prune_lattice path returns."""
    from paper_1808_00687_b200.pipeline import LatticePipeline
    from paper_1808_00687_b200.posteriors import cost_table
    g = synth.random_wfst(21, 300, 1200, 16, eps_fraction=0.05, final_fraction=0.1)
    cfg = DecodeConfig(beam=7.0, max_active=40, mode="fsd")
    batches = []
    for b in range(3):
        posts = [synth.random_posteriors(100 * b + i, 20 + 3 * i, 16) for i in range(5)]
        costs = [cost_table(p) for p in posts]
        T = np.asarray([len(c) for c in costs], np.int32)
        off = np.zeros(len(T), np.int64)
        np.cumsum(T[:-1], out=off[1:])
        batches.append((np.concatenate(costs), off, T,
                        np.concatenate([p.rows[:, 0] for p in posts])))
    dec = BatchDecoder(g, 0, max_utts_in_flight=4)
    with LatticePipeline(dec, lattice_beam=2.5) as pipe:
        futs = [pipe.submit(c, o, t, bl, cfg) for c, o, t, bl in batches]
        got = [f.result() for f in futs]
    ref = BatchDecoder(g, 0, max_utts_in_flight=4)
    for (c, o, t, bl), (out, lats) in zip(batches, got):
        rout = ref.decode_host(c, o, t, bl, cfg, "fsd", lattice=True)
        rl = ref.fetch_lattices(g)
        assert rout.decode_results() == out.decode_results()
        for a, b in zip(rl, lats):
            try:
                want = _key(L.prune_lattice(a, 2.5))
            except L.LatticeError:
                want = "error"
            assert ("error" if isinstance(b, L.LatticeError) else _key(b)) == want


def test_gpu_device_prune_matches_reference_golden(cuda):
    """Device lattice-beam pruning (stage one in prune_kernel, the path-exact split on the
    host) == the reference's prune_lattice on its own built lattice, at every golden beam."""
    beams = GC.prune_beams()
    n = 0
    for case in GC.cases():
        if not case.pruned:
            continue
        g = case.graph.to_wfst()
        cfg = DecodeConfig(beam=case.cfg.get("beam", INF), max_active=case.cfg.get("max_active"),
                           mode=case.cfg.get("mode", "lsd"))
        dec = BatchDecoder(g, 0, max_utts_in_flight=2)
        T = np.asarray([case.costs.shape[0]], np.int32)
        costs = case.costs if len(case.costs) else np.zeros((1, case.costs.shape[1]))
        blank = case.blank if len(case.blank) else np.zeros(1)
        for b, exp in zip(beams, case.pruned):
            dec.decode_host(costs, np.zeros(1, np.int64), T, blank, cfg, cfg.mode, lattice=True,
                            lattice_beam=b)
            got = dec.fetch_pruned_lattices(g, b)[0]
            key = "error" if isinstance(got, L.LatticeError) else _key(got)
            assert key == exp, (case.kind, case.seed, b)
            n += 1
    assert n > 200


def test_gpu_device_prune_batch_matches_host_prune(cuda):
    """Many utterances per launch: device-pruned lattices == host prune_lattice of the same
    device lattices (random graphs with epsilon arcs, several beams)."""
    from paper_1808_00687_b200.posteriors import cost_table
    for seed in range(3):
        g = synth.random_wfst(30 + seed, 400, 1600, 16, eps_fraction=0.08, selfloops=seed == 1,
                              final_fraction=0.1)
        posts = [synth.random_posteriors(500 * seed + i, 15 + 4 * i, 16, blank_fraction=0.3)
                 for i in range(9)]
        costs = [cost_table(p) for p in posts]
        blanks = [np.ascontiguousarray(p.rows[:, 0]) for p in posts]
        T = np.asarray([len(c) for c in costs], np.int32)
        off = np.zeros(len(T), np.int64)
        np.cumsum(T[:-1], out=off[1:])
        C_, B_ = np.concatenate(costs), np.concatenate(blanks)
        for mode in ("fsd", "lsd"):
            cfg = DecodeConfig(beam=8.0, max_active=60, mode=mode)
            dec = BatchDecoder(g, 0, max_utts_in_flight=4)
            dec.decode_host(C_, off, T, B_, cfg, mode, lattice=True)
            full = dec.fetch_lattices(g)
            for lb in (0.5, 3.0, 8.0):
                dec.decode_host(C_, off, T, B_, cfg, mode, lattice=True, lattice_beam=lb)
                got = dec.fetch_pruned_lattices(g, lb)
                for a, b in zip(full, got):
                    try:
                        want = _key(L.prune_lattice(a, lb))
                    except L.LatticeError:
                        want = "error"
                    assert ("error" if isinstance(b, L.LatticeError) else _key(b)) == want, (seed, mode, lb)


def test_gpu_lattices_with_negative_weights(cuda):
    """Negative arc weights (beam skip off): device lattices equal the oracle's build_lattice
    and device-pruned lattices equal the host prune_lattice of them."""
    from paper_1808_00687_b200.posteriors import cost_table
    from paper_1808_00687_b200.wfst import Wfst
    for seed in range(2):
        g0 = synth.random_wfst(60 + seed, 300, 1200, 16, eps_fraction=0.06, selfloops=True,
                               final_fraction=0.1)
        rng = np.random.default_rng(seed)
        w = g0.weight.copy()
        flip = rng.random(len(w)) < 0.3
        w[flip] = -np.round(rng.uniform(0.0, 0.5, int(flip.sum())), 6)
        g = Wfst.from_arrays(g0.num_states, g0.start, g0.src, g0.dst, g0.ilabel, g0.olabel, w,
                             g0.final_w)
        posts = [synth.random_posteriors(700 * seed + i, 12 + 5 * i, 16, blank_fraction=0.3)
                 for i in range(8)]
        costs = [cost_table(p) for p in posts]
        blanks = [np.ascontiguousarray(p.rows[:, 0]) for p in posts]
        cfg = DecodeConfig(beam=7.0, max_active=40, mode="lsd")
        out, lats = _decode_lattices(g, costs, blanks, cfg)
        for i, (c, b) in enumerate(zip(costs, blanks)):
            try:
                _, olat = O.decode(g, c, b, beam=7.0, max_active=40, mode="lsd",
                                   return_lattice=True)
                exp = olat.key() if not olat.empty else ("EMPTY",)
            except O.OracleLatticeError:
                with pytest.raises(L.LatticeError):
                    L._check(lats[i])
                continue
            assert lats[i].key() == exp, (seed, i)
        T = np.asarray([len(x) for x in costs], np.int32)
        off = np.zeros(len(T), np.int64)
        np.cumsum(T[:-1], out=off[1:])
        dec = BatchDecoder(g, 0, max_utts_in_flight=4)
        for lb in (1.0, 6.0):
            dec.decode_host(np.concatenate(costs), off, T, np.concatenate(blanks), cfg, "lsd",
                            lattice=True, lattice_beam=lb)
            got = dec.fetch_pruned_lattices(g, lb)
            for a, b in zip(lats, got):
                try:
                    want = _key(L.prune_lattice(a, lb))
                except L.LatticeError:
                    want = "error"
                assert ("error" if isinstance(b, L.LatticeError) else _key(b)) == want, (seed, lb)


def test_gpu_foreign_recorder_gets_the_protocol(cuda):
    """Any object with begin_step/emitting/epsilon/survivors/finish (here a minimal stand-in
    for the reference's LatticeRecorder) receives the decoded lattice step by step; the
    steps it collected rebuild the same lattice, and a PipelinedLatticeBuilder consumer is
    fed and closed."""
    import paper_1808_00687_b200 as P

    class Protocol:
        def __init__(self):
            self.steps, self.calls = [], []
            self.final_step = self.final_state = None
            self.reached_final = False

        def begin_step(self, k):
            self.steps.append(L.StepRecord())
            self.calls.append(("begin", k))

        def emitting(self, k, src, arc, ac):
            self.steps[k].emit.append((src, arc, ac))

        def epsilon(self, k, src, arc):
            self.steps[k].eps.add((src, arc))

        def survivors(self, k, states):
            self.steps[k].survivors = tuple(states)

        def finish(self, fs, fst, reached):
            self.final_step, self.final_state, self.reached_final = fs, fst, reached

    g = synth.random_wfst(9, 300, 1200, 12, eps_fraction=0.06, final_fraction=0.2)
    posts = [synth.random_posteriors(70 + i, 20 + 4 * i, 12) for i in range(4)]
    cfg = P.DecodeConfig(beam=7.0, max_active=40, mode="fsd")
    recs = [Protocol() for _ in posts]
    P.decode_batch(g, posts, cfg, recorder=recs)
    ours = [L.LatticeRecorder() for _ in posts]
    P.decode_batch(g, posts, cfg, recorder=ours)
    for rec, mine in zip(recs, ours):
        assert [c[1] for c in rec.calls] == list(range(rec.final_step + 1))
        assert _key(L.build_lattice(rec, g)) == _key(L.build_lattice(mine, g))
    builder = P.PipelinedLatticeBuilder(g)
    piped = L.LatticeRecorder(consumer=builder)
    P.decode(g, posts[0], cfg, recorder=piped)
    assert _key(builder.result_from(piped)) == _key(L.build_lattice(ours[0], g))
