"""Drop-in fidelity with the live reference objects (build container; skipped elsewhere):
the recorder protocol (lattice.py:112-135) in both directions, the reference's
PipelinedLatticeBuilder as a consumer and ours fed by the reference decoder, and the
reference's DecodeResult class (decoder.py:97-105) returned when the reference is loaded."""
import math

import numpy as np
import pytest

import refutil
from paper_1808_00687_b200 import _native as N
from paper_1808_00687_b200 import lattice as BL
from paper_1808_00687_b200.decoder import BatchOutput, DecodeResult, result_class
from paper_1808_00687_b200.wfst import Wfst

needs_ref = pytest.mark.skipif(not refutil.HAVE_REF, reason="reference not available")
INF = math.inf


def _instances(n=60):
    for seed in range(n):
        wfst, posts = refutil.random_instance(seed, max_states=14, max_arcs=40, max_frames=7,
                                              eps_fraction=0.2, blank_fraction=0.3,
                                              selfloops=seed % 2 == 0)
        cfg = dict(beam=(INF, 5.0, 2.5)[seed % 3], max_active=(None, 6, 3)[seed % 3],
                   mode="fsd" if seed % 2 else "lsd")
        yield seed, wfst, posts, cfg


@needs_ref
def test_our_recorder_and_builder_driven_by_the_reference_decoder():
    """Our LatticeRecorder takes the reference decoder's protocol calls; our build_lattice and
    our PipelinedLatticeBuilder (fed step by step on its thread) assemble exactly the
    reference's build_lattice."""
    L = refutil.ref()
    n = 0
    for seed, wfst, posts, cfg in _instances():
        c = L.decoder.DecodeConfig(**cfg)
        ref_rec = L.lattice.LatticeRecorder()
        L.decoder.decode(wfst, posts, c, recorder=ref_rec)
        try:
            want = L.lattice.build_lattice(ref_rec, wfst)
        except L.lattice.LatticeError:
            want = "error"
        mine_rec = BL.LatticeRecorder()
        L.decoder.decode(wfst, posts, c, recorder=mine_rec)
        builder = BL.PipelinedLatticeBuilder(wfst)
        piped_rec = BL.LatticeRecorder(consumer=builder)
        L.decoder.decode(wfst, posts, c, recorder=piped_rec)
        for get in (lambda: BL.build_lattice(mine_rec, wfst), lambda: builder.result_from(piped_rec)):
            try:
                got = get()
            except BL.LatticeError:
                got = "error"
            if want == "error" or got == "error":
                assert got == want, seed
            else:
                assert got == want, seed
                n += 1
    assert n > 50


@needs_ref
def test_replay_into_the_reference_recorder_rebuilds_the_lattice():
    """replay() (what decode does for a foreign recorder) drives the reference's own
    LatticeRecorder -- and through it the reference's PipelinedLatticeBuilder -- so that the
    reference's build_lattice returns the decoded lattice unchanged."""
    L = refutil.ref()
    n = 0
    for seed, wfst, posts, cfg in _instances():
        rec = L.lattice.LatticeRecorder()
        res = L.decoder.decode(wfst, posts, L.decoder.DecodeConfig(**cfg), recorder=rec)
        try:
            lat = L.lattice.build_lattice(rec, wfst)
        except L.lattice.LatticeError:
            continue
        mine = BL.Lattice.from_reference(lat)
        again = L.lattice.LatticeRecorder()
        BL.replay(mine, again, rec.final_step, rec.final_state, rec.reached_final)
        assert L.lattice.build_lattice(again, wfst) == lat, seed
        builder = L.lattice.PipelinedLatticeBuilder(wfst)
        piped = L.lattice.LatticeRecorder(consumer=builder)
        BL.replay(mine, piped, rec.final_step, rec.final_state, rec.reached_final)
        assert builder.result_from(piped) == lat, seed
        assert (again.final_step, again.final_state, again.reached_final) == \
            (rec.final_step, rec.final_state, res.reached_final)
        n += 1
    assert n > 40


@needs_ref
def test_results_are_the_reference_class_when_it_is_loaded():
    L = refutil.ref()
    assert result_class() is L.decoder.DecodeResult
    r = np.zeros(1, dtype=N.UTT_RESULT_DTYPE)
    r["total_cost"], r["search_steps"], r["tokens_expanded"] = 1.5, 3, 7
    r["reached_final"], r["died_at_step"], r["n_olabels"], r["n_ilabels"] = 1, -1, 2, 1
    ol = np.array([[4, 5]], np.int32)
    il = np.array([[9, 0]], np.int32)
    got = BatchOutput(r, ol, il, 2).decode_result(0)
    want = L.decoder.DecodeResult(total_cost=1.5, olabels=(4, 5), ilabels=(9,), search_steps=3,
                                  tokens_expanded=7, reached_final=True, died_at_step=None)
    assert type(got) is L.decoder.DecodeResult and got == want


def test_decode_rejects_objects_without_the_recorder_protocol():
    from paper_1808_00687_b200 import decode_batch, synth
    from paper_1808_00687_b200.decoder import DecodeConfig
    g = synth.random_wfst(1, 20, 40, 3)
    p = synth.random_posteriors(1, 4, 3)
    with pytest.raises(TypeError):
        decode_batch(g, [p], DecodeConfig(), recorder=[object()])
    assert result_class() in (DecodeResult, getattr(__import__("sys").modules.get(
        "lsd_wfst.decoder"), "DecodeResult", None))
