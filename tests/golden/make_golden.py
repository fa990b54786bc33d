"""Generate the golden decode / lattice fixtures by running the Python reference.

Run in the build container (it needs /root/reference):

    python tests/golden/make_golden.py

Writes ``tests/golden/cases.npz`` (graph CSR arrays + float64 cost tables + blank columns,
exactly as the reference scores them) and ``tests/golden/cases.json`` (configs and the
reference's outputs: DecodeResult fields, raw lattice, pruned lattices, lattice best path).
Floats are stored with ``float.hex`` so comparisons are bit-exact.  Instances come from the
reference's own generators and test envelopes:

* ``c1``  -- acceptance criterion 1 envelope (test_acceptance.py:65-83), FSD, beam off
* ``c5``  -- criterion 5 envelope (test_acceptance.py:235-273): FSD/LSD, beam, max-active,
             tie-heavy weight grids
* ``rnd`` -- tests/conftest.py:52-66 envelope with 30% blank frames, LSD, beam 7
* ``lat`` -- criterion 6 envelope (test_acceptance.py:302-348) with lattices
* ``toy`` -- config 1 (1k states / 10k arcs / 50 pdfs, 200 frames, beam 10), decode only
"""
from __future__ import annotations

import dataclasses
import json
import math
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import refutil  # noqa: E402

L = refutil.ref()
INF = math.inf


def fhex(x: float) -> str:
    return float(x).hex()


def graph_arrays(w):
    arcs = w.arcs
    return dict(
        row_ptr=np.asarray(w.arc_offsets, np.int32),
        eps_end=np.asarray(w.eps_split, np.int32),
        dst=np.asarray([a.dst for a in arcs], np.int32),
        ilabel=np.asarray([a.ilabel for a in arcs], np.int32),
        olabel=np.asarray([a.olabel for a in arcs], np.int32),
        weight=np.asarray([a.weight for a in arcs], np.float64),
        final_w=np.asarray([w.final_weight(s) for s in range(w.num_states)], np.float64),
    )


def result_json(r):
    return dict(total_cost=fhex(r.total_cost), olabels=list(r.olabels), ilabels=list(r.ilabels),
                search_steps=r.search_steps, tokens_expanded=r.tokens_expanded,
                reached_final=r.reached_final, died_at_step=r.died_at_step)


def lattice_store(arrays, prefix, lat):
    """Lattice -> npz arrays under ``prefix``; returns the JSON tag ("empty" / "arrays")."""
    if lat.start_id is None:
        return "empty"
    arrays[prefix + "_nodes"] = np.asarray([[n.state, n.step] for n in lat.nodes], np.int32).reshape(-1, 2)
    arrays[prefix + "_arcs_i"] = np.asarray([[a.from_id, a.to_id, a.ilabel, a.olabel, a.tie]
                                             for a in lat.arcs], np.int64).reshape(-1, 5)
    arrays[prefix + "_arcs_f"] = np.asarray([[a.graph_cost, a.acoustic_cost] for a in lat.arcs],
                                            np.float64).reshape(-1, 2)
    arrays[prefix + "_fin_i"] = np.asarray(list(lat.finals.keys()), np.int64)
    arrays[prefix + "_fin_w"] = np.asarray(list(lat.finals.values()), np.float64)
    return "arrays"


PRUNE_BEAMS = (0.0, 0.75, 2.5, 8.0, INF)


def main():
    arrays = {}
    cases = []

    def add(kind, seed, w, p, cfgk, with_lattice):
        idx = len(cases)
        ga = graph_arrays(w)
        for k, v in ga.items():
            arrays[f"{idx}_{k}"] = v
        arrays[f"{idx}_costs"] = refutil.ref_cost_table(p)
        arrays[f"{idx}_blank"] = np.ascontiguousarray(p.rows[:, p.blank_col], np.float64)
        cfg = L.decoder.DecodeConfig(**cfgk)
        rec = L.lattice.LatticeRecorder() if with_lattice else None
        r = L.decoder.decode(w, p, cfg, recorder=rec)
        case = dict(kind=kind, seed=seed, num_states=w.num_states, start=w.start,
                    cfg={k: (fhex(v) if isinstance(v, float) else v) for k, v in cfgk.items()},
                    result=result_json(r))
        if with_lattice:
            try:
                lat = L.lattice.build_lattice(rec, w)
            except L.lattice.LatticeError:
                case["lattice"] = "error"
            else:
                case["lattice"] = lattice_store(arrays, f"{idx}_lat", lat)
                pr = []
                for bi, beam in enumerate(PRUNE_BEAMS):
                    try:
                        pr.append(lattice_store(arrays, f"{idx}_lat_p{bi}",
                                                L.lattice.prune_lattice(lat, beam)))
                    except L.lattice.LatticeError:
                        pr.append("error")
                case["pruned"] = pr
                if not lat.is_empty:
                    c, ol, il = L.lattice.lattice_best_path(lat)
                    case["best_path"] = [fhex(c), list(ol), list(il)]
        cases.append(case)

    for seed in range(200):
        w, p = refutil.oracle_instance(seed)
        add("c1", seed, w, p, dict(mode="fsd", beam=INF, max_active=None), True)
    for seed in range(200):
        w, p, cfgk = refutil.equivalence_instance(seed)
        add("c5", seed, w, p, cfgk, seed % 4 == 0)
    for seed in range(60):
        w, p = refutil.random_instance(seed, blank_fraction=0.3)
        add("rnd", seed, w, p, dict(mode="lsd", beam=7.0, max_active=None), True)
    for seed in range(30):
        rng = random.Random(700 + seed)
        states = rng.randrange(3, 9)
        w = L.fixtures.make_random_wfst(rng, states, num_arcs=rng.randrange(states, 22),
                                        num_labels=3, eps_fraction=0.15 if seed % 2 else 0.0,
                                        selfloops=seed % 3 == 0, final_fraction=0.4)
        p = L.fixtures.make_random_posteriors(rng, rng.randrange(1, 5), 3, blank_fraction=0.3)
        for mode in ("fsd", "lsd"):
            add("lat", seed, w, p, dict(mode=mode, beam=INF, max_active=None), True)
    rng = random.Random(0)
    w = L.fixtures.make_random_wfst(rng, 1000, 10000, 50, selfloops=True, eps_fraction=0.05,
                                    final_fraction=0.05)
    p = L.fixtures.make_random_posteriors(rng, 200, 50)
    add("toy", 0, w, p, dict(mode="fsd", beam=10.0, max_active=None), False)

    np.savez_compressed(os.path.join(HERE, "cases.npz"), **arrays)
    with open(os.path.join(HERE, "cases.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "lsd_wfst 0.1.0",
                   "prune_beams": [fhex(b) for b in PRUNE_BEAMS], "cases": cases}, fh, separators=(",", ":"))
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
