"""Host-side throughput of SURVEY 8(f)'s "next" rows against the reference on this container's
CPU (the reference package is importable here, not on the GPU box):

  f1  lattice text I/O   format_lattice_text / parse_lattice_text (lattice.py:562-627)
  f2  WFST ingestion     parse_wfst_text + CSR build (wfst.py:315-378, :182)
  f3  POST1 ingestion    load_posteriors (posteriors.py:147-217) vs PosteriorBatch

Each row also checks that both sides produce the same result.  Writes one JSON object.
usage: python tools/ingest_bench.py [out.json]
"""
import json
import os
import random
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import refutil  # noqa: E402

from paper_1808_00687_b200 import lattice as L  # noqa: E402
from paper_1808_00687_b200 import posteriors as P  # noqa: E402
from paper_1808_00687_b200 import synth  # noqa: E402
from paper_1808_00687_b200 import wfst as W  # noqa: E402


def timed(fn, *a, **k):
    t = time.perf_counter()
    r = fn(*a, **k)
    return r, time.perf_counter() - t


def lattice_row(R, steps=1000, per_step=374, seed=0):
    """A config-3-sized trimmed lattice (~374 nodes per step after trim)."""
    rng = random.Random(seed)
    nodes, arcs = [], []
    for k in range(steps + 1):
        for j in range(per_step):
            nodes.append(R.lattice.LatticeNode(rng.randrange(1_000_000), k))   # (state, step)
    for k in range(1, steps + 1):
        for j in range(per_step):
            dst = k * per_step + j
            for _ in range(2):
                src = (k - 1) * per_step + rng.randrange(per_step)
                g, a = round(rng.uniform(0, 3), 6), rng.uniform(0, 20)
                arcs.append(R.lattice.LatticeArc(src, dst, rng.randrange(1, 3000), rng.randrange(1, 3000), g, a))
    finals = {steps * per_step + j: round(rng.uniform(0, 3), 6) for j in range(5)}
    ref = R.lattice.Lattice(nodes=tuple(nodes), arcs=tuple(arcs), start_id=0, finals=finals)
    ours = L.Lattice.from_reference(ref)
    want, t_ref_w = timed(R.lattice.format_lattice_text, ref)
    got, t_w = timed(L.format_lattice_text, ours)
    assert got == want
    back_ref, t_ref_p = timed(R.lattice.parse_lattice_text, want)
    back, t_p = timed(L.parse_lattice_text, want)
    assert back == back_ref
    mb = len(want) / 1e6
    return {"lattice": f"{len(nodes)} nodes, {len(arcs)} arcs, {mb:.1f} MB of text",
            "format_s": {"reference": round(t_ref_w, 3), "ours": round(t_w, 3),
                         "speedup": round(t_ref_w / t_w, 1)},
            "parse_s": {"reference": round(t_ref_p, 3), "ours": round(t_p, 3),
                        "speedup": round(t_ref_p / t_p, 1)},
            "identical": True}


def wfst_row(R, states=1_000_000, arcs=3_000_000):
    g = synth.hclg_like(0, states, arcs, 3000)
    text = W.format_wfst_text(g)
    ours, t = timed(W.parse_wfst_text, text)
    ref, t_ref = timed(R.wfst.parse_wfst_text, text)
    same = (ours.num_states == ref.num_states and ours.start == ref.start
            and np.array_equal(ours.dst, np.fromiter((a.dst for a in ref.arcs), np.int32, len(ref.arcs)))
            and np.array_equal(ours.ilabel, np.fromiter((a.ilabel for a in ref.arcs), np.int32, len(ref.arcs))))
    return {"graph": f"config-2 graph text: {states} states, {arcs} arcs, {len(text) / 1e6:.0f} MB",
            "parse_and_csr_s": {"reference": round(t_ref, 3), "ours": round(t, 3),
                                "speedup": round(t_ref / t, 1)},
            "same_csr": bool(same)}


def post1_row(R, n=16, frames=1000, labels=3000):
    d = tempfile.mkdtemp()
    paths = []
    for i in range(n):
        m = synth.random_posteriors(i + 1, frames, labels)
        pth = os.path.join(d, f"u{i}.post")
        P.save_posteriors(m, pth, binary=True)
        paths.append(pth)
    refs, t_ref = timed(lambda: [R.posteriors.load_posteriors(p) for p in paths])
    batch, t = timed(P.PosteriorBatch, paths)
    ok = all(np.array_equal(np.asarray(r.rows, dtype=np.float64).reshape(frames, labels + 1),
                            batch.table[o:o + frames]) for r, o in zip(refs, batch.offsets))
    gb = n * frames * (labels + 1) * 8 / 1e9
    for p in paths:
        os.unlink(p)
    return {"files": f"{n} POST1 files x {frames} frames x {labels + 1} columns ({gb:.2f} GB)",
            "read_s": {"reference": round(t_ref, 3), "ours": round(t, 3),
                       "speedup": round(t_ref / t, 1)},
            "ours_gb_per_s": round(gb / t, 2), "identical": bool(ok),
            "note": "ours: native reader straight into the batch table (page-locked on a GPU "
                    "host; pageable here, no GPU)"}


def main():
    R = refutil.ref()
    # one-time costs (library load, page-locked allocator) outside the timed calls
    W.parse_wfst_text("0 1 1 1 0.5\n1\n")
    L.parse_lattice_text(L.format_lattice_text(L.Lattice.from_reference(
        R.lattice.Lattice(nodes=(R.lattice.LatticeNode(0, 0),), arcs=(), start_id=0, finals={0: 0.0}))))
    d = tempfile.mkdtemp()
    P.save_posteriors(synth.random_posteriors(1, 3, 4), os.path.join(d, "w.post"), binary=True)
    P.PosteriorBatch([os.path.join(d, "w.post")])
    out = {"host": f"{os.cpu_count()} cores (this container's CPU; the reference is not on the GPU box)",
           "f1_lattice_text": lattice_row(R), "f3_post1": post1_row(R), "f2_wfst_text": wfst_row(R)}
    s = json.dumps(out, indent=1)
    print(s)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(s + "\n")


if __name__ == "__main__":
    main()
