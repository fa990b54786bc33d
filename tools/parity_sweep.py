"""Parity at the benchmarked sizes, every utterance: the public decode path (decode_batch:
posterior matrices in) on the GPU against the oracle (the C port of decoder.py,
reference-exact mode) on all host threads, all 7 DecodeResult fields.

usage: python tools/parity_sweep.py [configs...]   (default: 2 4 5; config 3 (lattices) on its
       first WB_SWEEP_C3 utterances, default 8; config 4 on its first
       WB_SWEEP_C4 utterances, default 128, config 5 on its first WB_SWEEP_C5, default 256:
       host memory for the posteriors and the oracle's cost tables)   -> one JSON line each
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1808_00687_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1808_00687_b200 import synth  # noqa: E402
from paper_1808_00687_b200.posteriors import PosteriorMatrix, cost_table  # noqa: E402


def sweep(cfg_id: str, utts: int | None = None) -> dict:
    cfg = dict(bench.CONFIGS[cfg_id])
    n = utts or cfg["utts"]
    g, L1, T, off, R = bench.make_workload(cfg, 0, n, cfg["frames"])
    posts = [PosteriorMatrix(synth.random_posterior_rows(i + 1, cfg["frames"], cfg["labels"],
                                                         blank_fraction=cfg["blank_fraction"]),
                             0, validate=False) for i in range(n)]
    dcfg = P.DecodeConfig(beam=cfg["beam"], max_active=cfg["max_active"] or None, mode=cfg["mode"])
    t = time.perf_counter()
    got = P.decode_batch(g, posts, dcfg)
    t_gpu = time.perf_counter() - t
    og = O.OracleGraph(g)
    t = time.perf_counter()
    want = O.decode_batch(og, [cost_table(p) for p in posts], [np.ascontiguousarray(p.rows[:, 0]) for p in posts],
                          beam=cfg["beam"], max_active=cfg["max_active"], mode=cfg["mode"],
                          n_threads=len(os.sched_getaffinity(0)))
    t_cpu = time.perf_counter() - t
    bad = [i for i, (r, o) in enumerate(zip(got, want))
           if (r.total_cost, r.olabels, r.ilabels, r.search_steps, r.tokens_expanded,
               r.reached_final, r.died_at_step) != o.astuple()]
    return {"config": cfg_id, "workload": cfg["name"], "utterances": n, "mismatches": len(bad),
            "mismatched_utts": bad[:20], "gpu_s": round(t_gpu, 2), "oracle_s": round(t_cpu, 2)}


def sweep_lattice(n: int) -> dict:
    """Config 3 at full length: the exact (trimmed) lattices and the device-pruned lattices
    (lattice-beam 8) of n bench utterances against the oracle's build_lattice / prune_lattice."""
    from paper_1808_00687_b200 import lattice as Lt
    from paper_1808_00687_b200.decoder import BatchDecoder
    from concurrent.futures import ThreadPoolExecutor
    cfg = dict(bench.CONFIGS["3"])
    g, L1, T, off, R = bench.make_workload(cfg, 0, n, cfg["frames"])
    posts = [PosteriorMatrix(synth.random_posterior_rows(i + 1, cfg["frames"], cfg["labels"]), 0,
                             validate=False) for i in range(n)]
    costs = np.concatenate([cost_table(p) for p in posts])
    blank = np.concatenate([np.ascontiguousarray(p.rows[:, 0]) for p in posts])
    dcfg = P.DecodeConfig(beam=cfg["beam"], max_active=cfg["max_active"], mode="fsd")
    dec = BatchDecoder(g, 0, max_utts_in_flight=n)
    t = time.perf_counter()
    out = dec.decode_host(costs, off, T, blank, dcfg, "fsd", lattice=True, lattice_beam=cfg["lattice_beam"])
    lats = dec.fetch_lattices(g)
    pruned = dec.fetch_pruned_lattices(g, cfg["lattice_beam"])
    t_gpu = time.perf_counter() - t
    og = O.OracleGraph(g)

    def one(i):
        r, olat = O.decode(og, cost_table(posts[i]), posts[i].rows[:, 0], beam=cfg["beam"],
                           max_active=cfg["max_active"], mode="fsd", return_lattice=True)
        try:
            want = O.prune_lattice(olat, cfg["lattice_beam"]).key()
        except O.OracleLatticeError:
            want = "error"
        return r, olat.key(), want
    t = time.perf_counter()
    with ThreadPoolExecutor(min(n, len(os.sched_getaffinity(0)))) as ex:
        ref = list(ex.map(one, range(n)))
    t_cpu = time.perf_counter() - t
    bad = []
    for i, (r, okey, want) in enumerate(ref):
        x = out.decode_results()[i]
        got = "error" if isinstance(pruned[i], Lt.LatticeError) else pruned[i].key()
        if ((x.total_cost, x.olabels, x.ilabels, x.search_steps, x.tokens_expanded, x.reached_final,
             x.died_at_step) != r.astuple() or lats[i].key() != okey or got != want):
            bad.append(i)
    return {"config": "3", "workload": cfg["name"], "utterances": n, "mismatches": len(bad),
            "mismatched_utts": bad, "compared": "decode fields + trimmed lattice + lattice-beam-8 pruned lattice",
            "raw_lattice_nodes": int(sum(l.num_nodes for l in lats)),
            "gpu_s": round(t_gpu, 2), "oracle_s": round(t_cpu, 2)}


def main():
    ids = sys.argv[1:] or ["2", "4", "5"]
    out = []
    for c in ids:
        if c == "3":
            out.append(sweep_lattice(int(os.environ.get("WB_SWEEP_C3", 8))))
        else:
            n = {"4": int(os.environ.get("WB_SWEEP_C4", 128)), "5": int(os.environ.get("WB_SWEEP_C5", 256))}.get(c)
            out.append(sweep(c, n))
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
