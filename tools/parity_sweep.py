"""Parity at the benchmarked sizes, every utterance: the public decode path (decode_batch:
posterior matrices in) on the GPU against the oracle (the C port of decoder.py,
reference-exact mode) on all host threads, all 7 DecodeResult fields.

usage: python tools/parity_sweep.py [configs...]   (default: 2 4 5; config 4 on its first
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


def main():
    ids = sys.argv[1:] or ["2", "4", "5"]
    out = []
    for c in ids:
        n = {"4": int(os.environ.get("WB_SWEEP_C4", 128)), "5": int(os.environ.get("WB_SWEEP_C5", 256))}.get(c)
        out.append(sweep(c, n))
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
