"""Randomised differential test: GPU decode (+ lattices, device-pruned lattices) vs the C oracle
in canonical mode, over random graphs / posteriors / configs.  Usage on the GPU box:
    python tools/stress.py SECONDS [SEED]"""
import os
import sys
import time

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import numpy as np

import paper_1808_00687_b200 as P
from oracle import oracle as O
from paper_1808_00687_b200 import lattice as L
from paper_1808_00687_b200 import synth
from paper_1808_00687_b200.decoder import BatchDecoder

limit = float(sys.argv[1]) if len(sys.argv) > 1 else 300
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t_end = time.time() + limit
it = 0
fails = 0
while time.time() < t_end:
    rng = np.random.default_rng(seed0 * 100003 + it)
    S = int(rng.integers(2, 3000))
    A = int(S * rng.uniform(1, 6))
    labels = int(rng.integers(1, 60))
    g = synth.random_wfst(int(rng.integers(1 << 30)), S, A, labels,
                          eps_fraction=float(rng.choice([0, 0.02, 0.1, 0.3])),
                          selfloops=bool(rng.random() < 0.4),
                          final_fraction=float(rng.uniform(0.01, 0.5)))
    if g.epsilon_cycle() is not None:
        it += 1
        continue
    L1 = int(g.max_ilabel) or 1
    n = int(rng.integers(1, 12))
    posts = [synth.random_posteriors(int(rng.integers(1 << 30)), int(rng.integers(0, 80)), L1,
                                     blank_fraction=float(rng.uniform(0, 0.9)))
             for _ in range(n)]
    mode = str(rng.choice(["fsd", "lsd"]))
    beam = float(rng.choice([np.inf, rng.uniform(0, 12)]))
    ma = None if rng.random() < 0.4 else int(rng.integers(1, 200))
    cfg = P.DecodeConfig(beam=beam, max_active=ma, mode=mode,
                         blank_threshold=float(rng.choice([0.98, 0.5])))
    lattice = rng.random() < 0.5
    lb = float(rng.choice([0.0, 1.0, 4.0, np.inf]))
    # WB_STRESS_CLUSTER=1: random cluster size per batch (lattice batches run one CTA per lane)
    K = int(rng.choice([1, 2, 4, 8])) if os.environ.get("WB_STRESS_CLUSTER") == "1" else 0
    dec = BatchDecoder(g, 0, cluster_ctas=K)
    costs = [P.cost_table(p) for p in posts]
    T = np.asarray([len(c) for c in costs], np.int32)
    off = np.zeros(n, np.int64)
    np.cumsum(T[:-1], out=off[1:])
    C_ = np.concatenate(costs) if T.sum() else np.zeros((1, L1 + 1))
    B_ = np.concatenate([p.rows[:, 0] for p in posts]) if T.sum() else np.zeros(1)
    out = dec.decode_host(C_, off, T, B_, cfg, mode, lattice=lattice,
                          lattice_beam=lb if lattice else None)
    got = out.decode_results()
    pr = dec.fetch_pruned_lattices(g, lb) if lattice else None
    for i, (c, p) in enumerate(zip(costs, posts)):
        kw = dict(beam=beam, max_active=ma, mode=mode, blank_threshold=cfg.blank_threshold,
                  canonical=True)
        try:
            if lattice:
                o, olat = O.decode(g, c, p.rows[:, 0], return_lattice=True, **kw)
            else:
                o, olat = O.decode(g, c, p.rows[:, 0], **kw), None
        except O.OracleLatticeError:
            o, olat = O.decode(g, c, p.rows[:, 0], **kw), "error"
        r = got[i]
        ok = (r.total_cost, r.olabels, r.ilabels, r.search_steps, r.tokens_expanded,
              r.reached_final, r.died_at_step) == o.astuple()
        if ok and lattice:
            if olat == "error":
                want = "error"
            else:
                try:
                    want = O.prune_lattice(olat, lb).key() if not olat.empty else ("EMPTY",)
                except O.OracleLatticeError:
                    want = "error"
            have = "error" if isinstance(pr[i], L.LatticeError) else pr[i].key()
            ok = have == want
        if not ok:
            fails += 1
            print("MISMATCH it", it, "utt", i, dict(S=S, A=A, labels=labels, mode=mode, beam=beam,
                                                      ma=ma, lattice=lattice, lb=lb), flush=True)
    it += 1
print(f"stress: {it} batches, {fails} mismatches", flush=True)
