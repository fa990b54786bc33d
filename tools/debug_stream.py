import sys, os, time, faulthandler
faulthandler.dump_traceback_later(100, exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1808_00687_b200 as P
from paper_1808_00687_b200 import synth
INF = float("inf")
for seed in range(12):
    for mode in ("fsd", "lsd"):
        rng = np.random.default_rng(seed)
        S = int(rng.integers(2, 60))
        g = synth.random_wfst(seed, S, int(S * rng.uniform(1, 4)), int(rng.integers(1, 6)),
                              eps_fraction=[0.0, 0.15, 0.3][seed % 3], selfloops=seed % 2 == 0,
                              final_fraction=0.3)
        L = int(g.max_ilabel) or 1
        posts = [synth.random_posteriors(seed * 100 + k, int(rng.integers(0, 12)), L,
                                         blank_fraction=0.3) for k in range(5)]
        for beam, ma in ((INF, None), (4.0, None), (INF, 3), (6.0, 5)):
            print(seed, mode, beam, ma, [p.num_frames for p in posts], flush=True)
            t = time.time()
            P.decode_batch(g, posts, P.DecodeConfig(beam=beam, max_active=ma, mode=mode))
            print("  ok", round(time.time() - t, 3), flush=True)
