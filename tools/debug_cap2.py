import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_1808_00687_b200 as P
from paper_1808_00687_b200 import synth, _native as N
from paper_1808_00687_b200.decoder import BatchDecoder, _native_config
g = synth.random_wfst(8, 2000, 7000, 30, eps_fraction=0.05, final_fraction=0.1)
posts = [synth.random_posteriors(70 + k, 60, 30) for k in range(5)]
T = np.asarray([p.num_frames for p in posts], np.int32)
off = np.zeros(len(T), np.int64); np.cumsum(T[:-1], out=off[1:])
costs = np.concatenate([P.cost_table(p) for p in posts])
blank = np.concatenate([p.rows[:, 0] for p in posts])
cfg = P.DecodeConfig(beam=9.0, max_active=150, mode="fsd")
mode = sys.argv[1]
if mode == "want":
    print(BatchDecoder(g, 0).decode_host(costs, off, T, blank, cfg, "fsd").results["status"])
tiny = BatchDecoder(g, 0, cand_capacity=16, arena_capacity=1024)
orig = tiny._grow
def grow(flags, **kw):
    print("grow", flags, {k: tiny.opts[k] for k in ("cand_capacity", "arena_capacity")}, flush=True)
    orig(flags, **kw)
    print("  ->", {k: tiny.opts[k] for k in ("cand_capacity", "arena_capacity")}, flush=True)
tiny._grow = grow
out = tiny.decode_host(costs, off, T, blank, cfg, "fsd", label_capacity=1)
print("done", out.results["status"])
