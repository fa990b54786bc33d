import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_1808_00687_b200 as P
from paper_1808_00687_b200 import synth, _native as N
from paper_1808_00687_b200.decoder import BatchDecoder, _native_config
cap, arena, lab = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = synth.random_wfst(8, 2000, 7000, 30, eps_fraction=0.05, final_fraction=0.1)
posts = [synth.random_posteriors(70 + k, 60, 30) for k in range(5)]
T = np.asarray([p.num_frames for p in posts], np.int32)
off = np.zeros(len(T), np.int64); np.cumsum(T[:-1], out=off[1:])
costs = np.concatenate([P.cost_table(p) for p in posts])
blank = np.concatenate([p.rows[:, 0] for p in posts])
cfg = P.DecodeConfig(beam=9.0, max_active=150, mode="fsd")
dec = BatchDecoder(g, 0, cand_capacity=cap, arena_capacity=arena, max_frames=64)
res = np.zeros(len(T), dtype=N.UTT_RESULT_DTYPE)
ol = np.zeros((len(T), max(lab, 1)), np.int32); il = ol.copy()
rc = N.load().wb_decode(dec._h, len(T), costs.ctypes.data, off.ctypes.data, T.ctypes.data,
                        costs.shape[1], blank.ctypes.data, C.byref(_native_config(cfg, "fsd")),
                        res.ctypes.data, ol.ctypes.data, il.ctypes.data, lab, N.WB_MEM_HOST, None)
print(cap, arena, lab, "rc", rc, N.load().wb_last_error(), res["status"].tolist(), res["capacity_flags"].tolist(), res["n_olabels"].tolist())
