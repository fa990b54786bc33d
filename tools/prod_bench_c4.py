"""Host producer throughput for config 4 (LSD: gather the non-blank rows, -log in place)."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402
__graft_entry__.build()
from paper_1808_00687_b200 import _native as N, synth  # noqa: E402

n, T, L = 256, 1500, 5000
t = time.perf_counter()
posts = [synth.random_posteriors(i + 1, T, L, blank_fraction=0.8) for i in range(n)]
print("generate %.1f s" % (time.perf_counter() - t))
need = [np.flatnonzero(~(p.rows[:, 0] > 0.98)).astype(np.int32) for p in posts]
R = sum(len(x) for x in need)
crow = np.zeros(n, np.int64)
np.cumsum([len(x) for x in need][:-1], out=crow[1:])
costs = np.empty((R, L + 1))
lib = N.load()
print("rows", R, "cores", len(os.sched_getaffinity(0)))
for bf in (32, 128):
    for nw in (8, 16):
        tasks = [(u, b) for b in range((300 + bf - 1) // bf) for u in range(n)]

        def work(u, b):
            lo, hi = b * bf, min(len(need[u]), (b + 1) * bf)
            if hi <= lo:
                return
            r0 = int(crow[u]) + lo
            idx = need[u][lo:hi]
            src = posts[u].rows
            lib.wb_gather_rows(src.ctypes.data, L + 1, idx.ctypes.data, hi - lo, 1, L,
                               costs[r0:].ctypes.data, L + 1, 1)
            dst = costs[r0:r0 + hi - lo, 1:]
            np.log(dst, out=dst)
            np.multiply(dst, -1.0, out=dst)
            costs[r0:r0 + hi - lo, 0] = np.inf
        t = time.perf_counter()
        with ThreadPoolExecutor(nw) as ex:
            for f in [ex.submit(work, u, b) for u, b in tasks]:
                f.result()
        print(f"block {bf:4d} workers {nw:3d}: {1e3 * (time.perf_counter() - t):7.1f} ms")
