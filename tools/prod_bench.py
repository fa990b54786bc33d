"""Host producer throughput of the streaming posterior path (numpy -log into a page-locked
table, frame-block tasks on a thread pool) without the kernel: is the host the bound?"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1808_00687_b200 import synth  # noqa: E402
from paper_1808_00687_b200.posteriors import cost_rows  # noqa: E402

n, T, L = 64, 1000, 3000
posts = [synth.random_posteriors(i + 1, T, L) for i in range(n)]
costs = np.empty((n * T, L + 1))
print("cores", len(os.sched_getaffinity(0)))
t = time.perf_counter()
np.log(posts[0].rows)
print("one utterance np.log: %.1f ms" % (1e3 * (time.perf_counter() - t)))
for bf in (32, 64, 128):
    for nw in (4, 8, 16):
        tasks = [(u, b) for b in range(T // bf) for u in range(n)]

        def work(u, b):
            cost_rows(posts[u], np.arange(b * bf, (b + 1) * bf), costs[u * T:(u + 1) * T], 1.0)
        t = time.perf_counter()
        with ThreadPoolExecutor(nw) as ex:
            for f in [ex.submit(work, u, b) for u, b in tasks]:
                f.result()
        print(f"block {bf:4d} workers {nw:3d}: {1e3 * (time.perf_counter() - t):7.1f} ms")
