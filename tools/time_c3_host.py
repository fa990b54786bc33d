"""Breakdown of the config-3 host path: decode_host, fetch_lattices, prune_lattices."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1808_00687_b200.decoder import BatchDecoder, DecodeConfig
from paper_1808_00687_b200.lattice import prune_lattices
cfg = bench.CONFIGS["3"]
utts = int(sys.argv[1]) if len(sys.argv) > 1 else cfg["utts"]
g, L1, T, off, R = bench.make_workload(cfg, 0, utts, cfg["frames"])
costs = torch.empty((R, L1), dtype=torch.float64, pin_memory=True)
blank = torch.empty(R, dtype=torch.float64, pin_memory=True)
bench.fill_inputs(cfg, 0, T, off, L1, costs.numpy(), blank.numpy())
dcfg = DecodeConfig(beam=cfg["beam"], max_active=cfg["max_active"], mode="fsd")
dec = BatchDecoder(g, 0, max_utts_in_flight=148)
for it in range(3):
    t0 = time.perf_counter()
    out = dec.decode_host(costs.numpy(), off, T, blank.numpy(), dcfg, "fsd", lattice=True)
    t1 = time.perf_counter()
    lats = dec.fetch_lattices(g)
    t2 = time.perf_counter()
    pr = prune_lattices(lats, 8.0)
    t3 = time.perf_counter()
    pr1 = prune_lattices(lats, 8.0, max_workers=1)
    t4 = time.perf_counter()
    print(f"decode_host {1e3*(t1-t0):.1f} ms (kernel {dec.last_kernel_ms():.1f})  fetch {1e3*(t2-t1):.1f}  "
          f"prune(threads={len(os.sched_getaffinity(0))}) {1e3*(t3-t2):.1f}  prune(1 thread) {1e3*(t4-t3):.1f}", flush=True)
