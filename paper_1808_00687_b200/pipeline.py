"""Pipelined lattice decoding (the reference's ``PipelinedLatticeBuilder``, lattice.py:252-292).

The paper runs lattice work on a second stream so it overlaps decoding; the
reference models that with a consumer thread that integrates step k while the decoder works on
step k+1.  Here the raw lattice is recorded and trimmed inside the decode kernel, so what is
left for the host -- canonical ordering, ``prune_lattice`` and ``lattice_best_path`` -- runs
on a thread pool for batch i while the GPU decodes batch i+1.

    pipe = LatticePipeline(BatchDecoder(wfst), lattice_beam=8.0)
    futs = [pipe.submit(costs, row_offset, num_frames, blank, cfg) for ... in batches]
    for f in futs:
        out, lattices = f.result()      # BatchOutput, [pruned Lattice | LatticeError]
    pipe.close()

One GPU thread owns the decoder (``decode_host`` + ``fetch_lattices`` run back to back, so a
batch's lattice pools are copied out before the next batch overwrites them); ctypes releases
the GIL during both, and the C++ prune releases it too, so host and device work overlap.
"""
from __future__ import annotations

import os
import threading
from concurrent.futures import Future, ThreadPoolExecutor

from .lattice import LatticeError, prune_lattice, split_lattice


class LatticePipeline:
    def __init__(self, decoder, lattice_beam: float | None = None, workers: int | None = None,
                 device_prune: bool = True):
        self.decoder = decoder
        self.lattice_beam = lattice_beam
        # stage one of prune_lattice in the decode launch (prune_kernel); host threads only
        # run the path-exact split
        self.device_prune = device_prune and lattice_beam is not None
        n = workers or max(1, len(os.sched_getaffinity(0)) - 1)
        self._gpu = ThreadPoolExecutor(1, thread_name_prefix="wb-decode")
        self._host = ThreadPoolExecutor(n, thread_name_prefix="wb-lattice")
        self._lock = threading.Lock()

    def _prune(self, lat):
        if isinstance(lat, tuple):       # device stage one done: (lattice, cutoff)
            try:
                return split_lattice(*lat)
            except LatticeError as exc:
                return exc
        if self.lattice_beam is None or isinstance(lat, LatticeError) or lat.start_id is None:
            return lat
        try:
            return prune_lattice(lat, self.lattice_beam)
        except LatticeError as exc:
            return exc

    def _decode(self, costs, row_offset, num_frames, blank, cfg, mode, fut: Future):
        try:
            dec = self.decoder
            if self.device_prune:
                out = dec.decode_host(costs, row_offset, num_frames, blank, cfg, mode or cfg.mode,
                                      lattice=True, lattice_beam=self.lattice_beam)
                lats = dec.fetch_pruned_lattices(dec.graph.wfst, self.lattice_beam, split=False)
            else:
                out = dec.decode_host(costs, row_offset, num_frames, blank, cfg, mode or cfg.mode,
                                      lattice=True)
                lats = dec.fetch_lattices(dec.graph.wfst)
        except BaseException as exc:  # surfaced through the future
            fut.set_exception(exc)
            return
        self._finish_batch(out, lats, fut)

    def _finish_batch(self, out, lats, fut: Future):
        parts = [self._host.submit(self._prune, lat) for lat in lats]

        def finish(_):
            if all(p.done() for p in parts) and not fut.done():
                with self._lock:
                    if not fut.done():
                        fut.set_result((out, [p.result() for p in parts]))
        if not parts:
            fut.set_result((out, []))
        for p in parts:
            p.add_done_callback(finish)

    def _decode_posts(self, posts, cfg, mode, fut: Future):
        try:
            dec = self.decoder
            if self.device_prune:
                out = dec.decode_posteriors(posts, cfg, mode or cfg.mode, lattice=True,
                                            lattice_beam=self.lattice_beam)
                lats = dec.fetch_pruned_lattices(dec.graph.wfst, self.lattice_beam, split=False)
            else:
                out = dec.decode_posteriors(posts, cfg, mode or cfg.mode, lattice=True)
                lats = dec.fetch_lattices(dec.graph.wfst)
        except BaseException as exc:  # surfaced through the future
            fut.set_exception(exc)
            return
        self._finish_batch(out, lats, fut)

    def submit_posteriors(self, posts, cfg, mode: str | None = None) -> Future:
        """Queue one batch given as posterior matrices (``decode_posteriors``)."""
        fut: Future = Future()
        self._gpu.submit(self._decode_posts, list(posts), cfg, mode, fut)
        return fut

    def submit(self, costs, row_offset, num_frames, blank, cfg, mode: str | None = None) -> Future:
        """Queue one batch; the future yields (BatchOutput, lattices)."""
        fut: Future = Future()
        self._gpu.submit(self._decode, costs, row_offset, num_frames, blank, cfg, mode, fut)
        return fut

    def close(self):
        self._gpu.shutdown(wait=True)
        self._host.shutdown(wait=True)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


__all__ = ["LatticePipeline"]
