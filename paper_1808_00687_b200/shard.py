"""Utterance sharding over GPUs.

Utterances are independent (``_search``, decoder.py:302-346 has no cross-utterance state), so
the multi-GPU path is a partition of the utterance list with a graph replica per rank and no
collective on the data path.  One process per GPU (``torch.distributed``, backend "nccl"; any
backend works since the only exchange is the optional final result gather).

``shard_utterances`` balances by frame count (longest-processing-time-first greedy: the
per-utterance decode time is proportional to its search steps), ``decode_sharded`` decodes
this rank's share through ``decode_batch`` and, if asked, gathers every rank's results back
into the caller's utterance order.
"""
from __future__ import annotations

import heapq
from typing import Callable, Sequence


def shard_utterances(lengths: Sequence[int], world: int) -> list[list[int]]:
    """Partition utterance indices over ``world`` ranks, balancing total frames.  Each
    rank's list is in ascending utterance order; the assignment is deterministic."""
    if world < 1:
        raise ValueError(f"world size must be >= 1, got {world}")
    order = sorted(range(len(lengths)), key=lambda i: (-int(lengths[i]), i))
    heap = [(0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + int(lengths[i]), r))
    return [sorted(x) for x in out]


def decode_sharded(wfst, posts_list, cfg, *, rank: int | None = None, world: int | None = None,
                   group=None, gather: bool = True,
                   decode_fn: Callable | None = None) -> list:
    """Decode this rank's share of ``posts_list``; with ``gather`` every rank returns the full
    result list in input order (``all_gather_object`` over ``group``).  ``decode_fn`` defaults
    to ``decode_batch`` on the current device."""
    import torch.distributed as dist
    if decode_fn is None:
        from .decoder import decode_batch as decode_fn
    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    posts_list = list(posts_list)
    shards = shard_utterances([p.num_frames for p in posts_list], world)
    mine = shards[rank]
    local = decode_fn(wfst, [posts_list[i] for i in mine], cfg) if mine else []
    if not gather or world == 1:
        return list(local) if world == 1 else list(zip(mine, local))
    parts: list = [None] * world
    dist.all_gather_object(parts, list(zip(mine, local)), group=group)
    out: list = [None] * len(posts_list)
    for part in parts:
        for i, r in part:
            out[i] = r
    return out


def decode_multi_device(wfst, posts_list, cfg, devices, mode: str | None = None) -> list:
    """One process, one host thread per device: utterances are balanced over
    ``devices`` by frame count, each thread drives its own graph replica and decoder through
    the C ABI (ctypes releases the GIL, so the devices run concurrently), results come back
    in input order.  A device may be listed twice (two decoders share it)."""
    import threading
    import torch
    from .decoder import BatchDecoder, as_wfst
    w = as_wfst(wfst)
    posts_list = list(posts_list)
    devices = list(devices)
    shards = shard_utterances([p.num_frames for p in posts_list], len(devices))
    out: list = [None] * len(posts_list)
    errors: list = []

    def run(k, dev):
        try:
            torch.cuda.set_device(dev)
            if not shards[k]:
                return
            dec = BatchDecoder(w, dev)
            res = dec.decode_posteriors([posts_list[i] for i in shards[k]], cfg,
                                        mode or cfg.mode).decode_results()
            for i, r in zip(shards[k], res):
                out[i] = r
        except BaseException as exc:  # re-raised in the caller
            errors.append(exc)
    threads = [threading.Thread(target=run, args=(k, d)) for k, d in enumerate(devices)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out


__all__ = ["decode_multi_device", "decode_sharded", "shard_utterances"]
