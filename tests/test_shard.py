"""Utterance sharding on CPU: the partition, and a world-size-2 gloo run of
decode_sharded whose gathered results equal a single-process decode (decode_fn = the oracle,
used here only as a deterministic stand-in decoder for the plumbing)."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1808_00687_b200.shard import shard_utterances


def test_partition_is_complete_and_balanced():
    rng = np.random.default_rng(0)
    lengths = rng.integers(10, 1000, size=257).tolist()
    for world in (1, 2, 3, 8):
        parts = shard_utterances(lengths, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(lengths)))
        loads = [sum(lengths[i] for i in p) for p in parts]
        assert max(loads) - min(loads) <= max(lengths)
        assert all(p == sorted(p) for p in parts)
    assert shard_utterances([], 4) == [[], [], [], []]
    with pytest.raises(ValueError):
        shard_utterances([1], 0)


def _oracle_decode(wfst, posts, cfg):
    from oracle import oracle as O
    from paper_1808_00687_b200.posteriors import cost_table
    return [O.decode(wfst, cost_table(p), p.rows[:, 0], beam=cfg.beam,
                     max_active=cfg.max_active, mode=cfg.mode).astuple() for p in posts]


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import torch.distributed as dist
    from paper_1808_00687_b200 import synth
    from paper_1808_00687_b200.decoder import DecodeConfig
    from paper_1808_00687_b200.shard import decode_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = synth.random_wfst(2, 200, 800, 10, eps_fraction=0.05, final_fraction=0.1)
        posts = [synth.random_posteriors(i, 5 + 3 * i, 10) for i in range(9)]
        cfg = DecodeConfig(beam=8.0, max_active=30, mode="fsd")
        got = decode_sharded(g, posts, cfg, decode_fn=_oracle_decode)
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_matches_single_process():
    import socket
    from paper_1808_00687_b200 import synth
    from paper_1808_00687_b200.decoder import DecodeConfig
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = synth.random_wfst(2, 200, 800, 10, eps_fraction=0.05, final_fraction=0.1)
    posts = [synth.random_posteriors(i, 5 + 3 * i, 10) for i in range(9)]
    want = _oracle_decode(g, posts, DecodeConfig(beam=8.0, max_active=30, mode="fsd"))
    assert out[0] == want and out[1] == want


def _gpu_worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import torch
    import torch.distributed as dist
    from paper_1808_00687_b200 import synth
    from paper_1808_00687_b200.decoder import DecodeConfig
    from paper_1808_00687_b200.shard import decode_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)   # one GPU here: both ranks decode on it (independent kernels)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = synth.random_wfst(3, 3000, 9000, 20, eps_fraction=0.05, final_fraction=0.1)
        posts = [synth.random_posteriors(50 + i, 20 + 9 * i, 20) for i in range(11)]
        cfg = DecodeConfig(beam=9.0, max_active=200, mode="fsd")
        got = decode_sharded(g, posts, cfg)   # the real device decoder on each rank's shard
        q.put((rank, [tuple(r.__dict__.values()) if hasattr(r, "__dict__") else r for r in got]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world2_device_decode_gather(cuda):
    """Two ranks (processes) shard the utterances, each decodes its share with the B200
    decoder, and the gloo gather gives every rank the full batch -- equal to the oracle."""
    import socket
    from oracle import oracle as O
    from paper_1808_00687_b200 import synth
    from paper_1808_00687_b200.posteriors import cost_table
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = synth.random_wfst(3, 3000, 9000, 20, eps_fraction=0.05, final_fraction=0.1)
    posts = [synth.random_posteriors(50 + i, 20 + 9 * i, 20) for i in range(11)]
    want = [O.decode(g, cost_table(p), p.rows[:, 0], beam=9.0, max_active=200,
                     mode="fsd").astuple() for p in posts]
    assert out[0] == want and out[1] == want
