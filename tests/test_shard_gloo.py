"""Multi-rank host logic on CPU (gloo, world size 2): the stream partition used by the
multi-GPU bench (paper_2511_11608_b200/shard.py) covers every stream exactly once, balances
bytes, and per-rank results are independent of placement (each rank encodes its own streams
with the CPU oracle; the gathered payload digests equal a single-process run)."""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_11608_b200 import shard

SMALL_MIX = {(1, 1, 4096, 2): (1, 1, 64, 2), (0, 1024, 196, 4): (0, 32, 16, 4), (1, 256, 4096, 2): (1, 8, 64, 2)}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _digest(sid, kind, rows, cols):
    from oracle import sif_oracle as O
    from oracle.synth import synth

    x = synth(kind, rows, cols, sid)
    blob = O.encode_bytes(x, O.Cfg(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01), sid)
    return hashlib.sha256(blob).hexdigest()


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mix = [SMALL_MIX[s] for s in shard.mixed_workload(n)]
    mine = shard.shard_streams([(r, c, b) for _, r, c, b in mix], world, rank)
    res = {i: _digest(i, mix[i][0], mix[i][1], mix[i][2]) for i in mine}
    out = [None] * world
    dist.all_gather_object(out, res)
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def test_partition_round_robin_and_lpt():
    assert shard.round_robin(10, 4, 1) == [1, 5, 9]
    parts = shard.lpt([5, 4, 3, 3, 3, 2, 2, 1], 3)
    assert sorted(i for p in parts for i in p) == list(range(8))
    loads = [sum([5, 4, 3, 3, 3, 2, 2, 1][i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= 1
    mix = shard.mixed_workload(8192)
    shapes = [(r, c, b) for _, r, c, b in mix]
    per = [shard.shard_streams(shapes, 8, r) for r in range(8)]
    assert sorted(i for p in per for i in p) == list(range(8192))
    bytes_ = [sum(shapes[i][0] * shapes[i][1] * shapes[i][2] for i in p) for p in per]
    assert max(bytes_) / min(bytes_) < 1.01


def test_gloo_world2_sharded_encode_matches_single_process():
    n = 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    merged = {}
    for d in out:
        assert not set(d) & set(merged), "a stream was assigned to two ranks"
        merged.update(d)
    assert sorted(merged) == list(range(n))
    mix = [SMALL_MIX[s] for s in shard.mixed_workload(n)]
    for i in range(n):
        assert merged[i] == _digest(i, *mix[i][:3]), i
