"""Partition of independent IF streams over ranks.

The codec is per-IF pure: a payload depends only on (x, cfg, seed) (atkf.py:44,
codec.py:186), never on batch composition or placement.  Multi-GPU runs therefore shard
streams (clients / requests) across ranks with no collective on the data path:

* homogeneous batches: round-robin by stream index (rank r gets i = r, r+W, ...);
* mixed shapes (BASELINE config "8192 mixed streams"): longest-processing-time first by
  HBM bytes (T * bytes per element), so each rank moves about the same number of bytes.

`shard_streams` is deterministic, so every rank computes the same assignment without
communicating.
"""

from __future__ import annotations

import heapq


def round_robin(n: int, world: int, rank: int) -> list[int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return list(range(rank, n, world))


def lpt(costs, world: int) -> list[list[int]]:
    """Longest-processing-time greedy: streams in decreasing cost (ties by index) go to the
    currently lightest rank (ties by rank id).  Returns the stream indices of every rank,
    each list in increasing stream order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-int(costs[i]), i))
    heap = [(0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + int(costs[i]), r))
    return [sorted(x) for x in out]


def shard_streams(shapes, world: int, rank: int) -> list[int]:
    """Stream indices owned by `rank`.  shapes: list of (rows, cols, bytes_per_element)."""
    if not shapes:
        return []
    if len({tuple(s) for s in shapes}) == 1:
        return round_robin(len(shapes), world, rank)
    costs = [int(r) * int(c) * int(b) for r, c, b in shapes]
    return lpt(costs, world)[rank]


def mixed_workload(n: int):
    """The BASELINE.json 'multi-device stress' mix: by sid mod 8,
    0-3 -> LLM decode token 1x4096 bf16, 4-6 -> ResNet IF 1024x196 fp32, 7 -> prefill
    chunk 256x4096 bf16.  Returns (kind, rows, cols, bytes_per_element) per sid."""
    out = []
    for sid in range(n):
        m = sid % 8
        if m <= 3:
            out.append((1, 1, 4096, 2))
        elif m <= 6:
            out.append((0, 1024, 196, 4))
        else:
            out.append((1, 256, 4096, 2))
    return out
