"""Debug aid: one synthetic stream (kind, rows, cols, sid) through the GPU encoder, alone
and inside a ListEncoder batch of other streams, compared block by block with the oracle.
    python tools/dbg_stream.py KIND ROWS COLS SID [batch sids...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2511_11608_b200 as sif
from oracle import sif_oracle as O
from oracle.synth import synth

kind, rows, cols, sid = (int(v) for v in sys.argv[1:5])
others = [int(v) for v in sys.argv[5:]]
BASE = dict(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
x = synth(kind, rows, cols, sid)
ref = O.encode_bytes(x, O.Cfg(**BASE), sid)
dt = torch.bfloat16 if kind == 1 else torch.float32


def diff(blob):
    if blob == ref:
        return "identical"
    ea, eb = O.deserialize(blob), O.deserialize(ref)
    out = []
    for i, (u, v) in enumerate(zip(ea.blocks_plus + ea.blocks_minus, eb.blocks_plus + eb.blocks_minus)):
        for f in ("q", "o", "v_min", "nnz"):
            if getattr(u, f) != getattr(v, f):
                out.append(f"block{i}.{f}: gpu {getattr(u, f)} ref {getattr(v, f)}")
        for f in ("row_ptr", "cols", "codes"):
            a, b = getattr(u, f), getattr(v, f)
            if a.shape != b.shape:
                out.append(f"block{i}.{f}: shape {a.shape} vs {b.shape}")
            elif not np.array_equal(a, b):
                k = np.flatnonzero(a != b)
                out.append(f"block{i}.{f}: {k.size} differ, first at {k[:5]} gpu {a[k[:5]]} ref {b[k[:5]]}")
    return "; ".join(out) or "header/CRC differ"


p = sif.encode(torch.from_numpy(x).cuda().to(dt), sif.CodecConfig(**BASE), seed=sid)
print("alone:", diff(p.to_bytes()))
mix = sif.shard.mixed_workload(8192)
xs, seeds = [], []
for o in others + [sid]:
    k, r, c, b = mix[o] if o != sid else (kind, rows, cols, 2 if kind == 1 else 4)
    t = torch.empty((r, c), dtype=torch.float32 if b == 4 else torch.bfloat16, device="cuda")
    sif.synthetic(k, r, c, o, out=t)
    xs.append(t)
    seeds.append(o)
if others:
    ps = sif.encode_list(xs, sif.CodecConfig(**BASE), seeds)
    print("in batch of", len(xs), ":", diff(ps[-1].to_bytes()))
