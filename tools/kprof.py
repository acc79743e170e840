"""Per-kernel times (CUDA events around each library launch) of one encode+decode of a
synthetic batch:  python tools/kprof.py KIND N K B DTYPE [key=value codec options...]
e.g.  python tools/kprof.py 1 2048 4096 32 bf16 s=0.9 lam=0.1"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_11608_b200 as sif

kind, N, K, B = (int(v) for v in sys.argv[1:5])
dt = torch.bfloat16 if sys.argv[5] == "bf16" else torch.float32
kw = dict(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
for a in sys.argv[6:]:
    k, v = a.split("=")
    kw[k] = float(v) if k in ("s", "lam", "delta") else int(v)
xs = torch.empty((B, N, K), dtype=dt, device="cuda")
for i in range(B):
    sif.synthetic(kind, N, K, i, out=xs[i])
enc = sif.BatchEncoder(xs, sif.CodecConfig(**kw), list(range(B)))
dec = sif.decoder_for(enc)
for _ in range(2):
    enc.run(); dec.run()
torch.cuda.synchronize()
L = sif._lib.load()
L.sif_profile_enable(1)
enc.run(); dec.run()
torch.cuda.synchronize()
L.sif_profile_enable(0)
ms = (ctypes.c_double * 64)(); cnt = (ctypes.c_int32 * 64)()
nk = L.sif_profile_read(ms, cnt, 64)
tot = 0.0
for k in range(max(0, nk)):
    if cnt[k]:
        tot += ms[k]
        print(f"{L.sif_profile_kernel_name(k).decode():22s} {ms[k] * 1e3:10.1f} us  x{cnt[k]}")
print(f"{'total':22s} {tot * 1e3:10.1f} us   codec {kw}")
enc.check(); dec.check()
