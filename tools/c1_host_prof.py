"""Where the C1 host-in/host-out round trip (encode(host x) -> decode -> .cpu()) spends its
time: wall-clock per stage over N calls, then a cProfile of the same loop."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2511_11608_b200 as sif  # noqa: E402
from paper_2511_11608_b200 import codec as C  # noqa: E402

N = 200
cfg = sif.CodecConfig(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
g = torch.Generator().manual_seed(0)
xh = torch.randn(1024, 196, generator=g)
xd = xh.cuda()
for _ in range(20):
    sif.decode(sif.encode(xh, cfg, seed=1)).cpu()
torch.cuda.synchronize()


def stage(name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(N):
        r = fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {1e6 * (time.perf_counter() - t) / N:9.1f} us", flush=True)
    return r


stage("h2d x.cuda()", lambda: xh.cuda())
p = stage("encode(device x)", lambda: sif.encode(xd, cfg, seed=1))
stage("encode(host x)", lambda: sif.encode(xh, cfg, seed=1))
stage("decode(p)", lambda: sif.decode(p))
y = sif.decode(p)
stage("y.cpu()", lambda: y.cpu())
stage("round trip host", lambda: sif.decode(sif.encode(xh, cfg, seed=1)).cpu())
stage("stream d2h (from_stream)", lambda: p.payload.buf[: p.payload.nbytes].cpu())
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    sif.decode(sif.encode(xh, cfg, seed=1)).cpu()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
