"""Phase timestamps (globaltimer, SIF_PROF_PTR) of enc_fused (and enc_select):
    python tools/phase_prof.py c2|c3|c4 [fused_min fused_max] [lam=X]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2511_11608_b200 as sif

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
lam = 0.0
args = [a for a in sys.argv[2:] if not a.startswith("lam=")]
for a in sys.argv[2:]:
    if a.startswith("lam="):
        lam = float(a[4:])
if len(args) >= 2:
    sif._lib.load().sif_set_fused_range(int(args[0]), int(args[1]))
kind, N, K, B, dt = {"c2": (0, 1024, 196, 256, torch.float32), "c3": (1, 1, 4096, 1024, torch.bfloat16),
                     "c4": (1, 2048, 4096, 32, torch.bfloat16)}[cfgname]
xs = torch.empty((B, N, K), dtype=dt, device="cuda")
for i in range(B):
    sif.synthetic(kind, N, K, i, out=xs[i])
cfg = sif.CodecConfig(s=0.9, lam=lam, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
prof = torch.zeros(B * 32, dtype=torch.int64, device="cuda")
os.environ["SIF_PROF_PTR"] = str(prof.data_ptr())
enc = sif.BatchEncoder(xs, cfg, list(range(B)))
for _ in range(3):
    enc.run()
torch.cuda.synchronize()
enc.check()
p = prof.cpu().numpy().reshape(B, 32).astype(np.float64)
sel = ["restream", "nz/hist", "tau-gather+select", "cls", "kept-counts", "cut-digits+A", "cut-gather", "cut-selects"]
fus = ["load", "select", "minmax", "abq", "layout", "pack", "crc"]
tok = ["load", "tau", "cand+sort", "ties+cuts", "members", "abq+layout", "pack"]
for title, names, i0 in (("enc_select phases", sel, 0), ("enc_post phases", fus, 16), ("enc_token phases", tok, 24)):
    ok = p[:, i0 + len(names)] > 0
    if not ok.any():
        continue
    t0 = p[ok, i0]
    print(f"{cfgname}: {title} (us), mean over {ok.sum()} IFs; IF total "
          f"{np.mean(p[ok, i0 + len(names)] - t0) / 1e3:.1f} us; span of the kernel "
          f"{(p[ok, i0 + len(names)].max() - t0.min()) / 1e3:.1f} us")
    for i, nm in enumerate(names):
        a, b = p[ok, i0 + i], p[ok, i0 + i + 1]
        m = (a > 0) & (b > 0)
        if m.any():
            print(f"  {nm:18s} {np.mean(b[m] - a[m]) / 1e3:9.2f}")
