"""Phase timestamps of enc_select (globaltimer, SIF_PROF_PTR): python tools/phase_prof.py c2|c3|c4"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_11608_b200 as sif

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
kind, N, K, B, dt = {"c2": (0, 1024, 196, 256, torch.float32), "c3": (1, 1, 4096, 1024, torch.bfloat16),
                     "c4": (1, 2048, 4096, 32, torch.bfloat16)}[cfgname]
xs = torch.empty((B, N, K), dtype=dt, device="cuda")
for i in range(B):
    sif.synthetic(kind, N, K, i, out=xs[i])
cfg = sif.CodecConfig(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
prof = torch.zeros(B * 16, dtype=torch.int64, device="cuda")
os.environ["SIF_PROF_PTR"] = str(prof.data_ptr())
enc = sif.BatchEncoder(xs, cfg, list(range(B)))
for _ in range(3):
    enc.run()
torch.cuda.synchronize()
enc.check()
p = prof.cpu().numpy().reshape(B, 16).astype(np.float64)
names = ["restream", "nz/hist", "tau-gather+select", "cls", "kept-counts", "cut-digits+A", "cut-gather", "cut-selects"]
ok = p[:, 8] > 0
print(f"{cfgname}: enc_select phases (us), mean over {ok.sum()} IFs; IF total {np.mean(p[ok,8]-p[ok,0])/1e3:.1f} us")
for i in range(8):
    a, b = p[ok, i], p[ok, i + 1]
    m = (a > 0) & (b > 0)
    if m.any():
        print(f"  {names[i]:18s} {np.mean(b[m]-a[m])/1e3:9.2f}")
