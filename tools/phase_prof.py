"""Per-phase encode timings (globaltimer stamps written by the kernel when SIF_PROF_PTR is set)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_11608_b200 as sif

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
B_override = int(os.environ.get("PROF_B", "0"))
kind, N, K, B, dt = {"c2": (0, 1024, 196, 256, torch.float32), "c3": (1, 1, 4096, 1024, torch.bfloat16),
                     "c4": (1, 2048, 4096, 32, torch.bfloat16)}[cfgname]
B = B_override or B
xs = torch.empty((B, N, K), dtype=dt, device="cuda")
for i in range(B):
    sif.synthetic(kind, N, K, i, out=xs[i])
cfg = sif.CodecConfig(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
prof = torch.zeros(B * 32, dtype=torch.int64, device="cuda")
os.environ["SIF_PROF_PTR"] = str(prof.data_ptr())
enc = sif.BatchEncoder(xs, cfg, list(range(B)))
for _ in range(3):
    enc.run()
torch.cuda.synchronize()
enc.check()
p = prof.cpu().numpy().reshape(B, 32).astype(np.float64)
names = ["sample", "stream", "select", "-", "kept", "-", "ms_cuts", "members", "minmax", "abq", "layout",
         "header", "rowptr", "pack", "crc", "end"]
p[:, 3] = p[:, 2]
p[:, 5] = p[:, 4]
d = np.diff(p[:, :16], axis=1) / 1e3  # us
print(f"{cfgname}: per-IF phase means (us) over {B} IFs; IF total {np.mean(p[:,15]-p[:,0])/1e3:.1f} us; "
      f"kernel span {(p[:,15].max()-p[:,0].min())/1e3:.1f} us")
for i in range(15):
    print(f"  {names[i]:8s} {d[:, i].mean():9.2f}  (max {d[:, i].max():.2f})")
