"""Small driver for ncu: one encode + one decode launch of the C2 batch (after warm-up)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_11608_b200 as sif

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
conf = {"c2": (0, 1024, 196, 256, torch.float32), "c3": (1, 1, 4096, 1024, torch.bfloat16),
        "c4": (1, 2048, 4096, 32, torch.bfloat16)}[cfgname]
kind, N, K, B, dt = conf
xs = torch.empty((B, N, K), dtype=dt, device="cuda")
for i in range(B):
    sif.synthetic(kind, N, K, i, out=xs[i])
cfg = sif.CodecConfig(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
enc = sif.BatchEncoder(xs, cfg, list(range(B))).run().check()
lens = enc.out_len.cpu().numpy()
dec = sif.BatchDecoder([enc.out.data_ptr() + i * enc.cap for i in range(B)], lens, N, K).run().check()
for _ in range(int(os.environ.get("REPS", "2"))):
    enc.run(); dec.run()
torch.cuda.synchronize()
print("ok")
