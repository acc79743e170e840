"""Check whether SM clocks are ramped during short kernels: time the same encode batch
cold, then after a 2 s busy loop, sampling nvidia-smi clocks."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_11608_b200 as sif

def clocks():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,pstate", "--format=csv,noheader"],
                          capture_output=True, text=True).stdout.strip()

B, N, K = 256, 1024, 196
xs = torch.empty((B, N, K), device="cuda")
for i in range(B):
    sif.synthetic(0, N, K, i, out=xs[i])
cfg = sif.CodecConfig(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
enc = sif.BatchEncoder(xs, cfg, list(range(B))).run().check()
torch.cuda.synchronize()
def timed(n=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        enc.run()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
print("idle clocks:", clocks())
print("cold encode ms:", timed(1))
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
t0 = time.time()
while time.time() - t0 < 2.0:
    (a @ a)
torch.cuda.synchronize()
print("after busy clocks:", clocks())
print("warm encode ms:", timed(20))
print("during-encode clocks:", end=" ")
for _ in range(50):
    enc.run()
print(clocks())
torch.cuda.synchronize()
