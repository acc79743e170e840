"""Throughput of consecutive encode+decode steps on one stream vs two streams with
double-buffered payloads (step i's decode overlaps step i+1's encode)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_11608_b200 as sif

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
kind, N, K, B, dt = {"c2": (0, 1024, 196, 256, torch.float32), "c3": (1, 1, 4096, 1024, torch.bfloat16),
                     "c4": (1, 2048, 4096, 32, torch.bfloat16)}[cfgname]
xs = torch.empty((B, N, K), dtype=dt, device="cuda")
for i in range(B):
    sif.synthetic(kind, N, K, i, out=xs[i])
cfg = sif.CodecConfig(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
pairs = []
for _ in range(2):
    enc = sif.BatchEncoder(xs, cfg, list(range(B))).run().check()
    lens = enc.out_len.cpu().numpy()
    dec = sif.BatchDecoder([enc.out.data_ptr() + i * enc.cap for i in range(B)], lens, N, K)
    dec.run().check()
    pairs.append((enc, dec))
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
graphs = []
for (enc, dec), st in zip(pairs, streams):
    with torch.cuda.stream(st):
        graphs.append(sif.capture_graph(lambda e=enc, d=dec: (e.run(), d.run())))
torch.cuda.synchronize()


def run(nsteps, two):
    cur = torch.cuda.current_stream()
    for st in streams:
        st.wait_stream(cur)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(cur)
    for st in streams:
        st.wait_stream(cur)
    for i in range(nsteps):
        k = i % 2 if two else 0
        with torch.cuda.stream(streams[k]):
            graphs[k].replay()
    for st in streams:
        cur.wait_stream(st)
    t1.record(cur)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / nsteps


for two in (False, True, False, True):
    run(5, two)
    print(cfgname, "two streams" if two else "one stream ", f"{run(40, two) * 1e3:.1f} us/step")
