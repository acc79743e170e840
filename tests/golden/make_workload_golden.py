"""Golden digests of the BENCHMARKED workloads, produced by running the REFERENCE.

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_workload_golden.py [--procs 8]

For every IF that `bench.py` times on up to 8 GPUs -- C2 (256 ResNet IFs per GPU, sids
0..2047), C3 (1024 decode tokens per GPU, sids 0..8191), C4 (32 prefill IFs per GPU, sids
0..255), C5 (the 8192 mixed streams, sids 0..8191) -- and for the BASELINE.md §4.2 C4 sweep (s x delta x lambda grid plus
fixed Q=[8,4,2], on the prefill IF of sid 0), the reference's own
`serialize(encode(DenseTensor(x), cfg, sid))` (codec.py:186, :283) and
`decode(deserialize(blob))` (codec.py:320, :254) are run and recorded as
(payload length, sha256[:16] of the payload, sha256[:16] of the decoded fp32 bits).
Inputs come from the integer-exact synthetic generator (`oracle/synth.py`), which is
bit-identical to the device generator the bench uses (`sif_gen_synthetic`).

Output: tests/golden/workloads.npz + tests/golden/workloads.json.  `tests/test_gpu_workloads.py`
checks the GPU codec against these digests for every IF; `bench.py` checks its own timed
payloads against them (`parity` in the JSON line).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

BASE = dict(s=0.9, lam=0.0, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
SWEEP_S = (0.5, 0.7, 0.8, 0.9, 0.95)
SWEEP_DELTA = (0.01, 0.05, 0.1, 0.2)
SWEEP_LAM = (0.0, 0.1)
FIXED_Q = (8, 4, 2)  # per plane, broadcast to M+ + M- = 6 blocks (codec.py:95-105)


def sweep_configs():
    out = []
    for s in SWEEP_S:
        for d in SWEEP_DELTA:
            for lam in SWEEP_LAM:
                out.append(dict(BASE, s=s, delta=d, lam=lam))
    out.append(dict(BASE, mode="fixed_q", fixed_q=FIXED_Q + FIXED_Q))
    return out


def workloads():
    """name -> list of (kind, rows, cols, sid, cfg)."""
    from paper_2511_11608_b200.shard import mixed_workload

    w = {
        # 8 ranks x the per-GPU batch: bench.py gives rank r the sids r*B .. r*B+B-1
        "c2": [(0, 1024, 196, i, BASE) for i in range(8 * 256)],
        "c3": [(1, 1, 4096, i, BASE) for i in range(8 * 1024)],
        "c4": [(1, 2048, 4096, i, BASE) for i in range(8 * 32)],
        "c4sweep": [(1, 2048, 4096, 0, c) for c in sweep_configs()],
        "c5": [(k, r, c, sid, BASE) for sid, (k, r, c, _b) in enumerate(mixed_workload(8192))],
    }
    return w


def _job(args):
    kind, rows, cols, sid, cfgd = args
    import slicer  # the reference
    from slicer import CodecConfig, DenseTensor

    from oracle.synth import synth

    x = synth(kind, rows, cols, sid)
    cfgd = dict(cfgd)
    if "fixed_q" in cfgd:
        cfgd["fixed_q"] = tuple(cfgd["fixed_q"])
    c = slicer.encode(DenseTensor(rows, cols, x), CodecConfig(**cfgd), sid)
    blob = slicer.serialize(c)
    y = slicer.decode(slicer.deserialize(blob))
    dec = np.ascontiguousarray(y.values, dtype=np.float32).reshape(-1).view(np.uint32).tobytes()
    return len(blob), hashlib.sha256(blob).digest()[:16], hashlib.sha256(dec).digest()[:16]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--only", default=None, help="comma-separated workload names")
    args = ap.parse_args()
    wl = workloads()
    names = args.only.split(",") if args.only else list(wl)
    out_npz = os.path.join(HERE, "workloads.npz")
    arrays = dict(np.load(out_npz)) if os.path.exists(out_npz) else {}
    meta_p = os.path.join(HERE, "workloads.json")
    meta = json.load(open(meta_p)) if os.path.exists(meta_p) else {}
    with mp.get_context("fork").Pool(args.procs) as pool:
        for name in names:
            jobs = wl[name]
            t0 = time.time()
            # big IFs first so the pool stays busy at the end
            order = sorted(range(len(jobs)), key=lambda i: -jobs[i][1] * jobs[i][2])
            res = pool.map(_job, [jobs[i] for i in order], chunksize=1)
            lens = np.zeros(len(jobs), dtype=np.int64)
            psha = np.zeros((len(jobs), 16), dtype=np.uint8)
            dsha = np.zeros((len(jobs), 16), dtype=np.uint8)
            for i, (n, a, b) in zip(order, res):
                lens[i] = n
                psha[i] = np.frombuffer(a, dtype=np.uint8)
                dsha[i] = np.frombuffer(b, dtype=np.uint8)
            arrays[f"{name}_len"] = lens
            arrays[f"{name}_payload_sha"] = psha
            arrays[f"{name}_dec_sha"] = dsha
            meta[name] = dict(n=len(jobs), jobs=[[k, r, c, sid, cfg] for k, r, c, sid, cfg in jobs]
                              if name in ("c4sweep",) else None,
                              shape_rule=("sids 0..n-1; shape/kind by shard.mixed_workload" if name == "c5"
                                          else f"kind {jobs[0][0]}, {jobs[0][1]}x{jobs[0][2]}, sids 0..{len(jobs) - 1}"),
                              cfg=None if name == "c4sweep" else BASE,
                              seconds=round(time.time() - t0, 1))
            print(f"{name}: {len(jobs)} IFs in {time.time() - t0:.1f} s", flush=True)
            np.savez_compressed(out_npz, **arrays)
            with open(meta_p, "w") as f:
                json.dump(dict(generator="tests/golden/make_workload_golden.py (reference slicer-codec, "
                                         "/root/reference/pkg/src)", **{k: v for k, v in meta.items()
                                                                        if k != "generator"}), f, indent=1)


if __name__ == "__main__":
    main()
