"""GPU parity on exactly the workloads bench.py times, plus fresh-input serving loops.

* Every IF of C2 (256), C3 (1024), C4 (32), C5 (8192 mixed streams) and every point of the
  BASELINE.md §4.2 C4 sweep (5 s x 4 delta x 2 lambda + fixed Q=[8,4,2]) is encoded and
  decoded on the GPU through the same classes the bench uses (BatchPipeline /
  ListEncoder) and compared with digests of the REFERENCE's own payload bytes and decoded
  fp32 bits (tests/golden/make_workload_golden.py ran slicer.encode/serialize/deserialize/
  decode, codec.py:186, :283, :320, :254).
* The serving loops (BatchPipeline, HostRoundTrip, ListRoundTrip) get NEW input data on
  every step; each step's payloads must equal the oracle's bytes for that step's data
  (the decoders read payload lengths on the device, so nothing is planned from a
  previous step).
"""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BASE = dict(s=0.9, lam=0.0, m_plus=3, m_minus=3, q_bit=8, delta=0.01)


@pytest.fixture(scope="module")
def wl():
    d = dict(np.load(os.path.join(GOLD, "workloads.npz")))
    with open(os.path.join(GOLD, "workloads.json")) as f:
        return d, json.load(f)


def _digests(out: torch.Tensor, offs, lens):
    """sha256[:16] of every payload (one D2H copy of the whole output buffer)."""
    host = out.reshape(-1).cpu().numpy()
    return [hashlib.sha256(host[o:o + n].tobytes()).digest()[:16] for o, n in zip(offs, lens)]


def _dec_digest(y: torch.Tensor) -> bytes:
    return hashlib.sha256(y.contiguous().cpu().numpy().reshape(-1).view(np.uint32).tobytes()).digest()[:16]


def _check(name, d, got_p, got_lens, got_d=None, idx=None):
    idx = list(range(len(got_p))) if idx is None else idx
    bad = [i for k, i in enumerate(idx)
           if got_lens[k] != d[f"{name}_len"][i] or got_p[k] != d[f"{name}_payload_sha"][i].tobytes()]
    assert not bad, f"{name}: {len(bad)} payloads differ from the reference, e.g. IF {bad[:8]}"
    if got_d is not None:
        badd = [i for k, i in enumerate(idx) if got_d[k] != d[f"{name}_dec_sha"][i].tobytes()]
        assert not badd, f"{name}: {len(badd)} decodes differ from the reference, e.g. IF {badd[:8]}"


def _homog(sif, kind, N, K, B, dtype, sid0=0):
    xs = torch.empty((B, N, K), dtype=dtype, device="cuda")
    for i in range(B):
        sif.synthetic(kind, N, K, sid0 + i, out=xs[i])
    return xs


def _pipeline_check(sif, name, wl, kind, N, K, B, dtype, depth):
    d, _ = wl
    xs = _homog(sif, kind, N, K, B, dtype)
    pipe = sif.BatchPipeline(xs, sif.CodecConfig(**BASE), list(range(B)), depth=depth, graphs=True)
    pipe.begin()
    for _ in range(depth + 1):
        pipe.step()
    pipe.end()
    torch.cuda.synchronize()
    pipe.check()
    for sl in pipe.slots:
        enc = sl["enc"]
        lens = enc.out_len.cpu().numpy()
        got = _digests(enc.out, [i * enc.cap for i in range(B)], lens)
        gd = [_dec_digest(sl["dec"].out[i]) for i in range(B)]
        _check(name, d, got, lens, gd)


def test_c2_every_if_matches_reference(sif, wl):
    """C2: all 256 ResNet IFs of the bench batch, through the bench's BatchPipeline."""
    _pipeline_check(sif, "c2", wl, 0, 1024, 196, 256, torch.float32, depth=2)


def test_c3_every_token_matches_reference(sif, wl):
    """C3: all 1024 decode-step tokens (1x4096 bf16)."""
    _pipeline_check(sif, "c3", wl, 1, 1, 4096, 1024, torch.bfloat16, depth=2)


def test_c4_every_if_matches_reference(sif, wl):
    """C4: all 32 prefill IFs (2048x4096 bf16) of the bench batch -- the multi-kernel select
    across the whole batch."""
    _pipeline_check(sif, "c4", wl, 1, 2048, 4096, 32, torch.bfloat16, depth=1)


def test_c4_sweep_matches_reference(sif, wl):
    """s in {0.5,0.7,0.8,0.9,0.95} x delta in {0.01,0.05,0.1,0.2} x
    lambda in {0, 0.1}, plus fixed Q=[8,4,2], on the C4 prefill IF (sid 0)."""
    d, meta = wl
    x = _homog(sif, 1, 2048, 4096, 1, torch.bfloat16)[0]
    got_p, got_l, got_d = [], [], []
    for kind, r, c, sid, cfg in meta["c4sweep"]["jobs"]:
        cfg = dict(cfg)
        if "fixed_q" in cfg:
            cfg["fixed_q"] = tuple(cfg["fixed_q"])
        p = sif.encode(x, sif.CodecConfig(**cfg), seed=sid)
        got_p.append(hashlib.sha256(p.to_bytes()).digest()[:16])
        got_l.append(p.nbytes)
        got_d.append(_dec_digest(sif.decode(p)))
    _check("c4sweep", d, got_p, got_l, got_d)


def test_c5_every_stream_matches_reference(sif, wl):
    """C5: all 8192 mixed streams, encoded by ListEncoder in shards like the bench's ranks
    (LPT partition for 8 ranks), decoded by the device-length decoder."""
    d, _ = wl
    mix = sif.shard.mixed_workload(8192)
    cfg = sif.CodecConfig(**BASE)
    for rank in range(8):
        mine = sif.shard.shard_streams([(r, c, b) for _k, r, c, b in mix], 8, rank)
        xs = []
        for sid in mine:
            kind, r, c, b = mix[sid]
            t = torch.empty((r, c), dtype=torch.float32 if b == 4 else torch.bfloat16, device="cuda")
            sif.synthetic(kind, r, c, sid, out=t)
            xs.append(t)
        enc = sif.ListEncoder(xs, cfg, mine)
        dec = sif.codec.decoder_for(enc)
        enc.run()
        dec.run()
        torch.cuda.synchronize()
        enc.check()
        dec.check()
        lens = enc.out_len.cpu().numpy()[: len(mine)]
        got = _digests(enc.out, enc.offs, lens)
        gd = [_dec_digest(y) for y in dec.outs]
        _check("c5", d, got, lens, gd, idx=mine)
        del enc, dec, xs
        torch.cuda.empty_cache()


# ------------------------------------------------------------------ fresh inputs per step
def _oracle_bytes(x, seed):
    from oracle import sif_oracle as O

    return O.encode_bytes(x, O.Cfg(**BASE), seed)


def test_batch_pipeline_refilled_inputs(sif):
    """BatchPipeline (CUDA graphs, 2 slots): xs gets new synthetic IFs before every step;
    every step's payloads and decodes equal the oracle's for that step's data."""
    from oracle import sif_oracle as O
    from oracle.synth import synth

    B, N, K = 6, 1024, 196
    seeds = [11 * i + 3 for i in range(B)]
    xs = torch.empty((B, N, K), dtype=torch.float32, device="cuda")
    pipe = sif.BatchPipeline(xs, sif.CodecConfig(**BASE), seeds, depth=2, graphs=True)
    for step in range(4):
        sids = [5000 + 100 * step + i for i in range(B)]
        for i, sid in enumerate(sids):
            sif.synthetic(0, N, K, sid, out=xs[i])
        slot = pipe.i % len(pipe.slots)
        pipe.begin()
        pipe.step()
        pipe.end()
        torch.cuda.synchronize()
        pipe.check()
        sl = pipe.slots[slot]
        ps = sl["enc"].payloads()
        for i, sid in enumerate(sids):
            ref = _oracle_bytes(synth(0, N, K, sid), seeds[i])
            assert ps[i].to_bytes() == ref, f"step {step} IF {i}: payload differs"
            assert np.array_equal(sl["dec"].out[i].cpu().numpy().view(np.uint32),
                                  O.decode_bytes(ref).view(np.uint32)), f"step {step} IF {i}: decode differs"


def test_host_round_trip_refilled_inputs(sif):
    """HostRoundTrip: the pinned host batch is refilled before every run (the bench's e2e
    path); every run's decoded host output and payloads equal the oracle's."""
    from oracle import sif_oracle as O
    from oracle.synth import synth

    B, N, K = 6, 1024, 196
    seeds = list(range(B))
    x_host = torch.empty((B, N, K), dtype=torch.float32).pin_memory()
    rt = sif.HostRoundTrip(x_host, sif.CodecConfig(**BASE), seeds, parts=3)
    for step in range(3):
        sids = [7000 + 100 * step + i for i in range(B)]
        xnp = [synth(0, N, K, sid) for sid in sids]
        for i in range(B):
            x_host[i].copy_(torch.from_numpy(xnp[i]))
        rt.run()
        torch.cuda.synchronize()
        rt.check()
        ps = [p for k in range(len(rt.parts)) for p in rt.payloads(k)]
        for i in range(B):
            ref = _oracle_bytes(xnp[i], seeds[i])
            assert ps[i].to_bytes() == ref, f"run {step} IF {i}: payload differs"
            assert np.array_equal(rt.y_host[i].numpy().view(np.uint32), O.decode_bytes(ref).view(np.uint32))


def test_list_round_trip_refilled_inputs(sif):
    """ListRoundTrip over mixed shapes, host inputs rewritten between runs."""
    from oracle import sif_oracle as O
    from oracle.synth import synth

    mix = sif.shard.mixed_workload(8)
    seeds = list(range(8))
    xs0 = [torch.zeros((r, c), dtype=torch.float32 if b == 4 else torch.bfloat16) for _k, r, c, b in mix]
    rt = sif.ListRoundTrip(xs0, sif.CodecConfig(**BASE), seeds, parts=2)
    for step in range(3):
        xnp = []
        for k, (kind, r, c, b) in enumerate(mix):
            x = synth(kind, r, c, 9000 + 10 * step + k)
            xnp.append(x)
            t = torch.from_numpy(x)
            if b == 2:
                t = t.to(torch.bfloat16)
            nb = t.numel() * t.element_size()
            rt.x_host[rt.in_off[k]: rt.in_off[k] + nb].copy_(t.reshape(-1).view(torch.uint8))
        rt.run()
        torch.cuda.synchronize()
        rt.check()
        for k in range(8):
            ref = _oracle_bytes(xnp[k], seeds[k])
            assert np.array_equal(rt.y(k).numpy().view(np.uint32), O.decode_bytes(ref).view(np.uint32)), (step, k)


def test_device_length_longer_than_buffer_is_rejected(sif):
    """A device-side length above the buffer capacity is refused (CapacityError-class status),
    never read past the buffer."""
    x = torch.from_numpy(np.arange(64, dtype=np.float32).reshape(8, 8)).cuda()
    p = sif.encode(x, sif.CodecConfig(s=0.5))
    bad = torch.tensor([p.nbytes + 64], dtype=torch.int64, device="cuda")
    dec = sif.BatchDecoder([p.buf.data_ptr()], [p.nbytes], 8, 8, len_ptrs=[bad.data_ptr()])
    dec.run()
    torch.cuda.synchronize()
    assert int(dec.status.item()) == 6  # SIF_ERR_CAPACITY
