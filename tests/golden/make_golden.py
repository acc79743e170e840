"""Generate golden vectors by running the REFERENCE implementation (slicer-codec 0.1.0).

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py            # writes tests/golden/*.npz + cases.json

Everything written here comes from `/root/reference/pkg/src/slicer` itself:
`atkf_filter` (atkf.py:44), `encode` (codec.py:186), `serialize` (codec.py:283),
`deserialize` (codec.py:320), `decode` (codec.py:254).  Inputs are either produced by
the reference's own fixture generator `random_tensor` (tensor.py:89) or by the
integer-exact synthetic generator in `oracle/synth.py` (bit-identical on the GPU).
"""

from __future__ import annotations

import hashlib
import json
import os
import struct
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import slicer  # noqa: E402  (the reference)
from slicer import CodecConfig, DenseTensor  # noqa: E402
from slicer.codec import MODE_FIXED  # noqa: E402

from oracle.synth import KIND_LLM, KIND_RESNET, bf16_rne, synth  # noqa: E402


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def cfg_dict(cfg: CodecConfig) -> dict:
    return dict(s=cfg.s, lam=cfg.lam, m_plus=cfg.m_plus, m_minus=cfg.m_minus, q_bit=cfg.q_bit,
                delta=cfg.delta, mode=cfg.mode, fixed_q=list(cfg.fixed_q))


def ref_error_kind(fn, *a):
    try:
        fn(*a)
        return None
    except slicer.SlicerError as e:  # the most-derived class name
        return type(e).__name__


def ref_error_msg(fn, *a):
    try:
        fn(*a)
        return None
    except slicer.SlicerError as e:
        return str(e)


def make_inputs(gen: np.random.Generator, kind: str, rows: int, cols: int, seed: int) -> np.ndarray:
    t = rows * cols
    if kind == "uniform":
        return slicer.random_tensor(rows, cols, seed, "uniform").values.copy()
    if kind == "gaussian":
        return slicer.random_tensor(rows, cols, seed, "gaussian").values.copy()
    if kind == "bf16ties":  # heavy exact ties + zeros (LLM-like)
        v = gen.normal(size=t).astype(np.float32)
        v[gen.random(t) < 0.2] = 0.0
        return bf16_rne(v)
    if kind == "coarse":  # very few distinct magnitudes -> giant tie sets
        v = gen.integers(-3, 4, size=t).astype(np.float32) * np.float32(0.5)
        return v
    if kind == "relu":
        v = gen.normal(size=t).astype(np.float32) - np.float32(0.3)
        return np.maximum(v, 0).astype(np.float32)
    if kind == "negheavy":
        v = gen.normal(size=t).astype(np.float32)
        v[v > 0] *= np.float32(0.25)
        return v
    if kind == "allequal":
        return np.full(t, 2.0, dtype=np.float32)
    if kind == "signed_zero":
        v = gen.normal(size=t).astype(np.float32)
        v[gen.random(t) < 0.3] = -0.0
        return v
    if kind == "wide_range":
        v = (gen.normal(size=t) * np.exp(gen.normal(size=t) * 6)).astype(np.float32)
        return v
    raise ValueError(kind)


def random_cfg(gen: np.random.Generator) -> CodecConfig:
    mp, mm = int(gen.integers(1, 5)), int(gen.integers(1, 5))
    if gen.random() < 0.2:
        q = tuple(int(v) for v in gen.integers(1, 17, size=mp + mm))
        return CodecConfig(s=float(gen.choice([0.0, 0.3, 0.5, 0.8, 0.9, 0.95, 1.0])),
                           lam=float(gen.choice([0.0, 0.1, 0.3, 0.7])), m_plus=mp, m_minus=mm,
                           q_bit=int(gen.choice([1, 2, 4, 8, 16])), mode=MODE_FIXED, fixed_q=q)
    return CodecConfig(s=float(gen.choice([0.0, 0.3, 0.5, 0.7, 0.8, 0.9, 0.95, 0.999, 1.0])),
                       lam=float(gen.choice([0.0, 0.0, 0.1, 0.3, 0.7, 0.95])),
                       m_plus=mp, m_minus=mm, q_bit=int(gen.choice([1, 2, 3, 4, 8, 12, 16])),
                       delta=float(gen.choice([0.0, 0.01, 0.05, 0.2, 1.0, 3.0])))


def run_case(x: np.ndarray, rows: int, cols: int, cfg: CodecConfig, seed: int) -> dict:
    dt = DenseTensor(rows, cols, x)
    at = slicer.atkf_filter(dt, cfg.s, cfg.lam, seed)
    c = slicer.encode(dt, cfg, seed)
    blob = slicer.serialize(c)
    dec = slicer.decode(slicer.deserialize(blob)).values
    return dict(kept=at.kept_indices.astype(np.int64), tau=at.tau, tau_plus=at.tau_plus,
                tau_minus=at.tau_minus, k_keep=at.k_keep, blob=blob,
                dec_bits=dec.view(np.uint32).copy(),
                q=[b.q for b in c.all_blocks], nnz=[b.nnz for b in c.all_blocks])


def corrupt_variants(blob: bytes, gen: np.random.Generator, rows: int) -> list[tuple[str, bytes]]:
    """Stream mutations exercising each deserialize/decode check (codec.py:235-252, :320-385)."""

    def refix(b: bytearray) -> bytes:
        b = bytes(b[:-4])
        return b + struct.pack("<I", zlib.crc32(b[4:]) & 0xFFFFFFFF)

    out = []
    b = bytearray(blob)
    out.append(("short", bytes(b[:20])))
    out.append(("magic", b"XSIF" + bytes(b[4:])))
    f = bytearray(b)
    f[len(f) // 2] ^= 0x40
    out.append(("crcflip", bytes(f)))
    v = bytearray(b)
    v[4] = 2
    out.append(("version", refix(v)))
    m = bytearray(b)
    m[27] = 7
    out.append(("mode", refix(m)))
    out.append(("trailing", refix(bytearray(b[:-4]) + b"\x00\x00\x00\x00" + b"\x00" * 4)))
    out.append(("truncated", refix(bytearray(b[: max(36, len(b) - 9)]) + b"\x00" * 4)))
    mode = b[27]
    pos = 32 + ((struct.unpack_from("<H", b, 28)[0] + struct.unpack_from("<H", b, 30)[0]) if mode == 1 else 0)
    # block 0: q out of range
    qb = bytearray(b)
    qb[pos] = 0
    out.append(("q0", refix(qb)))
    qb = bytearray(b)
    qb[pos] = 17
    out.append(("q17", refix(qb)))
    # row_ptr[0] != 0
    rp = bytearray(b)
    struct.pack_into("<I", rp, pos + 13, 1)
    out.append(("rowptr0", refix(rp)))
    # row_ptr[N] != nnz
    rp = bytearray(b)
    last = pos + 13 + 4 * rows
    struct.pack_into("<I", rp, last, struct.unpack_from("<I", rp, last)[0] + 1)
    out.append(("rowptrN", refix(rp)))
    # random payload byte flips after the header, CRC fixed (structural corruption or silent)
    for j in range(6):
        r = bytearray(b)
        if len(r) > 40:
            p = int(gen.integers(32, len(r) - 4))
            r[p] ^= int(gen.integers(1, 256))
            out.append((f"flip{j}", refix(r)))
    # o := NaN in block 0 -> NonFiniteError in decode (if the block is non-empty)
    nf = bytearray(b)
    struct.pack_into("<f", nf, pos + 1, float("nan"))
    out.append(("o_nan", refix(nf)))
    big = bytearray(b)
    struct.pack_into("<f", big, pos + 1, 3.0e38)
    out.append(("o_huge", refix(big)))
    return out


def main():
    gen = np.random.default_rng(20251111)
    cases = []
    arrays = {}

    def add(name, x, rows, cols, cfg, seed, extra=None, store_x=True):
        r = run_case(x, rows, cols, cfg, seed)
        i = len(cases)
        meta = dict(name=name, rows=rows, cols=cols, cfg=cfg_dict(cfg), seed=seed, tau=r["tau"],
                    tau_plus=r["tau_plus"], tau_minus=r["tau_minus"], k_keep=r["k_keep"],
                    q=r["q"], nnz=r["nnz"], payload_len=len(r["blob"]), payload_sha=sha(r["blob"]),
                    kept_sha=sha(r["kept"].tobytes()), dec_sha=sha(r["dec_bits"].tobytes()),
                    stored=store_x)
        if extra:
            meta.update(extra)
        if store_x:
            arrays[f"c{i}_x"] = x.astype(np.float32).view(np.uint32)
            arrays[f"c{i}_kept"] = r["kept"]
            arrays[f"c{i}_blob"] = np.frombuffer(r["blob"], dtype=np.uint8)
            arrays[f"c{i}_dec"] = r["dec_bits"]
        cases.append(meta)
        return r

    # 1. worked examples (tests/test_atkf.py:18-33, tests/test_codec.py:25-37)
    x6 = np.array([3, -1, 0.5, -4, 2, 0.1], dtype=np.float32)
    add("worked_1x6_lam0", x6, 1, 6, CodecConfig(s=0.5, lam=0.0, q_bit=4, delta=0.0), 1)
    add("worked_1x6_lam05", x6, 1, 6, CodecConfig(s=0.5, lam=0.5, q_bit=4, delta=0.0), 1)
    # 2. SURVEY Appendix C fixtures
    add("rt32_s7", slicer.random_tensor(32, 32, 7).values.copy(), 32, 32,
        CodecConfig(s=0.9, m_plus=2, m_minus=2, q_bit=8, delta=0.01), 5)
    add("rt16_s1", slicer.random_tensor(16, 16, 1).values.copy(), 16, 16,
        CodecConfig(s=0.8, m_plus=2, m_minus=2, q_bit=8, delta=0.01), 0)
    add("rt13x37_g", slicer.random_tensor(13, 37, 99, "gaussian").values.copy(), 13, 37,
        CodecConfig(s=0.7, lam=0.2, m_plus=3, m_minus=2, q_bit=8, delta=0.05), 3)
    add("rt9_fixed", slicer.random_tensor(9, 9, 8).values.copy(), 9, 9,
        CodecConfig(s=0.6, m_plus=2, m_minus=2, q_bit=8, mode=MODE_FIXED, fixed_q=(8, 4, 8, 4)), 0)
    # reference test shapes (tests/test_codec.py:185-190, :62-70)
    for rows, cols in ((1, 50), (50, 1)):
        add(f"shape_{rows}x{cols}", slicer.random_tensor(rows, cols, rows).values.copy(), rows, cols,
            CodecConfig(s=0.5, q_bit=8), 0)
    add("s1_header_only", slicer.random_tensor(4, 4, 2).values.copy(), 4, 4, CodecConfig(s=1.0), 0)
    add("allequal_1x10", np.full(10, 2.0, np.float32), 1, 10, CodecConfig(s=0.6), 12)
    add("tie_plane", np.array([9, 0, 5, 0, 0, 0, 0, 9], np.float32), 2, 4,
        CodecConfig(s=0.0, m_plus=2, m_minus=1, q_bit=4), 0)
    # 3. randomized sweep
    kinds = ["uniform", "gaussian", "bf16ties", "coarse", "relu", "negheavy", "allequal",
             "signed_zero", "wide_range"]
    for trial in range(260):
        kind = kinds[trial % len(kinds)]
        rows = int(gen.choice([1, 1, 2, 3, 7, 16, 31, 64, 100]))
        cols = int(gen.choice([1, 2, 3, 5, 17, 64, 196, 255, 256, 257, 600]))
        if rows * cols > 40000:
            cols = 40000 // rows
        x = make_inputs(gen, kind, rows, cols, 1000 + trial)
        cfg = random_cfg(gen)
        seed = int(gen.integers(0, 2**40)) if trial % 3 else int(trial)
        add(f"sweep{trial}_{kind}", x, rows, cols, cfg, seed)
    # 4. a few larger ones (stored x) exercising sampling/bracketing paths
    for trial, (rows, cols, kind) in enumerate([(256, 196, "relu"), (64, 1024, "bf16ties"),
                                               (128, 512, "gaussian"), (8, 8192, "coarse")]):
        x = make_inputs(gen, kind, rows, cols, 5000 + trial)
        for cfg in (CodecConfig(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01),
                    CodecConfig(s=0.5, lam=0.3, m_plus=4, m_minus=2, q_bit=6, delta=0.2)):
            add(f"large{trial}_{kind}", x, rows, cols, cfg, 77 + trial)
    # 5. bench-shaped synthetic IFs (x regenerated by oracle/synth.py, not stored)
    bench_cfg = CodecConfig(s=0.9, lam=0.0, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
    for sid in (0, 1):
        x = synth(KIND_RESNET, 1024, 196, sid)
        add(f"synth_resnet_sid{sid}", x.reshape(-1), 1024, 196, bench_cfg, sid,
            extra=dict(synth=dict(kind=KIND_RESNET, sid=sid)), store_x=False)
    for sid in (3, 4):
        x = synth(KIND_LLM, 1, 4096, sid)
        add(f"synth_llm_tok_sid{sid}", x.reshape(-1), 1, 4096, bench_cfg, sid,
            extra=dict(synth=dict(kind=KIND_LLM, sid=sid)))
    x = synth(KIND_LLM, 256, 4096, 9)
    add("synth_llm_prefill256_sid9", x.reshape(-1), 256, 4096, bench_cfg, 9,
        extra=dict(synth=dict(kind=KIND_LLM, sid=9)), store_x=False)

    # 6. corrupt streams: expected error class from reference deserialize+decode
    corrupt = []
    for ci in range(0, 40, 3):
        c = cases[ci]
        if not c["stored"]:
            continue
        blob = arrays[f"c{ci}_blob"].tobytes()
        for tag, bad in corrupt_variants(blob, gen, c["rows"]):
            kind = ref_error_kind(lambda d: slicer.decode(slicer.deserialize(d)), bad)
            j = len(corrupt)
            arrays[f"bad{j}"] = np.frombuffer(bad, dtype=np.uint8)
            corrupt.append(dict(case=ci, tag=tag, rows=c["rows"], cols=c["cols"], error=kind,
                                deser_error=ref_error_kind(slicer.deserialize, bad),
                                msg=ref_error_msg(lambda d: slicer.decode(slicer.deserialize(d)), bad),
                                deser_msg=ref_error_msg(slicer.deserialize, bad)))

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(dict(generator="tests/golden/make_golden.py", reference="slicer-codec 0.1.0",
                       cases=cases, corrupt=corrupt), f, indent=0)
    print(f"{len(cases)} cases, {len(corrupt)} corrupt streams")


if __name__ == "__main__":
    main()
