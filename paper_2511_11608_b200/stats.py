"""Payload bound and payload statistics.

    payload_upper_bound(shape, cfg, nnz_split)   planner.py:24-64 (bits, same arithmetic)
    stats(payload_or_bytes) -> dict             cli.py:191-250 (`slicer stats --json` fields)

`payload_upper_bound` is the reference's planner bound, reproduced exactly (it is the
number `slicer stats` prints).  It charges every block q_bit, so it is not an upper bound
in fixed-Q mode when a fixed q exceeds q_bit; output buffers are sized with
`max_payload_bytes` (sif_max_payload_bytes), which charges max(q_bit, max fixed q).

`stats` reads the header echo and the block table of a `.sif` stream that lives in device
memory (the block table comes from the GPU parse kernel, sif_decode_batched parse_only=1)
and returns the dictionary of `slicer stats --json`.
"""

from __future__ import annotations

import struct

from .codec import (
    CRC_BYTES,
    HEADER_BYTES,
    MODE_ABQ,
    MODE_FIXED,
    CodecConfig,
    CompressedIF,
    Payload,
    col_bits,
    deserialize,
    keep_count,
)
from .errors import ConfigError

_HEADER_AND_CRC_BITS = 8 * (HEADER_BYTES + CRC_BYTES)


def _block_meta_bits(n: int) -> int:
    return 8 * (13 + 4 * (n + 1)) + 14  # planner.py:26 (+14: section padding)


def payload_upper_bound(shape, cfg: CodecConfig, nnz_split=None) -> int:
    """planner.py:33-64: conservative payload size in bits, every block charged q_bit."""
    n, k = int(shape[0]), int(shape[1])
    keep = keep_count(cfg.s, n * k)
    if nnz_split is not None:
        nnz_p, nnz_m = (int(v) for v in nnz_split)
        if nnz_p < 0 or nnz_m < 0 or nnz_p + nnz_m != keep:
            raise ConfigError(f"nnz split {tuple(nnz_split)} inconsistent with k_keep={keep} at s={cfg.s}")
        n_blocks = max(1, min(cfg.m_plus, nnz_p)) + max(1, min(cfg.m_minus, nnz_m))
    else:
        n_blocks = max(2, min(keep, cfg.m_plus + cfg.m_minus), min(keep, cfg.m_plus) + 1,
                       min(keep, cfg.m_minus) + 1)
    bits = _HEADER_AND_CRC_BITS
    if cfg.mode == MODE_FIXED:
        bits += 8 * n_blocks
    bits += n_blocks * _block_meta_bits(n)
    bits += keep * (cfg.q_bit + col_bits(k))
    return bits


def header_fields(p: Payload) -> dict:
    """Header echo of a stream (codec.py:328-341): f32 fields widened as the reference does."""
    h = bytes(p.buf[: HEADER_BYTES].cpu().numpy().tobytes())
    _ver, n, k, s, lam, qb, dl, mode, mp, mm = struct.unpack_from("<HIIffBfBHH", h, 4)
    qv = ()
    if mode == 1:
        qv = tuple(int(v) for v in p.buf[HEADER_BYTES: HEADER_BYTES + mp + mm].cpu().tolist())
    return dict(rows=n, cols=k, s=s, lam=lam, q_bit=qb, delta=dl, mode=MODE_FIXED if mode == 1 else MODE_ABQ,
                m_plus=mp, m_minus=mm, q_vector=qv)


def stats(p) -> dict:
    """The `slicer stats --json` dictionary (cli.py:199-236) of a payload or `.sif` bytes."""
    if not isinstance(p, (Payload, CompressedIF)):
        p = deserialize(p)
    h = header_fields(p)
    blocks = p.blocks()
    total_nnz = sum(b["nnz"] for b in blocks)
    exact = p.payload_bits
    cfg = CodecConfig(s=h["s"], lam=h["lam"], m_plus=max(1, h["m_plus"]), m_minus=max(1, h["m_minus"]),
                      q_bit=h["q_bit"], delta=h["delta"], mode=h["mode"],
                      fixed_q=h["q_vector"] if h["mode"] == MODE_FIXED else ())
    b_ub = payload_upper_bound((h["rows"], h["cols"]), cfg)
    rows, cols = h["rows"], h["cols"]
    idx = {"plus": 0, "minus": 0}
    out_blocks = []
    for b in blocks:
        out_blocks.append({"plane": b["plane"], "index": idx[b["plane"]], "nnz": b["nnz"], "q": b["q"],
                           "scale": b["o"], "v_min": b["v_min"]})
        idx[b["plane"]] += 1
    return {
        "shape": [rows, cols],
        "sparsity_config": h["s"],
        "nonzeros": total_nnz,
        "actual_sparsity": 1.0 - total_nnz / (rows * cols),
        "payload_bits_exact": exact,
        "payload_bits_upper_bound": b_ub,
        "bits_per_element": exact / (rows * cols),
        "blocks": out_blocks,
    }
