"""CPU-side checks of the native library: it builds, loads, exports every symbol that
include/sif.h declares, and its host-side scalars agree with the oracle.  No kernels run."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import sif_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2511_11608_b200.build import build
    from paper_2511_11608_b200 import _lib

    build()
    return _lib.load()


def test_header_symbols_exported(lib):
    from paper_2511_11608_b200 import _lib

    hdr = open(os.path.join(ROOT, "include", "sif.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(sif_\w+)\s*\(", hdr, flags=re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(raw, name), name


def test_keep_count_and_col_bits_match_oracle(lib):
    rng = np.random.default_rng(3)
    for s in [0.0, 0.05, 0.1, 0.25, 0.3, 0.5, 0.7, 0.9, 0.95, 0.999, 1.0] + list(rng.random(200)):
        for t in [1, 6, 10, 100, 1000, 200704, 4096, 8388608, 12345677]:
            assert lib.sif_keep_count(float(s), t) == O.keep_count(float(s), t), (s, t)
    for k in [0, 1, 2, 3, 4, 5, 196, 255, 256, 257, 4096, 4097, 2**31, 2**32 - 1]:
        assert lib.sif_col_bits(k) == O.col_bits(k), k


def test_validate_cfg_mirrors_codecconfig(lib):
    import paper_2511_11608_b200 as sif

    with pytest.raises(sif.ConfigError):
        sif.CodecConfig(s=1.5)
    with pytest.raises(sif.ConfigError):
        sif.CodecConfig(s=0.5, lam=1.0)
    with pytest.raises(sif.ConfigError):
        sif.CodecConfig(s=0.5, q_bit=0)
    with pytest.raises(sif.ConfigError):
        sif.CodecConfig(s=0.5, mode=sif.MODE_FIXED, fixed_q=(8,), m_plus=1, m_minus=1)
    c, keep = sif.CodecConfig(s=0.5, mode=sif.MODE_FIXED, fixed_q=(8, 4), m_plus=1, m_minus=1)._c()
    assert lib.sif_validate_cfg(ctypes.byref(c)) == 0
    bad = sif.CodecConfig(s=0.5)
    cb, _ = bad._c()
    cb.q_bit = 17
    assert lib.sif_validate_cfg(ctypes.byref(cb)) == 1
    assert sif.broadcast_q([8, 4], 2, 2) == (8, 4, 8, 4)


def test_capacity_bound_is_sound_on_golden(lib, golden):
    import paper_2511_11608_b200 as sif

    meta, _ = golden
    for c in meta["cases"]:
        d = c["cfg"]
        cfg = sif.CodecConfig(s=d["s"], lam=d["lam"], m_plus=d["m_plus"], m_minus=d["m_minus"], q_bit=d["q_bit"],
                              delta=d["delta"], mode=d["mode"], fixed_q=tuple(d["fixed_q"]))
        assert sif.max_payload_bytes(c["rows"], c["cols"], cfg) >= c["payload_len"], c["name"]
