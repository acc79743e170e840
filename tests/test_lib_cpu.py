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


def _enc_plan(lib, shapes, cfg, dtype=1):
    """sif_enc_plan over fake (aligned, never dereferenced) device pointers: host-only."""
    from paper_2511_11608_b200 import _lib

    n = len(shapes)
    arr = (_lib.EncDesc * n)()
    for i, (r, c) in enumerate(shapes):
        arr[i].x = 0x10000 * (i + 1)
        arr[i].out = 0x100000000 + 0x10000 * i
        arr[i].out_cap = 1 << 20
        arr[i].seed = i
        arr[i].rows, arr[i].cols, arr[i].dtype = r, c, dtype
    cc, keep = cfg._c()
    p = _lib.Plan()
    st = lib.sif_enc_plan(arr, n, ctypes.byref(cc), ctypes.byref(p))
    return st, p


def test_encode_plan_routing_host_only(lib):
    """Size classes chosen by sif_enc_plan (no kernels): tokens (<= 4096 elements, lambda = 0,
    <= 8 blocks) take the one-CTA token path, others the chunk pipeline; more than
    SIF_MAX_BLOCKS planned blocks is a ConfigError (status 1); IFs of >= 2^31 elements are
    refused."""
    import paper_2511_11608_b200 as sif

    base = dict(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
    st, p = _enc_plan(lib, [(1, 4096)] * 5 + [(1024, 196)] * 2, sif.CodecConfig(**base))
    assert st == 0 and p.n == 7 and p.reserved == 5  # reserved: IFs on the token path
    st, p = _enc_plan(lib, [(1, 4096)] * 3, sif.CodecConfig(**{**base, "lam": 0.1}))
    assert st == 0 and p.reserved == 0  # lambda > 0: pipeline
    st, p = _enc_plan(lib, [(1, 4096)] * 3, sif.CodecConfig(**{**base, "m_plus": 5, "m_minus": 5}))
    assert st == 0 and p.reserved == 0  # 10 blocks: pipeline
    st, _ = _enc_plan(lib, [(64, 512)], sif.CodecConfig(**{**base, "m_plus": 32, "m_minus": 32}))
    assert st == 0  # 64 planned blocks: at the limit
    st, _ = _enc_plan(lib, [(64, 512)], sif.CodecConfig(**{**base, "m_plus": 40, "m_minus": 40}))
    assert st == 1  # 80 planned blocks > SIF_MAX_BLOCKS
    st, _ = _enc_plan(lib, [(1 << 16, 1 << 15)], sif.CodecConfig(**base))
    assert st == 8  # SIF_ERR_INVALID_ARG: 2^31 elements


def test_decode_plan_size_classes_host_only(lib):
    """sif_dec_plan (no kernels): streams of <= 4096 dense elements go to the one-CTA
    small-stream kernel (plan.n_fused), the rest to the four-kernel path; items are 1280
    elements for narrow batches, 4096 when some row is wider; sif_set_small_decode(0) routes
    everything to the four-kernel path; misaligned buffers are refused."""
    from paper_2511_11608_b200 import _lib

    def plan(shapes, align=16):
        arr = (_lib.DecDesc * len(shapes))()
        for i, (r, c) in enumerate(shapes):
            arr[i].inp = 0x10000 * (i + 1) + (0 if align == 16 else 2)
            arr[i].in_len = 4096
            arr[i].out = 0x100000000 + 0x100000 * i
            arr[i].rows, arr[i].cols = r, c
            arr[i].in_len_dev = None
        p = _lib.Plan()
        return lib.sif_dec_plan(arr, len(shapes), ctypes.byref(p)), p

    st, p = plan([(1, 4096)] * 4 + [(1024, 196)] * 3)
    assert st == 0 and p.n_fused == 4 and p.tiles == 1280
    st, p = plan([(1, 4096), (256, 4096)])
    assert st == 0 and p.n_fused == 1 and p.tiles == 4096
    assert lib.sif_set_small_decode(0) == 0
    try:
        st, p = plan([(1, 4096)] * 4)
        assert st == 0 and p.n_fused == 0
    finally:
        assert lib.sif_set_small_decode(4096) == 0
    assert lib.sif_set_small_decode(8192) == 8  # above the shared-memory buffer
    st, _ = plan([(1, 4096)], align=2)
    assert st == 8


def test_set_input_argument_checks_host_only(lib):
    """sif_enc_set_input / sif_dec_set_input refuse bad arguments before any launch."""
    from paper_2511_11608_b200 import _lib

    p = _lib.Plan()
    p.n = 1
    assert lib.sif_enc_set_input(None, None, 0, None, None, 0, None) == 8
    assert lib.sif_enc_set_input(ctypes.byref(p), ctypes.c_void_p(0x1000), 1, ctypes.c_void_p(0x1000),
                                 ctypes.c_void_p(0x2000), 0, None) == 8  # index out of range
    assert lib.sif_enc_set_input(ctypes.byref(p), ctypes.c_void_p(0x1000), 0, ctypes.c_void_p(0x1008),
                                 ctypes.c_void_p(0x2000), 0, None) == 8  # x not 16-byte aligned
    assert lib.sif_dec_set_input(ctypes.byref(p), ctypes.c_void_p(0x1000), 0, ctypes.c_void_p(0x1000), 64,
                                 None, ctypes.c_void_p(0x2000), None) == 8  # no device length slot
