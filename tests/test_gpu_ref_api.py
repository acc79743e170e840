"""The reference's codec API contract, through the `slicer`-named shim over the GPU codec
(paper_2511_11608_b200/compat/slicer): CompressedIF / EncodedBlock fields and equality
(codec.py:108-172), deserialize(serialize(c)) == c (codec.py:283-399), canonical v_max
(quant.py:76-85), degenerate blocks, hand-built CompressedIF objects decoded and
rejected exactly like the reference (codec.py:235-266), atkf_filter results (atkf.py:20-96).
Every value is compared with the pinned oracle or the reference's goldens."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def slicer():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test without a CUDA device")
    sys.path.insert(0, os.path.join(ROOT, "paper_2511_11608_b200", "compat"))
    try:
        import slicer as m
    finally:
        sys.path.pop(0)
    assert m.__file__.startswith(os.path.join(ROOT, "paper_2511_11608_b200", "compat")), m.__file__
    return m


def _oracle_blocks(blob):
    from oracle import sif_oracle as O

    c = O.deserialize(blob)
    return c, c.blocks_plus + c.blocks_minus


def test_worked_example_fields(slicer):
    x = slicer.DenseTensor(1, 6, np.array([3, -1, 0.5, -4, 2, 0.1], np.float32))
    c = slicer.encode(x, slicer.CodecConfig(s=0.5, lam=0.0, m_plus=1, m_minus=1, q_bit=4, delta=0.0), seed=1)
    assert (c.rows, c.cols, c.m_plus, c.m_minus, c.mode, c.q_vector) == (1, 6, 1, 1, "abq", ())
    [bp], [bm] = c.blocks_plus, c.blocks_minus
    assert (bp.nnz, bp.q, bp.o, bp.v_min, bp.degenerate) == (2, 1, 1.0, 2.0, False)
    assert list(bp.codes) == [1, 0] and list(bp.cols) == [0, 4] and list(bp.row_ptr) == [0, 2]
    assert (bm.nnz, bm.q, bm.v_min, bm.v_max, bm.degenerate) == (1, 1, 4.0, 4.0, True)
    assert bp.v_max == 3.0  # canonical: v_min + o * (2^q - 1)
    assert c.total_nnz == 3 and c.payload_bits == 8 * len(slicer.serialize(c))
    y = slicer.decode(c)
    assert isinstance(y, slicer.DenseTensor)
    assert list(y.values) == [3.0, 0.0, 0.0, -4.0, 2.0, 0.0]


def test_fields_match_oracle_and_round_trip(slicer):
    """Every field of every block of GPU-encoded streams equals the oracle's deserialize of
    the same bytes; deserialize(serialize(c)) == c; serialize(deserialize(b)) == b."""
    from oracle import sif_oracle as O

    cases = [((13, 37, 99, "gaussian"), dict(s=0.7, lam=0.2, m_plus=3, m_minus=2, q_bit=8, delta=0.05), 3),
             ((9, 9, 8, "uniform"), dict(s=0.6, m_plus=2, m_minus=2, q_bit=8, mode="fixed_q", fixed_q=(8, 4, 8, 4)), 0),
             ((4, 4, 2, "uniform"), dict(s=1.0, q_bit=8), 0),
             ((64, 196, 5, "uniform"), dict(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.2), 7)]
    for (r, cc, sd, dist), kw, seed in cases:
        x = slicer.random_tensor(r, cc, seed=sd, dist=dist)
        c = slicer.encode(x, slicer.CodecConfig(**kw), seed=seed)
        blob = slicer.serialize(c)
        ref = O.encode_bytes(x.values.reshape(r, cc), O.Cfg(**kw), seed)
        assert blob == ref
        oc, ob = _oracle_blocks(ref)
        assert (c.m_plus, c.m_minus, c.q_vector) == (len(oc.blocks_plus), len(oc.blocks_minus), tuple(oc.q_vector))
        for b, o in zip(c.all_blocks, ob):
            assert (b.q, np.float32(b.o), np.float32(b.v_min), b.nnz) == (o.q, np.float32(o.o), np.float32(o.v_min),
                                                                          len(o.codes))
            assert np.array_equal(b.row_ptr, o.row_ptr) and np.array_equal(b.cols, o.cols)
            assert np.array_equal(b.codes, o.codes)
        c2 = slicer.deserialize(blob)
        assert c2 == c and slicer.serialize(c2) == blob
        assert np.array_equal(slicer.decode(c2).values.view(np.uint32), O.decode_bytes(ref).reshape(-1).view(np.uint32))


def test_hand_built_objects_are_validated(slicer):
    """codec.py:235-251 on objects assembled from fields (the reference's own tests build
    them with type(c)(**{**c.__dict__, ...})): overlap and column order are rejected, an
    unchanged rebuild decodes like the original."""
    x = slicer.DenseTensor(2, 3, np.array([5, 0, 0, 0, 3, 0], np.float32))
    c = slicer.encode(x, slicer.CodecConfig(s=0.5, m_plus=2, m_minus=1, q_bit=4), seed=0)
    assert c.m_plus == 2
    same = type(c)(**c.__dict__)
    assert same == c
    assert slicer.decode(same) == slicer.decode(c)
    b0, b1 = c.blocks_plus
    clash = type(b1)(q=b1.q, o=b1.o, v_min=b1.v_min, v_max=b1.v_max, degenerate=b1.degenerate, row_ptr=b0.row_ptr,
                     cols=b0.cols, codes=b1.codes)
    with pytest.raises(slicer.CorruptStreamError, match="overlapping supports"):
        slicer.decode(type(c)(**{**c.__dict__, "blocks_plus": (b0, clash)}))
    y = slicer.DenseTensor(1, 4, np.array([5, 3, 0, 0], np.float32))
    c = slicer.encode(y, slicer.CodecConfig(s=0.5, q_bit=4), seed=0)
    [b] = c.blocks_plus
    rev = type(b)(q=b.q, o=b.o, v_min=b.v_min, v_max=b.v_max, degenerate=b.degenerate, row_ptr=b.row_ptr,
                  cols=b.cols[::-1].copy(), codes=b.codes)
    with pytest.raises(slicer.CorruptStreamError, match="strictly increasing"):
        slicer.decode(type(c)(**{**c.__dict__, "blocks_plus": (rev,)}))


def test_atkf_result_fields(slicer):
    x = slicer.DenseTensor(1, 6, np.array([3, -1, 0.5, -4, 2, 0.1], np.float32))
    r = slicer.atkf_filter(x, 0.5, 0.5, seed=1)
    assert (r.k_keep, r.tau, r.tau_plus, r.tau_minus) == (3, 2.0, 3.0, -1.0)
    assert list(r.filtered.values) == [3, 0, 0, -4, 2, 0]
    assert sorted(r.kept_indices.tolist()) == [0, 3, 4]
    z = slicer.atkf_filter(slicer.random_tensor(8, 8, seed=3), 1.0, 0.0, seed=1)
    assert z.k_keep == 0 and z.tau_is_fallback and not np.any(z.filtered.values)
    with pytest.raises(slicer.ConfigError):
        slicer.atkf_filter(x, -0.1, 0.0, seed=0)


def test_stream_errors(slicer):
    x = slicer.random_tensor(8, 8, seed=4)
    blob = bytearray(slicer.serialize(slicer.encode(x, slicer.CodecConfig(s=0.5, q_bit=8), seed=0)))
    bad = bytearray(blob)
    bad[len(bad) // 2] ^= 0x40
    with pytest.raises(slicer.StreamFormatError, match="CRC mismatch"):
        slicer.deserialize(bytes(bad))
    with pytest.raises(slicer.StreamFormatError, match="bad magic"):
        slicer.deserialize(b"XSIF" + bytes(blob[4:]))
    with pytest.raises(slicer.StreamFormatError, match="too short"):
        slicer.deserialize(bytes(blob[:20]))
