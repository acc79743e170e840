"""Pin the CPU oracle (oracle/sif_oracle.py) to golden vectors produced by the reference."""

import hashlib

import numpy as np
import pytest

from oracle import sif_oracle as O
from tests.golden_util import case_cfg, case_x


def _sha(b):
    return hashlib.sha256(b).hexdigest()


def test_oracle_matches_reference_payloads(golden):
    meta, arrays = golden
    for i, c in enumerate(meta["cases"]):
        x = case_x(i, c, arrays)
        cfg = case_cfg(c)
        blob = O.encode_bytes(x, cfg, c["seed"])
        assert len(blob) == c["payload_len"], c["name"]
        assert _sha(blob) == c["payload_sha"], c["name"]
        a = O.atkf(x.reshape(-1), cfg.s, cfg.lam, c["seed"])
        assert _sha(a.kept.tobytes()) == c["kept_sha"], c["name"]
        assert a.k_keep == c["k_keep"] and a.tau == c["tau"], c["name"]
        dec = O.decode_bytes(blob)
        assert _sha(dec.reshape(-1).view(np.uint32).tobytes()) == c["dec_sha"], c["name"]
        assert O.payload_bytes(O.deserialize(blob)) == len(blob)


def test_oracle_matches_reference_error_classes(golden):
    meta, arrays = golden
    for j, b in enumerate(meta["corrupt"]):
        data = arrays[f"bad{j}"].tobytes()
        _, kind = O.status_of(O.decode_bytes, data)
        assert kind == b["error"], (j, b)
        _, kind = O.status_of(O.deserialize, data)
        assert kind == b["deser_error"], (j, b)


def test_worked_example_hex():
    # full .sif hex of the 1x6 worked example.
    x = np.array([[3, -1, 0.5, -4, 2, 0.1]], dtype=np.float32)
    blob = O.encode_bytes(x, O.Cfg(s=0.5, q_bit=4, delta=0.0), seed=1)
    assert blob.hex() == (
        "53494631010001000000060000000000003f0000000004000000000001000100010000803f000000400200000000"
        "000000020000001080010000803f0000804001000000000000000100000060007fba913f")


def test_known_answers():
    # tests/test_quant.py:24-33, :84-86, :109-112 (reference known-answer tests)
    assert O.aiq(np.array([0.5, 1.5, 2.5]), 2)[0].tolist() == [0, 2, 3]
    assert O.aiq(np.array([0.5, 0.9, 1.5, 2.5]), 4)[0].tolist() == [0, 3, 8, 15]
    assert O.ds(np.array([0, 3, 8, 15]), 4, np.array([0, 1, 2, 3]), 2) == 0.25
    assert O.abq(np.array([0.5, 0.9, 1.5, 2.5]), 4, 0.1)[0] == 3
    assert O.col_bits(1) == 1 and O.col_bits(2) == 1 and O.col_bits(257) == 9
    a = O.atkf(np.array([3, -1, 0.5, -4, 2, 0.1], np.float32), 0.5, 0.5, 1)
    assert a.tau == 2.0 and a.tau_plus == 3.0 and a.tau_minus == -1.0
    assert a.kept.tolist() == [0, 3, 4]


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(0)
    for w in range(1, 33):
        v = rng.integers(0, 2 ** w, size=37, dtype=np.uint64).astype(np.uint32)
        assert np.array_equal(O.unpack_bits(O.pack_bits(v, w), 37, w), v)


def _structural():
    import os
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "structural.npz"))
    return d, [str(n) for n in d["names"]]


def test_oracle_structural_streams():
    """Hand-built streams (cross-plane overlap, corrupt CSR) decoded by the reference."""
    d, names = _structural()
    for n in names:
        data = d[f"{n}_blob"].tobytes()
        err = d[f"{n}_err"].tobytes().decode()
        _, kind = O.status_of(O.decode_bytes, data)
        if err:
            assert kind == err, n
        else:
            assert kind is None, (n, kind)
            y = O.decode_bytes(data)
            assert np.array_equal(y.reshape(-1).view(np.uint32), d[f"{n}_dec"].reshape(-1).view(np.uint32)), n


def _wide():
    import os

    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "wide.npz"))
    return d, [str(n) for n in d["names"]]


def test_oracle_matches_reference_many_blocks():
    """Many-block configurations (up to 64 effective blocks, tests/golden/make_wide_golden.py),
    including the two 1M-element cases pinned by SHA-256 of the reference's payload and decode."""
    from oracle.synth import synth

    d, names = _wide()
    for n in names:
        s, lam, mp, mm, qb, dl, seed = d[f"{n}_cfg"]
        cfg = O.Cfg(s=float(s), lam=float(lam), m_plus=int(mp), m_minus=int(mm), q_bit=int(qb), delta=float(dl))
        blob = O.encode_bytes(d[f"{n}_x"], cfg, int(seed))
        assert blob == d[f"{n}_blob"].tobytes(), n
        assert np.array_equal(O.decode_bytes(blob).reshape(-1).view(np.uint32), d[f"{n}_dec"].reshape(-1)), n
    for n in [str(x) for x in d["big_names"]]:
        kind, r, c = (int(v) for v in d[f"{n}_shape"])
        s, lam, mp, mm, qb, dl, seed = d[f"{n}_cfg"]
        cfg = O.Cfg(s=float(s), lam=float(lam), m_plus=int(mp), m_minus=int(mm), q_bit=int(qb), delta=float(dl))
        blob = O.encode_bytes(synth(kind, r, c, int(seed)).astype(np.float32), cfg, int(seed))
        assert hashlib.sha256(blob).hexdigest() == str(d[f"{n}_blob_sha"]), n
        y = np.ascontiguousarray(O.decode_bytes(blob), np.float32)
        assert hashlib.sha256(y.view(np.uint32).tobytes()).hexdigest() == str(d[f"{n}_dec_sha"]), n
