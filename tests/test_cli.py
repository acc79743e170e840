"""CLI drop-in: the reference CLI's transcript (tests/golden/cli.json,
made by tests/golden/make_cli_golden.py with slicer-codec 0.1.0) replayed through
`paper_2511_11608_b200.cli` on the GPU: same exit codes, same stdout (text and --json), the
same bytes in every written .tns / .sif file, and the same first stderr line on errors.
Covers gen (uniform + gaussian fixtures generated on the device), encode (ABQ, lambda,
fixed-Q), decode (--ref error statistics), stats (exact + upper-bound bits)."""

import hashlib
import json
import os

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


@pytest.mark.gpu
def test_cli_transcript_matches_reference(tmp_path, monkeypatch):
    from click.testing import CliRunner

    from paper_2511_11608_b200.cli import main

    with open(os.path.join(HERE, "golden", "cli.json")) as f:
        cases = json.load(f)
    monkeypatch.chdir(tmp_path)
    runner = CliRunner(mix_stderr=False)
    fails = []
    for c in cases:
        r = runner.invoke(main, c["args"], catch_exceptions=False)
        tag = " ".join(c["args"][:3])
        if r.exit_code != c["rc"]:
            fails.append(f"{tag}: rc {r.exit_code} vs {c['rc']} ({r.stderr.strip()[:200]})")
            continue
        if r.stdout != c["stdout"]:
            fails.append(f"{tag}: stdout differs:\n{r.stdout[:400]}\n--- reference:\n{c['stdout'][:400]}")
        if c["rc"] and r.stderr.splitlines()[:1] != c["stderr_first"]:
            fails.append(f"{tag}: stderr {r.stderr.splitlines()[:1]} vs {c['stderr_first']}")
        for name, meta in c["files"].items():
            if not os.path.exists(name):
                fails.append(f"{tag}: {name} missing")
            elif _sha(name) != meta["sha256"]:
                fails.append(f"{tag}: {name} differs ({os.path.getsize(name)} vs {meta['size']} bytes)")
    assert not fails, "\n".join(fails)


@pytest.mark.gpu
def test_fixture_tensors_and_tns_io(tmp_path):
    """random_tensor on the device vs the reference values pinned by the transcript's files,
    .tns round trip, and load_tensor's error classes (tensor.py:66-87)."""
    import struct

    import torch

    import paper_2511_11608_b200 as sif

    x = sif.random_tensor(32, 32, 7)
    p = tmp_path / "a.tns"
    sif.save_tensor(x, p)
    with open(os.path.join(HERE, "golden", "cli.json")) as f:
        ref = json.load(f)[0]["files"]["a.tns"]["sha256"]
    assert _sha(p) == ref
    y = sif.load_tensor(p)
    assert torch.equal(x, y)
    bad = tmp_path / "bad.tns"
    bad.write_bytes(b"TNS1" + struct.pack("<HII", 1, 1, 2) + struct.pack("<ff", 1.0, float("inf")))
    with pytest.raises(sif.NonFiniteError):
        sif.load_tensor(bad)
    bad.write_bytes(b"TNS1" + struct.pack("<HII", 1, 2, 2) + b"\0" * 8)
    with pytest.raises(sif.TensorFormatError, match="truncated payload"):
        sif.load_tensor(bad)
    bad.write_bytes(b"TNS1" + struct.pack("<HII", 1, 0, 2))
    with pytest.raises(sif.ShapeError):
        sif.load_tensor(bad)
    bad.write_bytes(b"TNS2" + struct.pack("<HII", 1, 1, 1) + b"\0" * 4)
    with pytest.raises(sif.TensorFormatError, match="bad magic"):
        sif.load_tensor(bad)
    with pytest.raises(ValueError):
        sif.random_tensor(2, 2, 0, "laplace")
    # large uniform tensor: spot values against the splitmix64 recurrence (rng.py:30-45)
    big = sif.random_tensor(1000, 1000, 123).reshape(-1).cpu()
    M = (1 << 64) - 1

    def mix(z):
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    import numpy as np

    for i in (0, 1, 2, 777, 999_999):
        u = mix((123 + (i + 1) * 0x9E3779B97F4A7C15) & M)
        assert big[i].item() == float(np.float32(-1.0 + 2.0 * (u / 2.0**64))), i


@pytest.mark.gpu
def test_calibrated_time_model(tmp_path):
    """calibrate() measures the three stage tables on the GPU and writes the reference's
    JSON schema (profiles.py:184-254); the planner estimate is positive and monotone in M."""
    import paper_2511_11608_b200 as sif
    from paper_2511_11608_b200.timemodel import calibrate

    m = calibrate(rows=256, cols=196, batch=8, s_grid=(0.5, 0.9), m_grid=((1, 1), (3, 3)), q_grid=(4, 8), reps=2)
    p = tmp_path / "tm.json"
    m.save(p)
    with open(p) as f:
        d = json.load(f)
    assert {"t_atkf", "t_ms", "t_abq", "m_buf_bytes"} <= set(d)
    m2 = sif.DeviceTimeModel.load(p)
    assert all(v > 0 for v in m2.t_atkf.values()) and all(v > 0 for v in m2.t_ms.values())
    assert all(v > 0 for v in m2.t_abq.values())
    est = m2.encode_time_estimate(sif.CodecConfig(s=0.9, m_plus=3, m_minus=3))
    assert est > 0
