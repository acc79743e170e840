"""Randomized parity sweep (GPU vs the pinned oracle): 400 seeded random IFs and codec
configurations, biased to the shapes and value distributions that select different device
paths -- single-chunk IFs (warp-per-IF select), multi-chunk IFs (CTA select), heavy ties
(bf16 grids, repeated values), ReLU zeros, one-signed planes, lambda > 0, fixed-Q, extreme
s / q_bit / delta.  Every payload must equal the oracle's bytes and every decode its bits."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _values(rng, kind, t):
    if kind == 0:
        return rng.standard_normal(t).astype(np.float32)
    if kind == 1:  # bf16 grid: many exact ties
        v = (rng.standard_normal(t) * 4).astype(np.float32)
        return (v.view(np.uint32) & 0xFFFF0000).view(np.float32)
    if kind == 2:  # few distinct values
        return rng.choice(np.array([-3, -1, -0.5, 0, 0.25, 1, 2, 7], np.float32), size=t)
    if kind == 3:  # ReLU-like
        return np.maximum(rng.standard_normal(t).astype(np.float32) - 0.5, 0).astype(np.float32)
    if kind == 4:  # one sign, integer valued
        return -rng.integers(1, 50, size=t).astype(np.float32)
    return np.full(t, np.float32(rng.choice([0.0, 1.5, -2.0])), np.float32)  # constant


def _case(rng):
    if rng.random() < 0.7:
        rows, cols = int(rng.integers(1, 33)), int(rng.integers(1, 129))
    else:
        rows, cols = int(rng.integers(8, 80)), int(rng.integers(64, 400))
    kind = int(rng.choice(6, p=[0.3, 0.25, 0.15, 0.15, 0.1, 0.05]))
    x = _values(rng, kind, rows * cols).reshape(rows, cols)
    s = float(rng.choice([0.0, 1.0, rng.random(), rng.random(), rng.uniform(0.8, 0.99)]))
    lam = 0.0 if rng.random() < 0.7 else float(rng.uniform(0, 0.9))
    mp, mm = int(rng.integers(1, 5)), int(rng.integers(1, 5))
    if rng.random() < 0.1:  # many blocks (up to SIF_MAX_BLOCKS = 64 effective)
        mp, mm = int(rng.integers(5, 33)), int(rng.integers(5, 33))
    qb = int(rng.choice([1, 2, 4, 8, 8, 8, 12, 16]))
    delta = float(rng.choice([0.0, 0.01, 0.01, 0.1, 1.0]))
    fixed = ()
    if rng.random() < 0.15:
        fixed = tuple(int(v) for v in rng.integers(1, 17, size=mp + mm))
    return x, kind, dict(s=s, lam=lam, m_plus=mp, m_minus=mm, q_bit=qb, delta=delta,
                         mode="fixed_q" if fixed else "abq", fixed_q=fixed), int(rng.integers(0, 1 << 62))


def test_random_sweep_matches_oracle(sif):
    from oracle import sif_oracle as O

    rng = np.random.default_rng(20261017)
    fails = []
    for i in range(400):
        x, kind, kw, seed = _case(rng)
        ref = O.encode_bytes(x, O.Cfg(**kw), seed)
        xt = torch.from_numpy(x).cuda()
        if kind == 1 and rng.random() < 0.5:
            xt = xt.to(torch.bfloat16)  # exact: the values are on the bf16 grid
        p = sif.encode(xt, sif.CodecConfig(**kw), seed=seed)
        got = sif.serialize(p)
        if got != ref:
            fails.append(f"case {i}: shape {x.shape} kind {kind} cfg {kw} seed {seed}: payload differs "
                         f"({len(got)} vs {len(ref)} bytes)")
            continue
        y = sif.decode(p).cpu().numpy()
        if not np.array_equal(y.view(np.uint32), O.decode_bytes(ref).view(np.uint32)):
            fails.append(f"case {i}: decode differs")
    assert not fails, "\n".join(fails[:10]) + f"\n({len(fails)} failures)"


def test_path_boundaries_match_oracle(sif):
    """Shapes and keep counts at the switch points of the device paths: one chunk (4096
    elements) vs two, the warp-select capacity (1024 candidates), decode row groups of 1280
    vs 1024-column segments, single rows and single columns."""
    from oracle import sif_oracle as O

    rng = np.random.default_rng(7)
    cases = [((1, 4096), 0.75), ((1, 4096), 0.76), ((1, 4096), 0.5), ((1, 4097), 0.9), ((2, 2048), 0.9),
             ((1, 1280), 0.5), ((1, 1281), 0.5), ((3, 1279), 0.2), ((2, 1280), 0.0), ((4096, 1), 0.9),
             ((64, 64), 0.75), ((1, 1), 0.0), ((1, 1), 1.0), ((1, 2), 0.5), ((1300, 1), 0.7),
             ((2561, 2), 0.9), ((3000, 3), 0.95), ((427, 3), 0.5), ((5, 1281), 0.9)]
    fails = []
    for (r, c), s in cases:
        for kind in (0, 1):
            x = _values(rng, kind, r * c).reshape(r, c)
            kw = dict(s=s, m_plus=3, m_minus=2, q_bit=8, delta=0.01)
            ref = O.encode_bytes(x, O.Cfg(**kw), 11)
            p = sif.encode(torch.from_numpy(x).cuda(), sif.CodecConfig(**kw), seed=11)
            if sif.serialize(p) != ref:
                fails.append(f"{(r, c)} s={s} kind={kind}: payload differs")
                continue
            y = sif.decode(p).cpu().numpy()
            if not np.array_equal(y.view(np.uint32), O.decode_bytes(ref).view(np.uint32)):
                fails.append(f"{(r, c)} s={s} kind={kind}: decode differs")
    assert not fails, "\n".join(fails)


def test_multi_kernel_select_path_matches_oracle(sif):
    """IFs with more than 128K candidates take the multi-kernel select (enc_gather<1/2>,
    enc_select<1/2>, one CTA per pending cut).  One C4-shaped prefill IF (2048x4096 bf16) and
    one fp32 IF with heavy ties, batched together, must match the oracle byte for byte; the
    ATKF-only entry point (atkf_filter) must keep the oracle's indices on the same IF."""
    from oracle import sif_oracle as O
    from oracle.synth import KIND_LLM, synth

    x1 = synth(KIND_LLM, 2048, 4096, 5)  # bf16 values widened to fp32
    rng = np.random.default_rng(3)
    x2 = rng.choice(np.array([-4, -2, -1, 1, 2, 3, 5], np.float32), size=(768, 2048)).astype(np.float32)
    cfgs = [dict(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01),
            dict(s=0.8, lam=0.0, m_plus=4, m_minus=2, q_bit=6, delta=0.2),
            dict(s=0.9, lam=0.3, m_plus=2, m_minus=3, q_bit=8, delta=0.05),  # lambda > 0: generic select
            dict(s=0.85, m_plus=3, m_minus=3, q_bit=8, mode="fixed_q", fixed_q=(9, 6, 4, 8, 5, 3)),
            dict(s=0.9, m_plus=32, m_minus=31, q_bit=8, delta=0.01),  # 63 blocks: in-CTA cut-bin gather
            dict(s=0.8, lam=0.1, m_plus=20, m_minus=24, q_bit=6, delta=0.1)]
    for kw in cfgs:
        refs = [O.encode_bytes(x, O.Cfg(**kw), sd) for x, sd in ((x1, 5), (x2, 6))]
        xs = [torch.from_numpy(x1).cuda().to(torch.bfloat16), torch.from_numpy(x2).cuda()]
        ps = sif.encode_list(xs, sif.CodecConfig(**kw), [5, 6])
        for p, ref, name in zip(ps, refs, ("prefill", "ties")):
            assert p.to_bytes() == ref, f"{name} {kw}: payload differs"
        ys = sif.decode_list(ps)
        for y, ref in zip(ys, refs):
            assert np.array_equal(y.cpu().numpy().view(np.uint32), O.decode_bytes(ref).view(np.uint32))
    a = sif.atkf_filter(torch.from_numpy(x1).cuda().to(torch.bfloat16), 0.9, 0.0, 5)
    ra = O.atkf(x1.reshape(-1), 0.9, 0.0, 5)
    assert np.array_equal(a.kept_indices.cpu().numpy(), ra.kept)
    assert a.tau == ra.tau


def test_bracket_miss_restream_matches_oracle():
    """The sampled tau bracket of enc_prep is speculative; when it misses (fewer than k
    elements above it) enc_select re-streams the IF with every nonzero as a candidate.  The
    miss is forced here (SIF_TEST_INJECT=1, read per launch by the library) on multi-chunk
    IFs, including one that then exceeds the multi-kernel threshold; payloads must still
    equal the oracle's.  Runs in a subprocess so the injection cannot leak."""
    import subprocess
    import sys

    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2511_11608_b200 as sif
from oracle import sif_oracle as O
rng = np.random.default_rng(11)
xs = [rng.standard_normal((300, 200)).astype(np.float32),
      np.maximum(rng.standard_normal((1024, 196)).astype(np.float32) - 0.3, 0).astype(np.float32),
      rng.choice(np.array([-3, -1, 1, 2, 4], np.float32), size=(600, 1024)).astype(np.float32)]
kw = dict(s=0.9, m_plus=3, m_minus=2, q_bit=8, delta=0.01)
ps = sif.encode_list([torch.from_numpy(x).cuda() for x in xs], sif.CodecConfig(**kw), [1, 2, 3])
for p, x, sd in zip(ps, xs, (1, 2, 3)):
    assert p.to_bytes() == O.encode_bytes(x, O.Cfg(**kw), sd), sd
print("ok")
"""
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SIF_TEST_INJECT="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]


def _tie_cut_if(a_big, rows, cols, seed):
    """A plus plane whose MS cut (rank base, M+ = 2) is the LAST element of a tie group
    larger than the exact-ranking capacity (1024): A distinct values above 1, 1500 copies
    of 1.0, A + 1498 distinct values below 1; everything else 0 and s chosen so exactly
    these are kept."""
    rng = np.random.default_rng(seed)
    big = (1.0 + (np.arange(a_big) + 1) * 2.0 ** -12).astype(np.float32)
    ties = np.ones(1500, np.float32)
    small = (0.1 + np.arange(a_big + 1498) * (0.8 / (a_big + 1498))).astype(np.float32)
    vals = np.concatenate([big, ties, small])
    x = np.zeros(rows * cols, np.float32)
    x[rng.permutation(rows * cols)[: vals.size]] = vals
    k = vals.size
    s = 1.0 - (k + 0.5) / (rows * cols)  # floor((1 - s) T + 1e-9) == k
    return x.reshape(rows, cols), s


def test_ms_cut_at_last_element_of_large_tie_group(sif):
    """Regression (found by the C5 workload parity, stream 6055): an MS cut that lands on
    the last member of a tie group with more than 1024 members must still place the block
    boundary at that member's flat index (msplit.py:64) -- single-CTA select and the
    multi-kernel select of large IFs, lambda = 0 and lambda > 0."""
    from oracle import sif_oracle as O

    for a_big, rows, cols in ((1000, 300, 200), (32000, 2048, 64)):
        x, s = _tie_cut_if(a_big, rows, cols, a_big)
        for lam in (0.0, 0.05):
            kw = dict(s=s, lam=lam, m_plus=2, m_minus=1, q_bit=8, delta=0.01)
            ref = O.encode_bytes(x, O.Cfg(**kw), 3)
            p = sif.encode(torch.from_numpy(x).cuda(), sif.CodecConfig(**kw), seed=3)
            assert p.to_bytes() == ref, (a_big, lam)


def test_per_if_back_end_matches_oracle(sif):
    """The opt-in per-IF encoder back end (sif_set_fused_range; enc_post) on C2-shaped IFs,
    a bracket-miss IF (fault injection off: heavy ties force many candidates), lambda > 0,
    fixed-Q, delta large enough to descend and 30 + 30 blocks: byte-identical to the oracle."""
    import ctypes

    from oracle import sif_oracle as O
    from oracle.synth import synth

    L = sif._lib.load()
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    L.sif_get_fused_range(ctypes.byref(lo), ctypes.byref(hi))
    L.sif_set_fused_range(4097, 1 << 20)
    try:
        rng = np.random.default_rng(17)
        xs = [synth(0, 1024, 196, 3), synth(1, 64, 4096, 4),
              rng.choice(np.array([-3, -1, 1, 2, 4], np.float32), size=(300, 200)).astype(np.float32),
              rng.standard_normal((100, 97)).astype(np.float32)]
        cfgs = [dict(s=0.9, m_plus=3, m_minus=3, q_bit=8, delta=0.01),
                dict(s=0.8, lam=0.2, m_plus=2, m_minus=3, q_bit=8, delta=0.05),
                dict(s=0.7, m_plus=4, m_minus=4, q_bit=6, delta=0.5),
                dict(s=0.85, m_plus=3, m_minus=3, q_bit=8, mode="fixed_q", fixed_q=(9, 6, 4, 8, 5, 3)),
                dict(s=0.8, m_plus=30, m_minus=30, q_bit=7, delta=0.3)]
        for kw in cfgs:
            ps = sif.encode_list([torch.from_numpy(x).cuda() for x in xs], sif.CodecConfig(**kw), [5, 6, 7, 8])
            for p, x, sd in zip(ps, xs, (5, 6, 7, 8)):
                assert p.to_bytes() == O.encode_bytes(x, O.Cfg(**kw), sd), (kw, x.shape)
    finally:
        L.sif_set_fused_range(lo.value, hi.value)


def test_stream_ring_tails_match_oracle(sif):
    """IFs whose size is not a whole number of 16-byte vectors (fp32 T % 4 != 0, bf16 T % 8
    != 0) and whose last chunk is a few elements long: the stream kernel's bulk-copy ring
    copies the tail with plain loads (nothing past the IF is read).  fp32 and bf16 inputs,
    lambda = 0 and lambda > 0."""
    from oracle import sif_oracle as O

    rng = np.random.default_rng(21)
    shapes = [(1, 4097), (3, 2731), (2, 4099), (5, 1639), (7, 1171), (1, 8195), (13, 631), (4099, 3)]
    fails = []
    for (r, c) in shapes:
        for dt in (torch.float32, torch.bfloat16):
            for lam in (0.0, 0.2):
                x = torch.from_numpy(_values(rng, 1, r * c).reshape(r, c)).to(dt)
                xf = x.float().numpy()
                kw = dict(s=0.8, lam=lam, m_plus=3, m_minus=3, q_bit=8, delta=0.01)
                ref = O.encode_bytes(xf, O.Cfg(**kw), 5)
                p = sif.encode(x.cuda(), sif.CodecConfig(**kw), seed=5)
                if sif.serialize(p) != ref:
                    fails.append(f"{(r, c)} {dt} lam={lam}: payload differs")
    assert not fails, "\n".join(fails)
