"""Integer-exact synthetic IF generator (NumPy side).  TEST/BENCH INFRASTRUCTURE ONLY.

Bit-identical to the device generator `sif_gen_synthetic` in
`paper_2511_11608_b200/csrc/sif_synth.cu`:

    u = splitmix(seed=sid, i)                       (rng.py:55-57 hash_index)
    z = sum_{j<4} ((u >> 16j) & 0xFFFF) - 131070     Irwin-Hall, sd ~ 37,837
    g = z * 2^-15                                    exact in fp32
    resnet: x[c, hw] = max(0, g + b_c),  b_c = -(c mod 4)/4
    llm:    x[t, h]  = bf16_rne(g * a_h), a_h = 32 on 8 outlier channels
            h = splitmix(sid ^ 0xA5, j) mod K (j < 8), else 1
"""

import numpy as np

from .sif_oracle import splitmix_keys

KIND_RESNET = 0
KIND_LLM = 1


def _gauss(sid: int, t: int) -> np.ndarray:
    u = splitmix_keys(sid, np.arange(t, dtype=np.uint64))
    z = np.zeros(t, dtype=np.int64)
    for j in range(4):
        z += ((u >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.int64)
    z -= 131070
    return (z.astype(np.float32) * np.float32(2.0 ** -15)).astype(np.float32)


def bf16_rne(x: np.ndarray) -> np.ndarray:
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


def synth(kind: int, n: int, k: int, sid: int) -> np.ndarray:
    """Returns an (n, k) float32 array (bf16-valued for the LLM kind)."""
    g = _gauss(sid, n * k).reshape(n, k)
    if kind == KIND_RESNET:
        bias = -(np.arange(n) % 4).astype(np.float32) / np.float32(4.0)
        return np.maximum(g + bias[:, None], np.float32(0.0)).astype(np.float32)
    if kind == KIND_LLM:
        a = np.ones(k, dtype=np.float32)
        out_ch = splitmix_keys(sid ^ 0xA5, np.arange(8, dtype=np.uint64)) % np.uint64(k)
        a[out_ch.astype(np.int64)] = 32.0
        return bf16_rne(g * a[None, :])
    raise ValueError(kind)
