"""CPU oracle for the SLICER IF codec (ATKF -> MS -> ABQ -> CSR -> .sif, and back).

TEST INFRASTRUCTURE ONLY.  Nothing in the product package (`paper_2511_11608_b200/`)
imports this module.  It is used by `tests/` as the parity checker, by
`__graft_entry__.smoke()` as the checker, and by `bench.py` as the CPU baseline
(the `cpu_baseline` leg and `--impl reference`).

This is a NumPy restatement of the reference algorithm in
`/root/reference/pkg/src/slicer/` (slicer-codec 0.1.0, pure Python + NumPy).  Each
function cites the reference file:line it follows.  The restatement is pinned by
`tests/golden/*.npz`, which were produced by running the reference itself in the
build container (`tests/golden/make_golden.py`); see `tests/test_oracle_golden.py`.

Differences from the reference are purely structural (vectorised bit packing instead
of the per-field BitWriter/BitReader loops, plain tuples instead of dataclasses);
the arithmetic (float64 ops, stable sorts, zlib CRC-32) is the same.
"""

from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

# --- constants (codec.py:44-54, quant.py:21) ---------------------------------------
MAGIC = b"SIF1"
VERSION = 1
MODE_ABQ = "abq"
MODE_FIXED = "fixed_q"
MODE_CODE = {MODE_ABQ: 0, MODE_FIXED: 1}
HEADER_BYTES = 32
BLOCK_META_BYTES = 13
CRC_BYTES = 4
Q_MAX = 16
GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


class OracleError(Exception):
    """Base of the oracle's error taxonomy; `kind` mirrors slicer/errors.py:4-37."""

    kind = "SlicerError"


class ConfigErr(OracleError):
    kind = "ConfigError"


class NonFiniteErr(OracleError):
    kind = "NonFiniteError"


class ShapeErr(OracleError):
    kind = "ShapeError"


class StreamFormatErr(OracleError):
    kind = "StreamFormatError"


class CorruptStreamErr(StreamFormatErr):
    kind = "CorruptStreamError"


# --- config (codec.py:61-92) ----------------------------------------------------------
@dataclass(frozen=True)
class Cfg:
    s: float
    lam: float = 0.0
    m_plus: int = 1
    m_minus: int = 1
    q_bit: int = 8
    delta: float = 0.01
    mode: str = MODE_ABQ
    fixed_q: tuple = ()

    def __post_init__(self):
        if not 0.0 <= self.s <= 1.0:
            raise ConfigErr("s out of range")
        if not 0.0 <= self.lam < 1.0:
            raise ConfigErr("lambda out of range")
        if self.m_plus < 1 or self.m_minus < 1:
            raise ConfigErr("block counts must be >= 1")
        if not 1 <= self.q_bit <= Q_MAX:
            raise ConfigErr("q_bit out of range")
        if self.delta < 0:
            raise ConfigErr("delta < 0")
        if self.mode not in MODE_CODE:
            raise ConfigErr("unknown mode")
        if self.mode == MODE_FIXED:
            if len(self.fixed_q) != self.m_plus + self.m_minus:
                raise ConfigErr("fixed_q length")
            if any(not 1 <= int(q) <= Q_MAX for q in self.fixed_q):
                raise ConfigErr("fixed_q entry out of range")


def col_bits(k: int) -> int:
    """codec.py:57-58."""
    return max(1, (k - 1).bit_length())


def keep_count(s: float, t: int) -> int:
    """atkf.py:31-34: floor((1-s)*T + 1e-9) in float64."""
    return int(np.floor((1.0 - s) * t + 1e-9))


# --- splitmix64 tie-break keys (rng.py:23-27, :60-68) ------------------------------
def splitmix_keys(seed: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def splitmix_key(seed: int, i: int) -> int:
    z = (seed + (i + 1) * GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


# --- ATKF (atkf.py:37-96) -----------------------------------------------------------
@dataclass
class Atkf:
    kept: np.ndarray  # sorted int64 flat indices
    tau: float
    tau_plus: float
    tau_minus: float
    k_keep: int
    tau_is_fallback: bool


def atkf(x: np.ndarray, s: float, lam: float, seed: int) -> Atkf:
    """Exact-cardinality asymmetric top-K; ties broken by splitmix64 key asc."""
    if not 0.0 <= s <= 1.0:
        raise ConfigErr("s")
    if not 0.0 <= lam < 1.0:
        raise ConfigErr("lam")
    v = x.reshape(-1).astype(np.float32)
    v64 = v.astype(np.float64)
    if not np.all(np.isfinite(v64)):  # atkf.py:49-51
        raise NonFiniteErr("input tensor contains NaN or Inf")
    t = v.size
    k = keep_count(s, t)
    mag = np.abs(v64)
    if k == 0:  # atkf.py:57-68
        tau = float(mag.max())
        return Atkf(np.empty(0, np.int64), tau, (1.0 + lam) * tau, -(1.0 - lam) * tau, 0, True)
    tau = float(np.partition(mag, t - k)[t - k])  # atkf.py:71
    tp = (1.0 + lam) * tau
    tm = -(1.0 - lam) * tau
    strict = (v64 > tp) | (v64 < tm)  # atkf.py:75

    def order(ix):  # atkf.py:37-41: |x| desc, splitmix key asc
        return ix[np.lexsort((splitmix_keys(seed, ix), -mag[ix]))]

    s_ix = np.flatnonzero(strict)
    if s_ix.size >= k:
        kept = order(s_ix)[:k]
    else:
        pool = order(np.flatnonzero(~strict))
        kept = np.concatenate([s_ix, pool[: k - s_ix.size]])
    return Atkf(np.sort(kept.astype(np.int64)), tau, tp, tm, k, False)


# --- magnitude split + CSR (msplit.py:48-133) --------------------------------------
def plane_blocks(filtered: np.ndarray, m: int, sign: float):
    """One sign plane: returns list of (flat_idx_csr_order, values_csr_order)."""
    plane = np.maximum(sign * filtered, np.float32(0.0))  # msplit.py:48-51
    nz = np.flatnonzero(plane)
    vals = plane[nz]
    o = np.lexsort((nz, -vals.astype(np.float64)))  # msplit.py:64: value desc, idx asc
    nz, vals = nz[o], vals[o]
    n = nz.size
    m_eff = max(1, min(m, n))  # msplit.py:68-80
    base = n // m_eff
    out = []
    for b in range(m_eff):
        lo = b * base
        hi = lo + base if b < m_eff - 1 else n
        f, w = nz[lo:hi], vals[lo:hi]
        so = np.argsort(f, kind="stable")  # msplit.py:93
        out.append((f[so].astype(np.int64), w[so]))
    return out


def csr_row_ptr(flat: np.ndarray, n_rows: int, k: int) -> np.ndarray:
    """msplit.py:97-100: exclusive prefix of per-row counts, u32[N+1]."""
    cnt = np.bincount(flat // k, minlength=n_rows) if flat.size else np.zeros(n_rows, np.int64)
    rp = np.zeros(n_rows + 1, dtype=np.uint64)
    rp[1:] = np.cumsum(cnt, dtype=np.uint64)
    return rp.astype(np.uint32)


# --- AIQ / DS / ABQ (quant.py:44-115) -------------------------------------------------
def aiq(values: np.ndarray, q: int):
    """Returns (codes u32, o64-rounded-to-f32, v_min f32, degenerate)."""
    vals = np.asarray(values, dtype=np.float64)
    v_min = np.float32(vals.min())
    v_max = np.float32(vals.max())
    levels = (1 << q) - 1
    if v_max == v_min:  # quant.py:54-56
        return np.zeros(vals.size, np.uint32), np.float32(1.0), v_min, True
    o64 = (np.float64(v_max) - np.float64(v_min)) / levels  # quant.py:59
    codes = np.floor((vals - np.float64(v_min)) / o64 + 0.5)  # quant.py:60-61
    codes = np.clip(codes, 0, levels).astype(np.uint32)  # quant.py:62
    return codes, np.float32(o64), v_min, False


def ds(ref: np.ndarray, q1: int, cand: np.ndarray, q2: int) -> float:
    """quant.py:88-99: mean |(ref >> (q1-q2)) - cand| (int64 sum, float64 divide)."""
    a = ref.astype(np.int64) >> (q1 - q2)
    return float(np.abs(a - cand.astype(np.int64)).sum() / ref.size)


def abq(values: np.ndarray, q_bit: int, delta: float):
    """quant.py:102-115: descend from q_bit, stop at the first DS > delta."""
    ref = aiq(values, q_bit)
    best_q, best = q_bit, ref
    for q in range(q_bit - 1, 0, -1):
        cand = aiq(values, q)
        if ds(ref[0], q_bit, cand[0], q) > delta:
            break
        best_q, best = q, cand
    return best_q, best


# --- encode (codec.py:175-232) -------------------------------------------------------
@dataclass
class Block:
    q: int
    o: np.float32
    v_min: np.float32
    row_ptr: np.ndarray
    cols: np.ndarray
    codes: np.ndarray

    @property
    def nnz(self):
        return int(self.codes.size)


@dataclass
class Encoded:
    rows: int
    cols: int
    s32: np.float32
    lam32: np.float32
    q_bit: int
    delta32: np.float32
    mode: str
    blocks_plus: list
    blocks_minus: list
    q_vector: tuple = field(default=())


def encode(x: np.ndarray, cfg: Cfg, seed: int = 0) -> Encoded:
    if x.ndim != 2 or x.shape[0] < 1 or x.shape[1] < 1:
        raise ShapeErr("IF must be a non-empty 2-D tensor")
    n, k = x.shape
    xf = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    if not np.all(np.isfinite(xf)):
        raise NonFiniteErr("tensor contains NaN or Inf")
    a = atkf(xf, cfg.s, cfg.lam, seed)
    filtered = np.zeros_like(xf)
    filtered[a.kept] = xf[a.kept]
    planes = []
    q_used = []
    for sign, m, segment in ((1.0, cfg.m_plus, cfg.fixed_q[: cfg.m_plus]),
                             (-1.0, cfg.m_minus, cfg.fixed_q[cfg.m_plus:])):
        blocks = []
        for i, (flat, vals) in enumerate(plane_blocks(filtered, m, sign)):
            qf = int(segment[i]) if cfg.mode == MODE_FIXED else None
            if vals.size == 0:  # codec.py:176-179
                q = cfg.q_bit if qf is None else qf
                codes, o, vmin = np.zeros(0, np.uint32), np.float32(1.0), np.float32(0.0)
            elif qf is not None:
                q = qf
                codes, o, vmin, _ = aiq(vals, q)
            else:
                q, (codes, o, vmin, _) = abq(vals, cfg.q_bit, cfg.delta)
            blocks.append(Block(q, o, vmin, csr_row_ptr(flat, n, k),
                                (flat % k).astype(np.uint32), codes))
            if cfg.mode == MODE_FIXED:
                q_used.append(q)
        planes.append(blocks)
    return Encoded(n, k, np.float32(cfg.s), np.float32(cfg.lam), cfg.q_bit, np.float32(cfg.delta),
                   cfg.mode, planes[0], planes[1], tuple(q_used))


def payload_bytes(e: Encoded) -> int:
    """codec.py:269-280 (in bytes)."""
    cb = col_bits(e.cols)
    total = HEADER_BYTES + (len(e.q_vector) if e.mode == MODE_FIXED else 0)
    for b in e.blocks_plus + e.blocks_minus:
        total += BLOCK_META_BYTES + 4 * (e.rows + 1) + (b.nnz * cb + 7) // 8 + (b.nnz * b.q + 7) // 8
    return total + CRC_BYTES


# --- bit packing (bitstream.py: MSB-first, zero pad to byte) -----------------------
def pack_bits(values: np.ndarray, w: int) -> bytes:
    if values.size == 0:
        return b""
    v = values.astype(np.uint64)
    if np.any(v >> np.uint64(w)):
        raise ValueError("value does not fit")
    shifts = np.arange(w - 1, -1, -1, dtype=np.uint64)
    bits = ((v[:, None] >> shifts[None, :]) & np.uint64(1)).astype(np.uint8).reshape(-1)
    return np.packbits(bits).tobytes()


def unpack_bits(buf: bytes, n: int, w: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0, np.uint32)
    bits = np.unpackbits(np.frombuffer(buf, dtype=np.uint8))[: n * w].reshape(n, w)
    weights = (np.uint64(1) << np.arange(w - 1, -1, -1, dtype=np.uint64))
    return (bits.astype(np.uint64) * weights[None, :]).sum(axis=1).astype(np.uint32)


# --- serialize (codec.py:283-317) ----------------------------------------------------
def serialize(e: Encoded) -> bytes:
    body = bytearray(struct.pack("<HIIffBfBHH", VERSION, e.rows, e.cols, e.s32, e.lam32, e.q_bit,
                                 e.delta32, MODE_CODE[e.mode], len(e.blocks_plus),
                                 len(e.blocks_minus)))
    if e.mode == MODE_FIXED:
        body += bytes(int(q) for q in e.q_vector)
    cb = col_bits(e.cols)
    for b in e.blocks_plus + e.blocks_minus:
        body += struct.pack("<BffI", b.q, b.o, b.v_min, b.nnz)
        body += b.row_ptr.astype("<u4").tobytes()
        body += pack_bits(b.cols, cb)
        body += pack_bits(b.codes, b.q)
    return MAGIC + bytes(body) + struct.pack("<I", zlib.crc32(bytes(body)) & 0xFFFFFFFF)


def encode_bytes(x: np.ndarray, cfg: Cfg, seed: int = 0) -> bytes:
    return serialize(encode(x, cfg, seed))


# --- deserialize (codec.py:320-399) --------------------------------------------------
def deserialize(data: bytes) -> Encoded:
    if len(data) < HEADER_BYTES + CRC_BYTES:
        raise StreamFormatErr("too short")
    if data[:4] != MAGIC:
        raise StreamFormatErr("bad magic")
    (crc,) = struct.unpack_from("<I", data, len(data) - 4)
    if zlib.crc32(data[4:-4]) & 0xFFFFFFFF != crc:
        raise StreamFormatErr("CRC mismatch")
    ver, n, k, s, lam, qb, dl, mc, mp, mm = struct.unpack_from("<HIIffBfBHH", data, 4)
    if ver != VERSION:
        raise StreamFormatErr("version")
    if mc not in (0, 1):
        raise StreamFormatErr("mode")
    mode = MODE_ABQ if mc == 0 else MODE_FIXED
    pos = HEADER_BYTES
    qv = ()
    if mode == MODE_FIXED:
        if len(data) < pos + mp + mm:
            raise StreamFormatErr("truncated Q vector")
        qv = tuple(data[pos: pos + mp + mm])
        pos += mp + mm
    cb = col_bits(k)
    blocks = []
    for _ in range(mp + mm):
        if len(data) < pos + BLOCK_META_BYTES + 4 * (n + 1):
            raise StreamFormatErr("truncated block header")
        q, o, vmin, nnz = struct.unpack_from("<BffI", data, pos)
        if not 1 <= q <= Q_MAX:
            raise CorruptStreamErr("bit-width out of range")
        pos += BLOCK_META_BYTES
        rp = np.frombuffer(data, dtype="<u4", count=n + 1, offset=pos).astype(np.uint32)
        pos += 4 * (n + 1)
        cbytes, qbytes = (nnz * cb + 7) // 8, (nnz * q + 7) // 8
        if len(data) - CRC_BYTES < pos + cbytes + qbytes:
            raise StreamFormatErr("truncated block payload")
        cols = unpack_bits(data[pos: pos + cbytes], nnz, cb)
        codes = unpack_bits(data[pos + cbytes: pos + cbytes + qbytes], nnz, q)
        pos += cbytes + qbytes
        blocks.append(Block(int(q), np.float32(o), np.float32(vmin), rp, cols, codes))
    if pos != len(data) - CRC_BYTES:
        raise StreamFormatErr("trailing bytes")
    return Encoded(n, k, np.float32(s), np.float32(lam), qb, np.float32(dl), mode,
                   blocks[:mp], blocks[mp:], qv)


# --- decode (codec.py:235-266, quant.py:67-73) --------------------------------------
def _csr_flat(b: Block, k: int) -> np.ndarray:
    cnt = np.diff(b.row_ptr.astype(np.int64))
    return np.repeat(np.arange(cnt.size, dtype=np.int64), cnt) * k + b.cols.astype(np.int64)


def decode(e: Encoded) -> np.ndarray:
    n, k = e.rows, e.cols
    flat = np.zeros(n * k, dtype=np.float64)
    for sign, blocks in ((1.0, e.blocks_plus), (-1.0, e.blocks_minus)):
        seen = np.zeros(n * k, dtype=bool)
        for b in blocks:  # codec.py:235-251
            rp = b.row_ptr.astype(np.int64)
            if rp.size != n + 1 or rp[0] != 0:
                raise CorruptStreamErr("bad row pointer array")
            if rp[-1] != b.nnz or np.any(np.diff(rp) < 0):
                raise CorruptStreamErr("row pointers inconsistent")
            if b.nnz and int(b.cols.max()) >= k:
                raise CorruptStreamErr("column out of range")
            c64 = b.cols.astype(np.int64)
            same_row = np.repeat(np.arange(n), np.diff(rp))
            if b.nnz > 1 and np.any((np.diff(c64) <= 0) & (same_row[1:] == same_row[:-1])):
                raise CorruptStreamErr("columns not strictly increasing")
            idx = _csr_flat(b, k)
            if np.any(seen[idx]):
                raise CorruptStreamErr("overlap")
            seen[idx] = True
        for b in blocks:
            if b.nnz == 0:
                continue
            vals = b.codes.astype(np.float64) * np.float64(b.o) + np.float64(b.v_min)
            flat[_csr_flat(b, k)] += sign * vals
    if n < 1 or k < 1:
        raise ShapeErr("degenerate shape")
    out = flat.astype(np.float32)
    if not np.all(np.isfinite(out)):
        raise NonFiniteErr("decoded tensor contains NaN or Inf")
    return out.reshape(n, k)


def decode_bytes(data: bytes) -> np.ndarray:
    return decode(deserialize(data))


def status_of(fn, *args):
    """Run fn and return (result, error-kind-or-None)."""
    try:
        return fn(*args), None
    except OracleError as err:
        return None, err.kind
