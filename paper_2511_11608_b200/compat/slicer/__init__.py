"""`slicer`-named shim over the B200 codec (paper_2511_11608_b200).

Code written against the reference package's codec API (slicer/__init__.py:15-25 --
CodecConfig, CompressedIF, EncodedBlock, broadcast_q, encode, decode, serialize,
deserialize, payload_bits_exact, atkf_filter, DenseTensor, random_tensor and the error
classes) runs unchanged on the GPU codec when `paper_2511_11608_b200/compat` is first on
sys.path.  The only conversion happens here: the reference's host DenseTensor
(tensor.py:19-56) in and out, torch CUDA tensors inside.  Everything the codec computes
(ATKF, MS, ABQ, packing, CRC, deserialize checks, decode) runs in the sm_100a kernels;
there is no CPU path behind this module.

Out of scope: planner, simulator, channel model -- importing those names
from this shim raises AttributeError.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

import paper_2511_11608_b200 as _g
from paper_2511_11608_b200.codec import (  # noqa: F401  (re-exported reference names)
    MODE_ABQ,
    MODE_FIXED,
    CodecConfig,
    CompressedIF,
    EncodedBlock,
    QuantSpec,
    broadcast_q,
    payload_bits_exact,
    serialize,
)
from paper_2511_11608_b200.errors import (  # noqa: F401
    ConfigError,
    CorruptStreamError,
    NonFiniteError,
    ShapeError,
    SlicerError,
    StreamFormatError,
    TensorFormatError,
)

from . import codec  # noqa: F401  (slicer.codec: MODE_FIXED, col_bits, payload_bits_exact)


@dataclass(frozen=True, eq=False)
class DenseTensor:
    """tensor.py:19-56: immutable rows x cols fp32 tensor (row-major, finite)."""

    rows: int
    cols: int
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        if self.rows < 1 or self.cols < 1:
            raise ShapeError(f"tensor shape must be positive, got {self.rows}x{self.cols}")
        vals = np.ascontiguousarray(self.values, dtype=np.float32).reshape(-1)
        if vals.size != self.rows * self.cols:
            raise ShapeError(f"value count {vals.size} does not match shape {self.rows}x{self.cols}")
        if not np.all(np.isfinite(vals)):
            raise NonFiniteError("tensor contains NaN or Inf")
        vals.flags.writeable = False
        object.__setattr__(self, "values", vals)

    @property
    def size(self) -> int:
        return self.rows * self.cols

    def as_matrix(self) -> np.ndarray:
        return self.values.reshape(self.rows, self.cols)

    def __eq__(self, other) -> bool:
        if not isinstance(other, DenseTensor):
            return NotImplemented
        return (self.rows == other.rows and self.cols == other.cols
                and np.array_equal(self.values.view(np.uint32), other.values.view(np.uint32)))

    __hash__ = None


def _to_device(x: DenseTensor) -> torch.Tensor:
    return torch.from_numpy(np.array(x.values, dtype=np.float32).reshape(x.rows, x.cols)).cuda()


def _to_host(y: torch.Tensor) -> DenseTensor:
    return DenseTensor(int(y.shape[0]), int(y.shape[1]), y.detach().cpu().numpy().reshape(-1))


def encode(x: DenseTensor, cfg: CodecConfig, seed: int = 0) -> CompressedIF:
    """codec.py:186 -> the GPU encoder."""
    return _g.encode(_to_device(x), cfg, seed)


def decode(c) -> DenseTensor:
    """codec.py:254 -> the GPU decoder (validation + dequantize + scatter)."""
    return _to_host(_g.decode(c))


def deserialize(data: bytes) -> CompressedIF:
    """codec.py:320 -> device-side checks, CompressedIF view."""
    return _g.deserialize(data)


@dataclass(frozen=True)
class AtkfResult:
    """atkf.py:20-28."""

    filtered: DenseTensor
    kept_indices: np.ndarray = field(repr=False)
    tau: float
    tau_plus: float
    tau_minus: float
    k_keep: int
    tau_is_fallback: bool = False


def atkf_filter(x: DenseTensor, s: float, lam: float, seed: int) -> AtkfResult:
    """atkf.py:44-96 -> the GPU select (sif_atkf_batched)."""
    r = _g.atkf_filter(_to_device(x), s, lam, seed)
    return AtkfResult(_to_host(r.filtered), r.kept_indices.cpu().numpy().astype(np.int64), r.tau, r.tau_plus,
                      r.tau_minus, r.k_keep, r.tau_is_fallback)


def random_tensor(rows: int, cols: int, seed: int, dist: str = "uniform") -> DenseTensor:
    """tensor.py:89-111, values generated on the device (sif_fixture_tensor)."""
    return _to_host(_g.random_tensor(rows, cols, seed, dist))


def save_tensor(t: DenseTensor, path) -> None:
    _g.save_tensor(_to_device(t), path)


def load_tensor(path) -> DenseTensor:
    return _to_host(_g.load_tensor(path))


def payload_upper_bound(shape, cfg) -> int:
    return _g.payload_upper_bound(shape, cfg)


__version__ = "0.1.0"
