"""`.tns` files and fixture tensors on the device.

Mirror of the reference's slicer/tensor.py:

    load_tensor(path) -> DenseTensor          tensor.py:66-87   load_tensor(path) -> CUDA fp32 (N, K)
    save_tensor(t, path)                      tensor.py:59-63   save_tensor(t, path)
    random_tensor(rows, cols, seed, dist)     tensor.py:90-111  random_tensor(...) -> CUDA fp32 (N, K)

`.tns` layout (little-endian): magic "TNS1" | version u16 = 1 | rows u32 | cols u32 |
rows*cols float32.  The payload is read into pinned host memory and copied to the device
asynchronously; the finiteness check of DenseTensor (tensor.py:35-36, :84-85) runs as a
kernel (sif_count_nonfinite).  Fixture values come from the counter-based splitmix64
stream (rng.py:30-52) evaluated per element on the device (sif_fixture_tensor): uniform
tensors are bit-identical to the reference's; gaussian tensors use CUDA log/sin/cos.
Error classes and messages follow the reference.
"""

from __future__ import annotations

import ctypes
import os
import struct

import torch

from . import _lib
from .errors import NonFiniteError, ShapeError, TensorFormatError

TNS_MAGIC = b"TNS1"
TNS_VERSION = 1
TNS_HEADER_BYTES = 14
_DISTS = {"uniform": 0, "gaussian": 1}
_MASK64 = (1 << 64) - 1


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def count_nonfinite(x: torch.Tensor) -> int:
    """Number of NaN/Inf elements of a CUDA fp32 tensor (one kernel + a 8-byte read)."""
    if not (x.is_cuda and x.dtype == torch.float32):
        raise TypeError("count_nonfinite expects a CUDA float32 tensor")
    x = x.contiguous()
    if x.data_ptr() % 16:
        x = x.clone()
    cnt = torch.empty(1, dtype=torch.int64, device=x.device)
    st = _lib.load().sif_count_nonfinite(x.data_ptr(), x.numel(), cnt.data_ptr(), _stream())
    if st:
        raise RuntimeError(f"sif_count_nonfinite failed with status {st}")
    return int(cnt.item())


def check_dense(x: torch.Tensor, what: str = "tensor") -> None:
    """DenseTensor invariants (tensor.py:27-36): 2-D, rows/cols >= 1, finite."""
    if x.dim() != 2 or x.shape[0] < 1 or x.shape[1] < 1:
        raise ShapeError(f"tensor shape must be positive, got {'x'.join(str(d) for d in x.shape)}")
    if count_nonfinite(x.to(torch.float32) if x.dtype != torch.float32 else x):
        raise NonFiniteError(f"{what} contains NaN or Inf")


def save_tensor(t: torch.Tensor, path) -> None:
    """tensor.py:59-63: header + little-endian fp32 values (device -> pinned host -> file)."""
    if not isinstance(t, torch.Tensor):
        raise TypeError("save_tensor expects a torch.Tensor")
    if t.dim() != 2 or t.shape[0] < 1 or t.shape[1] < 1:
        raise ShapeError(f"tensor shape must be positive, got {'x'.join(str(d) for d in t.shape)}")
    rows, cols = int(t.shape[0]), int(t.shape[1])
    v = t.detach().to(torch.float32).contiguous()
    host = torch.empty(v.numel(), dtype=torch.float32, pin_memory=v.is_cuda)
    host.copy_(v.reshape(-1))
    with open(path, "wb") as f:
        f.write(TNS_MAGIC)
        f.write(struct.pack("<HII", TNS_VERSION, rows, cols))
        f.write(memoryview(host.numpy()).cast("B"))


def load_tensor(path, device: str | torch.device = "cuda") -> torch.Tensor:
    """tensor.py:66-87, same checks in the same order; returns a CUDA fp32 (rows, cols)."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(TNS_HEADER_BYTES)
        if len(head) < TNS_HEADER_BYTES:
            raise TensorFormatError("file too short for a .tns header")
        if head[:4] != TNS_MAGIC:
            raise TensorFormatError(f"bad magic {head[:4]!r}")
        version, rows, cols = struct.unpack_from("<HII", head, 4)
        if version != TNS_VERSION:
            raise TensorFormatError(f"unsupported .tns version {version}")
        if rows < 1 or cols < 1:
            raise ShapeError(f"stored shape {rows}x{cols} is degenerate")
        expected = TNS_HEADER_BYTES + 4 * rows * cols
        if size < expected:
            raise TensorFormatError(f"truncated payload: need {expected} bytes, have {size}")
        host = torch.empty(rows * cols, dtype=torch.float32, pin_memory=True)
        f.readinto(memoryview(host.numpy()).cast("B"))
    x = host.to(device, non_blocking=True).view(rows, cols)
    if count_nonfinite(x):
        raise NonFiniteError("stored tensor contains NaN or Inf")
    return x


def random_tensor(rows: int, cols: int, seed: int, dist: str = "uniform",
                  device: str | torch.device = "cuda") -> torch.Tensor:
    """tensor.py:90-111 on the device: the reference's deterministic fixture values."""
    if rows < 1 or cols < 1:
        raise ShapeError(f"tensor shape must be positive, got {rows}x{cols}")
    if dist not in _DISTS:
        raise ValueError(f"unknown dist {dist!r}")
    x = torch.empty((rows, cols), dtype=torch.float32, device=device)
    st = _lib.load().sif_fixture_tensor(x.data_ptr(), rows * cols, int(seed) & _MASK64, _DISTS[dist], _stream())
    if st:
        raise RuntimeError(f"sif_fixture_tensor failed with status {st}")
    return x
