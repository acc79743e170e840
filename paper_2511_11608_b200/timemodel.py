"""Encode-time model calibrated on the GPU.

`DeviceTimeModel` mirrors the reference's table model (profiles.py:184-254: same JSON
schema, same nearest-grid-point lookups) that feeds the planner's encode-time estimate
(planner.py:67-75: t_atkf(s, lambda) + t_ms(M+, M-) + (M+ + M-) * t_abq(q_bit)).
`calibrate` fills the tables with measured per-IF times of this implementation's kernels
(per-kernel CUDA events, sif_profile_enable), mapped onto the reference's stages:

    t_atkf(s, lambda)  enc_prep + enc_stream + enc_select*/enc_gather*  (ATKF: tau, ties, MS cuts)
    t_ms(M+, M-)       enc_members + enc_layout + enc_pack + enc_crc   (MS blocks, CSR, .sif)
    t_abq(q)           (enc_abq<1> + enc_abq<0>) / (M+ + M-)     (per block, as the planner charges)

Times are per IF (batch time / batch size) for the calibrated IF shape and batch.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

from .errors import ConfigError

ATKF_KERNELS = ("enc_prep", "enc_stream", "enc_select_tiny", "enc_select<0>", "enc_gather<1>", "enc_select<1>",
                "enc_gather<2>", "enc_select<2>")
MS_KERNELS = ("enc_members", "enc_layout", "enc_pack", "enc_crc")
ABQ_KERNELS = ("enc_abq<1>", "enc_abq<0>")


def _nearest(grid, value):
    """profiles.py:179-181: nearest grid value, ties to the smaller grid point."""
    return min(sorted(set(grid)), key=lambda g: (abs(g - value), g))


@dataclass(frozen=True)
class DeviceTimeModel:
    t_atkf: dict  # (s, lambda) -> ms
    t_ms: dict  # (m_plus, m_minus) -> ms
    t_abq: dict  # q -> ms
    m_buf_bytes: float | None = None
    meta: dict | None = None  # calibration provenance (ignored by the reference reader)

    @staticmethod
    def zero() -> "DeviceTimeModel":
        return DeviceTimeModel(t_atkf={(0.0, 0.0): 0.0}, t_ms={(1, 1): 0.0}, t_abq={8: 0.0}, m_buf_bytes=0.0)

    @staticmethod
    def _lookup_pair(table: dict, a: float, b: float) -> float:
        key = (_nearest([k[0] for k in table], a), _nearest([k[1] for k in table], b))
        if key in table:
            return table[key]
        return table[min(table, key=lambda k: (abs(k[0] - a) + abs(k[1] - b), k))]

    def atkf_ms(self, s: float, lam: float) -> float:
        if not self.t_atkf:
            raise ConfigError("empty t_atkf table")
        return self._lookup_pair(self.t_atkf, s, lam)

    def ms_ms(self, m_plus: int, m_minus: int) -> float:
        if not self.t_ms:
            raise ConfigError("empty t_ms table")
        return self._lookup_pair(self.t_ms, m_plus, m_minus)

    def abq_ms(self, q: int) -> float:
        if not self.t_abq:
            raise ConfigError("empty t_abq table")
        return self.t_abq[_nearest(list(self.t_abq), q)]

    def buffer_bytes(self, dense_if_bits: int) -> float:
        if self.m_buf_bytes is None:
            return dense_if_bits / 8.0
        return self.m_buf_bytes

    def encode_time_estimate(self, cfg) -> float:
        """planner.py:67-75."""
        return self.atkf_ms(cfg.s, cfg.lam) + self.ms_ms(cfg.m_plus, cfg.m_minus) + \
            (cfg.m_plus + cfg.m_minus) * self.abq_ms(cfg.q_bit)

    @classmethod
    def from_dict(cls, d: dict) -> "DeviceTimeModel":
        return cls(
            t_atkf={(float(e["s"]), float(e.get("lambda", 0.0))): float(e["ms"]) for e in d.get("t_atkf", [])},
            t_ms={(int(e["m_plus"]), int(e["m_minus"])): float(e["ms"]) for e in d.get("t_ms", [])},
            t_abq={int(e["q"]): float(e["ms"]) for e in d.get("t_abq", [])},
            m_buf_bytes=None if d.get("m_buf_bytes") is None else float(d["m_buf_bytes"]),
            meta=d.get("meta"),
        )

    @classmethod
    def load(cls, path) -> "DeviceTimeModel":
        with open(path) as f:
            return cls.from_dict(json.load(f))

    def to_dict(self) -> dict:
        d = {
            "t_atkf": [{"s": s, "lambda": lam, "ms": ms} for (s, lam), ms in sorted(self.t_atkf.items())],
            "t_ms": [{"m_plus": a, "m_minus": b, "ms": ms} for (a, b), ms in sorted(self.t_ms.items())],
            "t_abq": [{"q": q, "ms": ms} for q, ms in sorted(self.t_abq.items())],
            "m_buf_bytes": self.m_buf_bytes,
        }
        if self.meta:
            d["meta"] = self.meta
        return d

    def save(self, path) -> None:
        with open(path, "w") as f:
            json.dump(self.to_dict(), f, indent=2)
            f.write("\n")


def _stage_ms(prof: dict, names) -> float:
    return sum(prof.get(k, {}).get("ms_total", 0.0) for k in names)


def profile_encode(xs, cfg, reps: int = 5) -> dict:
    """Per-kernel total ms and launch counts of `reps` encodes of the batch `xs` (warm)."""
    import ctypes

    import torch

    from . import _lib
    from .codec import BatchEncoder

    enc = BatchEncoder(xs, cfg, seeds=list(range(xs.shape[0])))
    enc.run()
    torch.cuda.synchronize()
    L = _lib.load()
    L.sif_profile_enable(1)
    try:
        for _ in range(reps):
            enc.run()
        torch.cuda.synchronize()
    finally:
        L.sif_profile_enable(0)
    ms = (ctypes.c_double * 32)()
    cnt = (ctypes.c_int32 * 32)()
    nk = L.sif_profile_read(ms, cnt, 32)
    if nk < 0:
        raise RuntimeError(f"sif_profile_read failed ({nk})")
    return {L.sif_profile_kernel_name(k).decode(): dict(ms_total=ms[k] / reps, launches=int(cnt[k]) // reps)
            for k in range(nk) if cnt[k]}


def calibrate(rows: int = 1024, cols: int = 196, batch: int = 64, kind: int = 0, dtype=None,
              s_grid=(0.5, 0.7, 0.9), lam_grid=(0.0,), m_grid=((1, 1), (2, 2), (3, 3), (4, 4)),
              q_grid=(4, 8, 16), delta: float = 0.01, reps: int = 5) -> DeviceTimeModel:
    """Measure the three stage tables on the current GPU for IFs of shape rows x cols
    (device synthetic generator `kind`).  Each grid axis varies alone
    around the base point (s=0.9, lambda=0, M=3/3, q_bit=8).  The stages are timed on the
    chunk pipeline, whose kernels map one-to-one onto the planner's stages (the fused
    per-IF kernel is switched off for the calibration and restored afterwards)."""
    import ctypes

    import torch

    from . import _lib

    L = _lib.load()
    tmin, tmax = ctypes.c_uint64(), ctypes.c_uint64()
    L.sif_get_fused_range(ctypes.byref(tmin), ctypes.byref(tmax))
    L.sif_set_fused_range(1, 0)
    try:
        return _calibrate(rows, cols, batch, kind, dtype, s_grid, lam_grid, m_grid, q_grid, delta, reps)
    finally:
        L.sif_set_fused_range(tmin.value, tmax.value)


def _calibrate(rows, cols, batch, kind, dtype, s_grid, lam_grid, m_grid, q_grid, delta, reps):
    import torch

    from .codec import CodecConfig, synthetic

    dtype = dtype or (torch.float32 if kind == 0 else torch.bfloat16)
    xs = torch.empty((batch, rows, cols), dtype=dtype, device="cuda")
    for i in range(batch):
        synthetic(kind, rows, cols, i, dtype=dtype, out=xs[i])
    base = dict(s=0.9, lam=0.0, m_plus=3, m_minus=3, q_bit=8, delta=delta)

    def run(**kw):
        c = dict(base)
        c.update(kw)
        return profile_encode(xs, CodecConfig(**c), reps), c

    t_atkf, t_ms, t_abq = {}, {}, {}
    for s in s_grid:
        for lam in lam_grid:
            p, _ = run(s=s, lam=lam)
            t_atkf[(float(s), float(lam))] = _stage_ms(p, ATKF_KERNELS) / batch
    for mp, mm in m_grid:
        p, _ = run(m_plus=mp, m_minus=mm)
        t_ms[(int(mp), int(mm))] = _stage_ms(p, MS_KERNELS) / batch
    for q in q_grid:
        p, c = run(q_bit=q)
        t_abq[int(q)] = _stage_ms(p, ABQ_KERNELS) / batch / (c["m_plus"] + c["m_minus"])
    meta = dict(device=torch.cuda.get_device_name(), if_shape=[rows, cols], batch=batch,
                dtype=str(dtype).replace("torch.", ""), kind=kind, delta=delta, reps=reps,
                units="ms per IF (batch time / batch)",
                stages=dict(t_atkf=list(ATKF_KERNELS), t_ms=list(MS_KERNELS), t_abq=list(ABQ_KERNELS)))
    return DeviceTimeModel(t_atkf=t_atkf, t_ms=t_ms, t_abq=t_abq, m_buf_bytes=None, meta=meta)
