"""Helpers shared by the oracle and GPU parity tests (reads committed fixtures only)."""

import numpy as np

from oracle.sif_oracle import Cfg
from oracle.synth import synth


def case_cfg(c):
    d = c["cfg"]
    return Cfg(s=d["s"], lam=d["lam"], m_plus=d["m_plus"], m_minus=d["m_minus"], q_bit=d["q_bit"],
               delta=d["delta"], mode=d["mode"], fixed_q=tuple(d["fixed_q"]))


def case_x(i, c, arrays):
    if c["stored"]:
        return arrays[f"c{i}_x"].view(np.float32).reshape(c["rows"], c["cols"])
    s = c["synth"]
    return synth(s["kind"], c["rows"], c["cols"], s["sid"])
