"""ctypes binding of the native codec library (include/sif.h).

The library must be built in-tree (`python -c "import __graft_entry__ as g; g.build()"`
or `python -m paper_2511_11608_b200.build`).  There is no CPU fallback: importing the
codec on a machine without the built library or without CUDA raises."""

import ctypes
import os

from ctypes import POINTER, c_double, c_int, c_int32, c_size_t, c_uint32, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsif.so")


class CodecCfgC(ctypes.Structure):
    _fields_ = [("s", c_double), ("lam", c_double), ("delta", c_double), ("m_plus", c_int32),
                ("m_minus", c_int32), ("q_bit", c_int32), ("mode", c_int32), ("fixed_q", c_void_p)]


class EncDesc(ctypes.Structure):
    _fields_ = [("x", c_void_p), ("out", c_void_p), ("out_cap", c_uint64), ("seed", c_uint64),
                ("rows", c_uint32), ("cols", c_uint32), ("dtype", c_uint32), ("reserved", c_uint32)]


class DecDesc(ctypes.Structure):
    _fields_ = [("inp", c_void_p), ("in_len", c_uint64), ("out", c_void_p), ("rows", c_uint32),
                ("cols", c_uint32), ("in_len_dev", c_void_p)]


class Plan(ctypes.Structure):
    _fields_ = [("n", c_int32), ("cluster", c_int32), ("threads", c_int32), ("smem_bytes", c_int32),
                ("cap_smem", c_int32), ("max_blocks", c_int32), ("tiles", c_int32), ("flags", c_int32),
                ("ws_bytes", c_uint64), ("ws_desc_off", c_uint64), ("ws_aux_off", c_uint64),
                ("ws_spill_off", c_uint64), ("n_fused", c_int32), ("reserved", c_int32)]


assert ctypes.sizeof(EncDesc) == 48 and ctypes.sizeof(DecDesc) == 40 and ctypes.sizeof(Plan) == 72

EXPORTS = {
    "sif_version": (c_int, []),
    "sif_keep_count": (c_uint64, [c_double, c_uint64]),
    "sif_col_bits": (c_uint32, [c_uint32]),
    "sif_validate_cfg": (c_int, [POINTER(CodecCfgC)]),
    "sif_max_payload_bytes": (c_uint64, [c_uint32, c_uint32, POINTER(CodecCfgC)]),
    "sif_status_string": (ctypes.c_char_p, [c_int]),
    "sif_set_fused_range": (c_int, [c_uint64, c_uint64]),
    "sif_get_fused_range": (c_int, [POINTER(c_uint64), POINTER(c_uint64)]),
    "sif_enc_plan": (c_int, [POINTER(EncDesc), c_int, POINTER(CodecCfgC), POINTER(Plan)]),
    "sif_enc_upload": (c_int, [POINTER(Plan), POINTER(EncDesc), POINTER(CodecCfgC), c_void_p, c_void_p]),
    "sif_enc_run": (c_int, [POINTER(Plan), POINTER(CodecCfgC), c_void_p, c_void_p, c_void_p, c_void_p]),
    "sif_encode_batched": (c_int, [POINTER(EncDesc), c_int, POINTER(CodecCfgC), c_void_p, c_size_t, c_void_p,
                                   c_void_p, c_void_p]),
    "sif_atkf_batched": (c_int, [POINTER(EncDesc), c_int, POINTER(CodecCfgC), c_void_p, c_size_t, c_void_p,
                                 c_void_p, c_void_p, c_void_p]),
    "sif_dec_plan": (c_int, [POINTER(DecDesc), c_int, POINTER(Plan)]),
    "sif_dec_upload": (c_int, [POINTER(Plan), POINTER(DecDesc), c_void_p, c_void_p]),
    "sif_dec_run": (c_int, [POINTER(Plan), c_int, c_void_p, c_void_p, c_void_p]),
    "sif_decode_batched": (c_int, [POINTER(DecDesc), c_int, c_int, c_void_p, c_size_t, c_void_p, c_void_p]),
    "sif_dec_table_offset": (c_uint64, [POINTER(Plan), POINTER(DecDesc), c_int]),
    "sif_set_small_decode": (c_int, [c_uint64]),
    "sif_routing_epoch": (c_uint64, []),
    "sif_enc_set_input": (c_int, [POINTER(Plan), c_void_p, c_int, c_void_p, c_void_p, c_uint64, c_void_p]),
    "sif_dec_set_input": (c_int, [POINTER(Plan), c_void_p, c_int, c_void_p, c_uint64, c_void_p, c_void_p, c_void_p]),
    "sif_gen_synthetic": (c_int, [c_void_p, c_uint32, c_uint32, c_uint32, c_uint32, c_uint64, c_void_p]),
    "sif_profile_enable": (c_int, [c_int]),
    "sif_profile_enabled": (c_int, []),
    "sif_profile_read": (c_int, [POINTER(c_double), POINTER(c_int32), c_int]),
    "sif_profile_kernel_name": (ctypes.c_char_p, [c_int]),
    "sif_fixture_tensor": (c_int, [c_void_p, c_uint64, c_uint64, c_int, c_void_p]),
    "sif_count_nonfinite": (c_int, [c_void_p, c_uint64, c_void_p, c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libsif.so and bind every symbol declared in include/sif.h (raises if absent)."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"native codec library not built: {path} (run __graft_entry__.build())")
    lib = ctypes.CDLL(path)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _lib = lib
    return lib
