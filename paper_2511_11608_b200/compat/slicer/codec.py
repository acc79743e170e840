"""`slicer.codec` names of the shim (codec.py:44-58 constants and helpers)."""

from paper_2511_11608_b200.codec import (  # noqa: F401
    BLOCK_FIXED_BYTES,
    CRC_BYTES,
    HEADER_BYTES,
    MODE_ABQ,
    MODE_FIXED,
    CodecConfig,
    CompressedIF,
    EncodedBlock,
    broadcast_q,
    col_bits,
    payload_bits_exact,
    serialize,
)
