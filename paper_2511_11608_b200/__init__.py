"""B200-native SLICER intermediate-feature codec (arxiv 2511.11608).

Drop-in for the reference codec path (slicer/codec.py): ATKF -> MS -> ABQ -> CSR
bit-pack -> .sif, and back, as sm_100a CUDA kernels behind a C ABI (include/sif.h).
"""

from .codec import (
    BLOCK_FIXED_BYTES,
    CRC_BYTES,
    HEADER_BYTES,
    MODE_ABQ,
    MODE_FIXED,
    AtkfResult,
    BatchDecoder,
    BatchEncoder,
    BatchPipeline,
    ListEncoder,
    ListRoundTrip,
    CodecConfig,
    CompressedIF,
    EncodedBlock,
    QuantSpec,
    HostRoundTrip,
    Payload,
    atkf_filter,
    broadcast_q,
    capture_graph,
    col_bits,
    decode,
    decode_batch,
    decode_list,
    decoder_for,
    deserialize,
    encode,
    encode_batch,
    encode_list,
    keep_count,
    max_payload_bytes,
    payload_bits_exact,
    serialize,
    synthetic,
)
from . import shard
from .stats import payload_upper_bound, stats
from .tensor import load_tensor, random_tensor, save_tensor
from .timemodel import DeviceTimeModel
from .errors import (
    CapacityError,
    ConfigError,
    CorruptStreamError,
    CudaError,
    NonFiniteError,
    ShapeError,
    SlicerError,
    StreamFormatError,
    TensorFormatError,
)

__version__ = "0.1.0"
