"""B200-native 3DES-ECB engine (arxiv 1305.4376 hot path, rebuilt for sm_100a).

Host API mirroring the reference's t3des API; the cipher runs only in the
CUDA kernels of libt3des_b200.so.
"""
from ._native import (  # noqa: F401
    VARIANT_AUTO,
    DECRYPT,
    ENCRYPT,
    VARIANT_BITSLICE,
    VARIANT_BITSLICE_LDG,
    VARIANT_BITSLICE_ALU,
    VARIANT_BITSLICE_DFMA,
    VARIANT_BITSLICE_SHRFMA,
    VARIANT_SPTABLE,
    EngineUnavailable,
    LIB_PATH,
)
from .api import (  # noqa: F401
    Backend,
    ChunkSpan,
    CudaError,
    DesKey,
    DispatchConfig,
    Engine,
    InputLengthError,
    IoError,
    KeyFormatError,
    KeyingOption,
    PaddingError,
    PaddingMode,
    StreamReport,
    TripleKey,
    TripleSchedule,
    decrypt_batch,
    decrypt_stream,
    encrypt_batch,
    encrypt_stream,
    engine,
    key_schedule,
    load_block,
    parse_hex_key,
    pkcs7_pad,
    pkcs7_unpad,
    plan_dispatch,
    store_block,
    to_hex,
    triple_schedule,
)
