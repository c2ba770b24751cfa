"""B200-native (sm_100a) implementation of the HyperOMS hot path.

The product is ``libhoms_b200.so`` (CUDA kernels behind the C ABI in ``include/homs_b200.h``);
this package is the Python host mirror of the reference's encoder/search interface.  Importing
it without the built library raises ImportError: there is no CPU fallback.
"""
from . import capi  # noqa: F401  (raises if the CUDA library is missing)
from .host import (  # noqa: F401
    CacheCorruptError, CacheFormatError, Codebook, ConfigError, Context, CudaError, EncodeOutcome,
    EncoderConfig, HomsError, InvariantError, Match, ParseError, PreprocessConfig, StaleCacheError, Tolerance,
    cache_parse, compute_fdr_curve, device_count, dimension, id_ranks, make_codebook, quantize_intensity, words_for,
)

__all__ = [
    "CacheCorruptError", "CacheFormatError", "Codebook", "ConfigError", "Context", "CudaError",
    "EncodeOutcome", "EncoderConfig", "HomsError", "InvariantError", "Match", "ParseError", "PreprocessConfig",
    "StaleCacheError", "Tolerance", "cache_parse", "compute_fdr_curve", "device_count", "dimension", "id_ranks",
    "make_codebook", "quantize_intensity", "words_for",
]
