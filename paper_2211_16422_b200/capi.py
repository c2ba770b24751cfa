"""ctypes declarations for include/homs_b200.h (the C ABI of libhoms_b200.so).

There is no fallback: if the shared object is missing this module raises ImportError telling
the user to build it.  Nothing here imports torch; device pointers are plain integers.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_ROOT = os.path.dirname(PKG_DIR)
LIB_PATH = os.environ.get("HOMS_B200_LIB") or os.path.join(PKG_DIR, "libhoms_b200.so")  # env: development A/B builds
HEADER_PATH = os.path.join(REPO_ROOT, "include", "homs_b200.h")

OK, ERR_CONFIG, ERR_INVARIANT, ERR_CUDA, ERR_ARGUMENT, ERR_STATE = range(6)
ERR_CACHE_FORMAT, ERR_CACHE_STALE, ERR_CACHE_CORRUPT, ERR_PARSE = 6, 7, 8, 9
TOL_PPM, TOL_DALTON = 0, 1
NO_HIT = 0xFFFFFFFF
MAX_TOPK = 64


class PreprocessConfigPod(C.Structure):
    _fields_ = [("min_mz", C.c_double), ("max_mz", C.c_double), ("bin_size", C.c_double),
                ("max_peaks", C.c_uint32), ("min_peaks", C.c_uint32),
                ("intensity_floor", C.c_double), ("scaling", C.c_uint32),
                ("reserved", C.c_uint32)]


class EncoderConfigPod(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("step_flips", C.c_uint32), ("levels", C.c_uint32),
                ("reserved", C.c_uint32), ("seed", C.c_uint64)]


class CacheLayoutPod(C.Structure):
    _fields_ = [("count", C.c_uint64), ("hv_offset", C.c_uint64), ("hv_bytes", C.c_uint64),
                ("stored_digest", C.c_uint64), ("id_bytes", C.c_uint64), ("peptide_bytes", C.c_uint64)]


class MgfInfoPod(C.Structure):
    _fields_ = [("n_lines", C.c_uint64), ("n_spectra", C.c_uint64), ("n_peaks", C.c_uint64),
                ("n_hard_numbers", C.c_uint64), ("error_line", C.c_uint64), ("error_code", C.c_uint32),
                ("reserved", C.c_uint32)]


class TolerancePod(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("reserved", C.c_uint32), ("value", C.c_double)]


def declared_functions() -> list[str]:
    """Names of every function include/homs_b200.h declares (used by the symbol-export test)."""
    with open(HEADER_PATH) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(homs_b200_[a-z0-9_]+)\s*\(", text)))


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: the CUDA library has not been built. Run "
        "`python -c 'import __graft_entry__ as g; g.build()'` from the repository root. "
        "This package has no CPU fallback.")

lib = C.CDLL(LIB_PATH)

_VP, _U64, _U32, _U8, _F64, _I = C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint8, C.c_double, C.c_int
_P = C.POINTER


def _decl(name, restype, argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = argtypes
    return fn


abi_version = _decl("homs_b200_abi_version", _I, [])
ctx_create = _decl("homs_b200_ctx_create", _I, [_I, _P(_VP)])
device_count = _decl("homs_b200_device_count", _I, [_P(_I)])
ctx_create_multi = _decl("homs_b200_ctx_create_multi", _I, [_P(_I), _I, _P(_VP)])
ctx_device_count = _decl("homs_b200_ctx_device_count", _I, [_VP])
ctx_destroy = _decl("homs_b200_ctx_destroy", None, [_VP])
last_error = _decl("homs_b200_last_error", C.c_char_p, [_VP])
ctx_set_stream = _decl("homs_b200_ctx_set_stream", _I, [_VP, _VP])
ctx_synchronize = _decl("homs_b200_ctx_synchronize", _I, [_VP])
ctx_launch_count = _decl("homs_b200_ctx_launch_count", _U64, [_VP])
ctx_set_engine = _decl("homs_b200_ctx_set_engine", _I, [_VP, _I])
ctx_last_engine = _decl("homs_b200_ctx_last_engine", _I, [_VP])
ctx_tensor_cta_pairs = _decl("homs_b200_ctx_tensor_cta_pairs", _I, [_VP])
ENGINE_AUTO, ENGINE_POPC, ENGINE_TENSOR, ENGINE_TENSOR_FP4, ENGINE_DIRECT = 0, 1, 2, 3, 4
ctx_profile = _decl("homs_b200_ctx_profile", _I, [_VP, _I])
ctx_kernel_time = _decl("homs_b200_ctx_kernel_time", _I, [_VP, _I, _P(_F64), _P(_U64)])
KERNEL_SEARCH, KERNEL_ENCODE, KERNEL_PREPROCESS = 0, 1, 2
tensor_peak_probe = _decl("homs_b200_tensor_peak_probe", _I, [_VP, _I, _F64, _P(_F64), _P(_F64)])

preprocess_validate = _decl("homs_b200_preprocess_validate", _I, [_P(PreprocessConfigPod)])
dimension = _decl("homs_b200_dimension", _U32, [_P(PreprocessConfigPod)])
encoder_validate = _decl("homs_b200_encoder_validate", _I, [_P(EncoderConfigPod)])
quantize_intensity = _decl("homs_b200_quantize_intensity", _I, [_F64, _U32, _P(_U32)])
make_codebook = _decl("homs_b200_make_codebook", _I, [_P(EncoderConfigPod), _U32, _VP, _VP])
compute_fdr_curve = _decl("homs_b200_compute_fdr_curve", _I, [_U64, _VP, _VP, _VP, _VP, _VP])

codebook_upload = _decl("homs_b200_codebook_upload", _I, [_VP, _U32, _U32, _U32, _VP, _VP])
encode_batch = _decl("homs_b200_encode_batch", _I,
                     [_VP, _P(PreprocessConfigPod), _U64, _VP, _VP, _VP, _VP, _VP])
encode_batch_dev = _decl("homs_b200_encode_batch_dev", _I,
                         [_VP, _P(PreprocessConfigPod), _U64, _U64, _VP, _VP, _VP, _VP, _VP])
preprocess_batch = _decl("homs_b200_preprocess_batch", _I,
                         [_VP, _P(PreprocessConfigPod), _U32, _U64, _VP, _VP, _VP, _VP, _VP, _VP])
encode_vectors = _decl("homs_b200_encode_vectors", _I, [_VP, _U64, _VP, _VP, _VP, _VP])
hamming_similarity = _decl("homs_b200_hamming_similarity", _I, [_VP, _U32, _U64, _VP, _VP, _VP])

library_upload = _decl("homs_b200_library_upload", _I,
                       [_VP, _U32, _U64, _VP, _VP, _VP, _VP, _U32, _U32])
library_upload_dev = _decl("homs_b200_library_upload_dev", _I,
                           [_VP, _U32, _U64, _VP, _VP, _VP, _VP, _U32, _U32])
library_bucket_count = _decl("homs_b200_library_bucket_count", _I, [_VP, _P(_U32)])
library_bucket_info = _decl("homs_b200_library_bucket_info", _I,
                            [_VP, _U32, _P(_U8), _P(_U64), _P(_U64), _P(_U64)])
library_bucket_export = _decl("homs_b200_library_bucket_export", _I, [_VP, _U32, _VP, _VP, _VP])

window_bounds = _decl("homs_b200_window_bounds", _I,
                      [_VP, _U64, _VP, _VP, _P(TolerancePod), _VP, _VP, _VP])
search_batch = _decl("homs_b200_search_batch", _I,
                     [_VP, _U32, _U64, _VP, _VP, _VP, _P(TolerancePod), _U32, _VP, _VP, _VP, _VP])
queries_upload = _decl("homs_b200_queries_upload", _I, [_VP, _U32, _U64, _VP, _VP, _VP])
queries_upload_dev = _decl("homs_b200_queries_upload_dev", _I, [_VP, _U32, _U64, _VP, _VP, _VP])
search_resident_dev = _decl("homs_b200_search_resident_dev", _I,
                            [_VP, _VP, _U64, _P(TolerancePod), _U32, _VP])
merge_candidates_dev = _decl("homs_b200_merge_candidates_dev", _I, [_VP, _U64, _U32, _U32, _VP, _VP])
candidates_decode = _decl("homs_b200_candidates_decode", _I, [_VP, _U64, _U32, _VP, _VP, _VP])
cascade_search = _decl("homs_b200_cascade_search", _I,
                       [_VP, _U32, _U64, _VP, _VP, _VP, _P(TolerancePod), _P(TolerancePod), _F64,
                        _VP, _VP, _VP, _VP, _VP, _VP, _P(_U64)])

library_build_from_spectra = _decl("homs_b200_library_build_from_spectra", _I,
                                   [_VP, _P(PreprocessConfigPod), _U64, _VP, _VP, _VP, _VP, _VP, _VP, _U32, _U32,
                                    _VP, _P(_U64)])
queries_from_spectra = _decl("homs_b200_queries_from_spectra", _I,
                             [_VP, _P(PreprocessConfigPod), _U64, _VP, _VP, _VP, _VP, _VP, _VP, _P(_U64)])
queries_from_mgf = _decl("homs_b200_queries_from_mgf", _I, [_VP, _P(PreprocessConfigPod), _VP, _P(_U64)])
search_resident = _decl("homs_b200_search_resident", _I, [_VP, _P(TolerancePod), _U32, _VP, _VP, _VP, _VP])
cascade_resident = _decl("homs_b200_cascade_resident", _I,
                         [_VP, _P(TolerancePod), _P(TolerancePod), _F64, _VP, _VP, _VP, _VP, _VP, _VP, _P(_U64)])

mgf_parse = _decl("homs_b200_mgf_parse", _I, [_VP, _VP, _U64, _P(MgfInfoPod)])
mgf_parse_dev = _decl("homs_b200_mgf_parse_dev", _I, [_VP, _VP, _U64, _P(MgfInfoPod)])
mgf_fetch = _decl("homs_b200_mgf_fetch", _I, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP])
mgf_device_csr = _decl("homs_b200_mgf_device_csr", _I,
                       [_VP, _P(_U64), _P(_U64), _P(_VP), _P(_VP), _P(_VP), _P(_VP), _P(_VP)])

fnv1a64_dev = _decl("homs_b200_fnv1a64_dev", _I, [_VP, _VP, _U64, _P(_U64)])
fnv1a64 = _decl("homs_b200_fnv1a64", _I, [_VP, _VP, _U64, _P(_U64)])
cache_parse = _decl("homs_b200_cache_parse", _I,
                    [_VP, _U64, _P(PreprocessConfigPod), _P(EncoderConfigPod), _P(CacheLayoutPod),
                     _VP, _VP, _VP, _VP, _VP, _VP, _VP])
library_load_cache = _decl("homs_b200_library_load_cache", _I,
                           [_VP, _VP, _U64, _P(PreprocessConfigPod), _P(EncoderConfigPod), _U32, _U32, _P(_U64)])
cache_write = _decl("homs_b200_cache_write", _I,
                    [_VP, _P(PreprocessConfigPod), _P(EncoderConfigPod), _U64, _VP, _VP, _VP, _VP, _VP, _VP,
                     _VP, _VP, _VP, _U64, _P(_U64)])
cache_write_dev = _decl("homs_b200_cache_write_dev", _I,
                        [_VP, _P(PreprocessConfigPod), _P(EncoderConfigPod), _U64, _VP, _VP, _VP, _VP, _VP, _VP,
                         _VP, _VP, _VP, _U64, _P(_U64)])
