"""Host-side mirror of the reference's encoder/search interface on top of the C ABI.

Names, argument meaning and error behaviour follow the reference (`homs`, paths under
/root/reference/proj/core/): PreprocessConfig (include/homs/preprocess.hpp:13-25), EncoderConfig /
Codebook / make_codebook (include/homs/codebook.hpp:12-59), encode_spectra (include/homs/
pipeline.hpp:45-48), build_index / select_candidates / search_batch / cascade_search (include/
homs/search.hpp:82-117), Tolerance (search.hpp:16-33), ConfigError / InvariantError (include/
homs/errors.hpp:16-56).  Spectra and hypervectors are numpy arrays instead of C++ objects:

* spectra: CSR triple ``(offsets u64[n+1], mz f64[], intensity f64[])``;
* hypervectors: ``u64[n, ceil(dim/64)]`` little-endian words (hypervector.hpp:12-15).

All compute happens in libhoms_b200.so on the GPU; this module only marshals arrays.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import capi


class HomsError(RuntimeError):
    """homs::Error (errors.hpp:10-13)."""


class ConfigError(HomsError):
    """homs::ConfigError (errors.hpp:16-19)."""


class InvariantError(HomsError):
    """homs::InvariantError (errors.hpp:53-56)."""


class CudaError(HomsError):
    pass


class ParseError(HomsError):
    """homs::ParseError (errors.hpp:22-32): str(e) == "line N: message"; .line is N."""

    @property
    def line(self) -> int:
        try:
            return int(str(self).split(":", 1)[0].split()[1])
        except Exception:
            return 0


class CacheFormatError(HomsError):
    """homs::CacheFormatError (errors.hpp:33-36)."""


class StaleCacheError(HomsError):
    """homs::StaleCacheError (errors.hpp:38-41)."""


class CacheCorruptError(HomsError):
    """homs::CacheCorruptError (errors.hpp:43-46)."""


_ERRORS = {capi.ERR_CONFIG: ConfigError, capi.ERR_INVARIANT: InvariantError,
           capi.ERR_CUDA: CudaError, capi.ERR_ARGUMENT: HomsError, capi.ERR_STATE: HomsError,
           capi.ERR_CACHE_FORMAT: CacheFormatError, capi.ERR_CACHE_STALE: StaleCacheError,
           capi.ERR_CACHE_CORRUPT: CacheCorruptError, capi.ERR_PARSE: ParseError}


def _check(rc: int, ctx=None) -> None:
    if rc != capi.OK:
        msg = (capi.last_error(ctx) or b"").decode(errors="replace")
        raise _ERRORS.get(rc, HomsError)(msg or f"homs_b200 error {rc}")


def _ptr(a) -> int:
    return 0 if a is None else a.ctypes.data


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def words_for(dim: int) -> int:
    return (dim + 63) // 64


@dataclass
class PreprocessConfig:
    min_mz: float = 101.0
    max_mz: float = 1500.0
    bin_size: float = 0.05
    max_peaks: int = 50
    min_peaks: int = 10
    intensity_floor: float = 0.01
    scaling: int = 0  # IntensityScaling: 0 none, 1 sqrt

    def pod(self) -> capi.PreprocessConfigPod:
        return capi.PreprocessConfigPod(self.min_mz, self.max_mz, self.bin_size, self.max_peaks,
                                        self.min_peaks, self.intensity_floor, self.scaling, 0)

    def validate(self) -> None:
        _check(capi.preprocess_validate(C.byref(self.pod())))


def dimension(cfg: PreprocessConfig) -> int:
    return int(capi.dimension(C.byref(cfg.pod())))


@dataclass
class EncoderConfig:
    dim: int = 8192
    step_flips: int = 4096
    levels: int = 16
    seed: int = 1

    def pod(self) -> capi.EncoderConfigPod:
        return capi.EncoderConfigPod(self.dim, self.step_flips, self.levels, 0, self.seed)

    def validate(self) -> None:
        _check(capi.encoder_validate(C.byref(self.pod())))


@dataclass
class Tolerance:
    kind: str = "ppm"  # "ppm" | "dalton"
    value: float = 20.0

    def pod(self) -> capi.TolerancePod:
        if self.kind in ("ppm", 0):
            k = capi.TOL_PPM
        elif self.kind in ("dalton", "da", 1):
            k = capi.TOL_DALTON
        else:
            raise ConfigError(f"unknown tolerance kind {self.kind!r}")
        return capi.TolerancePod(k, 0, float(self.value))

    def validate(self) -> None:  # search.cpp:13-15
        if not self.value > 0.0:
            raise ConfigError("tolerance value must be positive")


@dataclass
class Codebook:
    config: EncoderConfig
    spectrum_dims: int
    position: np.ndarray  # u64[spectrum_dims, W]
    level: np.ndarray     # u64[levels + 1, W]


def quantize_intensity(v: float, levels: int) -> int:
    out = C.c_uint32()
    _check(capi.quantize_intensity(float(v), int(levels), C.byref(out)))
    return out.value


def make_codebook(spectrum_dims: int, config: EncoderConfig) -> Codebook:
    """codebook.cpp:87-94; bit-identical streams (std::mt19937_64 + splitmix64 tags)."""
    W = words_for(config.dim)
    pos = np.zeros((spectrum_dims, W), np.uint64)
    lvl = np.zeros((config.levels + 1, W), np.uint64)
    _check(capi.make_codebook(C.byref(config.pod()), spectrum_dims, _ptr(pos), _ptr(lvl)))
    return Codebook(config, spectrum_dims, pos, lvl)


def compute_fdr_curve(score, is_decoy):
    """fdr.cpp:8-50 -> (input_index, fdr, q_value), each per sorted position."""
    score = _arr(score, np.float64)
    is_decoy = _arr(is_decoy, np.uint8)
    n = len(score)
    order = np.zeros(n, np.uint64)
    fdr = np.zeros(n, np.float64)
    q = np.zeros(n, np.float64)
    _check(capi.compute_fdr_curve(n, _ptr(score), _ptr(is_decoy), _ptr(order), _ptr(fdr), _ptr(q)))
    return order, fdr, q


def _blob(strings):
    enc = [x.encode() if isinstance(x, str) else bytes(x) for x in strings]
    off = np.zeros(len(enc) + 1, np.uint64)
    if enc:
        off[1:] = np.cumsum([len(e) for e in enc])
    return np.frombuffer(b"".join(enc) + b"\0", np.uint8).copy(), off


def cache_parse(image: bytes, preprocess: PreprocessConfig, encoder: EncoderConfig) -> dict:
    """Header + metadata of a cache image (cache.cpp:158-190); host only, no checksum.  Raises
    CacheFormatError / StaleCacheError / CacheCorruptError like read_cache."""
    buf = np.frombuffer(image, np.uint8)
    lay = capi.CacheLayoutPod()
    args = (_ptr(buf) if len(buf) else 0, len(buf), C.byref(preprocess.pod()), C.byref(encoder.pod()), C.byref(lay))
    _check(capi.cache_parse(*args, 0, 0, 0, 0, 0, 0, 0))
    n = lay.count
    mz = np.zeros(n, np.float64)
    charge = np.zeros(n, np.uint8)
    decoy = np.zeros(n, np.uint8)
    ipos, ppos = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
    ilen, plen = np.zeros(n, np.uint32), np.zeros(n, np.uint32)
    _check(capi.cache_parse(*args, _ptr(mz), _ptr(charge), _ptr(decoy), _ptr(ipos), _ptr(ilen), _ptr(ppos),
                            _ptr(plen)))
    ids = [bytes(image[int(p):int(p) + int(l)]).decode() for p, l in zip(ipos, ilen)]
    peps = [bytes(image[int(p):int(p) + int(l)]).decode() for p, l in zip(ppos, plen)]
    return dict(count=n, hv_offset=lay.hv_offset, hv_bytes=lay.hv_bytes, stored_digest=lay.stored_digest,
                precursor_mz=mz, charge=charge, is_decoy=decoy, ids=ids, peptides=peps)


def id_ranks(ids) -> np.ndarray:
    """Position of every entry in the library-wide sort by (id, ordinal): the integer stand-in for
    the reference's std::string comparison (search.cpp:43-45, :141-145)."""
    n = len(ids)
    if n == 0:
        return np.zeros(0, np.uint32)
    b = np.array([s.encode() if isinstance(s, str) else bytes(s) for s in ids], dtype="S")
    order = np.argsort(b, kind="stable")  # bytewise, shorter-is-smaller; stable => ordinal ties
    rank = np.empty(n, np.uint32)
    rank[order] = np.arange(n, dtype=np.uint32)
    return rank


@dataclass
class EncodeOutcome:  # pipeline.hpp:41-44, with positions instead of moved objects
    words: np.ndarray          # u64[n_encoded, W], input order, unprocessable rows removed
    kept: np.ndarray           # positions (into the input) of the encoded spectra
    unprocessable: int = 0


@dataclass
class Match:  # numeric core of Ssm (ssm.hpp:17-30)
    has_hit: np.ndarray
    raw_score: np.ndarray
    ordinal: np.ndarray
    first: np.ndarray = field(default=None)
    last: np.ndarray = field(default=None)


def device_count() -> int:
    n = C.c_int()
    _check(capi.device_count(C.byref(n)))
    return n.value


class Context:
    """Resident codebook, resident library index, resident queries -- on one CUDA device, or (devices=[...])
    on several devices of this process behind the same interface: the library is sharded by contiguous
    m/z slices over them, queries are replicated, per-device candidates are merged on the first device
    (homs_b200_ctx_create_multi; replaces the thread fan-out of parallel.hpp:20-48)."""

    def __init__(self, device: int = 0, devices=None):
        h = C.c_void_p()
        if devices is not None:
            devs = (C.c_int * len(devices))(*[int(d) for d in devices])
            rc = capi.ctx_create_multi(devs, len(devices), C.byref(h))
            device = int(devices[0]) if len(devices) else 0
        else:
            rc = capi.ctx_create(int(device), C.byref(h))
        if rc != capi.OK:
            msg = (capi.last_error(None) or b"").decode(errors="replace")
            raise _ERRORS.get(rc, HomsError)(msg)
        self._h = h
        self.device = device
        self.devices = list(devices) if devices is not None else [device]
        self.codebook: Codebook | None = None
        self.lib_dim = 0
        self.lib_n = 0
        self.lib_is_decoy: np.ndarray | None = None

    # -- lifetime ---------------------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            capi.ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def set_stream(self, cuda_stream: int | None) -> None:
        _check(capi.ctx_set_stream(self._h, cuda_stream or 0), self._h)

    def set_engine(self, engine: str | int) -> None:
        """Search engine: "auto" (tensor_fp4, or direct for narrow windows), "popc", "tensor_fp4"
        ("tensor" is an alias) or "direct".  Choose it before build_index: "popc" and "direct" skip the
        tensor image of the library."""
        code = {"auto": capi.ENGINE_AUTO, "popc": capi.ENGINE_POPC, "tensor": capi.ENGINE_TENSOR,
                "tensor_fp4": capi.ENGINE_TENSOR_FP4, "direct": capi.ENGINE_DIRECT}.get(engine, engine)
        _check(capi.ctx_set_engine(self._h, int(code)), self._h)

    def tensor_cta_pairs(self) -> bool:
        """True when the tensor engine searches the resident library on CTA pairs (cta_group::2)."""
        return int(capi.ctx_tensor_cta_pairs(self._h)) == 1

    def last_engine(self) -> str:
        """Engine the last search call ran on: "popc", "tensor", "tensor_fp4" or "direct"."""
        return {capi.ENGINE_POPC: "popc", capi.ENGINE_TENSOR: "tensor", capi.ENGINE_TENSOR_FP4: "tensor_fp4",
                capi.ENGINE_DIRECT: "direct"}.get(int(capi.ctx_last_engine(self._h)), "auto")

    def synchronize(self) -> None:
        _check(capi.ctx_synchronize(self._h), self._h)

    def launch_count(self) -> int:
        return int(capi.ctx_launch_count(self._h))

    def profile(self, enable: bool) -> None:
        _check(capi.ctx_profile(self._h, int(enable)), self._h)

    def kernel_time(self, which: int):
        """(total milliseconds, launches) of one hot kernel since the last call."""
        ms, cnt = C.c_double(), C.c_uint64()
        _check(capi.ctx_kernel_time(self._h, which, C.byref(ms), C.byref(cnt)), self._h)
        return ms.value, cnt.value

    def tensor_peak_probe(self, engine: str = "tensor_fp4", seconds: float = 0.5):
        """(ops/s, kernel ms) of the tensor engine's bare MMA issue loop on this device."""
        eng = {"tensor": capi.ENGINE_TENSOR_FP4, "tensor_fp4": capi.ENGINE_TENSOR_FP4}[engine]
        ops, ms = C.c_double(), C.c_double()
        _check(capi.tensor_peak_probe(self._h, eng, float(seconds), C.byref(ops), C.byref(ms)), self._h)
        return ops.value, ms.value

    # -- encoding ---------------------------------------------------------------------------
    def upload_codebook(self, cb: Codebook) -> None:
        pos = _arr(cb.position, np.uint64)
        lvl = _arr(cb.level, np.uint64)
        _check(capi.codebook_upload(self._h, cb.config.dim, cb.spectrum_dims, cb.config.levels,
                                    _ptr(pos), _ptr(lvl)), self._h)
        self.codebook = cb

    def encode_batch(self, offsets, mz, intensity, preprocess: PreprocessConfig, out=None):
        """Flat form of encode_spectra: (words u64[n, W] with zero rows for unprocessable
        spectra, ok u8[n]).  `out` = (words, ok) reuses caller arrays (e.g. pinned memory: the
        chunked H2D / kernel / D2H pipeline then overlaps fully)."""
        offsets = _arr(offsets, np.uint64)
        mz = _arr(mz, np.float64)
        intensity = _arr(intensity, np.float64)
        n = len(offsets) - 1
        W = words_for(self.codebook.config.dim) if self.codebook else 0
        if out is not None:
            words, ok = out
            if words.dtype != np.uint64 or words.shape != (n, W) or ok.dtype != np.uint8 or ok.shape != (n,) \
                    or not words.flags.c_contiguous:
                raise ValueError("encode_batch: out must be (uint64[n, W] C-contiguous, uint8[n])")
        else:
            words = np.empty((n, W), np.uint64)
            ok = np.empty(n, np.uint8)
        _check(capi.encode_batch(self._h, C.byref(preprocess.pod()), n, _ptr(offsets), _ptr(mz),
                                 _ptr(intensity), _ptr(words), _ptr(ok)), self._h)
        return words, ok

    def encode_spectra(self, offsets, mz, intensity, preprocess: PreprocessConfig,
                       threads: int = 1, batch_size: int = 0) -> EncodeOutcome:
        """pipeline.cpp:60-85.  `threads` / `batch_size` are accepted for signature parity and
        cannot change results."""
        words, ok = self.encode_batch(offsets, mz, intensity, preprocess)
        kept = np.flatnonzero(ok)
        return EncodeOutcome(words[kept], kept, int(len(ok) - len(kept)))

    def preprocess_batch(self, offsets, mz, intensity, preprocess: PreprocessConfig, levels: int):
        offsets = _arr(offsets, np.uint64)
        mz = _arr(mz, np.float64)
        intensity = _arr(intensity, np.float64)
        n = len(offsets) - 1
        bins = np.zeros((n, preprocess.max_peaks), np.uint32)
        lev = np.zeros((n, preprocess.max_peaks), np.uint32)
        cnt = np.zeros(n, np.uint32)
        _check(capi.preprocess_batch(self._h, C.byref(preprocess.pod()), levels, n, _ptr(offsets),
                                     _ptr(mz), _ptr(intensity), _ptr(bins), _ptr(lev), _ptr(cnt)),
               self._h)
        return bins, lev, cnt

    def encode(self, sv_offsets, bins, intensities) -> np.ndarray:
        """encoder.cpp:19-55 on already vectorized spectra (CSR of bins / intensities)."""
        sv_offsets = _arr(sv_offsets, np.uint64)
        bins = _arr(bins, np.uint32)
        intensities = _arr(intensities, np.float64)
        n = len(sv_offsets) - 1
        out = np.zeros((n, words_for(self.codebook.config.dim)), np.uint64)
        _check(capi.encode_vectors(self._h, n, _ptr(sv_offsets), _ptr(bins), _ptr(intensities),
                                   _ptr(out)), self._h)
        return out

    def hamming_similarity(self, dim: int, a, b) -> np.ndarray:
        a = _arr(a, np.uint64).reshape(-1, words_for(dim))
        b = _arr(b, np.uint64).reshape(-1, words_for(dim))
        if a.shape != b.shape:
            raise InvariantError("hamming_similarity: dimensionality mismatch")
        out = np.zeros(a.shape[0], np.uint32)
        _check(capi.hamming_similarity(self._h, dim, a.shape[0], _ptr(a), _ptr(b), _ptr(out)),
               self._h)
        return out

    # -- index ------------------------------------------------------------------------------
    def build_index(self, dim: int, words, precursor_mz, charge, ids=None, is_decoy=None,
                    shard_index: int = 0, shard_count: int = 1, id_rank=None) -> None:
        """search.cpp:17-60.  `ids` are the library ids (strings) used for tie-breaking."""
        precursor_mz = _arr(precursor_mz, np.float64)
        charge = _arr(charge, np.uint8)
        n = len(precursor_mz)
        words = _arr(words, np.uint64).reshape(n, -1) if n else np.zeros((0, words_for(dim)), np.uint64)
        if n and words.shape[1] != words_for(dim):
            raise InvariantError("build_index: mixed hypervector dimensionalities")
        if id_rank is None and ids is not None:
            id_rank = id_ranks(ids)
        rank = _arr(id_rank, np.uint32) if id_rank is not None else None
        _check(capi.library_upload(self._h, dim, n, _ptr(words), _ptr(precursor_mz), _ptr(charge),
                                   _ptr(rank), shard_index, shard_count), self._h)
        self._set_lib(dim, n, is_decoy)
        self.lib_precursor_mz = precursor_mz

    def build_index_dev(self, dim: int, d_words: int, n: int, precursor_mz, charge, ids=None,
                        is_decoy=None, shard_index: int = 0, shard_count: int = 1,
                        id_rank=None) -> None:
        """Same, hypervector rows already on the device (pointer to dense u64[n, W])."""
        precursor_mz = _arr(precursor_mz, np.float64)
        charge = _arr(charge, np.uint8)
        if id_rank is None and ids is not None:
            id_rank = id_ranks(ids)
        rank = _arr(id_rank, np.uint32) if id_rank is not None else None
        _check(capi.library_upload_dev(self._h, dim, n, d_words, _ptr(precursor_mz), _ptr(charge),
                                       _ptr(rank), shard_index, shard_count), self._h)
        self._set_lib(dim, n, is_decoy)
        self.lib_precursor_mz = precursor_mz

    def _set_lib(self, dim, n, is_decoy):
        self.lib_dim, self.lib_n = dim, n
        self.lib_is_decoy = (_arr(is_decoy, np.uint8) if is_decoy is not None
                             else np.zeros(n, np.uint8))

    def load_cache(self, image: bytes, preprocess: PreprocessConfig, encoder: EncoderConfig,
                   shard_index: int = 0, shard_count: int = 1) -> dict:
        """read_cache + build_index (pipeline.cpp:121-122): cache image -> resident index, checksum
        verified on the device.  Returns the parsed metadata (ids, peptides, ...)."""
        meta = cache_parse(image, preprocess, encoder)
        buf = np.frombuffer(image, np.uint8)
        cnt = C.c_uint64()
        _check(capi.library_load_cache(self._h, _ptr(buf), len(buf), C.byref(preprocess.pod()),
                                       C.byref(encoder.pod()), shard_index, shard_count, C.byref(cnt)), self._h)
        self._set_lib(encoder.dim, cnt.value, meta["is_decoy"])
        return meta

    def cache_write(self, preprocess: PreprocessConfig, encoder: EncoderConfig, words, precursor_mz, charge,
                    is_decoy, ids, peptides, d_words: int = 0) -> bytes:
        """write_cache (cache.cpp:122-156): the byte image of the cache file.  `d_words` != 0: the
        rows are on the device (dense u64[n, W]) and `words` is ignored."""
        mz = _arr(precursor_mz, np.float64)
        ch = _arr(charge, np.uint8)
        dec = _arr(is_decoy, np.uint8)
        n = len(mz)
        iblob, ioff = _blob(ids)
        pblob, poff = _blob(peptides)
        w = None if d_words else _arr(words, np.uint64)
        fn = capi.cache_write_dev if d_words else capi.cache_write
        args = (self._h, C.byref(preprocess.pod()), C.byref(encoder.pod()), n, d_words or _ptr(w), _ptr(mz),
                _ptr(ch), _ptr(dec), _ptr(iblob), _ptr(ioff), _ptr(pblob), _ptr(poff))
        size = C.c_uint64()
        _check(fn(*args, 0, 0, C.byref(size)), self._h)
        out = np.zeros(size.value, np.uint8)
        _check(fn(*args, _ptr(out), size.value, C.byref(size)), self._h)
        return out.tobytes()

    def fnv1a64(self, data) -> int:
        """FNV-1a-64 of host bytes, computed on the device (cache.cpp:18-29)."""
        buf = np.frombuffer(data, np.uint8) if not isinstance(data, np.ndarray) else data.view(np.uint8).ravel()
        out = C.c_uint64()
        _check(capi.fnv1a64(self._h, _ptr(buf) if len(buf) else 0, len(buf), C.byref(out)), self._h)
        return out.value

    def buckets(self):
        cnt = C.c_uint32()
        _check(capi.library_bucket_count(self._h, C.byref(cnt)), self._h)
        out = []
        W = words_for(self.lib_dim)
        for b in range(cnt.value):
            ch, size, sb, se = C.c_uint8(), C.c_uint64(), C.c_uint64(), C.c_uint64()
            _check(capi.library_bucket_info(self._h, b, C.byref(ch), C.byref(size), C.byref(sb),
                                            C.byref(se)), self._h)
            mz = np.zeros(size.value, np.float64)
            ordinal = np.zeros(size.value, np.uint32)
            words = np.zeros((se.value - sb.value, W), np.uint64)
            _check(capi.library_bucket_export(self._h, b, _ptr(mz), _ptr(ordinal), _ptr(words)),
                   self._h)
            out.append(dict(charge=ch.value, precursor_mz=mz, ordinal=ordinal, words=words,
                            shard_begin=sb.value, shard_end=se.value))
        return out

    # -- search -----------------------------------------------------------------------------
    def select_candidates(self, q_mz, q_charge, tol: Tolerance):
        """search.cpp:62-89 -> (first, last, has_bucket) in bucket coordinates."""
        q_mz = _arr(q_mz, np.float64)
        q_charge = _arr(q_charge, np.uint8)
        nq = len(q_mz)
        first = np.zeros(nq, np.uint64)
        last = np.zeros(nq, np.uint64)
        has = np.zeros(nq, np.uint8)
        _check(capi.window_bounds(self._h, nq, _ptr(q_mz), _ptr(q_charge), C.byref(tol.pod()),
                                  _ptr(first), _ptr(last), _ptr(has)), self._h)
        return first, last, has

    def search_batch(self, q_words, q_mz, q_charge, tol: Tolerance, k: int = 1,
                     query_dim: int | None = None, threads: int = 1, batch_size: int = 512) -> Match:
        """search.cpp:171-183 (k best per query; k = 1 is the reference).  Arrays are [nq, k]."""
        q_mz = _arr(q_mz, np.float64)
        q_charge = _arr(q_charge, np.uint8)
        nq = len(q_mz)
        dim = self.lib_dim if query_dim is None else query_dim
        q_words = _arr(q_words, np.uint64).reshape(nq, -1) if nq else np.zeros((0, 1), np.uint64)
        score = np.zeros((nq, k), np.uint32)
        ordinal = np.full((nq, k), capi.NO_HIT, np.uint32)
        first = np.zeros(nq, np.uint64)
        last = np.zeros(nq, np.uint64)
        _check(capi.search_batch(self._h, dim, nq, _ptr(q_words), _ptr(q_mz), _ptr(q_charge),
                                 C.byref(tol.pod()), k, _ptr(score), _ptr(ordinal), _ptr(first),
                                 _ptr(last)), self._h)
        return Match(ordinal != capi.NO_HIT, score, ordinal, first, last)

    def cascade_search(self, q_words, q_mz, q_charge, narrow: Tolerance, wide: Tolerance,
                       fdr_q: float, threads: int = 1, batch_size: int = 512) -> dict:
        """search.cpp:219-248.  Returns the accepted matches (narrow block, then wide block, each
        in query order) as arrays: query, ordinal, stage, raw_score, q_value."""
        q_mz = _arr(q_mz, np.float64)
        q_charge = _arr(q_charge, np.uint8)
        nq = len(q_mz)
        q_words = _arr(q_words, np.uint64).reshape(nq, -1) if nq else np.zeros((0, 1), np.uint64)
        query = np.zeros(nq, np.uint64)
        ordinal = np.zeros(nq, np.uint32)
        stage = np.zeros(nq, np.uint8)
        score = np.zeros(nq, np.uint32)
        qv = np.zeros(nq, np.float64)
        cnt = C.c_uint64()
        _check(capi.cascade_search(self._h, self.lib_dim, nq, _ptr(q_words), _ptr(q_mz),
                                   _ptr(q_charge), C.byref(narrow.pod()), C.byref(wide.pod()),
                                   float(fdr_q), _ptr(self.lib_is_decoy), _ptr(query),
                                   _ptr(ordinal), _ptr(stage), _ptr(score), _ptr(qv),
                                   C.byref(cnt)), self._h)
        m = cnt.value
        return dict(query=query[:m].copy(), ordinal=ordinal[:m].copy(), stage=stage[:m].copy(),
                    raw_score=score[:m].copy(), q_value=qv[:m].copy())

    # -- MGF text -> CSR -------------------------------------------------------
    def parse_mgf(self, text: bytes, decoy_prefix: str = "DECOY_", fetch: bool = True) -> dict:
        """parse_mgf (mgf.cpp:93-181) on the device.  Returns the spectra as CSR arrays plus ids /
        peptides / decoy flags built the way finalize_block does (mgf.cpp:66-76).  With
        fetch=False only the counts come back and the CSR stays resident (see mgf_device_csr)."""
        buf = np.frombuffer(text, np.uint8)
        info = capi.MgfInfoPod()
        _check(capi.mgf_parse(self._h, _ptr(buf) if len(buf) else 0, len(buf), C.byref(info)), self._h)
        n, npk = int(info.n_spectra), int(info.n_peaks)
        out = dict(n_spectra=n, n_peaks=npk, n_lines=int(info.n_lines), n_hard_numbers=int(info.n_hard_numbers))
        if not fetch:
            return out
        offsets = np.zeros(n + 1, np.uint64)
        mz, inten = np.zeros(npk, np.float64), np.zeros(npk, np.float64)
        prec, charge = np.zeros(n, np.float64), np.zeros(n, np.uint8)
        toff, tlen, soff, slen = (np.zeros(n, np.uint32) for _ in range(4))
        _check(capi.mgf_fetch(self._h, _ptr(offsets), _ptr(mz), _ptr(inten), _ptr(prec), _ptr(charge), _ptr(toff),
                              _ptr(tlen), _ptr(soff), _ptr(slen)), self._h)
        ids, peps = [], []
        pre = decoy_prefix.encode()
        decoy = np.zeros(n, np.uint8)
        for i in range(n):
            ident = text[int(toff[i]):int(toff[i]) + int(tlen[i])] if tlen[i] else b"spectrum_%d" % (i + 1)
            pep = text[int(soff[i]):int(soff[i]) + int(slen[i])]
            ids.append(ident)
            peps.append(pep)
            decoy[i] = bool(pre) and (ident.startswith(pre) or pep.startswith(pre))
        out.update(offsets=offsets, mz=mz, intensity=inten, precursor_mz=prec, charge=charge, is_decoy=decoy,
                   ids=ids, peptides=peps)
        return out

    def parse_mgf_dev(self, d_image: int, n_bytes: int) -> dict:
        """parse_mgf of an image already in device memory; the CSR stays resident."""
        info = capi.MgfInfoPod()
        _check(capi.mgf_parse_dev(self._h, d_image, n_bytes, C.byref(info)), self._h)
        return dict(n_spectra=int(info.n_spectra), n_peaks=int(info.n_peaks), n_lines=int(info.n_lines),
                    n_hard_numbers=int(info.n_hard_numbers))

    def mgf_fetch(self, n: int, n_peaks: int, out=None) -> dict:
        """Copies the resident CSR of the last parse to the host (`out`: dict of preallocated arrays)."""
        o = out or dict(offsets=np.zeros(n + 1, np.uint64), mz=np.zeros(n_peaks, np.float64),
                        intensity=np.zeros(n_peaks, np.float64), precursor_mz=np.zeros(n, np.float64),
                        charge=np.zeros(n, np.uint8), title_off=np.zeros(n, np.uint32),
                        title_len=np.zeros(n, np.uint32), seq_off=np.zeros(n, np.uint32),
                        seq_len=np.zeros(n, np.uint32))
        _check(capi.mgf_fetch(self._h, *[_ptr(o[k]) for k in ("offsets", "mz", "intensity", "precursor_mz", "charge",
                                                            "title_off", "title_len", "seq_off", "seq_len")]), self._h)
        return o

    def mgf_device_csr(self) -> dict:
        """Device pointers of the resident CSR of the last parse_mgf (valid until the next one)."""
        n, npk = C.c_uint64(), C.c_uint64()
        p = [C.c_void_p() for _ in range(5)]
        _check(capi.mgf_device_csr(self._h, C.byref(n), C.byref(npk), *[C.byref(x) for x in p]), self._h)
        return dict(n_spectra=n.value, n_peaks=npk.value, d_offsets=p[0].value or 0, d_mz=p[1].value or 0,
                    d_intensity=p[2].value or 0, d_precursor_mz=p[3].value or 0, d_charge=p[4].value or 0)

    # -- fused raw-spectra paths ---------------------------------------------
    def build_index_from_spectra(self, offsets, mz, intensity, preprocess: PreprocessConfig, precursor_mz,
                                 charge, ids=None, is_decoy=None, shard_index: int = 0, shard_count: int = 1,
                                 id_rank=None):
        """build_index(encode_spectra(spectra).encoded) without moving a hypervector to the host.
        Returns ok u8[n]; library ordinals count the processable spectra only (pipeline.cpp:75-83)."""
        offsets = _arr(offsets, np.uint64)
        mz = _arr(mz, np.float64)
        intensity = _arr(intensity, np.float64)
        precursor_mz = _arr(precursor_mz, np.float64)
        charge = _arr(charge, np.uint8)
        n = len(offsets) - 1
        if id_rank is None and ids is not None:
            id_rank = id_ranks(ids)
        rank = _arr(id_rank, np.uint32) if id_rank is not None else None
        ok = np.zeros(n, np.uint8)
        cnt = C.c_uint64()
        _check(capi.library_build_from_spectra(self._h, C.byref(preprocess.pod()), n, _ptr(offsets), _ptr(mz),
                                               _ptr(intensity), _ptr(precursor_mz), _ptr(charge), _ptr(rank),
                                               shard_index, shard_count, _ptr(ok), C.byref(cnt)), self._h)
        kept = np.flatnonzero(ok)
        dec = _arr(is_decoy, np.uint8)[kept] if is_decoy is not None else None
        self._set_lib(self.codebook.config.dim, int(cnt.value), dec)
        return ok

    def queries_from_spectra(self, offsets, mz, intensity, preprocess: PreprocessConfig, precursor_mz, charge):
        """encode_spectra with the result left resident as the query set.  Returns ok u8[n]."""
        offsets = _arr(offsets, np.uint64)
        mz = _arr(mz, np.float64)
        intensity = _arr(intensity, np.float64)
        precursor_mz = _arr(precursor_mz, np.float64)
        charge = _arr(charge, np.uint8)
        n = len(offsets) - 1
        ok = np.zeros(n, np.uint8)
        cnt = C.c_uint64()
        _check(capi.queries_from_spectra(self._h, C.byref(preprocess.pod()), n, _ptr(offsets), _ptr(mz),
                                         _ptr(intensity), _ptr(precursor_mz), _ptr(charge), _ptr(ok),
                                         C.byref(cnt)), self._h)
        self.resident_queries = int(cnt.value)
        return ok

    def queries_from_mgf(self, preprocess: PreprocessConfig, n_spectra: int) -> np.ndarray:
        """Known-charge filter + encode_spectra (pipeline.cpp:127-141) of the CSR the last parse_mgf left on the
        device; the result becomes the resident query set.  Returns state u8[n_spectra]: 0 = query, 1 = skipped
        (unknown charge), 2 = unprocessable."""
        state = np.zeros(n_spectra, np.uint8)
        cnt = C.c_uint64()
        _check(capi.queries_from_mgf(self._h, C.byref(preprocess.pod()), _ptr(state), C.byref(cnt)), self._h)
        self.resident_queries = int(cnt.value)
        return state

    def search_file(self, text: bytes, preprocess: PreprocessConfig, narrow: Tolerance, wide: Tolerance, fdr_q: float,
                    lib_ids, lib_peptides=None, decoy_prefix: str = "DECOY_") -> dict:
        """The query side of run_search (pipeline.cpp:119-150): MGF text in, accepted SSMs + statistics + the
        reference's TSV (write_ssm_tsv, :179-195) out.  The peaks never come back to the host; only titles,
        precursors and charges do (for the Ssm records)."""
        buf = np.frombuffer(text, np.uint8)
        info = capi.MgfInfoPod()
        _check(capi.mgf_parse(self._h, _ptr(buf) if len(buf) else 0, len(buf), C.byref(info)), self._h)
        n = int(info.n_spectra)
        state = self.queries_from_mgf(preprocess, n)
        acc = self.cascade_resident(narrow, wide, fdr_q)
        prec, charge = np.zeros(n, np.float64), np.zeros(n, np.uint8)
        toff, tlen = np.zeros(n, np.uint32), np.zeros(n, np.uint32)
        _check(capi.mgf_fetch(self._h, 0, 0, 0, _ptr(prec), _ptr(charge), _ptr(toff), _ptr(tlen), 0, 0), self._h)
        kept = np.flatnonzero(state == 0)
        lib_mz = self.lib_precursor_mz
        lines = ["query_id\tlibrary_id\tpeptide\tcharge\tquery_precursor_mz\tlibrary_precursor_mz\tmass_diff\tscore\t"
                 "stage\tq_value\n"]
        dim_d = float(self.lib_dim)
        for qi, o, st, sc, qv in zip(acc["query"], acc["ordinal"], acc["stage"], acc["raw_score"], acc["q_value"]):
            i = int(kept[int(qi)])
            qid = bytes(text[int(toff[i]):int(toff[i]) + int(tlen[i])]).decode() if tlen[i] else f"spectrum_{i + 1}"
            lid = lib_ids[int(o)]
            pep = lib_peptides[int(o)] if lib_peptides is not None else ""
            lines.append("%s\t%s\t%s\t%u\t%.5f\t%.5f\t%.5f\t%.6f\t%s\t%.6g\n" % (
                qid, lid, pep, charge[i], prec[i], lib_mz[int(o)], prec[i] - lib_mz[int(o)], float(sc) / dim_d,
                "narrow" if st == 0 else "wide", qv))
        stats = dict(total_queries=n, skipped_unknown_charge=int((state == 1).sum()), unprocessable=int((state == 2).sum()),
                     accepted_narrow=int((acc["stage"] == 0).sum()), accepted_wide=int((acc["stage"] == 1).sum()),
                     unidentified=int(len(kept) - len(acc["query"])))
        return dict(accepted=acc, stats=stats, tsv="".join(lines).encode(), kept=kept)

    def search_resident(self, tol: Tolerance, k: int = 1, nq: int | None = None) -> Match:
        """search_batch over the resident queries."""
        nq = self.resident_queries if nq is None else nq
        score = np.zeros((nq, k), np.uint32)
        ordinal = np.full((nq, k), capi.NO_HIT, np.uint32)
        first = np.zeros(nq, np.uint64)
        last = np.zeros(nq, np.uint64)
        _check(capi.search_resident(self._h, C.byref(tol.pod()), k, _ptr(score), _ptr(ordinal), _ptr(first),
                                    _ptr(last)), self._h)
        return Match(ordinal != capi.NO_HIT, score, ordinal, first, last)

    def cascade_resident(self, narrow: Tolerance, wide: Tolerance, fdr_q: float, nq: int | None = None) -> dict:
        """cascade_search over the resident queries."""
        nq = self.resident_queries if nq is None else nq
        query = np.zeros(nq, np.uint64)
        ordinal = np.zeros(nq, np.uint32)
        stage = np.zeros(nq, np.uint8)
        score = np.zeros(nq, np.uint32)
        qv = np.zeros(nq, np.float64)
        cnt = C.c_uint64()
        _check(capi.cascade_resident(self._h, C.byref(narrow.pod()), C.byref(wide.pod()), float(fdr_q),
                                     _ptr(self.lib_is_decoy), _ptr(query), _ptr(ordinal), _ptr(stage),
                                     _ptr(score), _ptr(qv), C.byref(cnt)), self._h)
        m = cnt.value
        return dict(query=query[:m].copy(), ordinal=ordinal[:m].copy(), stage=stage[:m].copy(),
                    raw_score=score[:m].copy(), q_value=qv[:m].copy())

    # -- device-resident pieces (multi-GPU composition, benchmarks) -------------------------
    def queries_upload(self, dim: int, q_words, q_mz, q_charge) -> int:
        q_mz = _arr(q_mz, np.float64)
        q_charge = _arr(q_charge, np.uint8)
        nq = len(q_mz)
        q_words = _arr(q_words, np.uint64)
        _check(capi.queries_upload(self._h, dim, nq, _ptr(q_words), _ptr(q_mz), _ptr(q_charge)),
               self._h)
        self.resident_queries = nq
        return nq

    def queries_upload_dev(self, dim: int, nq: int, d_words: int, d_mz: int, d_charge: int) -> None:
        _check(capi.queries_upload_dev(self._h, dim, nq, d_words, d_mz, d_charge), self._h)

    def search_resident_dev(self, tol: Tolerance, k: int, d_out: int, d_subset: int = 0,
                            n_subset: int = 0) -> None:
        _check(capi.search_resident_dev(self._h, d_subset, n_subset, C.byref(tol.pod()), k, d_out),
               self._h)

    def merge_candidates_dev(self, n: int, k: int, n_parts: int, d_parts: int, d_out: int) -> None:
        _check(capi.merge_candidates_dev(self._h, n, k, n_parts, d_parts, d_out), self._h)

    def candidates_decode(self, n: int, k: int, d_records: int):
        score = np.zeros((n, k), np.uint32)
        ordinal = np.zeros((n, k), np.uint32)
        _check(capi.candidates_decode(self._h, n, k, d_records, _ptr(score), _ptr(ordinal)),
               self._h)
        return score, ordinal

    def encode_batch_dev(self, preprocess: PreprocessConfig, n: int, n_peaks: int, d_offsets: int,
                         d_mz: int, d_intensity: int, d_out_words: int, d_out_ok: int) -> None:
        _check(capi.encode_batch_dev(self._h, C.byref(preprocess.pod()), n, n_peaks, d_offsets,
                                     d_mz, d_intensity, d_out_words, d_out_ok), self._h)
