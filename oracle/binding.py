"""ctypes binding shared by the two CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import this module; the product package never does.

Two shared objects expose the same flat C signatures under different prefixes:

* ``oracle/_ref/libhoms_ref.so`` (prefix ``hr_``)  -- the UNMODIFIED reference compiled from
  ``/root/reference/proj/core/src`` behind ``oracle/ref_shim.cpp`` (``kind="ref"``; the
  ``-march=x86-64-v3`` flavour is ``kind="ref_v3"``);
* ``oracle/libhoms_oracle.so`` (prefix ``ho_``) -- the plain-C restatement ``oracle/homs_oracle.c``
  (``kind="port"``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REFERENCE_ROOT = os.environ.get("HOMS_REFERENCE_ROOT", "/root/reference")

_LIBS = {
    "ref": (os.path.join(HERE, "_ref", "libhoms_ref.so"), "hr_"),
    "ref_v3": (os.path.join(HERE, "_ref", "libhoms_ref_v3.so"), "hr_"),
    "port": (os.path.join(HERE, "libhoms_oracle.so"), "ho_"),
}

PPM, DALTON = 0, 1


def tol_kind(kind) -> int:
    if kind in (0, "ppm"):
        return PPM
    if kind in (1, "da", "dalton"):
        return DALTON
    raise ValueError(f"unknown tolerance kind {kind!r}")


class PreCfg(C.Structure):
    """POD mirror of PreprocessConfig (reference preprocess.hpp:13-25)."""

    _fields_ = [
        ("min_mz", C.c_double),
        ("max_mz", C.c_double),
        ("bin_size", C.c_double),
        ("max_peaks", C.c_uint32),
        ("min_peaks", C.c_uint32),
        ("intensity_floor", C.c_double),
        ("scaling", C.c_uint32),
        ("pad_", C.c_uint32),
    ]

    def __init__(self, min_mz=101.0, max_mz=1500.0, bin_size=0.05, max_peaks=50, min_peaks=10,
                 intensity_floor=0.01, scaling=0):
        super().__init__(min_mz, max_mz, bin_size, max_peaks, min_peaks, intensity_floor,
                         scaling, 0)


class EncCfg(C.Structure):
    """POD mirror of EncoderConfig (reference codebook.hpp:12-23)."""

    _fields_ = [("dim", C.c_uint32), ("step_flips", C.c_uint32), ("levels", C.c_uint32),
                ("pad_", C.c_uint32), ("seed", C.c_uint64)]

    def __init__(self, dim=8192, step_flips=4096, levels=16, seed=1):
        super().__init__(dim, step_flips, levels, 0, seed)


class SynthCfg(C.Structure):
    """POD mirror of SynthConfig (reference synth.hpp:17-33)."""

    _fields_ = [
        ("n_library", C.c_uint64),
        ("n_query", C.c_uint64),
        ("peaks_per_spectrum", C.c_uint32),
        ("pad_", C.c_uint32),
        ("mz_min", C.c_double),
        ("mz_max", C.c_double),
        ("fraction_modified", C.c_double),
        ("precursor_shift_da", C.c_double),
        ("fraction_peaks_shifted", C.c_double),
        ("intensity_noise", C.c_double),
        ("decoy_ratio", C.c_double),
        ("seed", C.c_uint64),
    ]

    def __init__(self, n_library=1000, n_query=100, peaks_per_spectrum=50, mz_min=150.0,
                 mz_max=1300.0, fraction_modified=0.0, precursor_shift_da=79.97,
                 fraction_peaks_shifted=0.3, intensity_noise=0.05, decoy_ratio=1.0, seed=1):
        super().__init__(n_library, n_query, peaks_per_spectrum, 0, mz_min, mz_max,
                         fraction_modified, precursor_shift_da, fraction_peaks_shifted,
                         intensity_noise, decoy_ratio, seed)


def available(kind: str) -> bool:
    return os.path.exists(_LIBS[kind][0])


def build(kind: str = "all", quiet: bool = True) -> None:
    """Compile the checkers (``make -C oracle port|ref``).  ``ref`` needs /root/reference."""
    targets = []
    if kind in ("all", "port"):
        targets.append("port")
    if kind in ("all", "ref") and os.path.isdir(os.path.join(REFERENCE_ROOT, "proj", "core")):
        targets.append("ref")
    for t in targets:
        subprocess.run(["make", "-C", HERE, t, f"REF={REFERENCE_ROOT}"], check=True,
                       stdout=subprocess.DEVNULL if quiet else None)


def _p(a, ty):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ty))


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def words_for(dim: int) -> int:
    return (dim + 63) // 64


_FNV_LIB = None


def fnv1a64_words(words: np.ndarray) -> int:
    """FNV-1a-64 over the little-endian bytes of u64 words, the hash the reference cache uses
    for its hypervector block (reference cache.cpp:18-29); SURVEY.md section 8(c) fingerprints.
    Runs in C (ho_fnv1a64 of the port library)."""
    global _FNV_LIB
    if _FNV_LIB is None:
        _FNV_LIB = C.CDLL(_LIBS["port"][0])
        _FNV_LIB.ho_fnv1a64.restype = C.c_uint64
        _FNV_LIB.ho_fnv1a64.argtypes = [C.c_void_p, C.c_uint64]
    data = np.ascontiguousarray(words, dtype="<u8")
    return int(_FNV_LIB.ho_fnv1a64(data.ctypes.data, data.nbytes))


@dataclass
class Codebook:
    handle: int
    dim: int
    levels: int
    n_bins: int
    pos: np.ndarray  # [n_bins, W] u64
    lvl: np.ndarray  # [levels + 1, W] u64


class Oracle:
    def __init__(self, kind: str = "ref"):
        path, prefix = _LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.pre = prefix
        self._declare()

    # -- plumbing ---------------------------------------------------------------------------
    def _fn(self, name, restype, argtypes):
        f = getattr(self.lib, self.pre + name)
        f.restype = restype
        f.argtypes = argtypes
        return f

    def _declare(self):
        LL, VP, U64, U32, U8, F64, I = (C.c_longlong, C.c_void_p, C.c_uint64, C.c_uint32,
                                        C.c_uint8, C.c_double, C.c_int)
        P = C.POINTER
        f = self._fn
        self._last_error = f("last_error", C.c_char_p, [])
        self._dimension = f("dimension", LL, [P(PreCfg)])
        self._validate = f("validate_preprocess", LL, [P(PreCfg)])
        self._refvec = f("refine_vectorize", LL, [P(PreCfg), U64, P(F64), P(F64), U32, P(U32),
                                                  P(F64), P(U32)])
        self._quant = f("quantize_intensity", LL, [F64, U32])
        self._cb_create = f("codebook_create", VP, [U32, U32, U32, U64, U32])
        self._cb_from = f("codebook_from_words", VP, [U32, U32, U32, P(U64), P(U64)])
        self._cb_export = f("codebook_export", None, [VP, P(U64), P(U64)])
        self._cb_free = f("codebook_free", None, [VP])
        self._enc = f("encode_spectra", LL, [VP, P(PreCfg), U64, P(U64), P(F64), P(F64),
                                             C.c_uint, U64, P(U64), P(U8)])
        self._encvec = f("encode_vector", LL, [VP, U32, P(U32), P(F64), I, P(U64)])
        self._ham = f("hamming_similarity", LL, [U32, P(U64), P(U64), I])
        self._ix_create = f("index_create", VP, [U32, U64, P(U64), P(F64), P(U8), P(U8),
                                                 C.c_char_p, P(U64)])
        self._ix_free = f("index_free", None, [VP])
        self._ix_bcount = f("index_bucket_count", LL, [VP])
        self._ix_binfo = f("index_bucket_info", LL, [VP, U32, P(U8), P(U64)])
        self._ix_bexport = f("index_bucket_export", LL, [VP, U32, P(F64), P(U32), P(U64)])
        self._select = f("select_candidates", LL, [VP, U64, P(F64), P(U8), I, F64, P(U64),
                                                   P(U64), P(U8)])
        self._search = f("search_batch", LL, [VP, U64, P(U64), P(F64), P(U8), I, F64, C.c_uint,
                                              U64, I, P(U8), P(U32), P(U32), P(F64)])
        self._cascade = f("cascade_search", LL, [VP, U64, P(U64), P(F64), P(U8), I, F64, I, F64,
                                                 F64, C.c_uint, U64, P(U64), P(U32), P(U8),
                                                 P(U32), P(F64)])
        self._fdr = f("compute_fdr_curve", LL, [U64, P(F64), P(U8), P(U64), P(F64), P(F64)])
        self._synth_create = f("synth_create", VP, [P(SynthCfg)])
        self._synth_free = f("synth_free", None, [VP])
        self._synth_sizes = f("synth_sizes", None, [VP, I, P(U64)])
        self._synth_export = f("synth_export", None, [VP, I, P(U64), P(F64), P(F64), P(F64),
                                                      P(U8), P(U8), C.c_char_p, P(U64)])
        self._synth_truth = f("synth_truth", None, [VP, P(U64), P(U8)])
        UC = P(C.c_ubyte)
        self._cache_write = f("cache_write", LL, [P(PreCfg), P(EncCfg), U64, P(U64), P(F64), P(U8), P(U8),
                                                  C.c_char_p, P(U64), C.c_char_p, P(U64), UC, U64])
        self._cache_read = f("cache_read", LL, [UC, U64, P(PreCfg), P(EncCfg), P(U64), P(F64), P(U8), P(U8),
                                                C.c_char_p, P(U64), C.c_char_p, P(U64)])
        self._mgf_parse = f("mgf_parse", VP, [C.c_char_p, U64, C.c_char_p])
        self._mgf_free = f("mgf_free", None, [VP])
        self._mgf_sizes = f("mgf_sizes", None, [VP, P(U64)])
        self._mgf_export = f("mgf_export", None, [VP, P(U64), P(F64), P(F64), P(F64), P(U8), P(U8),
                                                  C.c_char_p, P(U64), C.c_char_p, P(U64)])
        self._mgf_write = f("mgf_write", LL, [U64, P(U64), P(F64), P(F64), P(F64), P(U8), C.c_char_p, P(U64),
                                              C.c_char_p, P(U64), C.c_char_p, U64])
        if self.kind == "port":
            self._topk = f("search_topk", LL, [VP, U64, P(U64), P(F64), P(U8), I, F64, U32,
                                               P(U32), P(U32)])

    def error(self) -> str:
        return (self._last_error() or b"").decode()

    def _check(self, rc):
        if rc is None or (isinstance(rc, int) and rc < 0):
            raise OracleError(self.error())
        return rc

    # -- preprocess -------------------------------------------------------------------------
    def dimension(self, cfg: PreCfg) -> int:
        return self._check(self._dimension(C.byref(cfg)))

    def validate_preprocess(self, cfg: PreCfg) -> None:
        self._check(self._validate(C.byref(cfg)))

    def refine_vectorize(self, cfg: PreCfg, mz, inten, levels=16):
        mz, inten = _f64(mz), _f64(inten)
        n = len(mz)
        bins = np.zeros(max(n, 1), np.uint32)
        vals = np.zeros(max(n, 1), np.float64)
        lev = np.zeros(max(n, 1), np.uint32)
        rc = self._check(self._refvec(C.byref(cfg), n, _p(mz, C.c_double), _p(inten, C.c_double),
                                      levels, _p(bins, C.c_uint32), _p(vals, C.c_double),
                                      _p(lev, C.c_uint32)))
        if rc == 0:
            return None
        return bins[:rc].copy(), vals[:rc].copy(), lev[:rc].copy()

    def quantize_intensity(self, v: float, levels: int) -> int:
        return self._check(self._quant(v, levels))

    # -- codebook ---------------------------------------------------------------------------
    def _wrap_codebook(self, h, dim, levels, n_bins) -> Codebook:
        if not h:
            raise OracleError(self.error())
        W = words_for(dim)
        pos = np.zeros((n_bins, W), np.uint64)
        lvl = np.zeros((levels + 1, W), np.uint64)
        self._cb_export(h, _p(pos, C.c_uint64), _p(lvl, C.c_uint64))
        return Codebook(h, dim, levels, n_bins, pos, lvl)

    def make_codebook(self, dim, step_flips, levels, seed, n_bins) -> Codebook:
        h = self._cb_create(dim, step_flips, levels, seed, n_bins)
        return self._wrap_codebook(h, dim, levels, n_bins)

    def codebook_from_words(self, dim, levels, pos, lvl) -> Codebook:
        pos, lvl = _u64(pos), _u64(lvl)
        n_bins = pos.shape[0]
        h = self._cb_from(dim, levels, n_bins, _p(pos, C.c_uint64), _p(lvl, C.c_uint64))
        return self._wrap_codebook(h, dim, levels, n_bins)

    def free_codebook(self, cb: Codebook) -> None:
        self._cb_free(cb.handle)
        cb.handle = None

    # -- encode -----------------------------------------------------------------------------
    def encode_spectra(self, cb: Codebook, cfg: PreCfg, offsets, mz, inten, threads=1, batch=64):
        offsets, mz, inten = _u64(offsets), _f64(mz), _f64(inten)
        n = len(offsets) - 1
        W = words_for(cb.dim)
        words = np.zeros((n, W), np.uint64)
        ok = np.zeros(n, np.uint8)
        rc = self._check(self._enc(cb.handle, C.byref(cfg), n, _p(offsets, C.c_uint64),
                                   _p(mz, C.c_double), _p(inten, C.c_double), threads, batch,
                                   _p(words, C.c_uint64), _p(ok, C.c_uint8)))
        assert rc == n - int(ok.sum())
        return words, ok

    def encode_vector(self, cb: Codebook, bins, intens, unpacked=False):
        bins, intens = _u32(bins), _f64(intens)
        out = np.zeros(words_for(cb.dim), np.uint64)
        self._check(self._encvec(cb.handle, len(bins), _p(bins, C.c_uint32),
                                 _p(intens, C.c_double), int(unpacked), _p(out, C.c_uint64)))
        return out

    def hamming_similarity(self, dim, a, b, bitwise=False) -> int:
        a, b = _u64(a), _u64(b)
        return self._check(self._ham(dim, _p(a, C.c_uint64), _p(b, C.c_uint64), int(bitwise)))

    # -- index / search ---------------------------------------------------------------------
    def build_index(self, dim, words, mz, charge, is_decoy=None, ids=None) -> "Index":
        words, mz, charge = _u64(words), _f64(mz), _u8(charge)
        n = len(mz)
        dec = _u8(is_decoy) if is_decoy is not None else None
        blob, off = encode_ids(ids) if ids is not None else (None, None)
        h = self._ix_create(dim, n, _p(words, C.c_uint64), _p(mz, C.c_double),
                            _p(charge, C.c_uint8), _p(dec, C.c_uint8), blob,
                            _p(off, C.c_uint64))
        if not h:
            raise OracleError(self.error())
        return Index(self, h, dim, n)

    def compute_fdr_curve(self, score, is_decoy):
        score, is_decoy = _f64(score), _u8(is_decoy)
        n = len(score)
        order = np.zeros(n, np.uint64)
        fdr = np.zeros(n, np.float64)
        q = np.zeros(n, np.float64)
        self._check(self._fdr(n, _p(score, C.c_double), _p(is_decoy, C.c_uint8),
                              _p(order, C.c_uint64), _p(fdr, C.c_double), _p(q, C.c_double)))
        return order, fdr, q

    # -- encoded-library cache (reference cache.cpp:122-211) ---------------------------------
    def cache_write(self, pre: PreCfg, enc: "EncCfg", words, mz, charge, is_decoy, ids, peptides) -> bytes:
        words, mz, charge, dec = _u64(words), _f64(mz), _u8(charge), _u8(is_decoy)
        n = len(mz)
        iblob, ioff = encode_ids(ids)
        pblob, poff = encode_ids(peptides)
        args = (C.byref(pre), C.byref(enc), n, _p(words, C.c_uint64), _p(mz, C.c_double),
                _p(charge, C.c_uint8), _p(dec, C.c_uint8), iblob, _p(ioff, C.c_uint64), pblob,
                _p(poff, C.c_uint64))
        size = self._check(self._cache_write(*args, None, 0))
        buf = (C.c_ubyte * size)()
        self._check(self._cache_write(*args, buf, size))
        return bytes(buf)

    def cache_read(self, image: bytes, pre: PreCfg, enc: "EncCfg") -> dict:
        """-> dict(words, mz, charge, is_decoy, ids, peptides); raises OracleError naming the
        reference exception class (CacheFormatError / StaleCacheError / CacheCorruptError)."""
        n_bytes = len(image)
        buf = (C.c_ubyte * max(1, n_bytes)).from_buffer_copy(image if n_bytes else b"\0")
        nul = (None,) * 8
        n = self._check(self._cache_read(buf, n_bytes, C.byref(pre), C.byref(enc), *nul))
        W = words_for(enc.dim)
        words = np.zeros((n, W), np.uint64)
        mz = np.zeros(n, np.float64)
        charge = np.zeros(n, np.uint8)
        dec = np.zeros(n, np.uint8)
        iblob = C.create_string_buffer(max(1, n_bytes))
        pblob = C.create_string_buffer(max(1, n_bytes))
        ioff = np.zeros(n + 1, np.uint64)
        poff = np.zeros(n + 1, np.uint64)
        self._check(self._cache_read(buf, n_bytes, C.byref(pre), C.byref(enc), _p(words, C.c_uint64),
                                     _p(mz, C.c_double), _p(charge, C.c_uint8), _p(dec, C.c_uint8), iblob,
                                     _p(ioff, C.c_uint64), pblob, _p(poff, C.c_uint64)))
        iraw, praw = iblob.raw, pblob.raw  # .raw copies the whole buffer: take it once
        ids = [iraw[int(ioff[i]):int(ioff[i + 1])].decode() for i in range(n)]
        peps = [praw[int(poff[i]):int(poff[i + 1])].decode() for i in range(n)]
        return dict(words=words, mz=mz, charge=charge, is_decoy=dec, ids=ids, peptides=peps)

    # -- synth ------------------------------------------------------------------------------
    def synth(self, cfg: SynthCfg) -> dict:
        h = self._synth_create(C.byref(cfg))
        if not h:
            raise OracleError(self.error())
        out = {}
        try:
            for which, name in ((0, "library"), (1, "queries")):
                sizes = np.zeros(3, np.uint64)
                self._synth_sizes(h, which, _p(sizes, C.c_uint64))
                n, npk, nid = (int(x) for x in sizes)
                offsets = np.zeros(n + 1, np.uint64)
                mz = np.zeros(npk, np.float64)
                inten = np.zeros(npk, np.float64)
                prec = np.zeros(n, np.float64)
                charge = np.zeros(n, np.uint8)
                decoy = np.zeros(n, np.uint8)
                blob = C.create_string_buffer(max(nid, 1))
                id_off = np.zeros(n + 1, np.uint64)
                self._synth_export(h, which, _p(offsets, C.c_uint64), _p(mz, C.c_double),
                                   _p(inten, C.c_double), _p(prec, C.c_double),
                                   _p(charge, C.c_uint8), _p(decoy, C.c_uint8), blob,
                                   _p(id_off, C.c_uint64))
                raw = blob.raw[:nid]
                ids = [raw[int(id_off[i]):int(id_off[i + 1])].decode() for i in range(n)]
                out[name] = dict(offsets=offsets, mz=mz, intensity=inten, precursor_mz=prec,
                                 charge=charge, is_decoy=decoy, ids=ids)
            nq = len(out["queries"]["precursor_mz"])
            src = np.zeros(nq, np.uint64)
            mod = np.zeros(nq, np.uint8)
            self._synth_truth(h, _p(src, C.c_uint64), _p(mod, C.c_uint8))
            out["truth"] = dict(source_index=src, modified=mod)
        finally:
            self._synth_free(h)
        return out


    # -- MGF text (src/mgf.cpp) -----------------------------------------------------------------
    def mgf_parse(self, text: bytes, decoy_prefix: str = "DECOY_") -> dict:
        """parse_mgf: CSR peaks + metadata; OracleError("ParseError: line N: ...") on a violation."""
        h = self._mgf_parse(text, len(text), decoy_prefix.encode())
        if not h:
            raise OracleError(self.error())
        try:
            sizes = np.zeros(4, np.uint64)
            self._mgf_sizes(h, _p(sizes, C.c_uint64))
            n, npk, nid, npep = (int(x) for x in sizes)
            offsets = np.zeros(n + 1, np.uint64)
            mz = np.zeros(npk, np.float64)
            inten = np.zeros(npk, np.float64)
            prec = np.zeros(n, np.float64)
            charge = np.zeros(n, np.uint8)
            decoy = np.zeros(n, np.uint8)
            iblob, pblob = C.create_string_buffer(max(nid, 1)), C.create_string_buffer(max(npep, 1))
            ioff, poff = np.zeros(n + 1, np.uint64), np.zeros(n + 1, np.uint64)
            self._mgf_export(h, _p(offsets, C.c_uint64), _p(mz, C.c_double), _p(inten, C.c_double),
                             _p(prec, C.c_double), _p(charge, C.c_uint8), _p(decoy, C.c_uint8), iblob,
                             _p(ioff, C.c_uint64), pblob, _p(poff, C.c_uint64))
            ri, rp = iblob.raw[:nid], pblob.raw[:npep]
            ids = [ri[int(ioff[i]):int(ioff[i + 1])] for i in range(n)]
            peps = [rp[int(poff[i]):int(poff[i + 1])] for i in range(n)]
            return dict(offsets=offsets, mz=mz, intensity=inten, precursor_mz=prec, charge=charge,
                        is_decoy=decoy, ids=ids, peptides=peps)
        finally:
            self._mgf_free(h)

    def mgf_write(self, offsets, mz, inten, precursor_mz, charge, ids, peptides=None) -> bytes:
        """write_mgf of the given spectra."""
        offsets, mz, inten = _u64(offsets), _f64(mz), _f64(inten)
        prec, charge = _f64(precursor_mz), _u8(charge)
        n = len(prec)
        iblob, ioff = encode_ids(ids)
        pblob, poff = encode_ids(peptides if peptides is not None else [b""] * n)
        args = (n, _p(offsets, C.c_uint64), _p(mz, C.c_double), _p(inten, C.c_double), _p(prec, C.c_double),
                _p(charge, C.c_uint8), iblob, _p(ioff, C.c_uint64), pblob, _p(poff, C.c_uint64))
        size = self._check(self._mgf_write(*args, None, 0))
        out = C.create_string_buffer(max(size, 1))
        self._check(self._mgf_write(*args, out, size))
        return out.raw[:size]


class OracleError(RuntimeError):
    pass


def encode_ids(ids):
    enc = [s.encode() if isinstance(s, str) else bytes(s) for s in ids]
    off = np.zeros(len(enc) + 1, np.uint64)
    if enc:
        off[1:] = np.cumsum([len(e) for e in enc])
    return b"".join(enc) + b"\0", off


class Index:
    def __init__(self, oracle: Oracle, handle, dim, n):
        self.o, self.h, self.dim, self.n = oracle, handle, dim, n

    def close(self):
        if self.h:
            self.o._ix_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def buckets(self):
        out = []
        W = words_for(self.dim)
        for b in range(self.o._ix_bcount(self.h)):
            ch = C.c_uint8()
            sz = C.c_uint64()
            self.o._ix_binfo(self.h, b, C.byref(ch), C.byref(sz))
            n = sz.value
            mz = np.zeros(n, np.float64)
            ordinal = np.zeros(n, np.uint32)
            words = np.zeros((n, W), np.uint64)
            self.o._ix_bexport(self.h, b, _p(mz, C.c_double), _p(ordinal, C.c_uint32),
                               _p(words, C.c_uint64))
            out.append(dict(charge=ch.value, precursor_mz=mz, ordinal=ordinal, words=words))
        return out

    def select_candidates(self, q_mz, q_charge, tol):
        q_mz, q_charge = _f64(q_mz), _u8(q_charge)
        nq = len(q_mz)
        first = np.zeros(nq, np.uint64)
        last = np.zeros(nq, np.uint64)
        has = np.zeros(nq, np.uint8)
        self.o._check(self.o._select(self.h, nq, _p(q_mz, C.c_double), _p(q_charge, C.c_uint8),
                                     tol_kind(tol[0]), float(tol[1]), _p(first, C.c_uint64),
                                     _p(last, C.c_uint64), _p(has, C.c_uint8)))
        return first, last, has

    def search_batch(self, q_words, q_mz, q_charge, tol, threads=1, batch=64, linear=False):
        q_words, q_mz, q_charge = _u64(q_words), _f64(q_mz), _u8(q_charge)
        nq = len(q_mz)
        has = np.zeros(nq, np.uint8)
        score = np.zeros(nq, np.uint32)
        ordinal = np.zeros(nq, np.uint32)
        mdiff = np.zeros(nq, np.float64)
        self.o._check(self.o._search(self.h, nq, _p(q_words, C.c_uint64), _p(q_mz, C.c_double),
                                     _p(q_charge, C.c_uint8), tol_kind(tol[0]), float(tol[1]),
                                     threads, batch, int(linear), _p(has, C.c_uint8),
                                     _p(score, C.c_uint32), _p(ordinal, C.c_uint32),
                                     _p(mdiff, C.c_double)))
        return has, score, ordinal, mdiff

    def search_topk(self, q_words, q_mz, q_charge, tol, k):
        """Full sort on the reference's 4-level key, first k (port only)."""
        q_words, q_mz, q_charge = _u64(q_words), _f64(q_mz), _u8(q_charge)
        nq = len(q_mz)
        score = np.zeros((nq, k), np.uint32)
        ordinal = np.zeros((nq, k), np.uint32)
        self.o._check(self.o._topk(self.h, nq, _p(q_words, C.c_uint64), _p(q_mz, C.c_double),
                                   _p(q_charge, C.c_uint8), tol_kind(tol[0]), float(tol[1]), k,
                                   _p(score, C.c_uint32), _p(ordinal, C.c_uint32)))
        return score, ordinal

    def query_flow(self, cb: "Codebook", cfg: "PreCfg", text: bytes, narrow, wide, fdr_q, threads=1, batch=64,
                   decoy_prefix: str = "DECOY_") -> dict:
        """The query side of the reference's run_search (pipeline.cpp:119-150) on an MGF image: parse_mgf ->
        known charges -> encode_spectra -> cascade_search -> write_ssm_tsv.  ref only.  Library peptides in
        the TSV are the decimal ordinals the shim tags entries with."""
        fn = self.o._fn("query_flow", C.c_longlong,
                        [C.c_void_p, C.c_void_p, C.POINTER(PreCfg), C.c_char_p, C.c_uint64, C.c_char_p, C.c_int,
                         C.c_double, C.c_int, C.c_double, C.c_double, C.c_uint, C.c_uint64, C.POINTER(C.c_double),
                         C.POINTER(C.c_uint64), C.c_char_p, C.c_uint64])
        sec = (C.c_double * 3)()
        stats = (C.c_uint64 * 6)()
        args = (self.h, cb.handle, C.byref(cfg), text, len(text), decoy_prefix.encode(), tol_kind(narrow[0]),
                float(narrow[1]), tol_kind(wide[0]), float(wide[1]), float(fdr_q), threads, batch)
        size = self.o._check(fn(*args, sec, stats, None, 0))
        buf = C.create_string_buffer(max(1, size))
        self.o._check(fn(*args, sec, stats, buf, size))
        names = ("total_queries", "skipped_unknown_charge", "unprocessable", "accepted_narrow", "accepted_wide",
                 "unidentified")
        return dict(tsv=buf.raw[:size], seconds=dict(parse=sec[0], encode=sec[1], cascade=sec[2]),
                    stats={k: int(v) for k, v in zip(names, stats)})

    def cascade_search(self, q_words, q_mz, q_charge, narrow, wide, fdr_q, threads=1, batch=64):
        q_words, q_mz, q_charge = _u64(q_words), _f64(q_mz), _u8(q_charge)
        nq = len(q_mz)
        query = np.zeros(nq, np.uint64)
        ordinal = np.zeros(nq, np.uint32)
        stage = np.zeros(nq, np.uint8)
        score = np.zeros(nq, np.uint32)
        qv = np.zeros(nq, np.float64)
        n = self.o._check(self.o._cascade(
            self.h, nq, _p(q_words, C.c_uint64), _p(q_mz, C.c_double), _p(q_charge, C.c_uint8),
            tol_kind(narrow[0]), float(narrow[1]), tol_kind(wide[0]), float(wide[1]),
            float(fdr_q), threads, batch, _p(query, C.c_uint64), _p(ordinal, C.c_uint32),
            _p(stage, C.c_uint8), _p(score, C.c_uint32), _p(qv, C.c_double)))
        return dict(query=query[:n].copy(), ordinal=ordinal[:n].copy(), stage=stage[:n].copy(),
                    raw_score=score[:n].copy(), q_value=qv[:n].copy())
