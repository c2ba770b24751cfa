"""Encoded-library cache (reference src/cache.cpp:98-211).

CPU: the C restatement against the golden file the reference wrote, the compiled reference when
present, the reference's error classes (test_cache.cpp:104-138), and the product's host-only parser.
GPU: device FNV-1a-64, cache image -> resident index (== build_index on the same entries),
byte-identical write_cache from host and device rows, checksum corruption caught on the device."""
import os

import numpy as np
import pytest

from oracle.binding import EncCfg, OracleError, PreCfg
from tests import _util as U

GOLDEN = U.GOLDEN


def _golden():
    with open(os.path.join(GOLDEN, "cache_small.homs"), "rb") as f:
        image = f.read()
    z = np.load(os.path.join(GOLDEN, "cache_small.npz"))
    ent = dict(words=z["words"], mz=z["mz"], charge=z["charge"], decoy=z["decoy"],
               ids=[x.decode() for x in z["ids"]], peptides=[x.decode() for x in z["peptides"]])
    p, e = z["pre"], z["enc"]
    return image, ent, p, e


def _opre(p):
    return PreCfg(float(p[0]), float(p[1]), float(p[2]), int(p[3]), int(p[4]), float(p[5]), int(p[6]))


def _ppre(hb, p):
    return hb.PreprocessConfig(float(p[0]), float(p[1]), float(p[2]), int(p[3]), int(p[4]), float(p[5]), int(p[6]))


CORRUPTIONS = (  # (mutation, reference exception class) -- test_cache.cpp:104-138
    (lambda b: b"XOMS" + b[4:], "CacheFormatError"),
    (lambda b: b[:4] + b"\x07" + b[5:], "CacheFormatError"),
    (lambda b: b[:8] + bytes([b[8] ^ 0x10]) + b[9:], "StaleCacheError"),       # profile byte
    (lambda b: b[:60] + bytes([b[60] ^ 1]) + b[61:], "StaleCacheError"),
    (lambda b: b[:-3], "CacheCorruptError"),                                   # truncated digest
    (lambda b: b[:200], "CacheCorruptError"),                                  # truncated metadata
    (lambda b: b[:3], "CacheCorruptError"),
    (lambda b: b"", "CacheCorruptError"),
    (lambda b: b[:77] + b"\xff\xff\xff\x7f" + b[81:], "CacheCorruptError"),    # first id length absurd
    (lambda b: b[:-20] + bytes([b[-20] ^ 0x40]) + b[-19:], "CacheCorruptError"),  # flipped block byte
    (lambda b: b[:-1] + bytes([b[-1] ^ 1]), "CacheCorruptError"),              # flipped digest byte
)


def _check_read(oracle, image, ent, opre, oenc):
    r = oracle.cache_read(image, opre, oenc)
    assert np.array_equal(r["words"], ent["words"]) and np.array_equal(r["mz"], ent["mz"])
    assert np.array_equal(r["charge"], ent["charge"]) and np.array_equal(r["is_decoy"], ent["decoy"])
    assert r["ids"] == ent["ids"] and r["peptides"] == ent["peptides"]


def test_port_reads_and_rewrites_the_reference_file(port):
    image, ent, p, e = _golden()
    opre, oenc = _opre(p), EncCfg(*[int(x) for x in e])
    _check_read(port, image, ent, opre, oenc)
    again = port.cache_write(opre, oenc, ent["words"], ent["mz"], ent["charge"], ent["decoy"], ent["ids"],
                             ent["peptides"])
    assert again == image  # byte-identical to what the reference wrote
    fp = U.fingerprints()["cache_small"]
    assert len(image) == fp["bytes"]
    for mutate, cls in CORRUPTIONS:
        with pytest.raises(OracleError, match="^" + cls):
            port.cache_read(mutate(image), opre, oenc)
    with pytest.raises(OracleError, match="^StaleCacheError"):
        port.cache_read(image, opre, EncCfg(int(e[0]), int(e[1]), int(e[2]), int(e[3]) + 1))
    assert port.cache_read(port.cache_write(opre, oenc, np.zeros((0, 5), np.uint64), [], [], [], [], []),
                           opre, oenc)["words"].shape == (0, 5)


def test_port_equals_live_reference(port, ref):
    image, ent, p, e = _golden()
    opre, oenc = _opre(p), EncCfg(*[int(x) for x in e])
    _check_read(ref, image, ent, opre, oenc)
    assert ref.cache_write(opre, oenc, ent["words"], ent["mz"], ent["charge"], ent["decoy"], ent["ids"],
                           ent["peptides"]) == image
    for mutate, cls in CORRUPTIONS:
        with pytest.raises(OracleError, match="^" + cls):
            ref.cache_read(mutate(image), opre, oenc)


def test_product_parser_host_only(hb):
    image, ent, p, e = _golden()
    pre, enc = _ppre(hb, p), hb.EncoderConfig(*[int(x) for x in e])
    m = hb.cache_parse(image, pre, enc)
    W = ent["words"].shape[1]
    assert m["count"] == len(ent["mz"]) and m["hv_bytes"] == len(ent["mz"]) * W * 8
    assert m["ids"] == ent["ids"] and m["peptides"] == ent["peptides"]
    assert np.array_equal(m["precursor_mz"], ent["mz"]) and np.array_equal(m["charge"], ent["charge"])
    assert np.array_equal(m["is_decoy"], ent["decoy"])
    block = np.frombuffer(image, np.uint8, m["hv_bytes"], m["hv_offset"]).view(np.uint64).reshape(-1, W)
    assert np.array_equal(block, ent["words"])
    classes = {"CacheFormatError": hb.CacheFormatError, "StaleCacheError": hb.StaleCacheError,
               "CacheCorruptError": hb.CacheCorruptError}
    for mutate, cls in CORRUPTIONS[:9]:  # the last two only fail the checksum, which needs the device
        with pytest.raises(classes[cls]):
            hb.cache_parse(mutate(image), pre, enc)


@pytest.mark.gpu
def test_device_fnv1a64(hb, ctx, port):
    import ctypes
    from oracle.binding import fnv1a64_words
    ho_fnv = port.lib.ho_fnv1a64
    ho_fnv.restype, ho_fnv.argtypes = ctypes.c_uint64, [ctypes.c_void_p, ctypes.c_uint64]
    rng = np.random.default_rng(8)
    assert ctx.fnv1a64(b"") == 1469598103934665603
    for n in (1, 7, 8, 255, 16383, 16384, 16385, 65536 + 3, 256 * 16384, 256 * 16384 + 1, 5_000_011):
        data = rng.integers(0, 256, n, dtype=np.uint8)
        want = int(ho_fnv(data.ctypes.data, n))
        assert ctx.fnv1a64(data) == want, n
    words = rng.integers(0, 2**64, 100_000, dtype=np.uint64)
    assert ctx.fnv1a64(words) == fnv1a64_words(words)
    zeros = np.zeros(70_000, np.uint8)
    assert ctx.fnv1a64(zeros) == int(ho_fnv(zeros.ctypes.data, 70_000))


@pytest.mark.gpu
def test_load_cache_equals_build_index(hb, best_oracle):
    rng = np.random.default_rng(12)
    dim, n, nq = 1024, 3000, 200
    words = U.random_hvs(rng, n, dim)
    words[2800:] = words[:200]
    mz = np.round(rng.uniform(400.0, 1200.0, n), 3)
    charge = rng.integers(0, 4, n).astype(np.uint8)
    decoy = (rng.uniform(0, 1, n) < 0.5).astype(np.uint8)
    ids = [f"c{rng.integers(0, 600)}" for _ in range(n)]
    peps = [f"PEP{i % 17}" for i in range(n)]
    pre, enc = hb.PreprocessConfig(), hb.EncoderConfig(dim, dim // 2, 16, 1)
    image = best_oracle.cache_write(PreCfg(), EncCfg(dim, dim // 2, 16, 1), words, mz, charge, decoy, ids, peps)
    qw = words[rng.integers(0, n, nq)]
    qmz = mz[rng.integers(0, n, nq)] + rng.choice([0.0, 0.002, 15.99], nq)
    qch = rng.integers(1, 4, nq).astype(np.uint8)
    with hb.Context(0) as a, hb.Context(0) as b:
        a.build_index(dim, words, mz, charge, ids=ids, is_decoy=decoy)
        meta = b.load_cache(image, pre, enc)
        assert meta["ids"] == ids and meta["peptides"] == peps
        for x, y in zip(a.buckets(), b.buckets()):
            assert x["charge"] == y["charge"] and np.array_equal(x["ordinal"], y["ordinal"])
            assert np.array_equal(x["words"], y["words"]) and np.array_equal(x["precursor_mz"], y["precursor_mz"])
        for tol in (hb.Tolerance("dalton", 500.0), hb.Tolerance("ppm", 20.0)):
            m1, m2 = a.search_batch(qw, qmz, qch, tol), b.search_batch(qw, qmz, qch, tol)
            assert np.array_equal(m1.ordinal, m2.ordinal) and np.array_equal(m1.raw_score, m2.raw_score)
        c1 = a.cascade_search(qw, qmz, qch, hb.Tolerance("ppm", 20.0), hb.Tolerance("dalton", 500.0), 0.05)
        c2 = b.cascade_search(qw, qmz, qch, hb.Tolerance("ppm", 20.0), hb.Tolerance("dalton", 500.0), 0.05)
        for k in c1:
            assert np.array_equal(c1[k], c2[k]), k
        # the two corruptions only the checksum can see are caught on the device
        for mutate, cls in CORRUPTIONS[9:]:
            with pytest.raises(hb.CacheCorruptError):
                b.load_cache(mutate(image), pre, enc)
        with pytest.raises(hb.StaleCacheError):
            b.load_cache(image, pre, hb.EncoderConfig(dim, dim // 2, 16, 2))
        # sharded load: the slices partition the library
        got = 0
        for g in range(3):
            b.load_cache(image, pre, enc, shard_index=g, shard_count=3)
            got += sum(x["shard_end"] - x["shard_begin"] for x in b.buckets())
        assert got == n


@pytest.mark.gpu
def test_cache_write_is_byte_identical(hb, ctx, best_oracle):
    import torch
    image, ent, p, e = _golden()
    pre, enc = _ppre(hb, p), hb.EncoderConfig(*[int(x) for x in e])
    args = (ent["mz"], ent["charge"], ent["decoy"], ent["ids"], ent["peptides"])
    assert ctx.cache_write(pre, enc, ent["words"], *args) == image
    d = torch.from_numpy(ent["words"].view(np.int64)).cuda()
    assert ctx.cache_write(pre, enc, None, *args, d_words=d.data_ptr()) == image
    # a larger file: encode on the device -> write from device rows -> the reference's writer agrees
    rng = np.random.default_rng(5)
    n, dim = 20_000, 2048
    words = U.random_hvs(rng, n, dim)
    mz = rng.uniform(300, 1300, n)
    ch = rng.integers(2, 4, n).astype(np.uint8)
    dec = np.zeros(n, np.uint8)
    ids = [f"L{i}" for i in range(n)]
    peps = [""] * n
    d = torch.from_numpy(words.view(np.int64)).cuda()
    mine = ctx.cache_write(hb.PreprocessConfig(), hb.EncoderConfig(dim, 1024, 16, 1), None, mz, ch, dec, ids, peps,
                           d_words=d.data_ptr())
    want = best_oracle.cache_write(PreCfg(), EncCfg(dim, 1024, 16, 1), words, mz, ch, dec, ids, peps)
    assert mine == want
    ctx.load_cache(mine, hb.PreprocessConfig(), hb.EncoderConfig(dim, 1024, 16, 1))
