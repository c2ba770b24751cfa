"""Helpers shared by the test modules (golden loading, config conversion, random inputs)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fingerprints():
    with open(os.path.join(GOLDEN, "fingerprints.json")) as f:
        return json.load(f)


def _nested(npz):
    out = {}
    for key in npz.files:
        parts = key.split("/")
        d = out
        for p in parts[:-1]:
            d = d.setdefault(p, {})
        d[parts[-1]] = npz[key]
    return out


def encode_cases():
    return _nested(np.load(os.path.join(GOLDEN, "encode_cases.npz")))


def search_cases():
    return _nested(np.load(os.path.join(GOLDEN, "search_cases.npz")))


def oracle_precfg(v):
    from oracle.binding import PreCfg
    return PreCfg(float(v[0]), float(v[1]), float(v[2]), int(v[3]), int(v[4]), float(v[5]), int(v[6]))


def product_precfg(v):
    import paper_2211_16422_b200 as hb
    return hb.PreprocessConfig(float(v[0]), float(v[1]), float(v[2]), int(v[3]), int(v[4]),
                               float(v[5]), int(v[6]))


def csr(spectra):
    offsets = np.zeros(len(spectra) + 1, np.uint64)
    if spectra:
        offsets[1:] = np.cumsum([len(s[0]) for s in spectra])
    mz = np.concatenate([np.asarray(s[0], np.float64) for s in spectra] + [np.zeros(0)])
    it = np.concatenate([np.asarray(s[1], np.float64) for s in spectra] + [np.zeros(0)])
    return offsets, mz, it


def random_hvs(rng, n, dim):
    W = (dim + 63) // 64
    w = rng.integers(0, 2**64, (n, W), dtype=np.uint64)
    if dim % 64:
        w[:, -1] &= np.uint64((1 << (dim % 64)) - 1)
    return w


TOLS = {"ppm150": ("ppm", 150.0), "da30": ("da", 30.0), "da500": ("da", 500.0), "da1": ("da", 1.0),
        "ppm20": ("ppm", 20.0)}


def product_tol(t):
    import paper_2211_16422_b200 as hb
    return hb.Tolerance("ppm" if t[0] == "ppm" else "dalton", t[1])


def mgf_cases():
    """[(text bytes, expected dict | error string)] generated from the reference (make_golden.py)."""
    with open(os.path.join(GOLDEN, "mgf_cases.json")) as f:
        raw = json.load(f)
    out = []
    for c in raw:
        text = bytes.fromhex(c["text"])
        if not c["ok"]:
            out.append((text, c["error"]))
            continue
        out.append((text, dict(offsets=np.array(c["offsets"], np.uint64),
                               mz=np.array(c["mz"], np.uint64).view(np.float64),
                               intensity=np.array(c["intensity"], np.uint64).view(np.float64),
                               precursor_mz=np.array(c["precursor_mz"], np.uint64).view(np.float64),
                               charge=np.array(c["charge"], np.uint8), is_decoy=np.array(c["is_decoy"], np.uint8),
                               ids=[bytes.fromhex(x) for x in c["ids"]],
                               peptides=[bytes.fromhex(x) for x in c["peptides"]])))
    return out


def fnv_hex(a) -> str:
    """FNV-1a-64 (cache.cpp:18-29) of an array's bytes, zero-padded to whole u64 words -- the fingerprint
    function of tests/golden/make_whole_config.py."""
    from oracle.binding import fnv1a64_words
    b = np.ascontiguousarray(a).view(np.uint8).ravel()
    if len(b) % 8:
        b = np.concatenate([b, np.zeros(8 - len(b) % 8, np.uint8)])
    return "%016x" % fnv1a64_words(b.view("<u8"))
