"""Synthetic workloads of the BASELINE.json shapes (numpy, deterministic, no dataset needed).

Shapes follow the reference's benchmark generator (src/synth.cpp:114-197: fragment m/z on a
0.01 Th grid in [150, 1300), intensities U[0.05, 1], precursors U[380, 1070], charge in {2, 3},
one decoy per target with the target's precursor/charge/intensities on fresh positions, queries
derived from targets with a planted +79.97 Da shift and 5 % intensity noise).

Two generators feed bench.py and the tests (`make(name, generator)`):

* "reference": the reference's OWN generator, `generate_benchmark(SynthConfig{...})`
  (src/synth.cpp:114-197) as compiled into oracle/_ref -- SURVEY.md section 8(d)'s exact inputs
  (configs 1-3 = seeds 1-3).  A data source, not a checker: nothing of the search/encode path runs
  in it.  Needs the built oracle/_ref (it travels to the GPU box as a built .so).
* "numpy": an independent vectorised generator of the same distribution (NOT the reference's
  streams); the fallback when oracle/_ref is absent, and the source of the encode / MGF workloads.

This module lives outside the product package on purpose: the reference arm of bench.py imports
it without mapping libhoms_b200.so.
"""
from __future__ import annotations

import numpy as np

GRID = 0.01
MZ_LO, MZ_HI = 150.0, 1300.0


def _distinct_grid_rows(rng: np.random.Generator, n: int, peaks: int) -> np.ndarray:
    """n rows of `peaks` distinct sorted grid indices in [lo, hi]."""
    lo, hi = int(round(MZ_LO / GRID)), int(round(MZ_HI / GRID)) - 1
    out = np.empty((n, peaks), np.int32)
    step = 200_000
    for a in range(0, n, step):
        b = min(n, a + step)
        rows = np.sort(rng.integers(lo, hi + 1, (b - a, peaks), dtype=np.int32), axis=1)
        while True:
            dup = (np.diff(rows, axis=1) == 0).any(axis=1)
            if not dup.any():
                break
            rows[dup] = np.sort(rng.integers(lo, hi + 1, (int(dup.sum()), peaks), dtype=np.int32), axis=1)
        out[a:b] = rows
    return out


def synth_library(n_targets: int, peaks: int = 50, decoy_ratio: float = 1.0, seed: int = 2) -> dict:
    rng = np.random.default_rng(seed)
    n_decoys = int(round(decoy_ratio * n_targets))
    n = n_targets + n_decoys
    idx = _distinct_grid_rows(rng, n, peaks)
    mz = idx.astype(np.float64) * GRID
    inten = np.empty((n, peaks), np.float64)
    inten[:n_targets] = 0.05 + 0.95 * rng.random((n_targets, peaks))
    src = np.arange(n_decoys) % n_targets
    inten[n_targets:] = inten[src]
    span = MZ_HI - MZ_LO
    prec = np.empty(n, np.float64)
    prec[:n_targets] = (MZ_LO + 0.2 * span) + (0.6 * span) * rng.random(n_targets)
    prec[n_targets:] = prec[src]
    charge = np.empty(n, np.uint8)
    charge[:n_targets] = rng.integers(2, 4, n_targets)
    charge[n_targets:] = charge[src]
    decoy = np.zeros(n, np.uint8)
    decoy[n_targets:] = 1
    ids = [f"LIB_{i + 1:06d}" for i in range(n_targets)] + [f"DECOY_{j + 1:06d}" for j in range(n_decoys)]
    offsets = np.arange(n + 1, dtype=np.uint64) * np.uint64(peaks)
    return dict(offsets=offsets, mz=mz.ravel(), intensity=inten.ravel(), precursor_mz=prec,
                charge=charge, is_decoy=decoy, ids=ids, n_targets=n_targets, peaks=peaks)


def synth_queries(lib: dict, n_query: int, fraction_modified: float = 0.6, shift: float = 79.97,
                  fraction_peaks_shifted: float = 0.3, noise: float = 0.05, seed: int = 2) -> dict:
    rng = np.random.default_rng(seed + 0x9E3779B9)
    peaks = lib["peaks"]
    src = rng.integers(0, lib["n_targets"], n_query)
    mz = lib["mz"].reshape(-1, peaks)[src].copy()
    inten = lib["intensity"].reshape(-1, peaks)[src].copy()
    charge = lib["charge"][src].copy()
    prec = lib["precursor_mz"][src].copy()
    modified = rng.random(n_query) < fraction_modified
    prec[modified] += shift / charge[modified]
    shifted = (rng.random((n_query, peaks)) < fraction_peaks_shifted) & modified[:, None]
    mz[shifted] += shift
    inten *= 1.0 + noise * (2.0 * rng.random((n_query, peaks)) - 1.0)
    order = np.argsort(mz, axis=1, kind="stable")
    mz = np.take_along_axis(mz, order, 1)
    inten = np.take_along_axis(inten, order, 1)
    # RawSpectrum invariant: strictly ascending m/z; merge the (rare) exact collisions
    counts = np.full(n_query, peaks, np.int64)
    dup_rows = np.flatnonzero((np.diff(mz, axis=1) == 0).any(axis=1))
    flat_mz, flat_in = [mz[i] for i in range(0)], []
    if len(dup_rows):
        keep = np.ones((n_query, peaks), bool)
        for r in dup_rows:
            m, v = mz[r], inten[r]
            j = 0
            for t in range(1, peaks):
                if m[t] == m[j]:
                    v[j] += v[t]
                    keep[r, t] = False
                else:
                    j = t
        counts = keep.sum(axis=1)
        flat_mz, flat_in = mz[keep], inten[keep]
    else:
        flat_mz, flat_in = mz.ravel(), inten.ravel()
    offsets = np.zeros(n_query + 1, np.uint64)
    offsets[1:] = np.cumsum(counts)
    return dict(offsets=offsets, mz=np.ascontiguousarray(flat_mz), intensity=np.ascontiguousarray(flat_in),
                precursor_mz=prec, charge=charge, source=src, modified=modified)


WORKLOADS = {
    # name: (n_targets, n_query, dim, peaks, seed)  -- BASELINE.json configs
    "config1": (5_000, 1_000, 2048, 50, 1),       # reference CPU test workload
    "iprg2012": (600_000, 16_000, 8192, 50, 2),   # 16k queries x 1.2M library, D = 8192
    "hek293": (2_150_000, 65_536, 8192, 50, 3),   # 4.3M library; query prefix of the 1M set
    "hek293_full": (2_150_000, 1_000_000, 8192, 50, 3),  # BASELINE config 3 at full size (seconds per step)
    "tiny": (2_000, 256, 2048, 50, 9),            # CI-sized
}


def reference_generator_available() -> bool:
    from oracle import binding as ob
    return ob.available("ref")


def make(name: str, generator: str = "auto"):
    """-> (library dict, query dict, dim, generator used).  Dicts carry CSR spectra (offsets, mz,
    intensity), precursor_mz, charge, is_decoy, ids; queries also `source` and `modified`."""
    n_targets, n_query, dim, peaks, seed = WORKLOADS[name]
    if generator == "auto":
        generator = "reference" if reference_generator_available() else "numpy"
    if generator == "reference":
        from oracle import binding as ob
        o = ob.Oracle("ref")
        s = o.synth(ob.SynthCfg(n_library=n_targets, n_query=n_query, peaks_per_spectrum=peaks,
                                fraction_modified=0.6, precursor_shift_da=79.97, fraction_peaks_shifted=0.3,
                                intensity_noise=0.05, decoy_ratio=1.0, seed=seed))
        lib, qry = s["library"], s["queries"]
        lib["n_targets"], lib["peaks"] = n_targets, peaks
        qry["source"] = s["truth"]["source_index"].astype(np.int64)
        qry["modified"] = s["truth"]["modified"].astype(bool)
        return lib, qry, dim, "reference"
    if generator != "numpy":
        raise ValueError(f"unknown generator {generator!r}")
    lib = synth_library(n_targets, peaks, 1.0, seed)
    qry = synth_queries(lib, n_query, seed=seed)
    return lib, qry, dim, "numpy"


# ---- BASELINE config 4: counter-based spectra -------------------------------------
# "10 M spectra x 150 distinct-grid peaks ... generated on device with a counter-based splitmix64 stream
# keyed by (seed = 4, spectrum, peak) so the CPU oracle can regenerate any sample."  Peak p of spectrum s
# is a pure function of (seed, s, p): bench.py generates the whole set ON THE GPU with the torch form
# (integer ops only, then exact int -> double conversions) and replays any sample on the host with the
# numpy form -- the two are bit-identical, which tests/test_host_logic.py checks.
#   stream(tag)[i] = finalise(base(tag) + (i + 1) * GOLDEN), base(tag) = finalise'(seed ^ finalise'(tag))
#   m/z:       the 0.01 Th grid of synth.cpp:25 on [150, 1300) cut into `peaks` equal strata; peak p sits at
#              cell 15000 + p * width + (top 32 bits of stream("mz")[s * peaks + p]) % width  (distinct, ascending)
#   intensity: 0.05 + 0.95 * (stream("in")[s * peaks + p] >> 11) * 2^-53   (U[0.05, 1), synth.cpp:69)
_GOLDEN = 0x9E3779B97F4A7C15
_C1, _C2 = 0xBF58476D1CE4E5B9, 0x94D049BB133111EB
_M64 = (1 << 64) - 1
_GRID_LO, _GRID_CELLS = 15000, 115000


def _mix_int(x: int) -> int:
    x = (x + _GOLDEN) & _M64
    x = ((x ^ (x >> 30)) * _C1) & _M64
    x = ((x ^ (x >> 27)) * _C2) & _M64
    return x ^ (x >> 31)


def _stream_base(seed: int, tag: int) -> int:
    return _mix_int(seed ^ _mix_int(tag))


def _signed(x: int) -> int:
    return x - (1 << 64) if x >= (1 << 63) else x


def config4_numpy(first: int, n: int, peaks: int = 150, seed: int = 4):
    """Spectra [first, first + n) of the config-4 set as host CSR arrays (offsets u64, mz f64, intensity f64)."""
    with np.errstate(over="ignore"):
        idx = np.arange(first * peaks, (first + n) * peaks, dtype=np.uint64) + np.uint64(1)

        def stream(tag):
            x = np.uint64(_stream_base(seed, tag)) + idx * np.uint64(_GOLDEN)
            x = (x ^ (x >> np.uint64(30))) * np.uint64(_C1)
            x = (x ^ (x >> np.uint64(27))) * np.uint64(_C2)
            return x ^ (x >> np.uint64(31))

        width = _GRID_CELLS // peaks
        p = (np.arange(n * peaks, dtype=np.uint64) % np.uint64(peaks))
        cell = np.uint64(_GRID_LO) + p * np.uint64(width) + (stream(0x6D7A) >> np.uint64(32)) % np.uint64(width)
        mz = cell.astype(np.float64) * 0.01
        u = (stream(0x696E) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        inten = 0.95 * u
        inten = inten + 0.05
    offsets = np.arange(n + 1, dtype=np.uint64) * np.uint64(peaks)
    return offsets, mz, inten


def config4_torch(first: int, n: int, device, peaks: int = 150, seed: int = 4):
    """The same spectra generated on `device` with torch integer ops (int64 wraps like uint64; logical
    shifts are arithmetic shifts with the sign extension masked off)."""
    import torch

    def lsr(x, s):
        return (x >> s) & ((1 << (64 - s)) - 1)

    idx = torch.arange(first * peaks, (first + n) * peaks, dtype=torch.int64, device=device) + 1

    def stream(tag):
        x = idx * _signed(_GOLDEN) + _signed(_stream_base(seed, tag))
        x = (x ^ lsr(x, 30)) * _signed(_C1)
        x = (x ^ lsr(x, 27)) * _signed(_C2)
        return x ^ lsr(x, 31)

    width = _GRID_CELLS // peaks
    p = torch.arange(n * peaks, dtype=torch.int64, device=device) % peaks
    cell = _GRID_LO + p * width + lsr(stream(0x6D7A), 32) % width
    mz = cell.to(torch.float64) * 0.01
    u = lsr(stream(0x696E), 11).to(torch.float64) * (2.0 ** -53)
    inten = 0.95 * u
    inten = inten + 0.05
    offsets = torch.arange(n + 1, dtype=torch.int64, device=device) * peaks
    return offsets, mz, inten
