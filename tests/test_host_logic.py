"""CPU: the C-ABI library loads and exports every declared symbol; host-only entry points
(configuration, codebook generation, FDR, id ranks) against the oracle and the golden fixtures."""
import ctypes

import numpy as np
import pytest

from oracle.binding import PreCfg, fnv1a64_words
from tests import _util as U


def test_library_exports_every_declared_symbol(hb):
    from paper_2211_16422_b200 import capi
    names = capi.declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(capi.lib, n)]
    assert not missing, missing
    assert capi.abi_version() == 2
    assert ctypes.sizeof(capi.PreprocessConfigPod) == 48
    assert ctypes.sizeof(capi.EncoderConfigPod) == 24
    assert ctypes.sizeof(capi.TolerancePod) == 16


def test_no_cpu_fallback(hb):
    """Without a CUDA device the product refuses to run instead of computing on the host."""
    try:
        c = hb.Context(0)
    except hb.CudaError as e:
        assert "no CPU fallback" in str(e) or "CUDA" in str(e)
        return
    c.close()
    pytest.skip("a CUDA device is present")


def test_product_never_imports_oracle():
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for sub in ("paper_2211_16422_b200", "include"):
        for dp, _, files in os.walk(os.path.join(root, sub)):
            for f in files:
                if f.endswith((".py", ".cu", ".cuh", ".h", ".hpp", ".cpp")):
                    text = open(os.path.join(dp, f)).read()
                    assert "oracle" not in text.replace("oracles.hpp", ""), os.path.join(dp, f)


def test_preprocess_validate(hb):  # preprocess.cpp:21-34, test_preprocess.cpp:60-80
    hb.PreprocessConfig().validate()
    for kw in (dict(min_mz=500.0, max_mz=500.0), dict(bin_size=0.0), dict(min_peaks=0),
               dict(max_peaks=5, min_peaks=6), dict(intensity_floor=1.0), dict(intensity_floor=-0.1)):
        with pytest.raises(hb.ConfigError):
            hb.PreprocessConfig(**kw).validate()


def test_dimension(hb):  # test_preprocess.cpp:40-58
    assert hb.dimension(hb.PreprocessConfig(0.0, 2000.0, 0.04)) == 50000
    assert hb.dimension(hb.PreprocessConfig()) == 27980
    assert hb.dimension(hb.PreprocessConfig(0.0, 10.0, 10.0)) == 1


def test_encoder_validate(hb):  # test_codebook.cpp:36-44
    hb.EncoderConfig().validate()
    for args in ((0, 1, 2), (100, 1, 2), (64, 0, 2), (64, 1, 1)):
        with pytest.raises(hb.ConfigError):
            hb.EncoderConfig(*args).validate()


def test_quantize_table(hb, port):  # test_encoder.cpp:44-48
    for v, q, want in ((1.0, 16, 16), (0.0, 16, 0), (0.26, 16, 4), (0.5, 2, 1), (0.97, 16, 16)):
        assert hb.quantize_intensity(v, q) == want
    for bad in (-0.1, 1.1, float("nan")):
        with pytest.raises(hb.InvariantError):
            hb.quantize_intensity(bad, 16)
    rng = np.random.default_rng(0)
    for v in rng.uniform(0, 1, 500):
        assert hb.quantize_intensity(v, 16) == port.quantize_intensity(v, 16)


def test_make_codebook_fingerprints(hb):
    fp = U.fingerprints()["codebook"]
    for dim in (1024, 2048, 8192):
        cb = hb.make_codebook(27980, hb.EncoderConfig(dim, dim // 2, 16, 1))
        assert f"{fnv1a64_words(cb.position):016x}" == fp[str(dim)]["position"]
        assert f"{fnv1a64_words(cb.level):016x}" == fp[str(dim)]["level"]


def test_make_codebook_equals_oracle_odd_shapes(hb, port):
    for dim, flips, levels, seed, n_bins in ((64, 1, 2, 0, 3), (192, 1, 5, 9, 17), (256, 0, 16, 5, 50),
                                             (8, 1, 2, 0, 3), (100, 7, 3, 2, 9), (1088, 500, 31, 4, 12)):
        cb = hb.make_codebook(n_bins, hb.EncoderConfig(dim, flips, levels, seed))
        ocb = port.make_codebook(dim, flips, levels, seed, n_bins)
        assert np.array_equal(cb.position, ocb.pos) and np.array_equal(cb.level, ocb.lvl)


def test_fdr_curve(hb, port):  # test_fdr.cpp:47-72 + random vs oracle
    order, fdr, q = hb.compute_fdr_curve([0.9, 0.8, 0.7, 0.6], [0, 0, 1, 0])
    assert list(order) == [0, 1, 2, 3]
    assert list(fdr) == [0.0, 0.0, 0.5, 1.0 / 3.0]
    assert list(q) == [0.0, 0.0, 1.0 / 3.0, 1.0 / 3.0]
    rng = np.random.default_rng(1)
    for n in (0, 1, 2, 17, 1000):
        score = np.round(rng.uniform(0, 1, n), 2)  # many ties
        decoy = (rng.uniform(0, 1, n) < 0.4).astype(np.uint8)
        a = hb.compute_fdr_curve(score, decoy)
        b = port.compute_fdr_curve(score, decoy)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_id_ranks(hb):
    ids = ["b", "a", "ab", "a", "", "B", "a\x7f", "DECOY_000010", "LIB_000002", "DECOY_000002"]
    rank = hb.id_ranks(ids)
    order = sorted(range(len(ids)), key=lambda i: (ids[i].encode(), i))
    want = np.empty(len(ids), np.uint32)
    want[order] = np.arange(len(ids))
    assert np.array_equal(rank, want)


def test_config4_counter_stream_replays_on_the_host():
    """the counter-based spectra bench.py generates with torch (on the device there,
    on the CPU here) are bit-identical to the numpy replay, distinct and ascending on the 0.01 Th grid,
    intensities in [0.05, 1); any window of the stream can be regenerated in isolation."""
    import torch
    import workload as wl
    o, mz, it = wl.config4_numpy(7_654_321, 4096, 150)
    o2, mz2, it2 = wl.config4_torch(7_654_321, 4096, "cpu", 150)
    assert np.array_equal(mz, mz2.numpy()) and np.array_equal(it, it2.numpy())
    assert np.array_equal(o.astype(np.int64), o2.numpy())
    rows = mz.reshape(-1, 150)
    assert (np.diff(rows, axis=1) > 0).all() and rows.min() >= 150.0 and rows.max() < 1300.0
    assert it.min() >= 0.05 and it.max() < 1.0
    # a window cut out of the middle is the same numbers
    _, mz3, it3 = wl.config4_numpy(7_654_321 + 1000, 10, 150)
    assert np.array_equal(mz3, mz[1000 * 150:1010 * 150]) and np.array_equal(it3, it[1000 * 150:1010 * 150])
    assert torch.equal(wl.config4_torch(5, 3, "cpu", 150)[1], torch.from_numpy(wl.config4_numpy(5, 3, 150)[1]))
