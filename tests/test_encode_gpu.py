"""GPU: preprocessing (K1) and encoding (K2) kernels against the oracle and the golden fixtures,
bit for bit, through the C ABI."""
import numpy as np
import pytest

from oracle.binding import PreCfg, SynthCfg, fnv1a64_words
from tests import _util as U

pytestmark = pytest.mark.gpu


def _upload(hb, ctx, dim, flips, levels, seed, n_bins):
    cb = hb.make_codebook(n_bins, hb.EncoderConfig(dim, flips, levels, seed))
    ctx.upload_codebook(cb)
    return cb


def test_golden_encode_cases(hb, ctx):
    for name, c in U.encode_cases().items():
        pre = U.product_precfg(c["precfg"])
        dim, flips, levels, seed = (int(x) for x in c["enccfg"])
        _upload(hb, ctx, dim, flips, levels, seed, hb.dimension(pre))
        words, ok = ctx.encode_batch(c["offsets"], c["mz"], c["intensity"], pre)
        assert np.array_equal(ok, c["ok"]), name
        assert np.array_equal(words, c["words"]), name
        bins, lev, cnt = ctx.preprocess_batch(c["offsets"], c["mz"], c["intensity"], pre, levels)
        for i in range(len(ok)):
            s, e = int(c["sv_offsets"][i]), int(c["sv_offsets"][i + 1])
            assert cnt[i] == e - s, (name, i)
            assert np.array_equal(bins[i, : cnt[i]], c["sv_bins"][s:e]), (name, i)
            assert np.array_equal(lev[i, : cnt[i]], c["sv_levels"][s:e]), (name, i)
        out = ctx.encode_spectra(c["offsets"], c["mz"], c["intensity"], pre, threads=4, batch_size=3)
        assert out.unprocessable == int((c["ok"] == 0).sum())
        assert np.array_equal(out.words, c["words"][c["ok"] == 1])


def test_reference_known_answers(hb, ctx):
    """test_encoder.cpp:85-130 (single peak XNOR, hand-built dim-8 codebook) and
    test_preprocess.cpp:82-215 through the device path."""
    cb = _upload(hb, ctx, 256, 128, 16, 8, 20)
    got = ctx.encode([0, 1], [7], [1.0])[0]
    assert np.array_equal(got, ~(cb.position[7] ^ cb.level[16]))

    def bits(*b):
        return np.array([sum(int(x) << i for i, x in enumerate(b))], np.uint64)
    pos = np.stack([bits(1, 0, 1, 0, 1, 0, 1, 0), bits(1, 1, 0, 0, 1, 1, 0, 0), bits(0, 0, 0, 0, 1, 1, 1, 1)])
    lvl = np.stack([bits(0, 0, 0, 0, 0, 0, 0, 0), bits(1, 0, 0, 1, 0, 1, 1, 0), bits(1, 1, 1, 1, 1, 1, 1, 1)])
    ctx.upload_codebook(hb.Codebook(hb.EncoderConfig(8, 1, 2, 0), 3, pos, lvl))
    got = ctx.encode([0, 2], [0, 2], [1.0, 0.4])[0]
    x0 = ~(pos[0] ^ lvl[2]) & np.uint64(0xFF)
    x1 = ~(pos[2] ^ lvl[1]) & np.uint64(0xFF)
    assert got[0] == (x0 & x1)[0]

    small = hb.PreprocessConfig(101.0, 1500.0, 0.05, 50, 1, 0.01)
    off, mz, it = U.csr([([200.0, 300.0, 400.0], [1000.0, 9.0, 10.0]),
                         ([100.99, 101.0, 1499.99, 1500.0], [5.0] * 4),
                         ([200.0 + i for i in range(60)], [float(100 - (i % 20)) for i in range(60)])])
    bins, lev, cnt = ctx.preprocess_batch(off, mz, it, small, 16)
    assert list(bins[0, : cnt[0]]) == [1980, 5980]
    assert list(bins[1, : cnt[1]]) == [0, 27979]
    order = sorted(range(60), key=lambda i: (-float(100 - (i % 20)), 200.0 + i))[:50]
    assert list(bins[2, : cnt[2]]) == sorted(int(np.floor((200.0 + i - 101.0) / 0.05 + 1e-9)) for i in order)
    cfg = hb.PreprocessConfig(100.0, 1500.0, 0.05, 50, 1)
    off, mz, it = U.csr([([100.00, 100.049, 100.05], [1.0, 1.0, 1.0]), ([200.00, 200.01], [0.4, 0.6])])
    bins, lev, cnt = ctx.preprocess_batch(off, mz, it, cfg, 16)
    assert list(bins[0, : cnt[0]]) == [0, 1] and list(lev[0, : cnt[0]]) == [16, 8]
    assert cnt[1] == 1 and lev[1, 0] == 16
    cfg = hb.PreprocessConfig(100.0, 1500.0, 0.05, 50, 1, 0.01, 1)
    off, mz, it = U.csr([([200.0, 300.0], [0.25, 1.0])])
    bins, lev, cnt = ctx.preprocess_batch(off, mz, it, cfg, 16)
    assert list(lev[0, :2]) == [8, 16]


def test_encode_errors(hb, ctx):
    with pytest.raises(hb.HomsError):
        ctx.encode_batch([0, 1], [200.0], [1.0], hb.PreprocessConfig())  # no codebook yet
    _upload(hb, ctx, 128, 16, 16, 12, 40)
    with pytest.raises(hb.InvariantError):  # encoder.cpp:20-22 dims mismatch (27980 != 40)
        ctx.encode_batch([0, 1], [200.0], [1.0], hb.PreprocessConfig())
    with pytest.raises(hb.InvariantError):  # encoder.cpp:23-25 empty vector
        ctx.encode([0, 0], [], [])
    with pytest.raises(hb.InvariantError):  # encoder.cpp:12-14
        ctx.encode([0, 1], [3], [1.5])
    with pytest.raises(hb.InvariantError):
        ctx.encode([0, 1], [40], [0.5])
    words, ok = ctx.encode_batch([0], [], [], hb.PreprocessConfig(100.0, 140.0, 1.0))
    assert words.shape[0] == 0


def test_non_finite_peaks(hb, ctx, best_oracle):
    """NaN m/z or intensity never passes the range / positivity filter (preprocess.cpp:45-49) and is
    dropped silently; an INFINITE kept intensity normalises to inf / inf = NaN, on which
    quantize_intensity throws out of the reference's encode_spectra (encoder.cpp:12-14,
    pipeline.cpp:67-72) -- the product reports the same InvariantError."""
    from oracle.binding import OracleError
    pre, opre = hb.PreprocessConfig(), PreCfg()
    dim = 1024
    cb = _upload(hb, ctx, dim, dim // 2, 16, 1, hb.dimension(pre))
    ocb = best_oracle.codebook_from_words(dim, 16, cb.position, cb.level)
    rng = np.random.default_rng(3)
    base_mz = np.sort(rng.choice(np.arange(20000, 120000), 16, replace=False)) * 0.01
    base_it = rng.uniform(0.1, 1.0, 16)
    with_nan = (base_mz.copy(), base_it.copy())
    with_nan[0][3] = np.nan
    with_nan[1][7] = np.nan
    off, mz, it = U.csr([(base_mz, base_it), with_nan, (base_mz[:11], base_it[:11])])
    words, ok = ctx.encode_batch(off, mz, it, pre)
    ow, ook = best_oracle.encode_spectra(ocb, opre, off, mz, it)
    assert ok.all() and np.array_equal(ok, ook) and np.array_equal(words, ow)

    # min_peaks (10) infinite peaks survive their own floor; each normalises to inf / inf
    with_inf = (base_mz.copy(), base_it.copy())
    with_inf[1][2:14] = np.inf
    off, mz, it = U.csr([(base_mz, base_it), with_inf])
    with pytest.raises(OracleError, match="outside"):
        best_oracle.encode_spectra(ocb, opre, off, mz, it)
    with pytest.raises(hb.InvariantError, match="quantize_intensity"):
        ctx.encode_batch(off, mz, it, pre)
    with pytest.raises(hb.InvariantError, match="quantize_intensity"):
        ctx.preprocess_batch(off, mz, it, pre, 16)
    with pytest.raises(hb.InvariantError, match="quantize_intensity"):
        ctx.build_index_from_spectra(off, mz, it, pre, np.array([500.0, 600.0]), np.array([2, 2], np.uint8))
    # a single infinite peak is the base peak: every finite peak falls below 1 % of it and is
    # dropped, the infinite one is kept alone -> below min_peaks, unprocessable, no error
    lone = base_it.copy()
    lone[4] = np.inf
    words, ok = ctx.encode_batch(*U.csr([(base_mz, lone)]), pre)
    ow, ook = best_oracle.encode_spectra(ocb, opre, *U.csr([(base_mz, lone)]))
    assert np.array_equal(ok, ook) and not ok.any()
    best_oracle.free_codebook(ocb)


def test_encode_fuzz_vs_oracle(hb, ctx, best_oracle):
    """Randomised differential test of refine_peaks -> vectorize -> quantize -> encode against the
    compiled reference: random preprocess configs (bin size, range, floor, max / min peaks, sqrt
    scaling), level counts and dimensions; spectra with out-of-range and non-positive peaks, m/z
    values on bin boundaries, tied intensities (top-N rule), bin collisions and too few peaks."""
    rng = np.random.default_rng(8192)
    seen_ok = seen_bad = 0
    for case in range(12):
        bin_size = float(rng.choice([0.05, 0.1, 1.0005, 0.01]))
        lo = float(rng.choice([101.0, 50.0, 200.5]))
        hi = lo + float(rng.choice([300.0, 1399.0]))
        max_peaks = int(rng.choice([8, 50, 150, 300]))
        min_peaks = int(rng.choice([1, 5, 10]))
        floor = float(rng.choice([0.0, 0.01, 0.2]))
        scaling = int(case % 2)
        levels = int(rng.choice([1, 16, 31]))
        dim = int(rng.choice([64, 1000, 2048, 4096]))
        pre = hb.PreprocessConfig(lo, hi, bin_size, max_peaks, min_peaks, floor, scaling)
        opre = PreCfg(lo, hi, bin_size, max_peaks, min_peaks, floor, scaling)
        cb = _upload(hb, ctx, dim, dim // 2, levels, case + 1, hb.dimension(pre))
        ocb = best_oracle.codebook_from_words(dim, levels, cb.position, cb.level)
        spectra = []
        for _ in range(150):
            p = int(rng.choice([0, 1, 3, 9, 10, 11, 40, 200, 700]))
            grid = rng.choice([bin_size, bin_size / 2, 0.013])
            m = np.sort(np.unique(np.round(rng.uniform(lo - 20.0, hi + 20.0, p) / grid) * grid))
            v = np.round(rng.uniform(-0.1, 1.0, len(m)), int(rng.choice([1, 2, 6])))
            spectra.append((m, v))
        off, mz, it = U.csr(spectra)
        words, ok = ctx.encode_batch(off, mz, it, pre)
        ow, ook = best_oracle.encode_spectra(ocb, opre, off, mz, it)
        best_oracle.free_codebook(ocb)
        seen_ok += int(ok.sum())
        seen_bad += int(len(ok) - ok.sum())
        assert np.array_equal(ok, ook), (case, pre)
        assert np.array_equal(words, ow), (case, pre)
    assert seen_ok > 500 and seen_bad > 500  # both outcomes are exercised


def test_level_rows_beyond_shared_memory(hb, ctx, best_oracle):
    """32 level rows of 4 KiB (D = 32768, Q = 30) exceed the 96 KB the encode kernel stages in shared
    memory: the level slabs (and the no-vote row) then come from global memory through L1."""
    rng = np.random.default_rng(12)
    dim, levels = 32768, 30
    pre, opre = hb.PreprocessConfig(max_peaks=40, min_peaks=3), PreCfg(max_peaks=40, min_peaks=3)
    cb = _upload(hb, ctx, dim, dim // 2, levels, 3, hb.dimension(pre))
    ocb = best_oracle.codebook_from_words(dim, levels, cb.position, cb.level)
    spectra = []
    for p in (0, 2, 3, 17, 33, 40, 41, 90):
        idx = np.sort(rng.choice(np.arange(11000, 140000), p, replace=False))
        spectra.append((idx * 0.01, np.round(rng.uniform(0.0, 1.0, p), 3)))
    off, mz, it = U.csr(spectra)
    words, ok = ctx.encode_batch(off, mz, it, pre)
    ow, ook = best_oracle.encode_spectra(ocb, opre, off, mz, it)
    best_oracle.free_codebook(ocb)
    assert np.array_equal(ok, ook) and ok.sum() >= 5
    assert np.array_equal(words, ow)


def test_encode_vectors_random_vs_oracle(hb, ctx, best_oracle):  # test_encoder.cpp:132-139, wider
    rng = np.random.default_rng(21)
    for dim, n_bins, levels, max_n in ((128, 40, 16, 12), (64, 9, 2, 9), (1088, 300, 31, 300),
                                       (4096, 500, 16, 200), (16384, 64, 16, 50)):
        cb = _upload(hb, ctx, dim, max(1, dim // 2), levels, 3, n_bins)
        ocb = best_oracle.codebook_from_words(dim, levels, cb.position, cb.level)
        offs, bins, vals = [0], [], []
        for _ in range(40):
            n = int(rng.integers(1, max_n + 1))
            b = np.sort(rng.choice(n_bins, min(n, n_bins), replace=False)).astype(np.uint32)
            v = rng.uniform(0, 1, len(b))
            v[rng.integers(0, len(b))] = 1.0
            bins.append(b)
            vals.append(v)
            offs.append(offs[-1] + len(b))
        got = ctx.encode(offs, np.concatenate(bins), np.concatenate(vals))
        for i in range(40):
            want = best_oracle.encode_vector(ocb, bins[i], vals[i])
            assert np.array_equal(got[i], want), (dim, i)
        best_oracle.free_codebook(ocb)


def test_config1_encode_fingerprints(hb, ctx, best_oracle):
    """config-1 library and query hypervector fingerprints."""
    fp = U.fingerprints()["config1"]
    s = best_oracle.synth(SynthCfg(n_library=5000, n_query=1000, fraction_modified=0.6, seed=1))
    L, Q = s["library"], s["queries"]
    pre = hb.PreprocessConfig()
    _upload(hb, ctx, 2048, 1024, 16, 1, hb.dimension(pre))
    lw, lok = ctx.encode_batch(L["offsets"], L["mz"], L["intensity"], pre)
    qw, qok = ctx.encode_batch(Q["offsets"], Q["mz"], Q["intensity"], pre)
    assert int(lok.sum()) == fp["library_encoded"] and int(qok.sum()) == 1000
    assert f"{fnv1a64_words(lw):016x}" == fp["library_hv_fnv"]
    assert f"{fnv1a64_words(qw):016x}" == fp["query_hv_fnv"]


def test_encode_ragged_and_large_spectra(hb, ctx, best_oracle):
    """Ragged inputs: empty spectra, thousands of raw peaks (top-N path), max_peaks > 255
    (16 counter planes), dimension sweep."""
    rng = np.random.default_rng(5)
    for dim, max_peaks in ((1024, 50), (2048, 150), (8192, 50), (16384, 400), (192, 20), (512, 3000)):
        pre = hb.PreprocessConfig(max_peaks=max_peaks, min_peaks=5)
        opre = PreCfg(max_peaks=max_peaks, min_peaks=5)
        cb = _upload(hb, ctx, dim, dim // 2, 16, 1, hb.dimension(pre))
        ocb = best_oracle.codebook_from_words(dim, 16, cb.position, cb.level)
        spectra = [(np.zeros(0), np.zeros(0))]
        for p in (1, 4, 5, 49, 50, 51, 333, 2500, 4000):
            idx = np.sort(rng.choice(np.arange(9000, 160000), p, replace=False))
            inten = np.round(rng.uniform(0, 1, p), 2)  # heavy ties
            spectra.append((idx * 0.01, inten))
        spectra.append((np.zeros(0), np.zeros(0)))
        off, mz, it = U.csr(spectra)
        words, ok = ctx.encode_batch(off, mz, it, pre)
        ow, ook = best_oracle.encode_spectra(ocb, opre, off, mz, it)
        assert np.array_equal(ok, ook), dim
        assert np.array_equal(words, ow), dim
        best_oracle.free_codebook(ocb)


def test_hamming_similarity(hb, ctx):  # test_encoder.cpp:50-79
    rng = np.random.default_rng(4)
    for dim in (8192, 16384, 65, 100, 184, 64):
        a = U.random_hvs(rng, 50, dim)
        b = U.random_hvs(rng, 50, dim)
        got = ctx.hamming_similarity(dim, a, b)
        want = dim - np.array([bin(int(x)).count("1") for x in (a ^ b).ravel()]).reshape(50, -1).sum(1)
        assert np.array_equal(got, want)
    x = U.random_hvs(rng, 1, 8192)
    mask = ~x
    assert ctx.hamming_similarity(8192, x, x)[0] == 8192
    assert ctx.hamming_similarity(8192, x, mask)[0] == 0
