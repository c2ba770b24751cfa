"""CPU: pins the plain-C restatement (oracle/homs_oracle.c) and, when it travelled with the
repo, the compiled reference (oracle/_ref) against
  (a) known answers the reference's own tests hold (file:line cited per test),
  (b) the committed golden fixtures generated from the reference (tests/golden/make_golden.py),
  (c) each other.
"""
import numpy as np
import pytest

from oracle.binding import OracleError, PreCfg, SynthCfg, fnv1a64_words
from tests import _util as U


@pytest.fixture(params=["port", "ref"])
def oracle(request, port):
    if request.param == "port":
        return port
    return request.getfixturevalue("ref")


def test_dimension_known_answers(oracle):  # test_preprocess.cpp:40-58
    assert oracle.dimension(PreCfg(0.0, 2000.0, 0.04)) == 50000
    assert oracle.dimension(PreCfg(101.0, 1500.0, 0.05)) == 27980
    assert oracle.dimension(PreCfg(0.0, 10.0, 10.0)) == 1


def test_quantize_table(oracle):  # test_encoder.cpp:44-48
    assert oracle.quantize_intensity(1.0, 16) == 16
    assert oracle.quantize_intensity(0.0, 16) == 0
    assert oracle.quantize_intensity(0.26, 16) == 4
    assert oracle.quantize_intensity(0.5, 2) == 1
    assert oracle.quantize_intensity(0.97, 16) == 16
    for bad in (-0.1, 1.1):
        with pytest.raises(OracleError):
            oracle.quantize_intensity(bad, 16)


def small_scale(**kw):  # test_preprocess.cpp:25-34
    d = dict(min_mz=101.0, max_mz=1500.0, bin_size=0.05, max_peaks=50, min_peaks=1, intensity_floor=0.01)
    d.update(kw)
    return PreCfg(**d)


def test_noise_floor_strict(oracle):  # test_preprocess.cpp:82-90
    r = oracle.refine_vectorize(small_scale(), [200.0, 300.0, 400.0], [1000.0, 9.0, 10.0])
    assert list(r[0]) == [1980, 5980]  # 200.0 and 400.0 survive, exactly 1% is kept


def test_range_half_open(oracle):  # test_preprocess.cpp:92-101
    r = oracle.refine_vectorize(small_scale(), [100.99, 101.0, 1499.99, 1500.0], [5.0] * 4)
    assert list(r[0]) == [0, 27979]


def test_top_n_ties_toward_lower_mz(oracle):  # test_preprocess.cpp:113-136
    mz = [200.0 + i for i in range(60)]
    inten = [float(100 - (i % 20)) for i in range(60)]
    r = oracle.refine_vectorize(small_scale(max_peaks=50), mz, inten)
    order = sorted(range(60), key=lambda i: (-inten[i], mz[i]))[:50]
    expect_bins = sorted(int(np.floor((mz[i] - 101.0) / 0.05 + 1e-9)) for i in order)
    assert list(r[0]) == expect_bins


def test_min_peaks_and_zero_intensity(oracle):  # test_preprocess.cpp:138-152
    assert oracle.refine_vectorize(small_scale(min_peaks=3), [200.0, 300.0], [1.0, 1.0]) is None
    r = oracle.refine_vectorize(small_scale(intensity_floor=0.0), [200.0, 300.0], [0.0, 1.0])
    assert len(r[0]) == 1


def test_vectorize_known_answers(oracle):  # test_preprocess.cpp:175-215
    cfg = PreCfg(100.0, 1500.0, 0.05, 50, 1)
    b, v, _ = oracle.refine_vectorize(cfg, [100.00, 100.049, 100.05], [1.0, 1.0, 1.0])
    assert list(b) == [0, 1] and list(v) == [1.0, 0.5]
    b, v, _ = oracle.refine_vectorize(cfg, [200.00, 200.01], [0.4, 0.6])
    assert len(b) == 1 and v[0] == 1.0
    cfg = PreCfg(100.0, 1500.0, 0.05, 50, 1, 0.01, 1)
    b, v, _ = oracle.refine_vectorize(cfg, [200.0, 300.0], [0.25, 1.0])
    assert list(v) == [0.5, 1.0]


def test_single_peak_is_xnor(oracle):  # test_encoder.cpp:85-102
    cb = oracle.make_codebook(256, 128, 16, 8, 20)
    got = oracle.encode_vector(cb, [7], [1.0])
    assert np.array_equal(got, ~(cb.pos[7] ^ cb.lvl[16]))


def test_hand_built_codebook(oracle):  # test_encoder.cpp:104-130
    def bits(*b):
        return np.array([sum(int(x) << i for i, x in enumerate(b))], np.uint64)
    pos = np.stack([bits(1, 0, 1, 0, 1, 0, 1, 0), bits(1, 1, 0, 0, 1, 1, 0, 0), bits(0, 0, 0, 0, 1, 1, 1, 1)])
    lvl = np.stack([bits(0, 0, 0, 0, 0, 0, 0, 0), bits(1, 0, 0, 1, 0, 1, 1, 0), bits(1, 1, 1, 1, 1, 1, 1, 1)])
    cb = oracle.codebook_from_words(8, 2, pos, lvl)
    a = oracle.encode_vector(cb, [0, 2], [1.0, 0.4])
    b = oracle.encode_vector(cb, [0, 2], [1.0, 0.4], unpacked=True)
    assert np.array_equal(a, b)
    # two peaks: bit set only where both XNORs agree (strict majority, tie -> 0)
    x0 = ~(pos[0] ^ lvl[2]) & np.uint64(0xFF)
    x1 = ~(pos[2] ^ lvl[1]) & np.uint64(0xFF)
    assert a[0] == (x0 & x1)[0]


def test_encode_equals_accumulator_oracle(oracle):  # test_encoder.cpp:132-139
    cb = oracle.make_codebook(128, 16, 16, 12, 40)
    rng = np.random.default_rng(13)
    for _ in range(100):
        n = int(rng.integers(1, 13))
        bins = np.sort(rng.choice(40, n, replace=False)).astype(np.uint32)
        vals = rng.uniform(0, 1, n)
        vals[rng.integers(0, n)] = 1.0
        assert np.array_equal(oracle.encode_vector(cb, bins, vals),
                              oracle.encode_vector(cb, bins, vals, unpacked=True))


def test_level_similarity_law(oracle):  # test_codebook.cpp:76-90
    cb = oracle.make_codebook(8192, 4096, 16, 1, 1)
    for a in range(17):
        for b in range(17):
            sim = oracle.hamming_similarity(8192, cb.lvl[a], cb.lvl[b])
            assert sim / 8192 == 1.0 - abs(a - b) / 32.0


def test_hamming_identities(oracle):  # test_encoder.cpp:50-79
    rng = np.random.default_rng(3)
    x = U.random_hvs(rng, 1, 8192)[0]
    assert oracle.hamming_similarity(8192, x, x) == 8192
    assert oracle.hamming_similarity(8192, x, ~x) == 0
    for dim in (65, 100, 184):
        a, b = U.random_hvs(rng, 2, dim)
        assert oracle.hamming_similarity(dim, a, b) == oracle.hamming_similarity(dim, a, b, bitwise=True)


def test_window_known_answers(oracle):  # test_search.cpp:116-171
    rng = np.random.default_rng(5)
    mz = [999.9799, 999.98, 1000.0, 1000.02, 1000.0201]
    ix = oracle.build_index(256, U.random_hvs(rng, 5, 256), mz, [2] * 5)
    f, l, has = ix.select_candidates([1000.0], [2], ("ppm", 20.0))
    assert (f[0], l[0]) == (1, 4)
    f, l, has = ix.select_candidates([1000.0], [2], ("da", 500.0))
    assert l[0] - f[0] == 5
    f, l, has = ix.select_candidates([1000.0, 1000.0], [5, 0], ("ppm", 20.0))
    assert not has.any() and (l == f).all()
    ix2 = oracle.build_index(256, U.random_hvs(rng, 4, 256), [499.99, 500.0, 1500.0, 1500.01], [2] * 4)
    f, l, _ = ix2.select_candidates([1000.0], [2], ("da", 500.0))
    assert (f[0], l[0]) == (1, 3)  # inclusive at both ends


def test_tie_breaks(oracle):  # test_search.cpp:205-243
    rng = np.random.default_rng(10)
    shared = U.random_hvs(rng, 1, 256)
    two = np.repeat(shared, 2, 0)
    q = (shared, [1000.0], [2])
    ix = oracle.build_index(256, two, [1000.30, 1000.10], [2, 2], ids=["far", "near"])
    assert ix.search_batch(*q, ("da", 1.0))[2][0] == 1
    ix = oracle.build_index(256, two, [999.75, 1000.25], [2, 2], ids=["zz", "aa"])
    assert ix.search_batch(*q, ("da", 1.0))[2][0] == 1  # equal |diff|: smaller id
    ix = oracle.build_index(256, two, [1000.0, 1000.0], [2, 2], ids=["dup", "dup"])
    assert ix.search_batch(*q, ("da", 1.0))[2][0] == 0  # equal id: first input position


def test_fdr_worked_example(oracle):  # test_fdr.cpp:47-72
    order, fdr, q = oracle.compute_fdr_curve([0.9, 0.8, 0.7, 0.6], [0, 0, 1, 0])
    assert list(order) == [0, 1, 2, 3]
    assert list(fdr) == [0.0, 0.0, 0.5, 1.0 / 3.0]
    assert list(q) == [0.0, 0.0, 1.0 / 3.0, 1.0 / 3.0]


def test_codebook_fingerprints(oracle):
    fp = U.fingerprints()["codebook"]
    for dim in (1024, 2048):
        cb = oracle.make_codebook(dim, dim // 2, 16, 1, 27980)
        assert f"{fnv1a64_words(cb.pos):016x}" == fp[str(dim)]["position"]
        assert f"{fnv1a64_words(cb.lvl):016x}" == fp[str(dim)]["level"]
        assert f"{int(cb.pos[0, 0]):016x}" == "29250ebab86306dc"
        assert f"{int(cb.lvl[0, 0]):016x}" == "e116dfefd04cb935"
        oracle.free_codebook(cb)


def test_config1_fingerprints(oracle):  # synth -> encode -> search -> cascade
    fp = U.fingerprints()["config1"]
    s = oracle.synth(SynthCfg(n_library=5000, n_query=1000, fraction_modified=0.6, seed=1))
    L, Q = s["library"], s["queries"]
    assert f"{fnv1a64_words(L['mz'].view(np.uint64)):016x}" == fp["synth_library_mz_fnv"]
    assert f"{fnv1a64_words(Q['mz'].view(np.uint64)):016x}" == fp["synth_query_mz_fnv"]
    cb = oracle.make_codebook(2048, 1024, 16, 1, 27980)
    n_lib = 10000 if oracle.kind != "port" else 1500  # the scalar port encodes ~5k spectra/s
    lw, lok = oracle.encode_spectra(cb, PreCfg(), L["offsets"][: n_lib + 1], L["mz"], L["intensity"], threads=8)
    qw, qok = oracle.encode_spectra(cb, PreCfg(), Q["offsets"], Q["mz"], Q["intensity"], threads=8)
    assert f"{fnv1a64_words(qw):016x}" == fp["query_hv_fnv"]
    if n_lib == 10000:
        assert f"{fnv1a64_words(lw):016x}" == fp["library_hv_fnv"]
        ix = oracle.build_index(2048, lw, L["precursor_mz"], L["charge"], L["is_decoy"], L["ids"])
        first, last, _ = ix.select_candidates(Q["precursor_mz"], Q["charge"], ("da", 500.0))
        assert int((last - first).sum()) == fp["open_candidates_total"]
        has, score, ordinal, _ = ix.search_batch(qw, Q["precursor_mz"], Q["charge"], ("da", 500.0), threads=8)
        assert int(has.sum()) == fp["open_hits"]
        assert f"{fnv1a64_words(ordinal.astype(np.uint64)):016x}" == fp["open_ordinal_fnv"]
        c = ix.cascade_search(qw, Q["precursor_mz"], Q["charge"], ("ppm", 20.0), ("da", 500.0), 0.01, threads=8)
        assert (len(c["query"]), int((c["stage"] == 0).sum()), int((c["stage"] == 1).sum())) == (1000, 385, 615)
        assert f"{fnv1a64_words(c['q_value'].view(np.uint64)):016x}" == fp["cascade_qvalue_fnv"]


def test_golden_encode_cases(oracle):
    for name, c in U.encode_cases().items():
        cfg = U.oracle_precfg(c["precfg"])
        dim, flips, levels, seed = (int(x) for x in c["enccfg"])
        cb = oracle.make_codebook(dim, flips, levels, seed, oracle.dimension(cfg))
        assert fnv1a64_words(cb.pos) == int(c["codebook_fnv"][0]), name
        words, ok = oracle.encode_spectra(cb, cfg, c["offsets"], c["mz"], c["intensity"])
        assert np.array_equal(ok, c["ok"]), name
        assert np.array_equal(words, c["words"]), name
        for i in range(len(ok)):
            a, b = int(c["offsets"][i]), int(c["offsets"][i + 1])
            r = oracle.refine_vectorize(cfg, c["mz"][a:b], c["intensity"][a:b], levels)
            assert (r is not None) == bool(ok[i])
            if r is not None:
                s, e = int(c["sv_offsets"][i]), int(c["sv_offsets"][i + 1])
                assert np.array_equal(r[0], c["sv_bins"][s:e]) and np.array_equal(r[2], c["sv_levels"][s:e])
        oracle.free_codebook(cb)


def test_golden_search_cases(oracle):
    for name, c in U.search_cases().items():
        dim = int(c["dim"][0])
        ids = [x.decode() for x in c["ids"]]
        ix = oracle.build_index(dim, c["words"], c["mz"], c["charge"], c["decoy"], ids)
        for bi, b in enumerate(ix.buckets()):
            assert b["charge"] == int(c[f"bucket{bi}"]["charge"][0])
            assert np.array_equal(b["ordinal"], c[f"bucket{bi}"]["ordinal"]), name
        for tname, tol in U.TOLS.items():
            g = c[tname]
            first, last, has_b = ix.select_candidates(c["q_mz"], c["q_charge"], tol)
            assert np.array_equal(first, g["first"]) and np.array_equal(last, g["last"]), (name, tname)
            assert np.array_equal(has_b, g["has_bucket"])
            has, score, ordinal, _ = ix.search_batch(c["q_words"], c["q_mz"], c["q_charge"], tol)
            assert np.array_equal(has, g["has"]) and np.array_equal(score, g["score"]), (name, tname)
            assert np.array_equal(ordinal, g["ordinal"]), (name, tname)
        for cname, narrow, wide, fq in (("c1", ("ppm", 150.0), ("da", 30.0), 0.05),
                                        ("c2", ("da", 0.3), ("da", 500.0), 0.5)):
            got = ix.cascade_search(c["q_words"], c["q_mz"], c["q_charge"], narrow, wide, fq)
            for k in got:
                assert np.array_equal(got[k], c[cname][k]), (name, cname, k)


def test_port_topk_first_is_top1(port):
    c = U.search_cases()["d256"]
    ix = port.build_index(256, c["words"], c["mz"], c["charge"], c["decoy"], [x.decode() for x in c["ids"]])
    score, ordinal = ix.search_topk(c["q_words"], c["q_mz"], c["q_charge"], ("da", 30.0), 5)
    assert np.array_equal(ordinal[:, 0], c["da30"]["ordinal"])
    assert np.array_equal(score[:, 0], c["da30"]["score"])
    assert (np.diff(score.astype(np.int64), axis=1) <= 0).all()


def test_port_equals_reference_random(port, ref):
    """Restatement vs the compiled reference on fresh random inputs (beyond the fixtures)."""
    rng = np.random.default_rng(99)
    for trial in range(4):
        cfg = PreCfg(max_peaks=int(rng.integers(5, 80)), min_peaks=int(rng.integers(1, 5)),
                     scaling=int(rng.integers(0, 2)), intensity_floor=float(rng.uniform(0, 0.2)))
        dim = int(rng.choice([64, 192, 1024, 4096]))
        cbp = port.make_codebook(dim, max(1, dim // 2), 16, trial, 27980)
        cbr = ref.make_codebook(dim, max(1, dim // 2), 16, trial, 27980)
        assert np.array_equal(cbp.pos, cbr.pos) and np.array_equal(cbp.lvl, cbr.lvl)
        spectra = []
        for _ in range(60):
            p = int(rng.integers(0, 150))
            mz = np.unique(np.round(rng.uniform(80, 1600, p), 2))
            spectra.append((mz, rng.uniform(0, 1, len(mz)) * (rng.uniform(0, 1, len(mz)) > 0.1)))
        off, mz, it = U.csr(spectra)
        wp, okp = port.encode_spectra(cbp, cfg, off, mz, it)
        wr, okr = ref.encode_spectra(cbr, cfg, off, mz, it, threads=3, batch=4)
        assert np.array_equal(okp, okr) and np.array_equal(wp, wr)


def test_golden_mgf_cases(oracle):
    """parse_mgf (mgf.cpp:93-181): the reference's own test cases (test_mgf.cpp), number-grammar corner
    cases and random mutations, expected results generated from the compiled reference."""
    from tests import _mgf_cases as M
    cases = U.mgf_cases()
    assert len(cases) == U.fingerprints()["mgf_cases"]["cases"]
    n_ok = 0
    for text, want in cases:
        if isinstance(want, str):
            with pytest.raises(OracleError) as e:
                oracle.mgf_parse(text)
            assert str(e.value) == want, text[:200]
        else:
            n_ok += 1
            assert M.same(want, oracle.mgf_parse(text)), text[:200]
    assert n_ok == U.fingerprints()["mgf_cases"]["parsed"]


def test_mgf_write_matches_reference_format(port):
    """write_mgf (mgf.cpp:183-208): "%.5f" precursor, "%.5f %.6f" peaks, CHARGE only when known."""
    text = port.mgf_write([0, 2, 2], [100.123456, 200.5], [1.5, 0.1234567], [500.123456, 600.0], [2, 0],
                          ["a", "b"], [b"PEP", b""])
    assert text == (b"BEGIN IONS\nTITLE=a\nPEPMASS=500.12346\nCHARGE=2+\nSEQ=PEP\n100.12346 1.500000\n"
                    b"200.50000 0.123457\nEND IONS\n\nBEGIN IONS\nTITLE=b\nPEPMASS=600.00000\nEND IONS\n\n")
    r = port.mgf_parse(text)
    assert r["ids"] == [b"a", b"b"] and list(r["charge"]) == [2, 0] and list(r["offsets"]) == [0, 2, 2]
