"""GPU: the fused raw-spectra entry points against the oracle's composition of the
reference calls they replace -- build_index(encode_spectra(library)), encode_spectra(queries),
search_batch, cascade_search -- bit for bit, with unprocessable spectra in both lists so that the
order-preserving compaction (pipeline.cpp:75-83) and the ordinal numbering are exercised."""
import numpy as np
import pytest

from oracle.binding import PreCfg, SynthCfg

pytestmark = pytest.mark.gpu


def _with_dropouts(spec, every, keep_peaks):
    """Copy of a synthetic spectrum list in which every `every`-th spectrum keeps only `keep_peaks`
    peaks (below min_peaks = 5 -> refine_peaks returns nullopt, preprocess.cpp:69)."""
    off = spec["offsets"].astype(np.int64)
    mz, it, new_off = [], [], [0]
    for i in range(len(off) - 1):
        a, b = off[i], off[i + 1]
        if i % every == every - 1:
            b = a + keep_peaks
        mz.append(spec["mz"][a:b])
        it.append(spec["intensity"][a:b])
        new_off.append(new_off[-1] + (b - a))
    out = dict(spec)
    out["offsets"] = np.asarray(new_off, np.uint64)
    out["mz"] = np.concatenate(mz)
    out["intensity"] = np.concatenate(it)
    return out


@pytest.fixture(scope="module")
def workload(best_oracle):
    synth = best_oracle.synth(SynthCfg(n_library=700, n_query=300, peaks_per_spectrum=40,
                                       fraction_modified=0.6, seed=77))
    return _with_dropouts(synth["library"], 9, 3), _with_dropouts(synth["queries"], 7, 2)


@pytest.fixture(params=["tensor_fp4", "popc"])
def fctx(hb, request):
    c = hb.Context(0)
    c.set_engine(request.param)
    yield c
    c.close()


def _oracle_side(best_oracle, hb, L, Q, dim):
    pre = hb.PreprocessConfig()
    ocb = best_oracle.make_codebook(dim, dim // 2, 16, 1, hb.dimension(pre))
    lw, lok = best_oracle.encode_spectra(ocb, PreCfg(), L["offsets"], L["mz"], L["intensity"])
    qw, qok = best_oracle.encode_spectra(ocb, PreCfg(), Q["offsets"], Q["mz"], Q["intensity"])
    lk, qk = np.flatnonzero(lok), np.flatnonzero(qok)
    ids = [L["ids"][i] for i in lk]
    oix = best_oracle.build_index(dim, lw[lk], L["precursor_mz"][lk], L["charge"][lk], L["is_decoy"][lk], ids)
    return oix, lok, qok, qw[qk], Q["precursor_mz"][qk], Q["charge"][qk]


@pytest.mark.parametrize("dim", [2048, 1000])
def test_fused_index_and_queries_match_composition(hb, fctx, best_oracle, workload, dim):
    L, Q = workload
    pre = hb.PreprocessConfig()
    fctx.upload_codebook(hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 1)))
    oix, lok, qok, oqw, oqmz, oqch = _oracle_side(best_oracle, hb, L, Q, dim)
    assert 0 < lok.sum() < len(lok) and 0 < qok.sum() < len(qok)  # both lists really have dropouts

    ok = fctx.build_index_from_spectra(L["offsets"], L["mz"], L["intensity"], pre, L["precursor_mz"],
                                       L["charge"], ids=L["ids"], is_decoy=L["is_decoy"])
    assert np.array_equal(ok, lok)
    assert fctx.lib_n == int(lok.sum())
    qk = fctx.queries_from_spectra(Q["offsets"], Q["mz"], Q["intensity"], pre, Q["precursor_mz"], Q["charge"])
    assert np.array_equal(qk, qok)
    assert fctx.resident_queries == int(qok.sum())

    for tol, otol in ((hb.Tolerance("dalton", 500.0), ("da", 500.0)), (hb.Tolerance("ppm", 20.0), ("ppm", 20.0))):
        got = fctx.search_resident(tol)
        has, score, ordinal, _ = oix.search_batch(oqw, oqmz, oqch, otol)
        assert np.array_equal(got.has_hit[:, 0], has.astype(bool))
        assert np.array_equal(got.raw_score[:, 0], score)
        assert np.array_equal(got.ordinal[:, 0], ordinal)  # ordinals count processable spectra only

    got = fctx.cascade_resident(hb.Tolerance("ppm", 20.0), hb.Tolerance("dalton", 500.0), 0.01)
    want = oix.cascade_search(oqw, oqmz, oqch, ("ppm", 20.0), ("da", 500.0), 0.01)
    for key in ("query", "ordinal", "stage", "raw_score"):
        assert np.array_equal(got[key], want[key]), key
    assert np.array_equal(got["q_value"].view(np.uint64), want["q_value"].view(np.uint64))
    assert len(got["query"]) > 0
    oix.close()


def test_fused_equals_unfused_product_path(hb, ctx, workload):
    """Same context, host round trip vs fused: identical resident state as seen through search."""
    L, Q = workload
    pre = hb.PreprocessConfig()
    dim = 2048
    ctx.upload_codebook(hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 1)))
    lib = ctx.encode_spectra(L["offsets"], L["mz"], L["intensity"], pre)
    qry = ctx.encode_spectra(Q["offsets"], Q["mz"], Q["intensity"], pre)
    ids = [L["ids"][i] for i in lib.kept]
    ctx.build_index(dim, lib.words, L["precursor_mz"][lib.kept], L["charge"][lib.kept], ids=ids)
    tol = hb.Tolerance("dalton", 500.0)
    a = ctx.search_batch(qry.words, Q["precursor_mz"][qry.kept], Q["charge"][qry.kept], tol, k=3)
    ctx.build_index_from_spectra(L["offsets"], L["mz"], L["intensity"], pre, L["precursor_mz"], L["charge"],
                                 ids=L["ids"])
    ctx.queries_from_spectra(Q["offsets"], Q["mz"], Q["intensity"], pre, Q["precursor_mz"], Q["charge"])
    b = ctx.search_resident(tol, k=3)
    assert np.array_equal(a.ordinal, b.ordinal) and np.array_equal(a.raw_score, b.raw_score)
    assert np.array_equal(a.first, b.first) and np.array_equal(a.last, b.last)


def test_fused_sharded_merge(hb, workload):
    """build_index_from_spectra on G shards + merge == the single-shard answer."""
    import torch
    L, Q = workload
    pre = hb.PreprocessConfig()
    dim = 2048
    cb = hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 1))
    tol = hb.Tolerance("dalton", 500.0)
    dev = torch.device("cuda", 0)
    answers = {}
    for G in (1, 3):
        parts = []
        for g in range(G):
            c = hb.Context(0)
            c.upload_codebook(cb)
            c.build_index_from_spectra(L["offsets"], L["mz"], L["intensity"], pre, L["precursor_mz"],
                                       L["charge"], ids=L["ids"], shard_index=g, shard_count=G)
            c.queries_from_spectra(Q["offsets"], Q["mz"], Q["intensity"], pre, Q["precursor_mz"], Q["charge"])
            nq = c.resident_queries
            rec = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
            c.search_resident_dev(tol, 1, rec.data_ptr())
            c.synchronize()
            parts.append(rec)
            if g == G - 1:
                gathered = torch.cat(parts)
                merged = torch.empty(nq * 16, dtype=torch.uint8, device=dev)
                c.merge_candidates_dev(nq, 1, G, gathered.data_ptr(), merged.data_ptr())
                answers[G] = c.candidates_decode(nq, 1, merged.data_ptr())
            c.close()
    assert np.array_equal(answers[1][0], answers[3][0]) and np.array_equal(answers[1][1], answers[3][1])


def test_fused_errors(hb, ctx):
    pre = hb.PreprocessConfig()
    with pytest.raises(hb.HomsError):  # no codebook
        ctx.build_index_from_spectra([0, 1], [200.0], [1.0], pre, [500.0], [2])
    ctx.upload_codebook(hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(256, 128, 16, 1)))
    with pytest.raises(hb.InvariantError):  # nothing processable -> "library is empty" (search.cpp:18)
        ctx.build_index_from_spectra([0, 1], [200.0], [1.0], pre, [500.0], [2])
    ok = ctx.queries_from_spectra([0, 1], [200.0], [1.0], pre, [500.0], [2])
    assert ok.tolist() == [0] and ctx.resident_queries == 0


def test_encode_batch_pipeline_many_chunks(hb, ctx, best_oracle):
    """More spectra than one pipeline chunk (64 Ki), ragged sizes incl. empty ones: the chunked
    three-stream path must produce exactly what the oracle produces, row for row."""
    rng = np.random.default_rng(11)
    n = 150_000
    pre = hb.PreprocessConfig()
    dim = 256
    ctx.upload_codebook(hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 3)))
    counts = rng.integers(0, 13, n)
    counts[rng.integers(0, n, 50)] = 70  # a few above max_peaks = 50
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(counts)
    total = int(off[-1])
    seg = np.repeat(np.arange(n), counts)
    mz = rng.uniform(90.0, 1600.0, total)
    mz = mz[np.lexsort((mz, seg))]  # ascending m/z inside every spectrum
    it = rng.uniform(0.0, 1.0, total) * (rng.random(total) > 0.05)
    words, ok = ctx.encode_batch(off, mz, it, pre)
    ocb = best_oracle.make_codebook(dim, dim // 2, 16, 3, hb.dimension(pre))
    ow, ook = best_oracle.encode_spectra(ocb, PreCfg(), off, mz, it, threads=8, batch=256)
    assert np.array_equal(ok, ook)
    assert 0 < ok.sum() < n
    assert np.array_equal(words, ow)
