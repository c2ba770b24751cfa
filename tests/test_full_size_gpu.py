"""GPU: BASELINE.json config 2 at FULL size (1.2 M library rows, D = 8192) through size-independent
properties -- the oracle cannot finish this size in seconds, so the checks are the ones the domain
offers: encode -> index -> search round trips (a library spectrum finds itself with score D),
monotonicity in the tolerance (test_search.cpp:280-296), consistency between k = 1 and k > 1,
agreement of the engines, and reported scores recomputed with hamming_similarity
(hypervector.hpp:70-81) from independently encoded rows."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _take(spec, rows, peaks):
    """CSR sub-list of fixed-width spectra."""
    off = np.arange(len(rows) + 1, dtype=np.uint64) * np.uint64(peaks)
    mz = spec["mz"].reshape(-1, peaks)[rows].ravel()
    it = spec["intensity"].reshape(-1, peaks)[rows].ravel()
    return off, mz, it


def test_iprg2012_full_size_properties(hb):
    import workload as wl
    n_targets, _, dim, peaks, seed = wl.WORKLOADS["iprg2012"]
    lib = wl.synth_library(n_targets, peaks, 1.0, seed)
    n = len(lib["precursor_mz"])
    assert n == 1_200_000
    pre = hb.PreprocessConfig()
    cb = hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 1))
    rank = hb.id_ranks(lib["ids"])
    rng = np.random.default_rng(5)
    open_tol, ppm_tol = hb.Tolerance("dalton", 500.0), hb.Tolerance("ppm", 20.0)

    with hb.Context(0) as c:
        c.upload_codebook(cb)
        ok = c.build_index_from_spectra(lib["offsets"], lib["mz"], lib["intensity"], pre, lib["precursor_mz"],
                                        lib["charge"], id_rank=rank, is_decoy=lib["is_decoy"])
        assert ok.all() and c.lib_n == n
        # the index: charge buckets partition the library, rows sorted by precursor m/z, ordinals a permutation
        buckets = c.buckets()
        assert sorted(b["charge"] for b in buckets) == [2, 3]
        assert sum(len(b["precursor_mz"]) for b in buckets) == n
        seen = np.zeros(n, bool)
        for b in buckets:
            assert (np.diff(b["precursor_mz"]) >= 0).all()
            assert np.array_equal(b["precursor_mz"], lib["precursor_mz"][b["ordinal"]])
            assert (lib["charge"][b["ordinal"]] == b["charge"]).all()
            seen[b["ordinal"]] = True
        assert seen.all()
        del buckets

        # (1) round trip: library spectra as queries find themselves with the maximal score
        pick = np.sort(rng.choice(n, 3072, replace=False))
        off, mz, it = _take(lib, pick, peaks)
        qok = c.queries_from_spectra(off, mz, it, pre, lib["precursor_mz"][pick], lib["charge"][pick])
        assert qok.all()
        for tol in (open_tol, ppm_tol):
            m = c.search_resident(tol)
            assert m.has_hit.all()
            assert (m.raw_score[:, 0] == dim).all()
            assert np.array_equal(m.ordinal[:, 0], pick.astype(np.uint32))
        # the open window of a charge-2/3 query is a large part of its bucket
        m_open = c.search_resident(open_tol)
        assert ((m_open.last - m_open.first) > 100_000).all()

        # (2) modified queries: widening the tolerance never lowers the best score, k = 1 is the head
        #     of k = 4, scores fall along k, ordinals are distinct
        qry = wl.synth_queries(lib, 4096, seed=seed)
        c.queries_from_spectra(qry["offsets"], qry["mz"], qry["intensity"], pre, qry["precursor_mz"], qry["charge"])
        prev = np.zeros(4096, np.uint32)
        for tol in (ppm_tol, hb.Tolerance("dalton", 1.0), hb.Tolerance("dalton", 50.0), open_tol):
            s = c.search_resident(tol)
            score = np.where(s.has_hit[:, 0], s.raw_score[:, 0], 0)
            assert (score >= prev).all()
            prev = score
        top1 = c.search_resident(open_tol)
        top4 = c.search_resident(open_tol, k=4)
        assert np.array_equal(top4.raw_score[:, 0], top1.raw_score[:, 0])
        assert np.array_equal(top4.ordinal[:, 0], top1.ordinal[:, 0])
        assert (np.diff(top4.raw_score.astype(np.int64), axis=1) <= 0).all()
        assert all(len(set(r)) == 4 for r in top4.ordinal[:256])
        # unmodified queries keep their precursor: the source target is inside even the 20 ppm window
        # and wins it (5 % intensity noise leaves it far above every other row)
        plain = np.flatnonzero(~qry["modified"])
        narrow = c.search_resident(ppm_tol)
        assert narrow.has_hit[plain, 0].all()
        assert np.array_equal(narrow.ordinal[plain, 0], qry["source"][plain].astype(np.uint32))

        # (3) reported scores == hamming_similarity of independently encoded rows
        sample = rng.choice(4096, 256, replace=False)
        q_enc = c.encode_spectra(*_sub(qry, sample), pre)
        hit_rows = top1.ordinal[sample, 0].astype(np.int64)
        l_enc = c.encode_spectra(*_take(lib, hit_rows, peaks), pre)
        assert len(q_enc.kept) == 256 and len(l_enc.kept) == 256
        assert np.array_equal(c.hamming_similarity(dim, q_enc.words, l_enc.words), top1.raw_score[sample, 0])

        # (4) the XOR+POPC engine agrees with the tensor engine at this size
        few = np.arange(512)
        c.queries_from_spectra(*_sub(qry, few), pre, qry["precursor_mz"][few], qry["charge"][few])
        tensor = c.search_resident(open_tol, k=2)
        c.set_engine("popc")
        popc = c.search_resident(open_tol, k=2)
        assert np.array_equal(tensor.ordinal, popc.ordinal) and np.array_equal(tensor.raw_score, popc.raw_score)


def _sub(spec, rows):
    """CSR sub-list of a ragged spectrum list."""
    off = spec["offsets"].astype(np.int64)
    parts_mz = [spec["mz"][off[i]:off[i + 1]] for i in rows]
    parts_it = [spec["intensity"][off[i]:off[i + 1]] for i in rows]
    new_off = np.zeros(len(rows) + 1, np.uint64)
    new_off[1:] = np.cumsum([len(p) for p in parts_mz])
    return new_off, np.concatenate(parts_mz), np.concatenate(parts_it)
