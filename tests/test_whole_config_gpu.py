"""GPU: WHOLE-config parity at the BASELINE shapes, on the reference generator's own inputs
(generate_benchmark(SynthConfig{...}), src/synth.cpp:114-197, seeds 2 and 3).

config 2 (iPRG2012 shape, 1.2 M library x 16 000 queries, D = 8192): every hypervector, the open +-500 Da
top-1 (has-hit, raw_score, ordinal) of ALL queries and the full cascade_search accepted list (ids, stage,
score, q-value bits) and counts -- against the live compiled reference (oracle/_ref, x86-64-v3 flavour) AND
the fingerprints committed in tests/golden/fingerprints.json (made from the reference by
tests/golden/make_whole_config.py).  The north-star's "FDR-filtered identification counts must be identical"
is checked here on the whole query set.

config 3 (HEK293 shape, 4.3 M library x 1 M queries): hypervector fingerprints of the whole library and
query set, open top-1 and cascade of a 2 048-query prefix against the reference over the full library.

Minutes of CPU time on the reference side: marked slow (still part of `-m gpu`)."""
import os
import time

import numpy as np
import pytest

from tests import _util as U

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _generate(name):
    import workload as wl
    if not wl.reference_generator_available():
        pytest.skip("oracle/_ref not built: the reference generator is unavailable")
    lib, qry, dim, gen = wl.make(name, "reference")
    assert gen == "reference"
    return lib, qry, dim


def _encode_all(hb, c, spec, pre, W, chunk=400_000):
    n = len(spec["offsets"]) - 1
    words = np.empty((n, W), np.uint64)
    ok = np.empty(n, np.uint8)
    off = spec["offsets"].astype(np.int64)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        p0, p1 = off[a], off[b]
        c.encode_batch((spec["offsets"][a:b + 1] - spec["offsets"][a]), spec["mz"][p0:p1], spec["intensity"][p0:p1], pre,
                       out=(words[a:b], ok[a:b]))
    return words, ok


def _reference(kind_pref=("ref_v3", "ref")):
    from oracle import binding as ob
    for kind in kind_pref:
        if ob.available(kind):
            return ob.Oracle(kind)
    pytest.skip("oracle/_ref not built")


def _check_golden(got: dict, want: dict, keys):
    for key in keys:
        assert got[key] == want[key], (key, got[key], want[key])


def test_config2_whole_parity(hb):
    want = U.fingerprints().get("whole_config", {}).get("config2")
    lib, qry, dim = _generate("iprg2012")
    n_lib, nq = len(lib["precursor_mz"]), len(qry["precursor_mz"])
    assert (n_lib, nq, dim) == (1_200_000, 16_000, 8192)
    W = dim // 64
    pre = hb.PreprocessConfig()
    cb = hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 1))
    open_tol, narrow_tol = hb.Tolerance("dalton", 500.0), hb.Tolerance("ppm", 20.0)
    cores = os.cpu_count() or 1

    with hb.Context(0) as c:
        c.upload_codebook(cb)
        lw, lok = _encode_all(hb, c, lib, pre, W)
        qw, qok = _encode_all(hb, c, qry, pre, W)
        assert lok.all() and qok.all()
        got = {"synth_library_mz_fnv": U.fnv_hex(lib["mz"]), "synth_query_mz_fnv": U.fnv_hex(qry["mz"]),
               "library_hv_fnv": U.fnv_hex(lw), "query_hv_fnv": U.fnv_hex(qw)}
        c.build_index(dim, lw, lib["precursor_mz"], lib["charge"], ids=lib["ids"], is_decoy=lib["is_decoy"])
        m = c.search_batch(qw, qry["precursor_mz"], qry["charge"], open_tol)
        cas = c.cascade_search(qw, qry["precursor_mz"], qry["charge"], narrow_tol, open_tol, 0.01)
        # the same through a multi-device context (aliases of device 0 when only one GPU is visible)
        devs = list(range(hb.device_count())) if hb.device_count() >= 2 else [0, 0]
    got.update(open_hits=int(m.has_hit.sum()), open_candidates_total=int((m.last - m.first).sum()),
               open_score_fnv=U.fnv_hex(m.raw_score[:, 0]), open_ordinal_fnv=U.fnv_hex(m.ordinal[:, 0]),
               cascade_accepted=int(len(cas["query"])), cascade_narrow=int((cas["stage"] == 0).sum()),
               cascade_wide=int((cas["stage"] == 1).sum()), cascade_query_fnv=U.fnv_hex(cas["query"]),
               cascade_ordinal_fnv=U.fnv_hex(cas["ordinal"]), cascade_score_fnv=U.fnv_hex(cas["raw_score"]),
               cascade_qvalue_fnv=U.fnv_hex(cas["q_value"]))
    if want:  # committed fingerprints, made from the reference alone
        _check_golden(got, want, ["synth_library_mz_fnv", "synth_query_mz_fnv", "library_hv_fnv", "query_hv_fnv", "open_hits",
                                  "open_candidates_total", "open_score_fnv", "open_ordinal_fnv", "cascade_accepted",
                                  "cascade_narrow", "cascade_wide", "cascade_query_fnv", "cascade_ordinal_fnv",
                                  "cascade_score_fnv", "cascade_qvalue_fnv"])

    with hb.Context(devices=devs) as grp:
        grp.build_index(dim, lw, lib["precursor_mz"], lib["charge"], ids=lib["ids"], is_decoy=lib["is_decoy"])
        gm = grp.search_batch(qw, qry["precursor_mz"], qry["charge"], open_tol)
        assert np.array_equal(gm.ordinal, m.ordinal) and np.array_equal(gm.raw_score, m.raw_score)
        gc = grp.cascade_search(qw, qry["precursor_mz"], qry["charge"], narrow_tol, open_tol, 0.01)
        assert all(np.array_equal(gc[k], cas[k]) for k in ("query", "ordinal", "stage", "raw_score"))

    # the live reference: its own encoder on a sample of spectra, its search / cascade on ALL queries over an
    # index built from the (fingerprint-checked) hypervectors
    ref = _reference()
    from oracle import binding as ob
    ocb = ref.make_codebook(dim, dim // 2, 16, 1, ref.dimension(ob.PreCfg()))
    pick = np.random.default_rng(2).choice(n_lib, 20_000, replace=False)
    pick.sort()
    peaks = lib["peaks"]
    s_off = np.arange(len(pick) + 1, dtype=np.uint64) * np.uint64(peaks)
    s_mz = lib["mz"].reshape(-1, peaks)[pick].ravel()
    s_it = lib["intensity"].reshape(-1, peaks)[pick].ravel()
    ow, ook = ref.encode_spectra(ocb, ob.PreCfg(), s_off, s_mz, s_it, threads=cores, batch=64)
    assert ook.all() and np.array_equal(ow, lw[pick])
    oq, _ = ref.encode_spectra(ocb, ob.PreCfg(), qry["offsets"], qry["mz"], qry["intensity"], threads=cores, batch=64)
    assert np.array_equal(oq, qw)
    t = time.time()
    ix = ref.build_index(dim, lw, lib["precursor_mz"], lib["charge"], lib["is_decoy"], lib["ids"])
    has, score, ordinal, _ = ix.search_batch(qw, qry["precursor_mz"], qry["charge"], ("da", 500.0), threads=cores, batch=8)
    assert np.array_equal(m.has_hit[:, 0], has.astype(bool))
    assert np.array_equal(m.raw_score[:, 0], score) and np.array_equal(m.ordinal[:, 0], ordinal)
    rc = ix.cascade_search(qw, qry["precursor_mz"], qry["charge"], ("ppm", 20.0), ("da", 500.0), 0.01, threads=cores, batch=8)
    ix.close()
    print(f"reference search + cascade of {nq} queries on {cores} cores: {time.time() - t:.0f}s")
    for key in ("query", "ordinal", "stage", "raw_score"):
        assert np.array_equal(cas[key], rc[key]), key
    assert np.array_equal(cas["q_value"].view(np.uint64), rc["q_value"].view(np.uint64))
    assert len(rc["query"]) == got["cascade_accepted"]


def test_config3_prefix_parity(hb):
    want = U.fingerprints().get("whole_config", {}).get("config3")
    lib, qry, dim = _generate("hek293_full")
    n_lib, nq = len(lib["precursor_mz"]), len(qry["precursor_mz"])
    assert (n_lib, nq, dim) == (4_300_000, 1_000_000, 8192)
    W = dim // 64
    pre = hb.PreprocessConfig()
    cb = hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 1))
    open_tol, narrow_tol = hb.Tolerance("dalton", 500.0), hb.Tolerance("ppm", 20.0)
    cores = os.cpu_count() or 1
    n = 2048
    with hb.Context(0) as c:
        c.upload_codebook(cb)
        lw, lok = _encode_all(hb, c, lib, pre, W)
        qw, qok = _encode_all(hb, c, qry, pre, W)
        assert lok.all() and qok.all()
        got = {"synth_library_mz_fnv": U.fnv_hex(lib["mz"]), "synth_query_mz_fnv": U.fnv_hex(qry["mz"]),
               "library_hv_fnv": U.fnv_hex(lw), "query_hv_fnv": U.fnv_hex(qw)}
        c.build_index(dim, lw, lib["precursor_mz"], lib["charge"], ids=lib["ids"], is_decoy=lib["is_decoy"])
        m = c.search_batch(qw[:n], qry["precursor_mz"][:n], qry["charge"][:n], open_tol)
        cas = c.cascade_search(qw[:n], qry["precursor_mz"][:n], qry["charge"][:n], narrow_tol, open_tol, 0.01)
        # all 1 M queries (several planning batches): the prefix must come out the same inside the big call
        big = c.search_batch(qw[:200_000], qry["precursor_mz"][:200_000], qry["charge"][:200_000], open_tol)
        assert np.array_equal(big.ordinal[:n], m.ordinal) and np.array_equal(big.raw_score[:n], m.raw_score)
    got.update(open_hits=int(m.has_hit.sum()), open_candidates_total=int((m.last - m.first).sum()),
               open_score_fnv=U.fnv_hex(m.raw_score[:, 0]), open_ordinal_fnv=U.fnv_hex(m.ordinal[:, 0]),
               cascade_accepted=int(len(cas["query"])), cascade_narrow=int((cas["stage"] == 0).sum()),
               cascade_wide=int((cas["stage"] == 1).sum()), cascade_query_fnv=U.fnv_hex(cas["query"]),
               cascade_ordinal_fnv=U.fnv_hex(cas["ordinal"]), cascade_score_fnv=U.fnv_hex(cas["raw_score"]),
               cascade_qvalue_fnv=U.fnv_hex(cas["q_value"]))
    if want:
        assert want["searched_queries"] == n
        _check_golden(got, want, ["synth_library_mz_fnv", "synth_query_mz_fnv", "library_hv_fnv", "query_hv_fnv", "open_hits",
                                  "open_candidates_total", "open_score_fnv", "open_ordinal_fnv", "cascade_accepted",
                                  "cascade_narrow", "cascade_wide", "cascade_query_fnv", "cascade_ordinal_fnv",
                                  "cascade_score_fnv", "cascade_qvalue_fnv"])
    ref = _reference()
    ix = ref.build_index(dim, lw, lib["precursor_mz"], lib["charge"], lib["is_decoy"], lib["ids"])
    has, score, ordinal, _ = ix.search_batch(qw[:n], qry["precursor_mz"][:n], qry["charge"][:n], ("da", 500.0),
                                             threads=cores, batch=8)
    assert np.array_equal(m.has_hit[:, 0], has.astype(bool))
    assert np.array_equal(m.raw_score[:, 0], score) and np.array_equal(m.ordinal[:, 0], ordinal)
    rc = ix.cascade_search(qw[:n], qry["precursor_mz"][:n], qry["charge"][:n], ("ppm", 20.0), ("da", 500.0), 0.01,
                           threads=cores, batch=8)
    ix.close()
    for key in ("query", "ordinal", "stage", "raw_score"):
        assert np.array_equal(cas[key], rc[key]), key
    assert np.array_equal(cas["q_value"].view(np.uint64), rc["q_value"].view(np.uint64))
