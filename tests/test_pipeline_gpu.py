"""GPU: the composed query-file flow (MGF text -> mgf_parse -> queries_from_mgf -> cascade_resident)
against the reference's own run_search stages (src/pipeline.cpp:119-150: parse_mgf, known-charge filter,
encode_spectra, cascade_search, write_ssm_tsv) run by the compiled reference on the same text: identical TSV
bytes and identical statistics, on one device and on a multi-device context."""
import numpy as np
import pytest

from oracle.binding import PreCfg, SynthCfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup(ref):
    synth = ref.synth(SynthCfg(n_library=3000, n_query=800, peaks_per_spectrum=50, fraction_modified=0.6, seed=31))
    L, Q = synth["library"], synth["queries"]
    q_charge = Q["charge"].copy()
    q_charge[[4, 77, 78, 500]] = 0          # unknown charge: skipped before encoding (pipeline.cpp:127-134)
    q_int = Q["intensity"].copy()
    for i in (9, 77, 300):                  # too few peaks: unprocessable (77 is also charge-less: counts as skipped)
        a, b = int(Q["offsets"][i]), int(Q["offsets"][i + 1])
        q_int[a + 4:b] = 0.0
    text = ref.mgf_write(Q["offsets"], Q["mz"], q_int, Q["precursor_mz"], q_charge, Q["ids"])
    # dirt the parser must cope with identically: comments, a title-less block, CRLF
    text = b"# exported\n" + text + b"BEGIN IONS\nPEPMASS=612.25\nCHARGE=2+\n" + \
        b"".join(b"%d.5 %d\r\n" % (200 + 13 * j, 1 + j % 7) for j in range(40)) + b"END IONS\n"
    return L, text


def _gpu_side(hb, c, L, dim):
    pre = hb.PreprocessConfig()
    cb = hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 1))
    c.upload_codebook(cb)
    ok = c.build_index_from_spectra(L["offsets"], L["mz"], L["intensity"], pre, L["precursor_mz"], L["charge"],
                                    ids=L["ids"], is_decoy=L["is_decoy"])
    assert ok.all()
    c.lib_precursor_mz = L["precursor_mz"]
    return pre


@pytest.mark.parametrize("devices", [None, [0, 0, 0]])
def test_query_file_flow_identical_tsv(hb, ref, setup, devices):
    L, text = setup
    dim = 2048
    ocb = ref.make_codebook(dim, dim // 2, 16, 1, ref.dimension(PreCfg()))
    lw, lok = ref.encode_spectra(ocb, PreCfg(), L["offsets"], L["mz"], L["intensity"], threads=8)
    assert lok.all()
    ix = ref.build_index(dim, lw, L["precursor_mz"], L["charge"], L["is_decoy"], L["ids"])
    want = ix.query_flow(ocb, PreCfg(), text, ("ppm", 20.0), ("da", 500.0), 0.01, threads=8)
    ix.close()
    assert want["stats"]["skipped_unknown_charge"] == 4 and want["stats"]["unprocessable"] == 2
    with (hb.Context(0) if devices is None else hb.Context(devices=devices)) as c:
        pre = _gpu_side(hb, c, L, dim)
        got = c.search_file(text, pre, hb.Tolerance("ppm", 20.0), hb.Tolerance("dalton", 500.0), 0.01, L["ids"],
                            [str(i) for i in range(len(L["ids"]))])
        assert got["stats"] == want["stats"]
        assert got["tsv"] == want["tsv"]
        assert len(got["tsv"].splitlines()) == 1 + want["stats"]["accepted_narrow"] + want["stats"]["accepted_wide"]
        # the pieces are also usable one by one; states line up with what the reference skipped / dropped
        info = c.parse_mgf(text, fetch=False)
        state = c.queries_from_mgf(pre, info["n_spectra"])
        assert info["n_spectra"] == want["stats"]["total_queries"] == 801
        assert sorted(np.flatnonzero(state == 1)) == [4, 77, 78, 500] and sorted(np.flatnonzero(state == 2)) == [9, 300]


def test_queries_from_mgf_needs_a_parse_and_a_codebook(hb):
    with hb.Context(0) as c:
        with pytest.raises(hb.HomsError):
            c.queries_from_mgf(hb.PreprocessConfig(), 0)
        c.upload_codebook(hb.make_codebook(hb.dimension(hb.PreprocessConfig()), hb.EncoderConfig(256, 128, 16, 1)))
        with pytest.raises(hb.HomsError):
            c.queries_from_mgf(hb.PreprocessConfig(), 0)
