"""GPU: MGF text -> CSR against the oracle's parse_mgf (the compiled reference when it
travelled, else the C restatement): same spectra bit for bit, same first ParseError text, on the
reference's own known answers (tests/test_mgf.cpp), number-grammar corner cases, unsorted / duplicate
peaks, and a few thousand random mutations of a valid file."""
import numpy as np
import pytest

from oracle.binding import OracleError, SynthCfg
from tests import _mgf_cases as M

pytestmark = pytest.mark.gpu


def _both(ctx, oracle, text, prefix="DECOY_"):
    try:
        want = ("ok", oracle.mgf_parse(text, prefix))
    except OracleError as e:
        want = ("err", str(e))
    import paper_2211_16422_b200 as hb
    try:
        got = ("ok", ctx.parse_mgf(text, prefix))
    except hb.ParseError as e:
        got = ("err", "ParseError: " + str(e))
    return got, want


def _assert_same(got, want, text):
    assert got[0] == want[0], (text[:400], got[1] if got[0] == "err" else "", want[1] if want[0] == "err" else "")
    if got[0] == "err":
        assert got[1] == want[1], text[:400]
    else:
        g = {k: got[1][k] for k in want[1]}
        assert M.same(want[1], g), text[:400]


def test_reference_known_answers(hb, ctx, best_oracle):
    """tests/test_mgf.cpp:22-131."""
    r = ctx.parse_mgf(b"BEGIN IONS\nTITLE=run1.scan42\nPEPMASS=500.25\nCHARGE=2+\n100.0 5.0\n200.5 7.25\nEND IONS\n")
    assert r["ids"] == [b"run1.scan42"] and r["precursor_mz"][0] == 500.25 and r["charge"][0] == 2
    assert not r["is_decoy"][0] and list(r["mz"]) == [100.0, 200.5] and list(r["intensity"]) == [5.0, 7.25]
    assert ctx.parse_mgf(b"BEGIN IONS\nPEPMASS=500\nCHARGE=+3\n100 1\nEND IONS\n")["charge"][0] == 3
    assert ctx.parse_mgf(b"BEGIN IONS\nPEPMASS=500\nCHARGE=4\n100 1\nEND IONS\n")["charge"][0] == 4
    assert ctx.parse_mgf(b"BEGIN IONS\nPEPMASS=500\n100 1\nEND IONS\n")["charge"][0] == 0
    assert ctx.parse_mgf(b"BEGIN IONS\nTITLE=DECOY_sp|P1|PEP\nPEPMASS=500\n100 1\nEND IONS\n")["is_decoy"][0]
    r = ctx.parse_mgf(b"BEGIN IONS\nTITLE=x\nSEQ=DECOY_PEPTIDE\nPEPMASS=500\n100 1\nEND IONS\n")
    assert r["is_decoy"][0] and r["peptides"] == [b"DECOY_PEPTIDE"]
    assert not ctx.parse_mgf(b"BEGIN IONS\nTITLE=DECOY_x\nPEPMASS=500\n100 1\nEND IONS\n", "XXX_")["is_decoy"][0]
    r = ctx.parse_mgf(b"BEGIN IONS\nPEPMASS=500\n100.0 5.0\n100.0 3.0\n99.5 1.0\nEND IONS\n")
    assert list(r["mz"]) == [99.5, 100.0] and list(r["intensity"]) == [1.0, 8.0]
    assert ctx.parse_mgf(b"")["n_spectra"] == 0 and ctx.parse_mgf(b"\n\n  \n# comment\n")["n_spectra"] == 0
    assert ctx.parse_mgf(b"BEGIN IONS\nPEPMASS=500.25 12345.6\n100 1\nEND IONS\n")["precursor_mz"][0] == 500.25
    r = ctx.parse_mgf(b"BEGIN IONS\nPEPMASS=500\n100.25 7.5 1\nEND IONS\n")
    assert list(r["mz"]) == [100.25] and list(r["intensity"]) == [7.5]
    r = ctx.parse_mgf(b"BEGIN IONS\nPEPMASS=500\n100 1\nEND IONS\nBEGIN IONS\nPEPMASS=600\n100 1\nEND IONS\n")
    assert r["ids"] == [b"spectrum_1", b"spectrum_2"]
    assert ctx.parse_mgf(b"MASS=Monoisotopic\nBEGIN IONS\nPEPMASS=500\n100 1\nEND IONS\n")["n_spectra"] == 1
    for text, line in ((b"BEGIN IONS\nTITLE=x\n100 1\nEND IONS\n", 1), (b"BEGIN IONS\nPEPMASS=500\n100 abc\nEND IONS\n", 3),
                       (b"BEGIN IONS\nPEPMASS=500\n100\nEND IONS\n", 3), (b"BEGIN IONS\nPEPMASS=0\n100 1\nEND IONS\n", 2),
                       (b"BEGIN IONS\nPEPMASS=500\nCHARGE=two\n100 1\nEND IONS\n", 3),
                       (b"BEGIN IONS\nPEPMASS=500\n-5 1\nEND IONS\n", 3), (b"BEGIN IONS\nPEPMASS=500\n100 -1\nEND IONS\n", 3),
                       (b"100 1\n", 1), (b"BEGIN IONS\nPEPMASS=500\nBEGIN IONS\nEND IONS\n", 3),
                       (b"BEGIN IONS\nPEPMASS=500\n100 1\n", 1), (b"END IONS\n", 1)):
        with pytest.raises(hb.ParseError) as e:
            ctx.parse_mgf(text)
        assert e.value.line == line, text
        _assert_same(*_both(ctx, best_oracle, text), text)


def test_number_grammar_and_exact_rounding(hb, ctx, best_oracle):
    """Every token of the corner-case list as m/z, as intensity and as PEPMASS: from_chars grammar,
    halfway cases that need the exact path, overflow / underflow, inf / nan."""
    hard = 0
    for t in M.TOKS + [b"0." + b"0" * 400 + b"1", b"1" + b"0" * 300, b"4.940656458412465441765687928682213723651e-324",
                       b"2.4703282292062327208828439643411068618e-324", b"2.4703282292062327208828439643411068619e-324",
                       b"0.500000000000000166533453693773481063544750213623046875",
                       b"9007199254740992.5", b"9007199254740993.5", b"1e23", b"8.5e-5", b"1.7976931348623157e308",
                       b"123456789.123456789e-30", b"-1e-5", b"1E5", b"1e+05", b"00012.500", b"1" * 900, b"0." + b"3" * 900]:
        for text in (b"BEGIN IONS\nPEPMASS=500\n" + t + b" 1\nEND IONS\n", b"BEGIN IONS\nPEPMASS=500\n5 " + t + b"\nEND IONS\n",
                     b"BEGIN IONS\nPEPMASS=" + t + b"\n5 1\nEND IONS\n", b"BEGIN IONS\nPEPMASS=1\nPEPMASS=" + t + b"\nPEPMASS=2\n5 1\nEND IONS\n"):
            got, want = _both(ctx, best_oracle, text)
            _assert_same(got, want, text)
    r = ctx.parse_mgf(b"BEGIN IONS\nPEPMASS=1e23\n0.1234567890123456789012345 1.00000000000000011102230246251565404236316680908203125\nEND IONS\n")
    assert r["n_hard_numbers"] == 2  # one peak line + one PEPMASS line went through the exact path


def test_structure_and_finalize(hb, ctx, best_oracle):
    rng = np.random.default_rng(3)
    blocks = []
    for b in range(300):  # unsorted peaks with duplicates, blank lines, CRLF, headers after peaks, repeated keys
        n = int(rng.integers(0, 90))
        grid = rng.integers(1000, 1400, n) / 10.0 if b % 3 else rng.integers(100000, 1300000, n) / 1000.0
        lines = [b"BEGIN IONS", b"PEPMASS=%d.%d" % (400 + b, b % 7)]
        if b % 4:
            lines.append(b"TITLE= t%d  " % b)
        if b % 5 == 0:
            lines.append(b"CHARGE=%d+" % (1 + b % 6))
        for j in range(n):
            lines.append(b"%.4f\t%.3f" % (grid[j], rng.random() * 100))
            if j % 17 == 0:
                lines.append(b"  ")
        if b % 6 == 0:
            lines += [b"SEQ=PEPTIDE%d" % b, b"PEPMASS=%d.25" % (700 + b), b"RTINSECONDS=12.5"]
        lines.append(b"END IONS")
        blocks.append((b"\r\n" if b % 2 else b"\n").join(lines))
    text = b"# header\nCOM=x\n\n" + b"\n\n".join(blocks) + b"\n"
    got, want = _both(ctx, best_oracle, text)
    assert want[0] == "ok" and want[1]["offsets"][-1] < sum(1 for _ in text.split(b"\n"))
    _assert_same(got, want, text)
    _assert_same(*_both(ctx, best_oracle, text.rstrip(b"\n")), text)  # no trailing newline
    # an error inside the block that is still open when a structural error / EOF stops the parser
    for tail in (b"BEGIN IONS\nPEPMASS=x\n5 1\n", b"BEGIN IONS\nPEPMASS=5\nCHARGE=0\nBEGIN IONS\n", b"BEGIN IONS\n5 1\nfoo\n",
                 b"BEGIN IONS\nPEPMASS=5\n5 1\nEND IONS\nEND IONS\n5 x\n", b"BEGIN IONS\nTITLE=a\n"):
        _assert_same(*_both(ctx, best_oracle, text + tail), tail)


def test_fuzz_against_oracle(hb, ctx, best_oracle):
    base = M.base_text(best_oracle)
    rng = np.random.default_rng(1)
    n_ok = n_err = 0
    for _ in range(3000):
        text = M.mutate(rng, base)
        got, want = _both(ctx, best_oracle, text)
        _assert_same(got, want, text)
        n_ok += want[0] == "ok"
        n_err += want[0] == "err"
    assert n_ok > 300 and n_err > 300


def test_write_then_parse_fixpoint_and_resident_encode(hb, ctx, best_oracle):
    """test_mgf.cpp:133-160 through the device parser; then the resident CSR feeds the encoder without
    a host round trip and gives the hypervectors of the host path."""
    import torch
    s = best_oracle.synth(SynthCfg(n_library=400, n_query=0, peaks_per_spectrum=60, seed=5))["library"]
    text = best_oracle.mgf_write(s["offsets"], s["mz"], s["intensity"], s["precursor_mz"], s["charge"], s["ids"])
    r = ctx.parse_mgf(text)
    assert [i.decode() for i in r["ids"]] == list(s["ids"]) and np.array_equal(r["charge"], s["charge"])
    assert np.array_equal(r["is_decoy"], s["is_decoy"]) and np.array_equal(r["offsets"], s["offsets"])
    again = best_oracle.mgf_write(r["offsets"], r["mz"], r["intensity"], r["precursor_mz"], r["charge"], r["ids"])
    assert again == text
    pre = hb.PreprocessConfig()
    dim = 1024
    ctx.upload_codebook(hb.make_codebook(hb.dimension(pre), hb.EncoderConfig(dim, dim // 2, 16, 1)))
    want, ok = ctx.encode_batch(r["offsets"], r["mz"], r["intensity"], pre)
    csr = ctx.mgf_device_csr()
    n = csr["n_spectra"]
    out = torch.empty((n, dim // 64), dtype=torch.int64, device="cuda:0")
    okd = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    ctx.encode_batch_dev(pre, n, csr["n_peaks"], csr["d_offsets"], csr["d_mz"], csr["d_intensity"], out.data_ptr(),
                         okd.data_ptr())
    ctx.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want) and np.array_equal(okd.cpu().numpy(), ok)


def test_golden_mgf_cases(hb, ctx):
    """The committed fixture generated from the compiled reference (tests/golden/make_golden.py)."""
    from tests import _util as U
    for text, want in U.mgf_cases():
        if isinstance(want, str):
            with pytest.raises(hb.ParseError) as e:
                ctx.parse_mgf(text)
            assert "ParseError: " + str(e.value) == want, text[:200]
        else:
            got = ctx.parse_mgf(text)
            assert M.same(want, {k: got[k] for k in want}), text[:200]
