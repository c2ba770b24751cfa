"""Generates the committed golden fixtures FROM THE UNMODIFIED REFERENCE.

Run in the build container (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

Every expected value below is produced by calling the reference's own functions through
oracle/_ref/libhoms_ref.so (oracle/ref_shim.cpp); nothing is computed by this repository's code.
The fixtures travel to the GPU box, /root/reference does not.

Outputs (tests/golden/):
  fingerprints.json   codebook / config-1 FNV-1a fingerprints and counts
  encode_cases.npz    spectra -> (ok, hypervector words, bins, levels) for several configs
  search_cases.npz    small libraries with clones / mirror pairs -> windows, top-1, cascade
  cache_small.homs    a cache file written by the reference's write_cache (+ cache_small.npz: its entries)
  mgf_cases.json      MGF texts (hex) -> the reference's parse_mgf result (doubles as u64 bit patterns) or
                      its ParseError text: test_mgf.cpp's cases, number-grammar corner cases, random mutations
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.binding import EncCfg, Oracle, PreCfg, SynthCfg, fnv1a64_words, words_for  # noqa: E402


def csr(spectra):
    offsets = np.zeros(len(spectra) + 1, np.uint64)
    offsets[1:] = np.cumsum([len(s[0]) for s in spectra])
    mz = np.concatenate([np.asarray(s[0], np.float64) for s in spectra]) if spectra else np.zeros(0)
    it = np.concatenate([np.asarray(s[1], np.float64) for s in spectra]) if spectra else np.zeros(0)
    return offsets, mz, it


def random_spectra(rng, n, lo_peaks, hi_peaks, mz_lo=90.0, mz_hi=1600.0, grid=None):
    out = []
    for _ in range(n):
        p = int(rng.integers(lo_peaks, hi_peaks + 1))
        if grid:
            idx = np.sort(rng.choice(np.arange(int(mz_lo / grid), int(mz_hi / grid)), p, replace=False))
            mz = idx.astype(np.float64) * grid
        else:
            mz = np.unique(rng.uniform(mz_lo, mz_hi, p))
        inten = rng.uniform(0.0, 1.0, len(mz))
        # sprinkle exact zeros, ties and tiny values to hit the floor / top-N tie rules
        if len(mz) > 4:
            inten[rng.integers(0, len(mz))] = 0.0
            j = rng.integers(0, len(mz), 3)
            inten[j] = inten[j[0]]
            inten[rng.integers(0, len(mz))] *= 0.009
        out.append((mz, inten))
    return out


def encode_cases(ref: Oracle):
    rng = np.random.default_rng(20240601)
    cases = {}
    configs = [
        # name, PreCfg kwargs, (dim, flips, levels, seed), n spectra, peaks range, grid
        ("default_d2048", dict(), (2048, 1024, 16, 1), 96, (0, 120), 0.01),
        ("sqrt_d256", dict(scaling=1, max_peaks=30, min_peaks=3), (256, 128, 16, 5), 64, (0, 80), None),
        ("coarse_d128", dict(min_mz=100.0, max_mz=600.0, bin_size=1.0005, max_peaks=20, min_peaks=1,
                             intensity_floor=0.05), (128, 16, 4, 12), 64, (0, 60), None),
        ("wide_d8192", dict(max_peaks=150, min_peaks=10), (8192, 4096, 16, 1), 24, (100, 220), 0.01),
        ("tiny_d64", dict(min_mz=100.0, max_mz=200.0, bin_size=0.5, max_peaks=300, min_peaks=1,
                          intensity_floor=0.0), (64, 7, 31, 3), 32, (1, 400), None),
    ]
    for name, pk, (dim, flips, levels, seed), n, (plo, phi), grid in configs:
        cfg = PreCfg(**pk)
        spectra = random_spectra(rng, n, plo, phi, mz_lo=cfg.min_mz - 10, mz_hi=cfg.max_mz + 20, grid=grid)
        # hand-made edge spectra: empty, all filtered, boundary m/z values, colliding peaks
        spectra.append((np.zeros(0), np.zeros(0)))
        spectra.append((np.array([cfg.min_mz - 1.0, cfg.max_mz]), np.array([1.0, 1.0])))
        edge_mz = np.array([cfg.min_mz, cfg.min_mz + cfg.bin_size * 0.98, cfg.min_mz + cfg.bin_size,
                            cfg.min_mz + 3 * cfg.bin_size, np.nextafter(cfg.max_mz, 0)])
        spectra.append((edge_mz, np.array([1.0, 1.0, 1.0, 0.01, 0.0100001])))
        offsets, mz, it = csr(spectra)
        n_bins = ref.dimension(cfg)
        cb = ref.make_codebook(dim, flips, levels, seed, n_bins)
        words, ok = ref.encode_spectra(cb, cfg, offsets, mz, it, threads=2, batch=7)
        bins_flat, lev_flat, sv_off = [], [], [0]
        for i in range(len(spectra)):
            a, b = int(offsets[i]), int(offsets[i + 1])
            r = ref.refine_vectorize(cfg, mz[a:b], it[a:b], levels)
            if r is not None:
                bins_flat.append(r[0])
                lev_flat.append(r[2])
                sv_off.append(sv_off[-1] + len(r[0]))
            else:
                sv_off.append(sv_off[-1])
        cases[name] = dict(
            precfg=np.array([cfg.min_mz, cfg.max_mz, cfg.bin_size, cfg.max_peaks, cfg.min_peaks,
                             cfg.intensity_floor, cfg.scaling], np.float64),
            enccfg=np.array([dim, flips, levels, seed], np.uint64),
            offsets=offsets, mz=mz, intensity=it, ok=ok, words=words,
            sv_offsets=np.array(sv_off, np.uint64),
            sv_bins=np.concatenate(bins_flat) if bins_flat else np.zeros(0, np.uint32),
            sv_levels=np.concatenate(lev_flat) if lev_flat else np.zeros(0, np.uint32),
            codebook_fnv=np.array([fnv1a64_words(cb.pos), fnv1a64_words(cb.lvl)], np.uint64),
        )
        ref.free_codebook(cb)
    flat = {}
    for name, d in cases.items():
        for k, v in d.items():
            flat[f"{name}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "encode_cases.npz"), **flat)
    return {k: int(v["ok"].sum()) for k, v in cases.items()}


def search_cases(ref: Oracle):
    rng = np.random.default_rng(777)
    flat = {}
    summary = {}
    for name, dim, n, nq in (("d256", 256, 600, 160), ("d64", 64, 200, 80), ("d1088", 1088, 300, 60)):
        W = words_for(dim)
        words = rng.integers(0, 2**64, (n, W), dtype=np.uint64)
        if dim % 64:
            words[:, -1] &= np.uint64((1 << (dim % 64)) - 1)
        mz = rng.uniform(400.0, 1200.0, n)
        charge = rng.integers(2, 4, n).astype(np.uint8)
        charge[rng.integers(0, n, 5)] = 0  # unknown-charge entries are parked
        decoy = (rng.uniform(0, 1, n) < 0.3).astype(np.uint8)
        ids = [f"ref_{i}" for i in range(n)]
        # clones: identical hypervector + precursor, different id  (acceptance_main.cpp:219-233)
        n_clone = 25
        src = rng.integers(0, n, n_clone)
        words = np.concatenate([words, words[src]])
        mz = np.concatenate([mz, mz[src]])
        charge = np.concatenate([charge, charge[src]])
        decoy = np.concatenate([decoy, decoy[src]])
        ids += [f"clone_{i}" for i in range(n_clone)]
        # mirror pairs: same hypervector at q -/+ delta with exactly representable delta
        n_mirror = 12
        centers = np.round(rng.uniform(500.0, 1100.0, n_mirror))
        mw = rng.integers(0, 2**64, (n_mirror, W), dtype=np.uint64)
        if dim % 64:
            mw[:, -1] &= np.uint64((1 << (dim % 64)) - 1)
        words = np.concatenate([words, mw, mw])
        mz = np.concatenate([mz, centers - 0.25, centers + 0.25])
        charge = np.concatenate([charge, np.full(2 * n_mirror, 2, np.uint8)])
        decoy = np.concatenate([decoy, np.zeros(2 * n_mirror, np.uint8)])
        ids += [f"zz_{i}" for i in range(n_mirror)] + [f"aa_{i}" for i in range(n_mirror)]
        # duplicate ids with identical precursor and vector: ordinal decides
        words = np.concatenate([words, words[:3], words[:3]])
        mz = np.concatenate([mz, mz[:3], mz[:3]])
        charge = np.concatenate([charge, charge[:3], charge[:3]])
        decoy = np.concatenate([decoy, [0, 0, 0, 1, 1, 1]]).astype(np.uint8)
        ids += ["dup0", "dup1", "dup2", "dup0", "dup1", "dup2"]
        nlib = len(mz)

        # queries: a third are library entries themselves, mirrors' centres, the rest random
        qw = rng.integers(0, 2**64, (nq, W), dtype=np.uint64)
        if dim % 64:
            qw[:, -1] &= np.uint64((1 << (dim % 64)) - 1)
        qmz = rng.uniform(400.0, 1200.0, nq)
        qch = rng.integers(2, 5, nq).astype(np.uint8)  # charge 4 has no bucket
        pick = rng.integers(0, nlib, nq // 3)
        qw[: nq // 3] = words[pick]
        qmz[: nq // 3] = mz[pick]
        qch[: nq // 3] = charge[pick]
        for j in range(n_mirror):
            qw[nq // 3 + j] = mw[j]
            qmz[nq // 3 + j] = centers[j]
            qch[nq // 3 + j] = 2
        qch[-3:] = 0  # unknown-charge queries

        ix = ref.build_index(dim, words, mz, charge, decoy, ids)
        flat.update({f"{name}/dim": np.array([dim]), f"{name}/words": words, f"{name}/mz": mz,
                     f"{name}/charge": charge, f"{name}/decoy": decoy,
                     f"{name}/ids": np.array(ids, dtype="S"), f"{name}/q_words": qw,
                     f"{name}/q_mz": qmz, f"{name}/q_charge": qch})
        for bi, b in enumerate(ix.buckets()):
            flat[f"{name}/bucket{bi}/charge"] = np.array([b["charge"]], np.uint8)
            flat[f"{name}/bucket{bi}/ordinal"] = b["ordinal"]
        for tname, tol in (("ppm150", ("ppm", 150.0)), ("da30", ("da", 30.0)), ("da500", ("da", 500.0)),
                           ("da1", ("da", 1.0)), ("ppm20", ("ppm", 20.0))):
            first, last, has_b = ix.select_candidates(qmz, qch, tol)
            has, score, ordinal, _ = ix.search_batch(qw, qmz, qch, tol, threads=3, batch=17)
            lin = ix.search_batch(qw, qmz, qch, tol, linear=True)
            # the reference's own property: indexed == exhaustive (test_search.cpp:245-278); the
            # test oracle breaks full ties by id only, so compare on (has, score, id)
            assert np.array_equal(has, lin[0]) and np.array_equal(score, lin[1])
            flat.update({f"{name}/{tname}/first": first, f"{name}/{tname}/last": last,
                         f"{name}/{tname}/has_bucket": has_b, f"{name}/{tname}/has": has,
                         f"{name}/{tname}/score": score, f"{name}/{tname}/ordinal": ordinal})
            summary[f"{name}/{tname}"] = int(has.sum())
        for cname, narrow, wide, fq in (("c1", ("ppm", 150.0), ("da", 30.0), 0.05),
                                        ("c2", ("da", 0.3), ("da", 500.0), 0.5)):
            c = ix.cascade_search(qw, qmz, qch, narrow, wide, fq, threads=2, batch=5)
            for k, v in c.items():
                flat[f"{name}/{cname}/{k}"] = v
            summary[f"{name}/{cname}"] = int(len(c["query"]))
        ix.close()
    np.savez_compressed(os.path.join(HERE, "search_cases.npz"), **flat)
    return summary


def fingerprints(ref: Oracle):
    out = {"codebook": {}, "note": "FNV-1a-64 exactly as reference cache.cpp:18-29 (state seeded with "
                                   "1469598103934665603) over little-endian u64 words"}
    cfg = PreCfg()
    n_bins = ref.dimension(cfg)
    for dim in (1024, 2048, 4096, 8192, 16384):
        cb = ref.make_codebook(dim, dim // 2, 16, 1, n_bins)
        out["codebook"][str(dim)] = {"position": f"{fnv1a64_words(cb.pos):016x}",
                                     "level": f"{fnv1a64_words(cb.lvl):016x}",
                                     "position0_word0": f"{int(cb.pos[0, 0]):016x}",
                                     "level0_word0": f"{int(cb.lvl[0, 0]):016x}"}
        if dim == 2048:
            cb2048 = cb
        else:
            ref.free_codebook(cb)
    # config 1
    s = ref.synth(SynthCfg(n_library=5000, n_query=1000, peaks_per_spectrum=50, decoy_ratio=1.0,
                           fraction_modified=0.6, precursor_shift_da=79.97,
                           fraction_peaks_shifted=0.3, intensity_noise=0.05, seed=1))
    L, Q = s["library"], s["queries"]
    lw, lok = ref.encode_spectra(cb2048, cfg, L["offsets"], L["mz"], L["intensity"], threads=8)
    qw, qok = ref.encode_spectra(cb2048, cfg, Q["offsets"], Q["mz"], Q["intensity"], threads=8)
    ix = ref.build_index(2048, lw, L["precursor_mz"], L["charge"], L["is_decoy"], L["ids"])
    first, last, _ = ix.select_candidates(Q["precursor_mz"], Q["charge"], ("da", 500.0))
    has, score, ordinal, _ = ix.search_batch(qw, Q["precursor_mz"], Q["charge"], ("da", 500.0), threads=8)
    nar = ix.search_batch(qw, Q["precursor_mz"], Q["charge"], ("ppm", 20.0), threads=8)
    c = ix.cascade_search(qw, Q["precursor_mz"], Q["charge"], ("ppm", 20.0), ("da", 500.0), 0.01, threads=8)
    out["config1"] = {
        "synth_library_mz_fnv": f"{fnv1a64_words(L['mz'].view(np.uint64)):016x}",
        "synth_query_mz_fnv": f"{fnv1a64_words(Q['mz'].view(np.uint64)):016x}",
        "library_encoded": int(lok.sum()), "library_unprocessable": int((lok == 0).sum()),
        "library_hv_fnv": f"{fnv1a64_words(lw):016x}", "query_hv_fnv": f"{fnv1a64_words(qw):016x}",
        "open_candidates_total": int((last - first).sum()), "open_hits": int(has.sum()),
        "open_score_fnv": f"{fnv1a64_words(score.astype(np.uint64)):016x}",
        "open_ordinal_fnv": f"{fnv1a64_words(ordinal.astype(np.uint64)):016x}",
        "narrow_hits": int(nar[0].sum()),
        "narrow_ordinal_fnv": f"{fnv1a64_words(nar[2].astype(np.uint64)):016x}",
        "cascade_accepted": int(len(c["query"])), "cascade_narrow": int((c["stage"] == 0).sum()),
        "cascade_wide": int((c["stage"] == 1).sum()),
        "cascade_ordinal_fnv": f"{fnv1a64_words(c['ordinal'].astype(np.uint64)):016x}",
        "cascade_qvalue_fnv": f"{fnv1a64_words(c['q_value'].view(np.uint64)):016x}",
    }
    ix.close()
    return out


def cache_case(ref: Oracle):
    """A cache file exactly as the reference writes it (cache.cpp:122-156): odd dimension count,
    empty / non-ASCII / long strings, unknown charge, decoys."""
    rng = np.random.default_rng(2211)
    n, dim = 37, 320
    words = rng.integers(0, 2**64, (n, words_for(dim)), dtype=np.uint64)
    mz = np.round(rng.uniform(300.0, 1400.0, n), 4)
    charge = rng.integers(0, 5, n).astype(np.uint8)
    decoy = (rng.uniform(0, 1, n) < 0.4).astype(np.uint8)
    ids = [f"LIB_{i:05d}" if i % 5 else "" for i in range(n)]
    ids[3], ids[4] = "d\u00e9j\u00e0-vu", "x" * 300
    peps = ["PEPTIDEK"[: 1 + i % 8] if i % 3 else "" for i in range(n)]
    pre = PreCfg(min_mz=100.5, max_peaks=64, min_peaks=3, scaling=1)
    enc = EncCfg(dim, 99, 7, 12345)
    image = ref.cache_write(pre, enc, words, mz, charge, decoy, ids, peps)
    back = ref.cache_read(image, pre, enc)
    assert np.array_equal(back["words"], words) and back["ids"] == ids and back["peptides"] == peps
    with open(os.path.join(HERE, "cache_small.homs"), "wb") as f:
        f.write(image)
    np.savez_compressed(os.path.join(HERE, "cache_small.npz"), words=words, mz=mz, charge=charge, decoy=decoy,
                        ids=np.array([x.encode() for x in ids], dtype="S"),
                        peptides=np.array([x.encode() for x in peps], dtype="S"),
                        pre=np.array([100.5, 1500.0, 0.05, 64, 3, 0.01, 1]), enc=np.array([dim, 99, 7, 12345]))
    return dict(bytes=len(image), fnv_of_file=f"{fnv1a64_words(np.frombuffer(image + bytes(-len(image) % 8), np.uint64)):016x}")


def mgf_cases(ref: Oracle):
    from oracle.binding import OracleError
    sys.path.insert(0, os.path.dirname(HERE))
    import _mgf_cases as M
    texts = [b"BEGIN IONS\nTITLE=run1.scan42\nPEPMASS=500.25\nCHARGE=2+\n100.0 5.0\n200.5 7.25\nEND IONS\n",
             b"BEGIN IONS\nPEPMASS=500\nCHARGE=+3\n100 1\nEND IONS\n", b"BEGIN IONS\nPEPMASS=500\n100 1\nEND IONS\n",
             b"BEGIN IONS\nTITLE=x\nSEQ=DECOY_PEPTIDE\nPEPMASS=500\n100 1\nEND IONS\n",
             b"BEGIN IONS\nPEPMASS=500\n100.0 5.0\n100.0 3.0\n99.5 1.0\nEND IONS\n", b"", b"\n\n  \n# comment\n",
             b"BEGIN IONS\nPEPMASS=500.25 12345.6\n100 1\nEND IONS\n", b"BEGIN IONS\nPEPMASS=500\n100.25 7.5 1\nEND IONS\n",
             b"BEGIN IONS\nPEPMASS=500\n100 1\nEND IONS\nBEGIN IONS\nPEPMASS=600\n100 1\nEND IONS\n",
             b"MASS=Monoisotopic\nBEGIN IONS\nPEPMASS=500\n100 1\nEND IONS\n", b"BEGIN IONS\nTITLE=x\n100 1\nEND IONS\n",
             b"BEGIN IONS\nPEPMASS=500\n100 abc\nEND IONS\n", b"BEGIN IONS\nPEPMASS=500\n100\nEND IONS\n",
             b"BEGIN IONS\nPEPMASS=0\n100 1\nEND IONS\n", b"BEGIN IONS\nPEPMASS=500\nCHARGE=two\n100 1\nEND IONS\n",
             b"BEGIN IONS\nPEPMASS=500\n-5 1\nEND IONS\n", b"BEGIN IONS\nPEPMASS=500\n100 -1\nEND IONS\n", b"100 1\n",
             b"BEGIN IONS\nPEPMASS=500\nBEGIN IONS\nEND IONS\n", b"BEGIN IONS\nPEPMASS=500\n100 1\n", b"END IONS\n"]
    for t in M.TOKS:
        texts.append(b"BEGIN IONS\nPEPMASS=" + t + b"\n" + t + b" 1\n5 " + t + b"\nEND IONS\n")
        texts.append(b"BEGIN IONS\nPEPMASS=7\n5 " + t + b"\nEND IONS\n")
        texts.append(b"BEGIN IONS\nPEPMASS=7\n" + t + b" 1\nEND IONS\n")
    base = M.base_text(ref)
    rng = np.random.default_rng(2024)
    texts += [M.mutate(rng, base) for _ in range(120)]
    cases, n_ok = [], 0
    for t in texts:
        try:
            r = ref.mgf_parse(t)
            n_ok += 1
            cases.append(dict(text=t.hex(), ok=True, offsets=r["offsets"].tolist(),
                              mz=r["mz"].view(np.uint64).tolist(), intensity=r["intensity"].view(np.uint64).tolist(),
                              precursor_mz=r["precursor_mz"].view(np.uint64).tolist(), charge=r["charge"].tolist(),
                              is_decoy=r["is_decoy"].tolist(), ids=[i.hex() for i in r["ids"]],
                              peptides=[p.hex() for p in r["peptides"]]))
        except OracleError as e:
            cases.append(dict(text=t.hex(), ok=False, error=str(e)))
    with open(os.path.join(HERE, "mgf_cases.json"), "w") as f:
        json.dump(cases, f)
    return dict(cases=len(cases), parsed=n_ok, errors=len(cases) - n_ok)


def main():
    ref = Oracle("ref")
    if "--mgf-only" in sys.argv:  # adds the MGF fixture without regenerating the others
        with open(os.path.join(HERE, "fingerprints.json")) as f:
            fp = json.load(f)
        fp["mgf_cases"] = mgf_cases(ref)
        with open(os.path.join(HERE, "fingerprints.json"), "w") as f:
            json.dump(fp, f, indent=1, sort_keys=True)
        print(fp["mgf_cases"])
        return
    if "--cache-only" in sys.argv:  # adds the cache fixture without regenerating the others
        with open(os.path.join(HERE, "fingerprints.json")) as f:
            fp = json.load(f)
        fp["cache_small"] = cache_case(ref)
        with open(os.path.join(HERE, "fingerprints.json"), "w") as f:
            json.dump(fp, f, indent=1, sort_keys=True)
        print(fp["cache_small"])
        return
    fp = fingerprints(ref)
    fp["cache_small"] = cache_case(ref)
    fp["mgf_cases"] = mgf_cases(ref)
    fp["encode_cases_ok"] = encode_cases(ref)
    fp["search_cases_hits"] = search_cases(ref)
    with open(os.path.join(HERE, "fingerprints.json"), "w") as f:
        json.dump(fp, f, indent=1, sort_keys=True)
    print(json.dumps(fp, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
