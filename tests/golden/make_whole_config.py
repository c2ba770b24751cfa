"""Golden fingerprints of BASELINE configs 2 and 3 at FULL size, computed from the reference itself
(oracle/_ref: the unmodified sources of /root/reference compiled in place; the -march=x86-64-v3 flavour,
built with -ffp-contract=off, for speed).  CPU only; minutes to tens of minutes.

    python tests/golden/make_whole_config.py config2 [config3]

Writes the `whole_config` section of tests/golden/fingerprints.json: FNV-1a-64 (cache.cpp:18-29) of the
generator's output, of the encoded hypervectors, of the open top-1 (score, ordinal) arrays and of the
cascade's accepted list, plus the accepted counts.  tests/test_whole_config_gpu.py checks the CUDA path
against these AND against the live reference; bench.py checks its result digest against `bench_result_digest`.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import binding as ob  # noqa: E402
from tests._util import fnv_hex  # noqa: E402
import workload as wl  # noqa: E402

CONFIGS = {
    # name: (workload, queries of the prefix searched on the CPU -- None = all)
    "config2": ("iprg2012", None),
    "config3": ("hek293_full", 2048),
}


def fnv(a) -> str:
    return "%016x" % ob.fnv1a64_words(np.ascontiguousarray(a).view(np.uint8).view("<u8") if a.dtype != np.uint64 else a)


def pad8(a: np.ndarray) -> np.ndarray:
    """bytes of an array, zero-padded to a multiple of 8, as u64 words (for arrays of u32 / u8)."""
    b = np.ascontiguousarray(a).view(np.uint8).ravel()
    if len(b) % 8:
        b = np.concatenate([b, np.zeros(8 - len(b) % 8, np.uint8)])
    return b.view("<u8")


def run(name: str) -> dict:
    workload, prefix = CONFIGS[name]
    cores = os.cpu_count() or 1
    t = time.time()
    lib, qry, dim, gen = wl.make(workload, "reference")
    assert gen == "reference"
    out = {"workload": workload, "dim": dim, "library": len(lib["precursor_mz"]), "queries": len(qry["precursor_mz"]),
           "synth_library_mz_fnv": fnv(lib["mz"].view(np.uint64)), "synth_query_mz_fnv": fnv(qry["mz"].view(np.uint64)),
           "synth_library_precursor_fnv": fnv(lib["precursor_mz"].view(np.uint64)),
           "synth_query_precursor_fnv": fnv(qry["precursor_mz"].view(np.uint64))}
    print(f"[{name}] generated in {time.time() - t:.0f}s", flush=True)
    o = ob.Oracle("ref_v3" if ob.available("ref_v3") else "ref")
    pre = ob.PreCfg()
    cb = o.make_codebook(dim, dim // 2, 16, 1, o.dimension(pre))
    t = time.time()
    lw, lok = o.encode_spectra(cb, pre, lib["offsets"], lib["mz"], lib["intensity"], threads=cores, batch=64)
    qw, qok = o.encode_spectra(cb, pre, qry["offsets"], qry["mz"], qry["intensity"], threads=cores, batch=64)
    print(f"[{name}] encoded in {time.time() - t:.0f}s", flush=True)
    out.update(library_encoded=int(lok.sum()), queries_encoded=int(qok.sum()),
               library_hv_fnv=fnv(lw), query_hv_fnv=fnv(qw))
    assert lok.all() and qok.all()
    ix = o.build_index(dim, lw, lib["precursor_mz"], lib["charge"], lib["is_decoy"], lib["ids"])
    n = len(qok) if prefix is None else prefix
    out["searched_queries"] = n
    t = time.time()
    has, score, ordinal, _ = ix.search_batch(qw[:n], qry["precursor_mz"][:n], qry["charge"][:n], ("da", 500.0),
                                             threads=cores, batch=8)
    print(f"[{name}] open search of {n} queries in {time.time() - t:.0f}s", flush=True)
    first, last, _ = ix.select_candidates(qry["precursor_mz"][:n], qry["charge"][:n], ("da", 500.0))
    out.update(open_hits=int(has.sum()), open_candidates_total=int((last - first).sum()),
               open_score_fnv=fnv(pad8(score)), open_ordinal_fnv=fnv(pad8(ordinal)))
    t = time.time()
    c = ix.cascade_search(qw[:n], qry["precursor_mz"][:n], qry["charge"][:n], ("ppm", 20.0), ("da", 500.0), 0.01,
                          threads=cores, batch=8)
    print(f"[{name}] cascade of {n} queries in {time.time() - t:.0f}s", flush=True)
    out.update(cascade_accepted=int(len(c["query"])), cascade_narrow=int((c["stage"] == 0).sum()),
               cascade_wide=int((c["stage"] == 1).sum()), cascade_query_fnv=fnv(c["query"].astype("<u8")),
               cascade_ordinal_fnv=fnv(pad8(c["ordinal"])), cascade_score_fnv=fnv(pad8(c["raw_score"])),
               cascade_qvalue_fnv=fnv(c["q_value"].view(np.uint64)))
    if prefix is None:  # what bench.py's result_digest must equal on this workload (sha256 of ordinal + score bytes)
        digest = hashlib.sha256(np.where(has.astype(bool), ordinal, 0xFFFFFFFF).astype(np.uint32).reshape(-1, 1).tobytes() +
                                np.where(has.astype(bool), score, 0).astype(np.uint32).reshape(-1, 1).tobytes()).hexdigest()[:16]
        out["bench_result_digest"] = {f"{workload}/reference/D{dim}/da500/k1": digest}
    ix.close()
    return out


def main():
    path = os.path.join(HERE, "fingerprints.json")
    with open(path) as f:
        fp = json.load(f)
    for name in sys.argv[1:] or ["config2"]:
        res = run(name)
        fp.setdefault("bench_result_digest", {}).update(res.pop("bench_result_digest", {}))
        fp.setdefault("whole_config", {})[name] = res
        with open(path, "w") as f:
            json.dump(fp, f, indent=1, sort_keys=True)
            f.write("\n")
        print(json.dumps(res, indent=1), flush=True)


if __name__ == "__main__":
    main()
