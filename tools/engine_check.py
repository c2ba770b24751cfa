#!/usr/bin/env python
"""Development check (GPU): the tensor engine against the POPC engine on random hypervectors,
including clone / mirror rows that force score ties.  Prints one line per case; exit code 1 on the
first mismatch.  The pytest suite holds the real parity tests; this is the fast loop."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2211_16422_b200 as hb  # noqa: E402


ENGINES = ("popc", "direct", "tensor_fp4")


def random_hvs(rng, n, dim):
    W = (dim + 63) // 64
    w = rng.integers(0, 2**64, (n, W), dtype=np.uint64)
    if dim % 64:
        w[:, -1] &= np.uint64((1 << (dim % 64)) - 1)
    return w


def case(name, dim, n_lib, nq, tol, seed, clones=0):
    rng = np.random.default_rng(seed)
    lw = random_hvs(rng, n_lib, dim)
    mz = rng.uniform(380.0, 1070.0, n_lib)
    ch = rng.integers(2, 4, n_lib).astype(np.uint8)
    src = rng.integers(0, n_lib, nq)
    qw = lw[src].copy()
    flips = rng.integers(0, 2**64, qw.shape, dtype=np.uint64) & rng.integers(0, 2**64, qw.shape, dtype=np.uint64) \
        & rng.integers(0, 2**64, qw.shape, dtype=np.uint64)
    qw ^= flips
    if dim % 64:
        qw[:, -1] &= np.uint64((1 << (dim % 64)) - 1)
    qmz = mz[src] + rng.choice([0.0, 0.001, 79.97, -15.99], nq)
    qch = ch[src].copy()
    if nq > 3:
        qch[0] = 0
        qch[1] = 7
    for i in range(clones):  # identical hypervectors at mirrored / equal precursor offsets
        a = int(rng.integers(0, n_lib))
        b = int(rng.integers(0, n_lib))
        lw[b] = lw[a]
        ch[b] = ch[a]
        mz[b] = mz[a] if i % 2 else 2 * qmz[i % nq] - mz[a]
    ids = [f"lib{(i * 7919) % n_lib:07d}" for i in range(n_lib)]
    out = {}
    for eng in ENGINES:
        with hb.Context(0) as ctx:
            ctx.set_engine(eng)
            ctx.build_index(dim, lw, mz, ch, ids=ids)
            t = time.time()
            m = ctx.search_batch(qw, qmz, qch, tol)
            dt = time.time() - t
            out[eng] = (m.raw_score.copy(), m.ordinal.copy(), dt)
    all_ok = True
    for eng in ENGINES[1:]:
        ok = np.array_equal(out["popc"][0], out[eng][0]) and np.array_equal(out["popc"][1], out[eng][1])
        nbad = int(((out["popc"][1] != out[eng][1]) | (out["popc"][0] != out[eng][0])).sum())
        print(f"{name:22s} dim={dim:5d} lib={n_lib:7d} nq={nq:6d} tol={tol.kind}:{tol.value:g} "
              f"hits={int((out['popc'][1] != 0xFFFFFFFF).sum()):6d} popc={out['popc'][2]*1e3:8.1f}ms "
              f"{eng}={out[eng][2]*1e3:8.1f}ms {'OK' if ok else 'MISMATCH ' + str(nbad)}", flush=True)
        if not ok:
            bad = np.flatnonzero((out["popc"][1] != out[eng][1]).ravel() | (out["popc"][0] != out[eng][0]).ravel())[:8]
            for i in bad:
                print("   q", i, "popc", out["popc"][0].ravel()[i], out["popc"][1].ravel()[i], eng,
                      out[eng][0].ravel()[i], out[eng][1].ravel()[i])
        all_ok &= ok
    return all_ok


def main():
    T = hb.Tolerance
    ok = True
    ok &= case("tiny", 128, 300, 5, T("dalton", 500.0), 1)
    ok &= case("one-tile", 1024, 2000, 128, T("dalton", 500.0), 2)
    ok &= case("ragged", 2048, 10_000, 1000, T("dalton", 500.0), 3, clones=40)
    ok &= case("narrow ppm", 2048, 10_000, 1000, T("ppm", 20.0), 4, clones=40)
    ok &= case("narrow da", 2048, 50_000, 3000, T("dalton", 1.0), 5, clones=100)
    ok &= case("dim 64", 64, 5000, 700, T("dalton", 30.0), 6, clones=20)
    ok &= case("dim 192 (pad K)", 192, 5000, 700, T("dalton", 30.0), 7, clones=20)
    ok &= case("dim 100 (tail bits)", 100, 3000, 300, T("dalton", 50.0), 8, clones=20)
    ok &= case("D8192", 8192, 100_000, 4000, T("dalton", 500.0), 9, clones=50)
    ok &= case("D16384", 16384, 20_000, 1500, T("dalton", 500.0), 10, clones=10)
    print("ALL OK" if ok else "FAILED")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
