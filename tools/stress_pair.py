#!/usr/bin/env python
"""Stress of the CTA-pair hand-offs (development aid): many searches with the shortest possible work items, so that
the cross-CTA item FIFO, the stage relay and the accumulator hand-back turn over as often as they can; every run
must reproduce the first one bit for bit, and the first one the single-CTA form's answer.

    HOMS_B200_TC_MAX_STRIP=1 HOMS_B200_TC_ITEMS_PER_SM=100000 python tools/stress_pair.py [--runs 300]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=300)
    ap.add_argument("--dims", default="2048,8192")
    args = ap.parse_args()
    import paper_2211_16422_b200 as hb
    from tests import _util as U

    rng = np.random.default_rng(5)
    for dim in [int(x) for x in args.dims.split(",")]:
        n, nq = 60000, 3000
        words = U.random_hvs(rng, n, dim)
        mz = np.round(rng.uniform(400.0, 1400.0, n), 3)
        charge = rng.integers(2, 4, n).astype(np.uint8)
        qw = U.random_hvs(rng, nq, dim)
        qw[:500] = words[rng.integers(0, n, 500)]
        qmz = np.round(rng.uniform(380.0, 1420.0, nq), 3)
        qch = rng.integers(2, 4, nq).astype(np.uint8)
        tol = hb.Tolerance("dalton", 500.0)
        ref = {}
        for pair in ("0", "1"):
            os.environ["HOMS_B200_TC_PAIR"] = pair
            with hb.Context(0) as c:
                c.set_engine("tensor_fp4")
                c.build_index(dim, words, mz, charge)
                runs = args.runs if pair == "1" else 3
                for k in (1, 8):
                    first = None
                    for i in range(runs):
                        m = c.search_batch(qw, qmz, qch, tol, k=k)
                        got = (m.ordinal.copy(), m.raw_score.copy())
                        if first is None:
                            first = got
                        assert np.array_equal(got[0], first[0]) and np.array_equal(got[1], first[1]), (dim, pair, k, i)
                    if pair == "0":
                        ref[k] = first
                    else:
                        assert np.array_equal(first[0], ref[k][0]) and np.array_equal(first[1], ref[k][1]), (dim, k)
                print(f"D={dim} pair={pair} pairs_active={c.tensor_cta_pairs()}: {runs} runs x k in (1, 8) identical", flush=True)
    print("stress ok")


if __name__ == "__main__":
    main()
