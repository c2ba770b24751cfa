#!/usr/bin/env python
"""Hottest SASS instructions of a kernel by warp-stall samples, from `ncu -i X.ncu-rep --page source --csv`.

Used to find where the single-thread roles of tc_search_kernel spend their time (DESIGN.md 4 K4a: the MMA thread of
round 1 was issuing, not waiting).  Prints every instruction with at least `min_pct` percent of the samples and the
sample totals of the regions between the marker instructions (UBLKCP = producer, UTCOMMA = MMA thread, LDTM = drain).

    python tools/ncu_source_hot.py source.csv [min_pct]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    min_pct = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
    head = next(r for r in rows if "Source" in r and "# Samples" in r)
    i_src, i_n = head.index("Source"), head.index("# Samples")
    data = []
    for r in rows[rows.index(head) + 1:]:
        try:
            data.append((int(r[i_n]), r[i_src]))
        except (ValueError, IndexError):
            data.append((0, r[i_src] if len(r) > i_src else ""))
    total = sum(n for n, _ in data)
    print(f"total samples {total}, {len(data)} instructions")
    marks = {k: [i for i, (_, s) in enumerate(data) if k in s] for k in ("UBLKCP", "LDTM", "UTCOMMA")}
    print("markers:", {k: (v[0], v[-1]) if v else None for k, v in marks.items()})
    for i, (n, s) in enumerate(data):
        if total and 100.0 * n / total >= min_pct:
            print(f"{i:6d} {n:8d} {100.0 * n / total:5.1f}%  {s[:110]}")


if __name__ == "__main__":
    main()
