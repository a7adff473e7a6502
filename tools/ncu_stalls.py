#!/usr/bin/env python
"""Stall-reason breakdown per CUDA source line of an ncu SASS source page.
usage: tools/ncu_stalls.py <sass.csv> <cubin> <mangled kernel> [top]"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_lines as T  # noqa: E402


def main():
    path, cubin, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 15
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    base = min(int(r[0], 16) for r in data)
    m = T.line_map(cubin, fn)
    agg = collections.defaultdict(lambda: collections.Counter())
    tot = collections.Counter()
    for r in data:
        k = m.get(int(r[0], 16) - base, ("?", 0))
        for i in cols:
            v = int(r[i] or 0)
            agg[k][hdr[i][6:]] += v
            tot[hdr[i][6:]] += v
    n = sum(tot.values())
    print("all:", ", ".join(f"{k} {100 * v / n:.1f}%" for k, v in tot.most_common(8)))
    for k, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
        s = sum(c.values())
        print(f"{k[0]}:{k[1]:<5} {100 * s / n:5.1f}%  " +
              ", ".join(f"{a} {100 * v / s:.0f}%" for a, v in c.most_common(4)))


if __name__ == "__main__":
    main()
