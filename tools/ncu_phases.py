#!/usr/bin/env python
"""Instructions and stall samples of a kernel per loop phase: every SASS
instruction is attributed (via nvdisasm -g line info) to the CUDA source line
it came from, and a line to the nearest enclosing `// (n)` phase marker of
the kernel it is inlined into (or to the device function it sits in).
usage: tools/ncu_phases.py <sass.csv> <cubin> <mangled kernel> [top]"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_lines as T  # noqa: E402
import ncu_regions as R  # noqa: E402


def main():
    path, cubin, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    iE = hdr.index("Instructions Executed")
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    base = min(int(r[0], 16) for r in data)
    m = T.line_map(cubin, fn)
    ins, smp = collections.Counter(), collections.Counter()
    why = collections.defaultdict(collections.Counter)
    for r in data:
        loc = m.get(int(r[0], 16) - base)
        reg = R.region(*loc) if loc else "?"
        ins[reg] += int(r[iE] or 0)
        smp[reg] += int(r[iS] or 0)
        for i in cols:
            why[reg][hdr[i][6:]] += int(r[i] or 0)
    ti, ts = sum(ins.values()), sum(smp.values())
    print(f"warp-instructions {ti}  stall samples {ts}")
    for reg, v in smp.most_common(top):
        w = ", ".join(f"{k} {100 * c / max(1, smp[reg]):.0f}%" for k, c in why[reg].most_common(3))
        print(f"{100 * ins[reg] / ti:5.1f}% instr {100 * v / ts:5.1f}% stall  {reg[:70]}  [{w}]")


if __name__ == "__main__":
    main()
