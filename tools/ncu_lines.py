#!/usr/bin/env python
"""Attribute an ncu SASS source page (CSV) to CUDA source lines.

usage: tools/ncu_lines.py <sass.csv from `ncu -i X --page source --csv --print-source=sass`>
                          <cubin> <mangled kernel name> [top]
Line info comes from `nvdisasm -g` (build with -lineinfo)."""
import collections
import csv
import re
import subprocess
import sys


def line_map(cubin, fn):
    out = subprocess.run(["nvdisasm", "-g", "-fun", fn, cubin], capture_output=True, text=True).stdout
    if not out.strip():
        out = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
    cur, m, infn = None, {}, False
    for ln in out.splitlines():
        if re.match(r"\s*\.text\.", ln) or ln.startswith(".text."):
            infn = fn in ln
        h = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if h:
            cur = (h.group(1).split("/")[-1], int(h.group(2)))
            continue
        a = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s", ln)
        if a and infn:
            m[int(a.group(1), 16)] = cur
    return m


def main():
    path, cubin, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = rows[2:]
    iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    base = min(int(r[0], 16) for r in data)
    m = line_map(cubin, fn)
    agg = collections.defaultdict(lambda: [0, 0])
    for r in data:
        off = int(r[0], 16) - base
        key = m.get(off, ("?", 0))
        agg[key][0] += int(r[iS] or 0)
        agg[key][1] += int(r[iE] or 0)
    ts = sum(v[0] for v in agg.values())
    te = sum(v[1] for v in agg.values())
    print(f"samples {ts}  warp-instructions {te}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0]:22s}:{k[1]:<5d} stall {100 * v[0] / ts:5.1f}%  instr {100 * v[1] / te:5.1f}%")


if __name__ == "__main__":
    main()
