#!/usr/bin/env python
"""Instruction / stall-sample shares of a kernel grouped by enclosing source
region (nearest preceding function or `// (n)` phase marker).
usage: tools/ncu_regions.py <sass.csv> <cubin> <mangled kernel> [top]"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_lines as T  # noqa: E402

SRC = {n: open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "paper_1711_11407_b200", "csrc", n)).read().split("\n")
       for n in ("fpssft.cu", "fpssft_device.cuh", "fpssft_team.cuh", "fpssft_large.cuh",
                                "fpssft_guard.cuh", "fpssft_regfft.cuh", "fpssft_synth.cuh")}


def region(f, ln):
    src = SRC.get(f)
    if src is None:
        return f
    for i in range(min(ln, len(src)) - 1, -1, -1):
        t = src[i]
        if t.startswith(("__device__", "__global__", "struct ")) or t.strip().startswith("// ("):
            return f"{f}:{i + 1} {t.strip()[:64]}"
    return f


def main():
    path, cubin, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    base = min(int(r[0], 16) for r in data)
    m = T.line_map(cubin, fn)
    agg = collections.defaultdict(lambda: [0, 0])
    for r in data:
        k = m.get(int(r[0], 16) - base, ("?", 0))
        key = region(*k) if k[0] != "?" else "?"
        agg[key][0] += int(r[iS] or 0)
        agg[key][1] += int(r[iE] or 0)
    ts = sum(v[0] for v in agg.values())
    te = sum(v[1] for v in agg.values())
    print(f"samples {ts}  warp-instructions {te}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100 * v[1] / te:5.1f}% instr {100 * v[0] / ts:5.1f}% stall  {k}")


if __name__ == "__main__":
    main()
