#!/usr/bin/env python
"""Local-memory (STL/LDL) instructions of one kernel per CUDA source line.
usage: tools/spills.py <nvdisasm -g output> <mangled kernel name>"""
import collections
import re
import sys

cur, cnt, infn = None, collections.Counter(), False
for ln in open(sys.argv[1]):
    if re.match(r"\s*\.text\.", ln) or ln.startswith(".text."):
        infn = sys.argv[2] in ln
    h = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if h:
        cur = (h.group(1).split("/")[-1], int(h.group(2)))
        continue
    if infn and re.search(r"\b(STL|LDL)", ln):
        cnt[cur] += 1
for k, v in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print(v, k)
