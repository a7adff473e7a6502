#!/bin/bash
# A/B timing of library builds (under gpurun): tools/ab.sh "<bench args>" rounds a.so b.so ...
# prints one line per run: build ms_per_step kernel_ms (+ parity when the bench ran it)
ARGS="$1"; R="$2"; shift 2
for r in $(seq $R); do for so in "$@"; do
  FPSSFT_LIB=$so timeout 600 python bench.py $ARGS 2>/dev/null | python -c '
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d.get("parity") or {}
print(sys.argv[1], round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms"],4), d["clocks"].get("sm_mhz"),
      (p.get("identical_support"), p.get("instances"), p.get("pass")) if p else "",
      "batch-major %.4f" % d["batch_major"]["ms_per_step"] if d.get("batch_major") else "")' $so
done; done
