#!/bin/bash
# A/B timing of synth512_kernel builds (under gpurun): tools/ab_synth.sh rounds a.so b.so ...
R="$1"; shift
for r in $(seq $R); do for so in "$@"; do
  echo -n "$so  "; FPSSFT_LIB=$so timeout 300 python tools/synth_profile.py --reps 20 2>&1 | tail -1
done; done
