#!/bin/bash
# One-GPU evidence run (under gpurun): GPU tests, bench lines for every config
# and the reference arm, the ncu launch list of the headline bench and
# `ncu --set full` captures of each config's dominant kernel.  Outputs land in
# gpurun_out/evidence/; tools/summarize_profiles.py turns them into profiles/.
set -u
O=gpurun_out/evidence
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 600 python tools/bench_imaging.py --reps 5 > $O/imaging.jsonl 2>&1
: > $O/bench_lines.jsonl
timeout 900 python bench.py >> $O/bench_lines.jsonl 2> $O/bench_c2.err
timeout 900 python bench.py --impl reference >> $O/bench_lines.jsonl 2> $O/bench_ref.err
for c in 1 3 4 5; do
  timeout 1200 python bench.py --config $c >> $O/bench_lines.jsonl 2> $O/bench_c$c.err
done
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --load-seconds 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv $B > $O/ncu_launches.log 2>&1
N="ncu --set full --import-source on --clock-control none -k regex:recover -s 3 -c 1"
timeout 900 $N -o $O/cfg2 $B --config 2 > $O/ncu_cfg2.log 2>&1
timeout 900 $N -o $O/cfg3 $B --config 3 > $O/ncu_cfg3.log 2>&1
timeout 900 $N -o $O/cfg4 $B --config 4 > $O/ncu_cfg4.log 2>&1
timeout 900 $N -o $O/cfg5_recover $B --config 5 --batch 2048 --no-synth > $O/ncu_cfg5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:synth -c 1 \
  -o $O/cfg5_synth python tools/synth_profile.py --reps 1 > $O/ncu_synth.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage_lines -s 1 -c 1 \
  -o $O/cfg2_stage python tools/stage_profile.py 2 > $O/ncu_stage.log 2>&1
# reports are ~25 MB each (gpurun brings back <= 64 MiB): keep CSV exports
for r in $O/*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source=sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
  rm -f $r
done
ls -la $O
