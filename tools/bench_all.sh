#!/bin/bash
# bench.py lines for every config and the reference arm (under gpurun).
O=gpurun_out/evidence
mkdir -p $O
: > $O/bench_lines.jsonl
timeout 900 python bench.py >> $O/bench_lines.jsonl 2> $O/bench_c2.err
timeout 900 python bench.py --impl reference >> $O/bench_lines.jsonl 2> $O/bench_ref.err
for c in 1 3 4 5; do
  timeout 1200 python bench.py --config $c >> $O/bench_lines.jsonl 2> $O/bench_c$c.err
done
wc -l $O/bench_lines.jsonl
