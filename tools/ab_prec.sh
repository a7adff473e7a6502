mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu-baseline --no-batch-major --steps 10 --warmup 3 --load-seconds 0"
for c in 3 5; do for p in fp32 fp32-guarded fp64; do
  echo "cfg$c $p $(timeout 600 $B --config $c --precision $p 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["roofline"]["kernel_ms"], d["run"]["arithmetic"])')"
done; done
