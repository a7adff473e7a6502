for b in 512 1024 2048 4096 8192; do
  timeout 300 python bench.py --batch $b --no-e2e --no-cpu-baseline --no-batch-major --steps 20 --warmup 5 --load-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'batch': $b, 'ms_per_step': d['ms_per_step'], 'value': d['value']}))"
done
