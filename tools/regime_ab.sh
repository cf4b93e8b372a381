for env in "" "PHC_DEBUG_NO_LATENCY_PATH=1"; do
for w in tiny c2 c3; do
  env $env timeout 300 python bench.py --workload $w --steps 300 --warmup 10 --no-flush --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', d['config']['workload'], round(d['ms_per_step']*1e3,2), 'us/step', {k: round(v*1e3,2) for k,v in d['kernels_ms_per_step'].items()})"
done; done
