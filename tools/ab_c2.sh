# A/B of single-point DD latency (c2, tiny) between the default library and a variant
for r in 1 2 3; do
for lib in libphc.so ${1:-libphc_ddchain.so}; do
for w in c2 tiny; do
  PHC_LIB=paper_1109_0545_b200/$lib timeout 300 python bench.py --workload $w --steps 300 --warmup 10 --no-flush --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config']['workload'], round(d['ms_per_step']*1e3,2), {k: round(v*1e3,2) for k,v in d.get('kernels_ms_per_step',{}).items()})"
done; done; done
