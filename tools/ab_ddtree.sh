for r in 1 2 3; do
for lib in libphc.so libphc_ddtree.so; do
  PHC_LIB=paper_1109_0545_b200/$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done; done
for lib in libphc.so libphc_ddtree.so; do
for w in c2 tiny; do
  PHC_LIB=paper_1109_0545_b200/$lib timeout 300 python bench.py --workload $w --steps 300 --warmup 10 --no-flush --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config']['workload'], round(d['ms_per_step']*1e3,2))"
done; done
