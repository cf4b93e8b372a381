# A/B of the QD layouts (large single, large x4096, c3 x1024 homotopy/plain) between the default library and a variant
V=${1:-libphc_swz.so}
for r in 1 2; do
for lib in libphc.so $V; do
  PHC_LIB=paper_1109_0545_b200/$lib timeout 300 python bench.py --workload large --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib large1', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],4))"
done; done
for lib in libphc.so $V; do
  PHC_LIB=paper_1109_0545_b200/$lib timeout 600 python bench.py --workload large_batch --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib large_batch', round(d['value'],1), round(d['roofline']['frac'],4))"
  PHC_LIB=paper_1109_0545_b200/$lib python tools/homotopy_timing.py 2>&1 | grep '"c3", "points": 1024'
done
