# A/B of the default library against a variant: batch DD, large QD x4096 and single point
# usage: bash tools/ab_lib.sh libphc_variant.so
V=${1:-libphc_f2s.so}
for r in 1 2; do
for lib in libphc.so $V; do
  PHC_LIB=paper_1109_0545_b200/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib batch', round(d['value']), round(d['roofline']['frac'],4))"
  PHC_LIB=paper_1109_0545_b200/$lib timeout 300 python bench.py --workload large --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib large1', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],4))"
done; done
for lib in libphc.so $V; do
  PHC_LIB=paper_1109_0545_b200/$lib timeout 600 python bench.py --workload large_batch --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib large_batch', round(d['value'],1), round(d['roofline']['frac'],4))"
  PHC_LIB=paper_1109_0545_b200/$lib timeout 300 python tools/newton_timing.py 2>&1 | grep -E '"c3"|"large"'
done
