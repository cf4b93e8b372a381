# Re-measure the bench lines, the launch list and one ncu capture of the dominant kernel
# (tag = round/capture suffix, e.g. r01k); outputs under gpurun_out/
T=${1:-r01x}
python bench.py > gpurun_out/bench_${T}.json 2> gpurun_out/bench_${T}.err
python bench.py --workload large_batch --steps 3 --warmup 3 > gpurun_out/bench_${T}_large.json 2> gpurun_out/bench_${T}_large.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}_batch.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:block_kernel -s 1 -c 1 -o gpurun_out/batch8k_${T} python tools/prof_run.py batch 8192 2 > /dev/null 2>&1
