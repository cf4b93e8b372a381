set -x
python bench.py > gpurun_out/bench_r01j.json 2> gpurun_out/bench_r01j.err
python bench.py --workload large_batch --steps 3 --warmup 3 > gpurun_out/bench_r01j_large.json 2> gpurun_out/bench_r01j_large.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01j_batch.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:block_kernel -s 1 -c 1 -o gpurun_out/batch8k_r01j python tools/prof_run.py batch 8192 2 > /dev/null 2>&1
{ echo "## tools/latency.py"; python tools/latency.py; echo "## tools/newton_timing.py"; python tools/newton_timing.py; echo "## tools/homotopy_timing.py"; python tools/homotopy_timing.py; echo "## tools/common_timing.py"; python tools/common_timing.py; echo "## tools/track_timing.py"; python tools/track_timing.py; } > gpurun_out/next_rows_r01b.txt 2>&1
