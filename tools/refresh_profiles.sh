# Re-measure the default bench line, its launch list and one ncu capture of each bench kernel
# (tag = round/capture suffix, e.g. r02i); outputs under gpurun_out/ (summarise with
# tools/ncu_summary.py, copy what is judged into profiles/).  Each ncu run follows a plain run
# of the same command that exited 0 (B200_PROFILING.md).
set -e
T=${1:-r02x}
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/plain_${T}.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_${T}_default.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/prof_run.py large_batch 64 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:block_kernel -s 1 -c 1 -o gpurun_out/large64_${T} \
    python tools/prof_run.py large_batch 64 2 > /dev/null 2>&1
python tools/prof_run.py batch 8192 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:block_kernel -s 1 -c 1 -o gpurun_out/batch8k_${T} \
    python tools/prof_run.py batch 8192 2 > /dev/null 2>&1
