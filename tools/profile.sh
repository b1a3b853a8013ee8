#!/bin/bash
# Profiling recipe (run under gpurun from the repo root).  Outputs to gpurun_out/.
#   1. launch list of a short bench run (per-launch device time; shares, not absolutes)
#   2. one `ncu --set full` capture each of the copy kernel and the fused reclaim kernel
set -x
mkdir -p gpurun_out
make -C oracle >/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --preemptions 20 > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_reclaim_copy -s 1 -c 1 \
    -o gpurun_out/prof_copy -f python bench.py --steps 2 --warmup 1 --preemptions 5 > gpurun_out/prof_copy.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_reclaim$|k_reclaimENS" -s 1 -c 1 \
    -o gpurun_out/prof_reclaim -f python bench.py --steps 2 --warmup 1 --preemptions 5 > gpurun_out/prof_reclaim.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_offline_decode -s 3 -c 1 \
    -o gpurun_out/prof_offline -f python bench.py --steps 2 --warmup 1 --preemptions 5 > gpurun_out/prof_offline.log 2>&1
ls -la gpurun_out
