#!/bin/bash
# Profiling recipe (run under gpurun from the repo root).  Outputs go to gpurun_out/:
#   launches.csv      every launch of a short bench run with its device time
#   prof_<k>.ncu-rep  one `ncu --set full` capture of each hot kernel
set -x
mkdir -p gpurun_out
make -C oracle >/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --preemptions 20 > gpurun_out/launches_bench.log 2>&1
for k in k_reclaim_copy k_reclaim k_offline_decode k_offline_reserve k_apply; do
  ncu --set full --clock-control none --import-source on -k regex:"^${k}$" -s 2 -c 1 \
      -o gpurun_out/prof_${k} -f python bench.py --steps 2 --warmup 1 --preemptions 5 > gpurun_out/prof_${k}.log 2>&1
done
ls -la gpurun_out
