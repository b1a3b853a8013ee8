#!/bin/bash
# Profiling recipe (run under gpurun from the repo root).  Outputs go to gpurun_out/:
#   launches.csv      every launch of a short bench run with its device time (profile mode: no
#                     concurrent offline kernel -- ncu serialises kernels, so a gated kernel
#                     running beside the reclaim would run to completion first)
#   prof_<k>.ncu-rep  one `ncu --set full` capture of each hot kernel
set -x
mkdir -p gpurun_out
make -C oracle >/dev/null
ARGS="--steps 2 --warmup 1 --preemptions 5 --skip-realtime --skip-fanout"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS --profile-mode > gpurun_out/launches_bench.log 2>&1
for k in ${KERNELS:-k_reclaim_copy_tma k_reclaim_fused k_offline_decode k_offline_gemm_pair k_restore_scatter k_apply k_offline_reserve}; do
  ncu --set full --clock-control none --import-source on -k regex:"^${k}$" -s 2 -c 1 \
      -o gpurun_out/prof_${k} -f python bench.py $ARGS > gpurun_out/prof_${k}.log 2>&1
done
ls -la gpurun_out
