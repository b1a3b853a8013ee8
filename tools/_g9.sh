timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_reclaim_fused -s 3 -c 1 -o gpurun_out/prof_reclaim_fused -f python tools/bench_decision.py > gpurun_out/g9_ncu.log 2>&1; echo ncu $?
tail -3 gpurun_out/g9_ncu.log
