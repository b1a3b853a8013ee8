timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_copy_gate.py tests/test_reference_suites.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/bench_decision.py --sweep > gpurun_out/g6_decision.jsonl 2>&1; cat gpurun_out/g6_decision.jsonl
timeout 300 tools/_bin/valve_ops table 1024 1,4,15,36,64 > gpurun_out/g6_valve_ops_1024.json 2>&1; cat gpurun_out/g6_valve_ops_1024.json
timeout 2400 python tools/rt_tenant_sweep.py "16:64,16:-1,-1:32,-1:-1" 30 > gpurun_out/g6_sweep.jsonl 2>&1; cut -c1-400 gpurun_out/g6_sweep.jsonl
