set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_copy_gate.py tests/test_gpu_copy_tickets.py tests/test_reference_suites.py -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 300 python tools/bench_decision.py --sweep > gpurun_out/g4_decision.jsonl 2>&1; cat gpurun_out/g4_decision.jsonl
timeout 300 tools/_bin/valve_ops table 1024 1,4,15,36,64 > gpurun_out/g4_valve_ops_1024.json 2>&1; cat gpurun_out/g4_valve_ops_1024.json
timeout 300 tools/_bin/valve_ops table 128 1,4,15,64 > gpurun_out/g4_valve_ops_128.json 2>&1; cat gpurun_out/g4_valve_ops_128.json
timeout 300 oracle/_ref/ref_ops table 1024 1,4,15,36,64 > gpurun_out/g4_ref_ops_1024.json 2>&1; cat gpurun_out/g4_ref_ops_1024.json
timeout 300 oracle/_ref/ref_ops table 128 1,4,15,64 > gpurun_out/g4_ref_ops_128.json 2>&1; cat gpurun_out/g4_ref_ops_128.json
timeout 300 tools/_bin/valve_ops e2e 1024 36 20 3 > gpurun_out/g4_e2e.json 2>&1; cat gpurun_out/g4_e2e.json
timeout 900 python tools/rt_coupling.py 200 10 > gpurun_out/g4_coupling.jsonl 2>&1; cat gpurun_out/g4_coupling.jsonl | cut -c1-600
