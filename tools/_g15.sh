timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_suites.py tests/test_cpp_driver.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/bench_decision.py --sweep > gpurun_out/g15_decision.jsonl 2>&1; cut -c1-330 gpurun_out/g15_decision.jsonl
timeout 600 python tools/decision_under_copy.py > gpurun_out/g15_under_copy.jsonl 2>&1; cat gpurun_out/g15_under_copy.jsonl
