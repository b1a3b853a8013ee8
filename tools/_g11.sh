timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_copy_gate.py tests/test_gpu_copy_tickets.py tests/test_reference_suites.py tests/test_cpp_driver.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/bench_decision.py --sweep > gpurun_out/g11_decision.jsonl 2>&1; cut -c1-460 gpurun_out/g11_decision.jsonl
timeout 300 python tools/copy_sweep.py > gpurun_out/g11_copy_sweep.jsonl 2>&1; cat gpurun_out/g11_copy_sweep.jsonl
