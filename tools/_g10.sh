timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_copy_gate.py tests/test_reference_suites.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/bench_decision.py --sweep > gpurun_out/g10_decision.jsonl 2>&1; cut -c1-420 gpurun_out/g10_decision.jsonl
timeout 2400 python bench.py > gpurun_out/g10_bench.json 2> gpurun_out/g10_bench.err; echo bench $?
tail -5 gpurun_out/g10_bench.err
