timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g13_pytest.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/g13_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python tools/bench_decision.py --sweep > gpurun_out/g13_decision.jsonl 2>&1; cut -c1-300 gpurun_out/g13_decision.jsonl
