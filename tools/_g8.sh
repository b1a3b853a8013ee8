timeout 300 python tools/bench_decision.py --sweep > gpurun_out/g8_decision.jsonl 2>&1; cat gpurun_out/g8_decision.jsonl
for L in low high mid spread low; do timeout 300 python tools/rt_coupling.py 50 8 $L 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['spread'], d['mean_ms'], min(d['iter_ms']), max(d['iter_ms']))"; done
