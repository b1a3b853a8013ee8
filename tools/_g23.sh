timeout 900 python tools/pool_op_latency.py 2>&1 | tail -6
