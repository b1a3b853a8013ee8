timeout 900 python tools/pool_op_latency.py 2>&1 | tail -6
CUDA_DEVICE_MAX_CONNECTIONS=8 timeout 900 python tools/pool_op_latency.py 2>&1 | tail -6
