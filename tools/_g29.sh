timeout 1500 python - <<'PY' > gpurun_out/g29_rt.log 2>&1
import json, sys
sys.path.insert(0, '.')
from paper_2604_07874_b200 import realtime as RT
r = RT.measure(horizon=30, tail_s=10, repeats=1, policies=())
a = r["valve"]
print("valve", a["ttft_delta_pct"], a["tpot_delta_pct"], json.dumps(a["slow_iterations"]))
PY
tail -2 gpurun_out/g29_rt.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 3 --warmup 3 --handles 256 --rt-horizon-multi 8 --c4-layers 2 --c4-horizon 6 > gpurun_out/g29_bench2.json 2> gpurun_out/g29_bench2.err; echo bench2 $?
tail -c 3000 gpurun_out/g29_bench2.json; grep -i "error\|Traceback\|failed" gpurun_out/g29_bench2.err | head
