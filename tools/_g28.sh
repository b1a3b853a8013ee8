CUDA_MODULE_LOADING=EAGER timeout 1500 python - <<'PY' > gpurun_out/g28_rt.log 2>&1
import json, sys
sys.path.insert(0, '.')
from paper_2604_07874_b200 import realtime as RT
r = RT.measure(horizon=30, tail_s=10, repeats=1, policies=())
a = r["valve"]
print("valve", a["ttft_delta_pct"], a["tpot_delta_pct"], json.dumps(a["slow_iterations"]))
print("solo", json.dumps(r["standalone"]["slow_iterations"]))
PY
tail -3 gpurun_out/g28_rt.log
