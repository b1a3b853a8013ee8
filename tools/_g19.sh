
timeout 1500 python - <<'PY' > gpurun_out/g19_rt.log 2>&1
import json, sys
sys.path.insert(0, '.')
from paper_2604_07874_b200 import realtime as RT
r = RT.measure(horizon=60, tail_s=15, repeats=1, policies=())
json.dump(r, open("gpurun_out/g19_rt.json", "w"))
a = r["valve"]
print("valve", a["ttft_delta_pct"], a["tpot_delta_pct"], json.dumps(a["slow_iterations"]))
PY
tail -c 5000 gpurun_out/g19_rt.log
