timeout 1500 python - <<'PY' > gpurun_out/g17_rt.log 2>&1
import json, sys
sys.path.insert(0, '.')
from paper_2604_07874_b200 import realtime as RT
r = RT.measure(horizon=60, tail_s=15, repeats=1, policies=("channel+prism",))
json.dump(r, open("gpurun_out/g17_rt.json", "w"))
for p in ("valve", "channel+prism"):
    a = r[p]
    print(p, a["ttft_delta_pct"], a["tpot_delta_pct"], json.dumps(a["slow_iterations"])[:3000])
print("solo", json.dumps(r["standalone"]["slow_iterations"])[:2000])
PY
tail -c 6000 gpurun_out/g17_rt.log
