timeout 1500 python - <<'PY' > gpurun_out/g27_rt.log 2>&1
import json, sys
sys.path.insert(0, '.')
from paper_2604_07874_b200 import realtime as RT
r = RT.measure(horizon=30, tail_s=10, repeats=1, policies=("channel+prism",))
print("solo", r["standalone"]["decode_gpu_ms_mean"], json.dumps(r["standalone"]["clocks"]))
for p in ("valve", "channel+prism"):
    a = r[p]
    print(p, a["ttft_delta_pct"], a["tpot_delta_pct"], a["decode_gpu_ms_mean"], json.dumps(a["clocks"]))
PY
tail -5 gpurun_out/g27_rt.log
nvidia-smi -q -d CLOCK | head -40
