mkdir -p gpurun_out/rt34
timeout 1500 python - <<'PY' > gpurun_out/g34_rt.log 2>&1
import json, sys
sys.path.insert(0, '.')
from paper_2604_07874_b200 import realtime as RT
r = RT.measure(horizon=60, tail_s=10, repeats=1, policies=("channel+prism",), log_dir="gpurun_out/rt34")
print("solo", r["standalone"]["decode_gpu_ms_mean"])
for p in ("valve", "channel+prism"):
    a = r[p]; print(p, a["ttft_delta_pct"], a["tpot_delta_pct"], a["decode_gpu_ms_mean"], a["slow_iterations"]["n"])
PY
tail -4 gpurun_out/g34_rt.log
