timeout 900 python -m pytest tests/test_gpu_copy_gate.py tests/test_gpu_copy_tickets.py tests/test_realtime_logs.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 1500 python - <<'PY' > gpurun_out/g18_rt.log 2>&1
import json, sys
sys.path.insert(0, '.')
from paper_2604_07874_b200 import realtime as RT
r = RT.measure(horizon=60, tail_s=15, repeats=2, policies=("channel+prism",))
json.dump(r, open("gpurun_out/g18_rt.json", "w"))
print("aa", r["aa_noise_ttft_pct"], r["aa_noise_tpot_pct"])
for p in ("valve", "channel+prism"):
    a = r[p]
    print(p, a["ttft_delta_pct"], a["tpot_delta_pct"], a["per_run_ttft_delta_pct"], a["releases"], a["deferred_releases"], a["reclaims"], json.dumps(a["slow_iterations"])[:1500])
print("solo", json.dumps(r["standalone"]["slow_iterations"])[:800])
PY
tail -c 5000 gpurun_out/g18_rt.log
