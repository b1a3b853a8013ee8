mkdir -p gpurun_out/rt7
timeout 1200 python - <<'PY' > gpurun_out/g7_rt.log 2>&1
import json, sys
sys.path.insert(0, '.')
from paper_2604_07874_b200 import realtime as RT
r = RT.measure(horizon=30, tail_s=10, repeats=1, policies=("channel+prism",), cfg=RT.RtConfig(decode_ctas=-1, gemm_ctas=-1), log_dir="gpurun_out/rt7")
print(json.dumps({k: r[k] for k in ("aa_noise_ttft_pct", "aa_noise_tpot_pct")}), json.dumps({p: {k: r[p][k] for k in ("ttft_delta_pct", "tpot_delta_pct", "decode_gpu_ms_mean", "releases", "reclaims")} for p in ("valve", "channel+prism")}))
PY
tail -2 gpurun_out/g7_rt.log
for f in solo1 colo0 channel_prism0; do echo "== $f"; python tools/rt_steps.py gpurun_out/rt7/solo0_steps.json gpurun_out/rt7/${f}_steps.json; done
