"""Online step slowdown vs the offline tenant's intensity on the C2 trace (realtime.measure, one
A B A pair per point): decode graph device time, TTFT / TPOT deltas, power and temperatures.
usage: python tools/rt_tenant_sweep.py "16:64,16:-1,-1:32,-1:-1" [horizon]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_07874_b200 import realtime as RT  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "16:64,16:-1,-1:32,-1:-1"
horizon = float(sys.argv[2]) if len(sys.argv) > 2 else 30.0
for point in spec.split(","):
    dec, gemm = (int(x) for x in point.split(":"))
    cfg = RT.RtConfig(decode_ctas=dec, gemm_ctas=gemm)
    r = RT.measure(horizon=horizon, tail_s=10.0, repeats=1, policies=(), cfg=cfg)
    v, s = r["valve"], r["standalone"]
    print(json.dumps({"decode_ctas": dec, "gemm_ctas": gemm, "ttft": v["ttft_delta_pct"], "tpot": v["tpot_delta_pct"],
                      "aa_ttft": r["aa_noise_ttft_pct"], "aa_tpot": r["aa_noise_tpot_pct"],
                      "decode_gpu_ms": [s["decode_gpu_ms_mean"], v["decode_gpu_ms_mean"]],
                      "decode_iter_ms": [s["decode_iter_ms_mean"], v["decode_iter_ms_mean"]],
                      "offline_tokens_per_s": v["offline_tokens_per_s"], "reclaims": v["reclaims"],
                      "clocks_solo": s["clocks"], "clocks_colo": v["clocks"]}), flush=True)
