"""TTFT/TPOT deltas vs the offline tenant's intensity -- one JSON line per point.

Points are (decode-pass CTAs, GEMM CTAs or -1 for no GEMM tenant); the GEMM tenant is the Qwen2-7B
gate/up projection over 2048 tokens (bench.py --rt-gemm default).  A tensor-heavy tenant in the
gaps holds the GPU at its power cap; the online tenant then starts its busy period at reduced SM
clocks -- fewer GEMM CTAs trade harvested TFLOP/s for online latency."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_07874_b200 import realtime as RT  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "148:-1,148:0,148:74"
repeats = int(sys.argv[2]) if len(sys.argv) > 2 else 2
# optional trace: "spike_rate,period_s,width_s" (default: the pair_06 shape 6/s, 8 s, 1 s)
trace = dict(zip(("spike", "period", "width"), (float(x) for x in sys.argv[3].split(",")))) if len(sys.argv) > 3 else {}
for point in spec.split(","):
    dec, gemm = (int(x) for x in point.split(":"))
    r = RT.measure_deltas(horizon=24.0, offline_ctas=dec, repeats=repeats, **trace,
                          offline_gemm=None if gemm < 0 else (2048, 37888, 3584), offline_gemm_ctas=max(gemm, 0))
    clk = r["clocks_per_run"]["colocated"]
    print(json.dumps({"trace": r["trace"], "decode_ctas": dec, "gemm_ctas": gemm, "ttft": r["ttft_delta_pct"], "tpot": r["tpot_delta_pct"],
                      "ttft_runmean": r["ttft_delta_runmean_pct"], "tpot_runmean": r["tpot_delta_runmean_pct"],
                      "aa_ttft": r["aa_noise_ttft_pct"], "aa_tpot": r["aa_noise_tpot_pct"],
                      "prefill_ms": r["prefill_ms_median"], "decode_ms": r["decode_iter_ms_median"],
                      "offline_gbs": r["offline_gbs_harvested"], "gemm": r["offline_gemm"],
                      "colo_sm_mhz": [c and c["sm_mhz_median"] for c in clk],
                      "colo_power_w": [c and c["power_w_median"] for c in clk],
                      "plan_deviations": r.get("plan_deviations")}), flush=True)
