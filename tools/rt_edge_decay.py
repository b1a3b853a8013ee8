"""Online decode slowdown vs time since the busy edge, per offline-tenant intensity: for each
(decode-pass CTAs : GEMM CTAs) point, one replayed A B A run of valve and channel+prism on the C2
trace; per-step device time of the colocated arm over the paired standalone step, bucketed by the
time since the step's busy edge.  One JSON line per point.
usage: python tools/rt_edge_decay.py "16:64,16:32,16:-1,-1:-1" [horizon]"""
import bisect
import json
import os
import statistics
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_07874_b200 import realtime as RT  # noqa: E402

BUCKETS = ((0, 20e3, "<20ms"), (20e3, 100e3, "20-100ms"), (100e3, 500e3, "100-500ms"), (500e3, 1e12, ">500ms"))


def decay(solo, colo):
    out = {}
    k = min(len(solo["decode_gpu_us"]), len(colo["decode_gpu_us"]))
    bs, ts = colo["busy_starts"], colo["decode_t_us"]
    for lo, hi, name in BUCKETS:
        v = []
        for i in range(k):
            j = bisect.bisect_right(bs, ts[i]) - 1
            dt = ts[i] - bs[j] if j >= 0 else -1
            if lo <= dt < hi:
                v.append(colo["decode_gpu_us"][i] / solo["decode_gpu_us"][i])
        out[name] = [len(v), round(statistics.mean(v), 4) if v else None]
    return out


spec = sys.argv[1] if len(sys.argv) > 1 else "16:64,16:32,16:-1,-1:-1"
horizon = float(sys.argv[2]) if len(sys.argv) > 2 else 30.0
for point in spec.split(","):
    dec, gemm = (int(x) for x in point.split(":"))
    d = tempfile.mkdtemp()
    r = RT.measure(horizon=horizon, tail_s=10.0, repeats=1, policies=("channel+prism",),
                   cfg=RT.RtConfig(decode_ctas=dec, gemm_ctas=gemm), log_dir=d)
    ld = lambda n: json.load(open(os.path.join(d, f"{n}_steps.json")))  # noqa: E731
    solo = ld("solo0")
    print(json.dumps({"decode_ctas": dec, "gemm_ctas": gemm,
                      "valve": {"ttft": r["valve"]["ttft_delta_pct"], "tpot": r["valve"]["tpot_delta_pct"],
                                "offline_tokens_per_s": r["valve"]["offline_tokens_per_s"],
                                "step_ratio_by_time_since_busy_edge": decay(solo, ld("colo0"))},
                      "channel+prism": {"ttft": r["channel+prism"]["ttft_delta_pct"],
                                        "tpot": r["channel+prism"]["tpot_delta_pct"],
                                        "step_ratio_by_time_since_busy_edge": decay(solo, ld("channel_prism0"))},
                      "aa": {"ttft": r["aa_noise_ttft_pct"], "tpot": r["aa_noise_tpot_pct"],
                             "step_ratio_by_time_since_busy_edge": decay(solo, ld("solo1"))},
                      "power_w_median_colo": (r["valve"]["clocks"][0] or {}).get("power_w_median")}), flush=True)
