"""TTFT/TPOT deltas vs offline harvest intensity (offline CTAs) -- one JSON line per point."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_07874_b200 import realtime as RT  # noqa: E402

for ctas in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,148,74").split(",")]:
    r = RT.measure_deltas(horizon=24.0, offline_ctas=ctas)
    print(json.dumps({"offline_ctas": ctas, "ttft": r["ttft_delta_pct"], "tpot": r["tpot_delta_pct"],
                      "prefill_ms": r["prefill_ms_median"], "decode_ms": r["decode_iter_ms_median"],
                      "offline_gbs": r["offline_gbs_harvested"]}), flush=True)
