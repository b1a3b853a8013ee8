"""Long paired TTFT/TPOT measurement (more A/B repeats than bench.py's default) with the bench's
tenant configuration; prints one JSON line (profiles/r1_realtime_long.json)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_07874_b200 import realtime as RT  # noqa: E402

repeats = int(sys.argv[1]) if len(sys.argv) > 1 else 8
# argv[2] = "qwen2-7b:<tokens>" runs the offline model's projection chain instead of one GEMM shape
gemm = ("qwen2-7b", int(sys.argv[2].split(":")[1])) if len(sys.argv) > 2 else (2048, 37888, 3584)
r = RT.measure_deltas(horizon=24.0, offline_ctas=16, repeats=repeats, offline_gemm=gemm, offline_gemm_ctas=64)
print(json.dumps(r))
