"""C2/C3 real-time colocation run (paper_2604_07874_b200.realtime.measure): one JSON line.

usage: python tools/realtime_c2.py [--horizon S] [--repeats N] [--policies a,b] [--tail S]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    from paper_2604_07874_b200 import realtime as RT

    ap = argparse.ArgumentParser()
    ap.add_argument("--horizon", type=float, default=60.0)
    ap.add_argument("--tail", type=float, default=30.0)
    ap.add_argument("--repeats", type=int, default=2)
    ap.add_argument("--handles", type=int, default=0)
    ap.add_argument("--policies", default="valve-fifo,channel+static,channel+prism")
    ap.add_argument("--log-dir", default="")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    pols = tuple(p for p in a.policies.split(",") if p)
    r = RT.measure(horizon=a.horizon, tail_s=a.tail, repeats=a.repeats, handles=a.handles, policies=pols,
                   log_dir=a.log_dir or None)
    line = json.dumps(r)
    print(line, flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")
