"""Measured online TTFT/TPOT deltas: the same online trace standalone vs colocated with the gated
offline tenant (paper_2604_07874_b200.realtime.measure_deltas).  Prints one JSON line."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    from paper_2604_07874_b200 import realtime as RT

    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--horizon", type=float, default=24.0)
    ap.add_argument("--base", type=float, default=0.3)
    ap.add_argument("--spike", type=float, default=6.0)
    ap.add_argument("--handles", type=int, default=64)
    ap.add_argument("--seed", type=int, default=2604)
    ap.add_argument("--repeats", type=int, default=2)
    ap.add_argument("--offline-ctas", type=int, default=148)
    ap.add_argument("--gemm", default="", help="m,n,k of the gated offline GEMM tenant (empty: decode only)")
    a = ap.parse_args()
    gemm = tuple(int(x) for x in a.gemm.split(",")) if a.gemm else None
    print(json.dumps(RT.measure_deltas(a.horizon, a.base, a.spike, handles=a.handles, layers=a.layers,
                                       seed=a.seed, repeats=a.repeats,
                                       offline_ctas=a.offline_ctas, offline_gemm=gemm)))
