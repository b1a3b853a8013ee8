"""Per-request breakdown of a paired real-time run (events.jsonl logs written by realtime.measure):
where the colocated arm's TTFT goes -- prefill durations, decode iterations, queueing -- for the
requests with the largest increases.  usage: python tools/rt_analyze.py SOLO.jsonl COLO.jsonl"""
import json
import sys
from collections import defaultdict


def load(path):
    recs = [json.loads(line) for line in open(path)]
    ev = defaultdict(dict)
    for r in recs:
        if r.get("class") == "online" or r["kind"] in ("prefill_start", "prefill_end", "first_token"):
            rid = r.get("request_id")
            if rid is None:
                continue
            ev[rid][r["kind"]] = r
    return recs, ev


def main(solo, colo):
    rs, es = load(solo)
    rc, ec = load(colo)
    rows = []
    for rid, s in es.items():
        c = ec.get(rid)
        if not c or "first_token" not in s or "first_token" not in c:
            continue
        arr = s["arrival"]["time_us"]
        ts, tc = s["first_token"]["time_us"] - arr, c["first_token"]["time_us"] - arr
        ps = s["prefill_end"]["time_us"] - s["prefill_start"]["time_us"]
        pc = c["prefill_end"]["time_us"] - c["prefill_start"]["time_us"]
        qs, qc = s["prefill_start"]["time_us"] - arr, c["prefill_start"]["time_us"] - arr
        rows.append((100.0 * (tc - ts) / ts, rid, ts, tc, ps, pc, qs, qc))
    rows.sort(reverse=True)
    print(f"pairs {len(rows)}  mean ttft delta {sum(r[0] for r in rows) / len(rows):.2f} %")
    print("pct     rid  ttft_s  ttft_c  pre_s  pre_c  queue_s queue_c (ms)")
    for r in rows[:15] + [None] + rows[-5:]:
        if r is None:
            print("...")
            continue
        print(f"{r[0]:6.1f} {r[1]:5d} " + " ".join(f"{x / 1e3:7.1f}" for x in r[2:]))
    dp = [r[5] - r[4] for r in rows]
    print(f"prefill duration delta: mean {sum(dp) / len(dp) / 1e3:.2f} ms, max {max(dp) / 1e3:.2f} ms")
    kinds = defaultdict(int)
    for r in rc:
        kinds[r["kind"]] += 1
    print(dict(kinds))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
