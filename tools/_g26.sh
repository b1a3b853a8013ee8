mkdir -p gpurun_out/rt26
timeout 1500 python - <<'PY' > gpurun_out/g26_rt.log 2>&1
import json, sys
sys.path.insert(0, '.')
from paper_2604_07874_b200 import realtime as RT
r = RT.measure(horizon=60, tail_s=15, repeats=1, policies=("channel+prism",), log_dir="gpurun_out/rt26")
print("aa", r["aa_noise_ttft_pct"], r["aa_noise_tpot_pct"])
print("solo", r["standalone"]["decode_gpu_ms_mean"], r["standalone"]["decode_sm_mhz_mean"])
for p in ("valve", "channel+prism"):
    a = r[p]
    print(p, a["ttft_delta_pct"], a["tpot_delta_pct"], a["decode_gpu_ms_mean"], a["decode_sm_mhz_mean"])
PY
tail -5 gpurun_out/g26_rt.log
python - <<'PY'
import json
def ld(n): return json.load(open(f"gpurun_out/rt26/{n}_steps.json"))
s = ld("solo0")
for n in ("solo1", "colo0", "channel_prism0"):
    c = ld(n)
    k = min(len(s["decode_gpu_us"]), len(c["decode_gpu_us"]))
    import statistics
    rat = [c["decode_gpu_us"][i] / s["decode_gpu_us"][i] for i in range(k)]
    mh = [c["decode_sm_mhz"][i] - s["decode_sm_mhz"][i] for i in range(k)]
    lo = [i for i in range(k) if c["decode_sm_mhz"][i] < 1900]
    print(n, "ratio mean %.4f" % statistics.mean(rat), "mhz solo %.0f colo %.0f" % (statistics.mean(s["decode_sm_mhz"][:k]), statistics.mean(c["decode_sm_mhz"][:k])),
          "steps<1900MHz colo %d solo %d" % (len(lo), sum(1 for i in range(k) if s["decode_sm_mhz"][i] < 1900)),
          "ratio on low-clock steps %.4f" % (statistics.mean([rat[i] for i in lo]) if lo else 0),
          "ratio on full-clock steps %.4f" % statistics.mean([rat[i] for i in range(k) if i not in set(lo)]))
PY
