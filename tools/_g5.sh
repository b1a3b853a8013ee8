timeout 600 python tools/rt_coupling.py 200 6 > gpurun_out/g5_coupling.jsonl 2>&1; timeout 600 python tools/rt_coupling.py 200 6 spread >> gpurun_out/g5_coupling.jsonl 2>&1; cut -c1-80,400-700 gpurun_out/g5_coupling.jsonl
timeout 900 python tools/realtime_c2.py --horizon 30 --tail 10 --repeats 1 --policies channel+static --out gpurun_out/g5_rt.json > gpurun_out/g5_rt.log 2>&1; echo rt $?
python - <<'PY'
import json
r=json.load(open('gpurun_out/g5_rt.json'))
print('aa', r['aa_noise_ttft_pct'], r['aa_noise_tpot_pct'])
s=r['standalone']; print('solo', s['decode_iter_ms_mean'], s['decode_gpu_ms_mean'], s['step_gap_us_mean'])
for p in ('valve','channel+static'):
    a=r[p]; print(p, a['ttft_delta_pct'], a['tpot_delta_pct'], a['decode_iter_ms_mean'], a['decode_gpu_ms_mean'], a['step_gap_us_mean'])
PY
