mkdir -p gpurun_out/rt14
timeout 2700 python tools/realtime_c2.py --horizon 60 --tail 15 --repeats 4 --policies valve-fifo,channel+static,channel+prism --log-dir gpurun_out/rt14 --out gpurun_out/g14_rt_long.json > gpurun_out/g14_rt.log 2>&1; echo rt $?
python - <<'PY'
import json
r=json.load(open('gpurun_out/g14_rt_long.json'))
print('aa', r['aa_noise_ttft_pct'], r['aa_noise_tpot_pct'])
for p in ('valve','valve-fifo','channel+static','channel+prism'):
    a=r[p]; print(p, round(a['ttft_delta_pct'],2), round(a['tpot_delta_pct'],2), [round(x,1) for x in a['per_run_ttft_delta_pct']], [round(x,2) for x in a['per_run_tpot_delta_pct']], a['decode_gpu_ms_mean'])
PY
