set -x
timeout 300 python -m pytest tests/test_gpu_tp.py -x -q -p no:cacheprovider 2>&1 | tail -5
mkdir -p gpurun_out/rt2
timeout 1200 python tools/realtime_c2.py --horizon 30 --tail 10 --repeats 1 --policies channel+prism --log-dir gpurun_out/rt2 --out gpurun_out/g2_rt.json > gpurun_out/g2_rt.log 2>&1; echo "rt rc $?"
python tools/rt_analyze.py gpurun_out/rt2/solo0.jsonl gpurun_out/rt2/colo0.jsonl
python tools/rt_analyze.py gpurun_out/rt2/solo0.jsonl gpurun_out/rt2/solo1.jsonl
python tools/rt_analyze.py gpurun_out/rt2/solo0.jsonl gpurun_out/rt2/channel_prism0.jsonl
