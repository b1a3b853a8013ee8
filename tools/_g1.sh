set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/g1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc $?"; tail -3 gpurun_out/g1_smoke.log
timeout 1200 python tools/realtime_c2.py --horizon 30 --tail 10 --repeats 1 --out gpurun_out/g1_rt.json > gpurun_out/g1_rt.log 2>&1; echo "rt rc $?"; tail -c 3000 gpurun_out/g1_rt.log
