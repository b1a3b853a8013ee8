set -x
timeout 300 python -m pytest tests/test_gpu_tp.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/c4_tp.py --tp 2 --layers 2 --horizon 8 --handles 16 --ctx 512 --out gpurun_out/g3_c4.json > gpurun_out/g3_c4.log 2>&1; echo "c4 rc $?"; tail -c 2500 gpurun_out/g3_c4.log
mkdir -p gpurun_out/rt3
timeout 1800 python tools/realtime_c2.py --horizon 60 --tail 15 --repeats 2 --log-dir gpurun_out/rt3 --out gpurun_out/g3_rt.json > gpurun_out/g3_rt.log 2>&1; echo "rt rc $?"
tail -c 600 gpurun_out/g3_rt.log
