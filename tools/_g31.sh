timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 bench.py --gpus 2 --steps 3 --warmup 3 --handles 128 > gpurun_out/g31_bench2.json 2> gpurun_out/g31_bench2.err; echo bench2 $?
grep "bench" gpurun_out/g31_bench2.err | tail -20; tail -c 800 gpurun_out/g31_bench2.json
