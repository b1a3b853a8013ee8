timeout 2400 python bench.py > gpurun_out/g38_bench.json 2> gpurun_out/g38_bench.err; echo bench $?
timeout 600 python bench.py --impl reference > gpurun_out/g38_ref.json 2>&1; echo ref $?
mkdir -p gpurun_out/rt38
timeout 2700 python tools/realtime_c2.py --horizon 60 --tail 15 --repeats 4 --policies valve-fifo,channel+static,channel+prism --log-dir gpurun_out/rt38 --out gpurun_out/g38_rt_long.json > gpurun_out/g38_rt.log 2>&1; echo rt $?
