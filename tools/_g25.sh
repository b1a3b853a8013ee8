timeout 2400 python bench.py > gpurun_out/g25_bench.json 2> gpurun_out/g25_bench.err; echo bench $?
tail -3 gpurun_out/g25_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/g25_ref.json 2>&1; echo ref $?; tail -1 gpurun_out/g25_ref.json | cut -c1-400
