mkdir -p gpurun_out/r2
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; tail -c 400 gpurun_out/r2/bench.json
