# GPU battery: tests, smoke, one bench line (with sweep)
mkdir -p gpurun_out/r2
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/r2/gpu_tests.log 2>&1; tail -30 gpurun_out/r2/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; tail -2 gpurun_out/r2/smoke.log
timeout 1500 python bench.py --steps 5 --warmup 3 --oracle-seconds 5 > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; tail -c 400 gpurun_out/r2/bench.json; tail -5 gpurun_out/r2/bench.err
