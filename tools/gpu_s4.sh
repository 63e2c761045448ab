# session re-entry check: full GPU tests, smoke, short bench line
mkdir -p gpurun_out/s4
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/s4/gpu_tests.log 2>&1; tail -3 gpurun_out/s4/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4/smoke.log 2>&1; tail -1 gpurun_out/s4/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-sweep > gpurun_out/s4/bench.json 2> gpurun_out/s4/bench.err; tail -c 600 gpurun_out/s4/bench.json
