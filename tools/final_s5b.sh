# Session-5 second battery: the tree with the forked weight solves — GPU tests, smoke, bench line,
# launch list, step split, serial-rules comparison, then compute-sanitizer over the small cases.
mkdir -p gpurun_out/s5b
timeout 1200 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/s5b/gpu_tests.log 2>&1; tail -3 gpurun_out/s5b/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s5b/smoke.log 2>&1; tail -1 gpurun_out/s5b/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s5b/bench.json 2> gpurun_out/s5b/bench.err; tail -c 300 gpurun_out/s5b/bench.json
WQ_RULES_FORK=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/s5b/bench_serial_rules.json 2> gpurun_out/s5b/bench_serial.err; tail -c 200 gpurun_out/s5b/bench_serial_rules.json
timeout 300 python bench.py --steps 10 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/s5b/bench_fork_rules.json 2> gpurun_out/s5b/bench_fork.err; tail -c 200 gpurun_out/s5b/bench_fork_rules.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s5b/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/s5b/ncu_launch.log 2>&1
bash tools/gpu_sanitize.sh
ls -la gpurun_out/s5b/
