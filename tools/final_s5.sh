# Round-2 session-5 GPU battery on the restored tree: full GPU tests, smoke, bench line, reference arm,
# launch list, ncu capture of the headline z-line assembly, step split.
mkdir -p gpurun_out/s5
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/s5/gpu_tests.log 2>&1; tail -3 gpurun_out/s5/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s5/smoke.log 2>&1; tail -1 gpurun_out/s5/smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/s5/bench.json 2> gpurun_out/s5/bench.err; tail -c 300 gpurun_out/s5/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s5/ref.json 2> gpurun_out/s5/ref.err; tail -c 300 gpurun_out/s5/ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s5/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/s5/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zline -c 3 -o gpurun_out/s5/zline_p4 python tools/run_step.py --p 4 --steps 1 > gpurun_out/s5/ncu_full.log 2>&1; tail -1 gpurun_out/s5/ncu_full.log
timeout 900 python tools/time_step.py --p 4 --reps 7 > gpurun_out/s5/time_step_p4.json 2>&1
ls -la gpurun_out/s5/
