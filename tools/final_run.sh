# Round-end GPU battery: full GPU tests, smoke, bench line, launch list, full capture of the z-line launches.
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final/gpu_tests.log 2>&1; tail -1 gpurun_out/final/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; tail -c 300 gpurun_out/final/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-e2e --no-cpu > gpurun_out/final/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_zline -c 3 -o gpurun_out/final/zline_p4 python tools/run_step.py --p 4 --steps 1 > gpurun_out/final/ncu_full.log 2>&1; tail -1 gpurun_out/final/ncu_full.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_coefz -c 1 -o gpurun_out/final/coefz_p4 python tools/run_step.py --p 4 --steps 1 > gpurun_out/final/ncu_coef.log 2>&1; tail -1 gpurun_out/final/ncu_coef.log
