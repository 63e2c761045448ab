# Round-2 closing battery (session 4): GPU tests, smoke, bench line with sweep, reference arm,
# launch list, 2D kernel timings and capture
mkdir -p gpurun_out/final2
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/final2/gpu_tests.log 2>&1; tail -3 gpurun_out/final2/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; tail -1 gpurun_out/final2/smoke.log
timeout 1800 python bench.py --steps 10 --warmup 3 > gpurun_out/final2/bench.json 2> gpurun_out/final2/bench.err; tail -c 300 gpurun_out/final2/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final2/ref.json 2> gpurun_out/final2/ref.err; tail -c 200 gpurun_out/final2/ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final2/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/final2/ncu_launch.log 2>&1
timeout 300 python tools/time_kernels.py --d 2 --nel 1000 --p 2,4,6,8,10 --kernels 5 --reps 5 > gpurun_out/final2/t2d_stiff.jsonl 2>&1
timeout 300 python tools/time_kernels.py --d 2 --nel 1000 --p 2,4,6,8,10 --kernels 5 --reps 5 --matrix mass > gpurun_out/final2/t2d_mass.jsonl 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sf2l -c 1 -o gpurun_out/final2/sf2l_p4 python tools/time_kernels.py --d 2 --nel 1000 --p 4 --kernels 5 --reps 1 > gpurun_out/final2/ncu_sf2.log 2>&1
ls -la gpurun_out/final2/
