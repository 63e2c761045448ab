mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rules or coef or small or C1 or folded" > gpurun_out/r2/chk_tests.log 2>&1; tail -2 gpurun_out/r2/chk_tests.log
timeout 600 python tools/time_step.py --p 4 --reps 7 > gpurun_out/r2/time_step_p4.json 2>&1; cat gpurun_out/r2/time_step_p4.json | head -30
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/chk_launch.csv python tools/time_step.py --p 4 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/chk_launch.csv | head -14
