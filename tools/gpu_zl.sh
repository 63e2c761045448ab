# z-line iteration battery: z-line parity tests, kernel timings, per-launch list
mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "${PYTEST_K:-uniform_lines or graded or full_parity_small or repeatable or slabs or C1}" > gpurun_out/r2/zl_tests.log 2>&1; tail -3 gpurun_out/r2/zl_tests.log
timeout 600 python tools/time_kernels.py --p ${ZL_P:-2,3,4,5,6} --kernels 3 --reps 5 > gpurun_out/r2/zl_time.jsonl 2>&1; cat gpurun_out/r2/zl_time.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/zl_launch.csv python tools/time_kernels.py --p ${ZL_P:-2,3,4,5,6} --kernels 3 --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/zl_launch.csv
