# d <= 2 sum-factorised kernel parity + timing; z-line boundary lines via ZHP (measurement switch WQ_ZL_BND)
mkdir -p gpurun_out/s5
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sf2 or SF2 or C1 or small or coefficients" > gpurun_out/s5/parity.log 2>&1; tail -3 gpurun_out/s5/parity.log
timeout 600 python tools/time_kernels.py --d 2 --nel 1000 --p 2,4,6 --kernels 5,1 --reps 5 > gpurun_out/s5/t2d_stiff.jsonl 2>&1
timeout 600 python tools/time_kernels.py --d 2 --nel 1000 --p 2,4,6 --kernels 5,1 --reps 5 --matrix mass > gpurun_out/s5/t2d_mass.jsonl 2>&1
cat gpurun_out/s5/t2d_*.jsonl | cut -c1-200
for B in zline zhp; do
  WQ_ZL_BND=$B timeout 900 python tools/time_kernels.py --p 2,3,4,6 --kernels 3 --reps 5 > gpurun_out/s5/zl_bnd_$B.jsonl 2>&1
  WQ_ZL_BND=$B timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5/launch_$B.csv python tools/time_kernels.py --p 2,3,4,6 --kernels 3 --reps 1 > /dev/null 2>&1
done
cat gpurun_out/s5/zl_bnd_*.jsonl | cut -c1-160
