# d = 2 line kernel: parity + timing against the row variant and the direct kernel
mkdir -p gpurun_out/s7
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sf2 or SF2 or C1 or small or coefficients or slabs" > gpurun_out/s7/parity.log 2>&1; tail -3 gpurun_out/s7/parity.log
timeout 600 python tools/time_kernels.py --d 2 --nel 1000 --p 2,4,6,8,10 --kernels 5,1 --reps 5 > gpurun_out/s7/t2d_stiff.jsonl 2>&1
timeout 600 python tools/time_kernels.py --d 2 --nel 1000 --p 2,4,6,8,10 --kernels 5,1 --reps 5 --matrix mass > gpurun_out/s7/t2d_mass.jsonl 2>&1
WQ_SF2_ROWS=1 timeout 600 python tools/time_kernels.py --d 2 --nel 1000 --p 4 --kernels 5 --reps 5 > gpurun_out/s7/t2d_rows.jsonl 2>&1
cat gpurun_out/s7/t2d_*.jsonl | cut -c1-200
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sf2l -c 1 -o gpurun_out/s7/sf2l_p4 python tools/time_kernels.py --d 2 --nel 1000 --p 4 --kernels 5 --reps 1 > gpurun_out/s7/ncu.log 2>&1; tail -2 gpurun_out/s7/ncu.log
