mkdir -p gpurun_out/s13
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sf2 or C1" > gpurun_out/s13/parity.log 2>&1; tail -2 gpurun_out/s13/parity.log
timeout 300 python tools/time_kernels.py --d 2 --nel 1000 --p 2,4,6,8,10 --kernels 5 --reps 5 > gpurun_out/s13/t2d_stiff.jsonl 2>&1
timeout 300 python tools/time_kernels.py --d 2 --nel 1000 --p 2,4,6,8,10 --kernels 5 --reps 5 --matrix mass > gpurun_out/s13/t2d_mass.jsonl 2>&1
cat gpurun_out/s13/t2d_*.jsonl | cut -c1-150
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sf2l -c 1 -o gpurun_out/s13/sf2l_p4 python tools/time_kernels.py --d 2 --nel 1000 --p 4 --kernels 5 --reps 1 > gpurun_out/s13/ncu.log 2>&1; tail -1 gpurun_out/s13/ncu.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sf2l -c 1 -o gpurun_out/s13/sf2l_p8m python tools/time_kernels.py --d 2 --nel 1000 --p 8 --kernels 5 --reps 1 --matrix mass > gpurun_out/s13/ncu2.log 2>&1; tail -1 gpurun_out/s13/ncu2.log
