python tools/time_kernels.py --p 2,3,4,5,6,7,8,10 --kernels 3,4,2 --reps 3 2>&1 | tee gpurun_out/r2/times_stiff.log
python tools/time_kernels.py --p 2,4,6,8,10 --kernels 4,2 --reps 3 --matrix mass 2>&1 | tee gpurun_out/r2/times_mass.log
