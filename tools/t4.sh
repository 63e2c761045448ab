mkdir -p gpurun_out/r2
PYTEST_K="4-" timeout 900 bash tools/gpu_quick.sh
timeout 600 python tools/time_kernels.py --p 2,3,4,6,8 --kernels 4 --reps 3
timeout 600 python tools/time_kernels.py --p 4,8 --kernels 4 --reps 3 --matrix mass
