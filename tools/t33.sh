timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "repeatable or slabs" 2>&1 | tail -1
PYTEST_K="4-" timeout 900 bash tools/gpu_quick.sh | tail -1
timeout 900 python tools/time_kernels.py --p 7,8,9,10 --kernels 4 --reps 2 2>&1 | grep cfg | cut -c1-120
timeout 900 python tools/time_kernels.py --p 4,5,6,7,8,9,10 --kernels 4 --reps 2 --matrix mass 2>&1 | grep cfg | cut -c1-120
timeout 900 python tools/time_kernels.py --p 2,3,4 --kernels 2 --reps 2 --matrix mass 2>&1 | grep cfg | cut -c1-120
