timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "repeatable or slabs" 2>&1 | tail -2
PYTEST_K="4-" timeout 900 bash tools/gpu_quick.sh | tail -1
timeout 900 python tools/time_kernels.py --p 4,6,7,8,9 --kernels 4 --reps 3 2>&1 | grep -v "^$" | cut -c1-140
timeout 900 python tools/time_kernels.py --p 5,6,7 --kernels 4 --reps 3 --matrix mass 2>&1 | grep -v "^$" | cut -c1-140
