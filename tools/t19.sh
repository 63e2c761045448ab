PYTEST_K="4-" timeout 900 bash tools/gpu_quick.sh | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "slabs" 2>&1 | tail -1
timeout 900 python tools/time_kernels.py --p 2,3,4,5,6,7,8,9 --kernels 4 --reps 3 2>&1 | grep -v "^$" | cut -c1-140
timeout 900 python tools/time_kernels.py --p 4,5,6,7 --kernels 4 --reps 3 --matrix mass 2>&1 | grep -v "^$" | cut -c1-140
