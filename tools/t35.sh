timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "repeatable or slabs" 2>&1 | tail -1
for B in 1 4 8 16; do echo "B $B"; WQ_ZHP_BLOCK=$B timeout 600 python tools/time_kernels.py --p 5,8,10 --kernels 4 --reps 2 2>&1 | grep cfg | cut -c1-100;
WQ_ZHP_BLOCK=$B timeout 600 python tools/time_kernels.py --p 6,10 --kernels 4 --reps 2 --matrix mass 2>&1 | grep cfg | cut -c1-100; done
