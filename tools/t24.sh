timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "repeatable or slabs" 2>&1 | tail -1
WQ_ZHP_D=3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "repeatable or slabs" 2>&1 | tail -1
for D in 2 3 4; do for P in 6 8; do echo "D $D"; WQ_ZHP_D=$D timeout 300 python tools/time_kernels.py --p $P --kernels 4 --reps 3 2>&1 | grep cfg | cut -c1-120; done; done
