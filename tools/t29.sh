timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "repeatable or slabs" 2>&1 | tail -1
for A in 0 1 2 3; do echo "abl $A"; WQ_ZHP_ABLATE=$A timeout 300 python tools/time_kernels.py --p 8 --kernels 4 --reps 3 2>&1 | grep cfg | cut -c1-100; done
timeout 900 python tools/time_kernels.py --p 10 --kernels 2,4 --reps 2 2>&1 | grep cfg | cut -c1-120
timeout 900 python tools/time_kernels.py --p 8,9,10 --kernels 2,4 --reps 2 --matrix mass 2>&1 | grep cfg | cut -c1-120
