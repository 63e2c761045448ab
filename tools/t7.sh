timeout 600 python tools/time_kernels.py --p 1,2,3,4,5,6,7,8,9,10 --kernels 4,2 --reps 3 --matrix mass 2>&1 | grep -v "^$" | cut -c1-150
timeout 600 python tools/time_kernels.py --p 7,9,10 --kernels 4,2 --reps 3 2>&1 | grep -v "^$" | cut -c1-150
